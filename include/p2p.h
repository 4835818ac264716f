/*
 * p2p.h -- C ABI of the B200-native MLFMA near-field (P2P) operator.
 *
 * The operation (§3 L61-79 and §4.1; kernel per SPEC.md L150-158;
 * SURVEY.md §8 hot-path sentence):
 *
 *     phi_t = sum_{s : box(s) in E1(box(t)), r_ts >= eps}  q_s * ln(1/r_ts)
 *
 * where the leaf level L gives a 2^(L-1) x 2^(L-1) grid of boxes on the unit
 * square ("The number of boxes is equal to 4^{L-1}"), box(p) =
 * (min(floor(x*2^(L-1)), 2^(L-1)-1), same for y), and E1(b) is
 * b plus its <= 8 adjacent boxes, clipped at the domain edge (PAPER.md L88,
 * "The number 9 ... adjacent neighboring boxes").
 *
 * Life cycle: p2p_plan_create (host-side plan build: level selection, box
 * assignment, Morton sort, CSR offsets, tiles, partition, NR/R layout, upload)
 * or p2p_plan_create_device (the same plan built by GPU kernels from device
 * coordinates) -> p2p_apply (per matrix-vector product; stream-ordered,
 * allocation-free) -> p2p_destroy.  Beyond the paper's kernel and grid
 * (SURVEY.md §8(f)): the 2D Helmholtz kernel, 3D octree kernels and an adaptive
 * (CT-driven) quadtree layout -- see p2p_kernel and p2p_layout below.
 *
 * Conventions:
 *  - Every entry point returns a p2p_status; nothing throws or exits.  On
 *    failure p2p_last_error() returns a thread-local human-readable detail.
 *  - "Host" pointers are ordinary CPU memory; "device" pointers are CUDA
 *    global memory on the plan's device (e.g. torch.Tensor.data_ptr()).
 *  - Plan order ("P2P_ORDER_PLAN") is the Morton order of the leaf boxes, and
 *    within a box the original index order (stable sort; "in the
 *    order of the boxes' morton index").  It is the fast path: no permutation.
 *  - One apply may be in flight per plan at a time (the plan owns workspace), unless the plan
 *    was given more workspace slots (p2p_plan_set_workspaces).
 *  - Multi-GPU (part_world > 1): plans from the global point set (p2p_plan_create) or from each
 *    rank's own points (p2p_box_counts / p2p_partition_route / p2p_plan_create_local); the halo
 *    exchange by the caller's collective (p2p_halo_pack + p2p_apply_dist*) or by the library's
 *    device-synchronised peer-memory kernels (p2p_peer_* / p2p_apply_peer_sync / p2p_gather).
 *  - There is no CPU fallback: a plan created with device < 0 is host-only
 *    (plan building, introspection and export work; apply returns
 *    P2P_ERROR_NO_DEVICE).
 */
#ifndef P2P_B200_H
#define P2P_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define P2P_ABI_VERSION 1

typedef struct p2p_plan_s *p2p_plan; /* opaque; owned by the library */

typedef enum {
    P2P_SUCCESS = 0,
    P2P_ERROR_INVALID_ARGUMENT = 1,     /* n = 0, non-finite or out-of-[0,1] coordinate, L+i < 1 */
    P2P_ERROR_CONSTRUCTION_FAILURE = 2, /* CT loop exceeded l_max */
    P2P_ERROR_LAYOUT_CORRUPT = 3,       /* internal offsets inconsistent */
    P2P_ERROR_OUT_OF_MEMORY = 4,        /* host or device allocation failed */
    P2P_ERROR_CUDA = 5,                 /* a CUDA runtime call failed; detail in p2p_last_error() */
    P2P_ERROR_NOT_SUPPORTED = 6,        /* valid request outside this build's envelope (e.g. L > 15) */
    P2P_ERROR_NO_DEVICE = 7             /* apply on a host-only plan, or no CUDA device */
} p2p_status;

/* Kernel functions G(r) of phi_t = sum_{s in E1(t), r >= eps} q_s G(r_ts):
 *   LAPLACE_2D   (the paper's): G = ln(1/r), real q and phi.
 *   HELMHOLTZ_2D (beyond the paper's kernel; R23):
 *                G = (i/4) H0^(1)(kappa r) = (-Y0(kappa r) + i J0(kappa r)) / 4, the 2D
 *                free-space Green's function of the oscillatory ("high-frequency", PAPER.md
 *                L17, L299) MLFMA problems; kappa = desc.wavenumber > 0; q and phi complex,
 *                interleaved (re, im) pairs in the plan precision (C99 complex / torch
 *                complex64 / complex128 layout).  TILED layout; partitions (halo exchange,
 *                distributed applies) move (re, im) pairs.
 *   LAPLACE_3D / HELMHOLTZ_3D (R24): the operator on an octree
 *                leaf grid of the unit cube -- boxes 2^(L-1) per side (L <= 9), E1 = the 3x3x3 block
 *                clipped at the faces, 3D Morton order (x bit 3i, y 3i+1, z 3i+2); G = 1/(4 pi r)
 *                (real) or e^{i kappa r}/(4 pi r) (complex, interleaved (re, im)).  Coordinates
 *                are [n][3] (src_xy / tgt_xy hold x, y, z); explicit level only; NONREDUNDANT
 *                layout (one CTA per target box stages its 27 neighbour boxes); one partition;
 *                host plan build. */
typedef enum {
    P2P_KERNEL_LAPLACE_2D = 0,
    P2P_KERNEL_HELMHOLTZ_2D = 1,
    P2P_KERNEL_LAPLACE_3D = 2,
    P2P_KERNEL_HELMHOLTZ_3D = 3
} p2p_kernel;

/* Source layouts (§3.2 Indexing = non-redundant; §3.3 Repetition =
 * redundant), re-derived for B200:
 *   NR    = Morton-sorted points + CSR box offsets, gathered per tile into
 *           shared memory at run time (no copy of any point);
 *   R     = per target box, the packed halo of its E1 sources (coordinates
 *           copied at plan time, weights refreshed per apply by a pack
 *           kernel), read as one contiguous TMA bulk copy per tile;
 *   TILED = per CTA tile, its region (tile + one-box ring) packed at plan
 *           time, rebased to the region origin: redundancy only on the ring,
 *           ((W+2)/W)^2, streamed by one TMA bulk copy per tile; weights are
 *           gathered in-kernel through a per-entry index. */
typedef enum {
    P2P_LAYOUT_NONREDUNDANT = 0,
    P2P_LAYOUT_REDUNDANT = 1,
    P2P_LAYOUT_TILED = 2,
    /* The paper's own layouts and kernels, reproduced as written (fp64,
     * one partition, weights/potentials in either order, no accumulate with P2P_ORDER_PLAN):
     *   PAPER_INDEXING (§3.2): the seven arrays -- source and target coordinates and
     *     source weights in the caller's order, per-box target index lists and per-box E1
     *     source index lists (boxes in Morton order) with their offsets; one GPU thread per box
     *     loops its targets x neighbour sources through the indices (global memory only, as in
     *     the paper: "none of ... Shared Memory ... were employed", L61).  Eq. 3 bytes.
     *   PAPER_REPETITION (§3.3): one fixed-stride record of 3 + 27*C doubles per target
     *     (caller's order) = [x_t, y_t, count (integer in the low 4 bytes of its slot), then
     *     (x_s, y_s, q_s) per E1 source]; C = max(ct, t) (ct of the descriptor, t the largest box
     *     occupancy); one GPU thread per target; each apply first writes q into the records
     *     (the paper's per-execution collection of potentials).  Eq. 8 bytes (with C = ct). */
    P2P_LAYOUT_PAPER_INDEXING = 3,
    P2P_LAYOUT_PAPER_REPETITION = 4,
    /* a CT-driven ADAPTIVE quadtree -- a box is split while
     * it holds more than desc.ct sources or targets and its level is below desc.l_max (desc.level
     * is ignored); E1 becomes the U-list: the leaves whose closed squares touch the target's leaf
     * (the 3x3 block on a uniform tree).  One CTA per target leaf stages its U-list's sources.
     * LAPLACE_2D, one partition, host plan build. */
    P2P_LAYOUT_ADAPTIVE = 5
} p2p_layout;

/* fp64 is paper-faithful ("stored as Double"); fp32 uses
 * box-local coordinates and the SFU lg2. */
typedef enum { P2P_FP64 = 0, P2P_FP32 = 1 } p2p_precision;

typedef enum {
    P2P_ORDER_PLAN = 0, /* q and phi in plan (Morton) order */
    P2P_ORDER_USER = 1  /* q and phi in the caller's original point order */
} p2p_order;

typedef struct {
    uint32_t struct_size;  /* = sizeof(p2p_plan_desc); set by p2p_plan_desc_init */
    int32_t abi_version;   /* = P2P_ABI_VERSION */
    int64_t n_src, n_tgt;  /* global point counts, >= 1 */
    const double *src_xy;  /* host, [n_src][2] interleaved x,y in [0,1]^2; copied, caller keeps ownership */
    const double *tgt_xy;  /* host, [n_tgt][2]; may alias src_xy (collocated) */
    int32_t level;         /* > 0: leaf level L (grid 2^(L-1) per side); 0: CT loop */
    int32_t ct;            /* CT loop clustering threshold (default 15) */
    int32_t l_start;       /* CT loop start level (default 3) */
    int32_t l_max;         /* CT loop cap (default 15 in this build; SPEC.md L122 caps at 16) */
    int32_t level_delta;   /* i of PAPER.md Eq. 37 (L' = L + i), applied after the CT loop */
    int32_t kernel;        /* p2p_kernel */
    double epsilon;        /* minimum separation (default 1e-12) */
    int32_t layout;        /* p2p_layout */
    int32_t precision;     /* p2p_precision */
    int32_t device;        /* CUDA device ordinal; -1 = host-only plan (no upload, no apply) */
    int32_t tile_log2;     /* -1 = auto; else CTA tile side 2^tile_log2 leaf boxes */
    void *stream;          /* cudaStream_t for plan-time uploads (NULL = default stream) */
    int32_t part_world;    /* number of Morton-range partitions (ranks); 1 = whole problem */
    int32_t part_rank;     /* partition owned by this plan, 0 <= part_rank < part_world */
    double wavenumber;     /* HELMHOLTZ_2D: kappa > 0 (radians per unit length); ignored for LAPLACE_2D */
} p2p_plan_desc;

/* Fill *desc with defaults (level 0 -> CT loop, ct 15, l_start 3, l_max 15,
 * epsilon 1e-12, NR, fp32, device 0, auto tile, 1 partition, LAPLACE_2D, wavenumber 0). */
void p2p_plan_desc_init(p2p_plan_desc *desc);

/* Build a plan.  Copies the host inputs; allocates all device memory and
 * workspace on desc->device; uploads on desc->stream and synchronises it.
 * *out is set to NULL on failure.  Errors: INVALID_ARGUMENT, CONSTRUCTION_FAILURE,
 * NOT_SUPPORTED, OUT_OF_MEMORY, CUDA. */
p2p_status p2p_plan_create(const p2p_plan_desc *desc, p2p_plan *out);

/* Build the same plan ON THE GPU from device-resident coordinates (SURVEY.md §8(f) NEXT-2:
 * the paper's "collection", its dominant cost -- PAPER.md §3.2, §3.3, alpha ~ 0.82 of
 * the total at L337-343 -- done by sm_100a kernels: Morton codes, stable radix sort, CSR offsets,
 * box statistics, tiles, the NR / TILED layouts and the launch queue).
 *   d_src_xy, d_tgt_xy: device, [n][2] interleaved fp64 x,y in [0,1]^2 on desc->device (may
 *                       alias); read during the call only (the caller keeps ownership).
 *   desc->src_xy / tgt_xy are ignored; every other field means what it means for
 *   p2p_plan_create, and the plan (every exported array, the info, every apply result) is
 *   bit-identical to the one p2p_plan_create builds from the same coordinates.
 * Work runs on desc->stream and the call synchronises it.  Scope: layouts NONREDUNDANT and
 * TILED, part_world = 1.  Errors: as p2p_plan_create, plus NOT_SUPPORTED (other layouts,
 * part_world > 1), NO_DEVICE (device < 0 or no GPU). */
p2p_status p2p_plan_create_device(const p2p_plan_desc *desc, const double *d_src_xy, const double *d_tgt_xy,
                                  p2p_plan *out);

/* phi = A q on the plan's device, asynchronously on `stream` (cudaStream_t,
 * NULL = default stream).
 *   d_q   : device, weights in the plan precision (float or double; HELMHOLTZ_2D: complex,
 *           i.e. 2 values (re, im) per point -- every count below is then in complex elements).
 *           ORDER_PLAN: n_src elements in global plan order.
 *           ORDER_USER: n_src elements in the caller's point order.
 *   d_out : device, results in the plan precision.
 *           ORDER_PLAN: n_tgt_local elements = this partition's targets in plan order.
 *           ORDER_USER: n_tgt elements in the caller's order; only this
 *           partition's targets are written.
 *   accumulate: 0 -> overwrite, 1 -> d_out += phi (near + far).
 * The caller keeps ownership of d_q/d_out; they must not alias.
 * Errors: INVALID_ARGUMENT (NULL pointers, bad order), NO_DEVICE, CUDA. */
p2p_status p2p_apply(p2p_plan plan, const void *d_q, void *d_out, int32_t order,
                     int32_t accumulate, void *stream);

/* Applies in flight: by default a plan has one workspace (gathered weights, partial results,
 * staging for host buffers, the tile queue), so applies on one plan must be serialised on one
 * stream (applies on different plans may overlap freely).  p2p_plan_set_workspaces(plan, n)
 * (1 <= n <= 8) gives the plan n workspace slots, rotated over p2p_apply / p2p_apply_host /
 * p2p_apply_host_async calls: up to n applies of one plan may then be in flight on different
 * streams -- e.g. step k's D2H overlapping step k+1's H2D and kernel; each apply waits on the
 * device (an event) for the apply that last used its slot, so no host synchronisation is
 * needed.  Calls from several host threads on one plan must still be serialised.  Single-
 * partition NR / R / TILED / 3D / ADAPTIVE plans (NOT_SUPPORTED for part_world > 1 and the
 * paper's layouts).  Extra device memory: n - 1 copies of the workspace. */
p2p_status p2p_plan_set_workspaces(p2p_plan plan, int32_t n);

/* Same operation with HOST buffers (h_q: n_src weights, h_out: n_tgt_local
 * (ORDER_PLAN) or n_tgt (ORDER_USER) results).  Copies h_q to the device,
 * applies, copies the result back and synchronises `stream`.  For full copy
 * bandwidth pass page-locked (pinned) memory.  With accumulate = 1, h_out is
 * read first. */
p2p_status p2p_apply_host(p2p_plan plan, const void *h_q, void *h_out, int32_t order,
                          int32_t accumulate, void *stream);

/* Asynchronous variant of p2p_apply_host: enqueues the H2D copy, the apply and
 * the D2H copy on `stream` and returns; h_q / h_out must stay valid (and, for
 * overlap, be pinned) until the caller synchronises the stream.  Applies on
 * different plans and streams overlap their copies with each other's kernels. */
p2p_status p2p_apply_host_async(p2p_plan plan, const void *h_q, void *h_out, int32_t order,
                                int32_t accumulate, void *stream);

/* Distributed apply (part_world > 1, weights NOT replicated): phi for this
 * partition's targets (plan order, n_tgt_local) from
 *   d_q_owned: device, n_src_owned weights this partition owns, in plan order
 *              (global plan indices [src_owned_begin, src_owned_begin + n_src_owned));
 *   d_q_halo : device, n_halo weights received from the other partitions, grouped
 *              by owner rank ascending and, within an owner, by global plan
 *              index ascending (the order p2p_halo_pack produces on the owner).
 * The halo weight exchange itself is the caller's collective (NCCL via a
 * torch ProcessGroup). */
p2p_status p2p_apply_dist(p2p_plan plan, const void *d_q_owned, const void *d_q_halo,
                          void *d_out, int32_t accumulate, void *stream);

/* p2p_apply_dist in two phases, to overlap the halo exchange with work that does
 * not need it (issue both on the same stream, interior first):
 *   p2p_apply_dist_interior: stages d_q_owned and runs the TILED tiles whose
 *     regions hold owned sources only (p2p_plan_info.interior_launches queue
 *     entries; every tile when part_world = 1; none for NR / R);
 *   p2p_apply_dist_boundary: stages d_q_halo and runs the remaining tiles.
 * The caller's exchange of d_q_halo may be in flight during the interior phase;
 * d_q_owned must stay valid until the boundary phase is enqueued. */
p2p_status p2p_apply_dist_interior(p2p_plan plan, const void *d_q_owned, void *d_out, int32_t accumulate,
                                   void *stream);
p2p_status p2p_apply_dist_boundary(p2p_plan plan, const void *d_q_halo, void *d_out, int32_t accumulate,
                                   void *stream);

/* Distributed apply with the halo read straight from the owners' device memory (SURVEY.md
 * §8(e): the peer-memory alternative to the NCCL exchange -- over NVLink / NVSwitch on a B200
 * node these are P2P loads, no send buffer, no collective, one gather kernel):
 *   d_peer_q: HOST array of part_world DEVICE pointers; d_peer_q[r] = rank r's owned weights
 *             (its n_src_owned elements in plan order), mapped into this process with
 *             p2p_ipc_open (or any peer-accessible pointer); d_peer_q[part_rank] is ignored
 *             (d_q_owned is used).  Read during the call's stream work only.
 *   The caller orders the peers: their buffers must hold this apply's weights before the
 *   gather runs and must not change until it has finished (e.g. barriers around the apply).
 * part_world <= 16.  Errors: INVALID_ARGUMENT (NULL pointers, part_world > 16), NO_DEVICE, CUDA. */
p2p_status p2p_apply_dist_peer(p2p_plan plan, const void *d_q_owned, const void *const *d_peer_q, void *d_out,
                               int32_t accumulate, void *stream);

/* Result gather (allgatherv) over peer memory: d_global (device, n_tgt
 * elements, global plan order) receives every rank's shard, d_peer_out[r] = rank r's n_tgt_local
 * results (plan order; mapped with p2p_ipc_open; d_peer_out[part_rank] may be this rank's own
 * output).  Device-to-device copies on `stream` (NVLink reads on a node).  The caller orders the
 * peers (every shard written before the call's copies run). */
p2p_status p2p_gather_peer(p2p_plan plan, const void *const *d_peer_out, void *d_global, void *stream);

/* Device-synchronised peer-memory exchange: the halo weight exchange (a6) and the result
 * allgatherv (a11) as one-sided NVLink reads between the ranks' HBM, ordered by signal words
 * in device memory -- no host barrier, no collective library; every step is a stream-ordered
 * kernel, so an apply can be captured in a CUDA graph.  Set-up (once per plan, collective):
 *   p2p_peer_buffers: allocates (first call) and returns this rank's published send buffer
 *     (n_send weights), published result buffer (n_tgt_local results) and signal block
 *     (zero-initialised, device-synchronised before return); export them with p2p_ipc_export.
 *   p2p_peer_connect: every rank's three pointers as mapped in this process (HOST arrays of
 *     part_world DEVICE pointers; p2p_ipc_open for the peers, this rank's own for part_rank) and
 *     displ[o] = the offset of this rank's segment in rank o's send buffer (the sum of rank o's
 *     halo_counts send entries for ranks < part_rank).  The caller must ensure every rank's
 *     p2p_peer_buffers returned before any rank's first apply (e.g. the handle all-gather).
 * p2p_apply_peer_sync: as p2p_apply_dist, with the halo pulled from the owners: publish this
 *   rank's send buffer once every reader has finished the previous apply, pull the halo on an
 *   internal stream (waiting for each owner's signal) while the interior tiles run, then the
 *   boundary tiles.  Every rank must call it the same number of times (epochs are counted on
 *   the device).  d_q_owned / d_out as p2p_apply_dist.
 * p2p_gather (allgatherv, a11): d_global (device, n_tgt results, global plan
 *   order) receives every rank's n_tgt_local results d_local (plan order); collective.
 * p2p_peer_check: host-synchronous; P2P_ERROR_CUDA if a wait for a peer's signal gave up after
 *   20 s (a peer that stopped calling), else SUCCESS.
 * Applies on one plan must be serialised on one stream (the plan's workspace and signal words
 * are shared).  part_world <= 16; NR, R and TILED 2D plans (Laplace, Helmholtz).
 * Errors: INVALID_ARGUMENT (NULL pointers, no connect), NOT_SUPPORTED (other layouts), CUDA. */
p2p_status p2p_peer_buffers(p2p_plan plan, void **d_pub_w, void **d_pub_o, void **d_sig);
p2p_status p2p_peer_connect(p2p_plan plan, const void *const *peer_pub_w, const void *const *peer_pub_o,
                            const void *const *peer_sig, const int64_t *displ);
p2p_status p2p_apply_peer_sync(p2p_plan plan, const void *d_q_owned, void *d_out, int32_t accumulate,
                               void *stream);
p2p_status p2p_gather(p2p_plan plan, const void *d_local, void *d_global, void *stream);
p2p_status p2p_peer_check(p2p_plan plan);

/* Partitioned plans from each rank's OWN points (north_star: "a one-time
 * exchange distributes halo source points"): no rank ever holds the global point set.
 *   1. p2p_box_counts: per-box counts of n points (host [n][2] in [0,1]^2) at leaf level `level`
 *      -> counts[4^(level-1)] (Morton order, overwritten).  Every rank counts the points it
 *      holds; the caller sums the counts over the ranks (an allreduce): the GLOBAL counts.
 *   2. p2p_partition_route: from the global counts alone, the partition the global builder
 *      would make, and for each passed point the bit mask of the ranks that need it (sources:
 *      the owner of its box and every rank with an owned tile whose region (tile + one-box
 *      ring) holds the box -- the halo; targets: the owner of its box).  desc: level > 0,
 *      layout NR / R / TILED, part_world <= 32, part_rank = the caller, n_src / n_tgt /
 *      src_xy / tgt_xy = the passed points (may be 0 / NULL); *_ids = their global ids
 *      (distinct int64 per set: they fix the order of points inside a box, as the caller's
 *      point index does for p2p_plan_create).
 *   3. the caller sends every point (coordinates + id) to the ranks in its mask (an all-to-all);
 *   4. p2p_plan_create_local: the partition's plan from what arrived -- every point of every
 *      box the rank needs, once (else INVALID_ARGUMENT naming the box) -- with the same
 *      desc fields and global counts.  The plan (tiles, local order, halo, send lists) equals
 *      p2p_plan_create's with the global point set for this part_rank, so applies are
 *      bit-identical.  ORDER_USER and the host-buffer applies are NOT_SUPPORTED on it (there is
 *      no global user order on one rank); p2p_plan_export(SRC_PERM / TGT_PERM) give indices into
 *      the passed arrays.  Host build only; `device` as p2p_plan_create. */
p2p_status p2p_box_counts(int32_t level, int64_t n, const double *xy, int32_t *counts);
p2p_status p2p_partition_route(const p2p_plan_desc *desc, const int64_t *src_ids, const int64_t *tgt_ids,
                               const int32_t *src_counts, const int32_t *tgt_counts, int64_t n_src_global,
                               int64_t n_tgt_global, uint32_t *src_mask, uint32_t *tgt_mask);
p2p_status p2p_plan_create_local(const p2p_plan_desc *desc, const int64_t *src_ids, const int64_t *tgt_ids,
                                 const int32_t *src_counts, const int32_t *tgt_counts, int64_t n_src_global,
                                 int64_t n_tgt_global, p2p_plan *out);

/* CUDA IPC for p2p_apply_dist_peer.  p2p_ipc_export: the 64-byte handle (host buffer) of the
 * allocation holding d_ptr and d_ptr's byte offset in it (pointers from sub-allocating
 * allocators, e.g. torch's, are fine).  p2p_ipc_open: map a peer's handle on `device` and
 * return the mapping + offset; p2p_ipc_close releases it (pass the pointer p2p_ipc_open gave). */
p2p_status p2p_ipc_export(const void *d_ptr, void *handle64, int64_t *offset);
p2p_status p2p_ipc_open(const void *handle64, int64_t offset, int32_t device, void **d_ptr);
p2p_status p2p_ipc_close(void *d_ptr, int64_t offset);

/* Gather this partition's owned weights that the other partitions need into
 * d_send (device, n_send elements), grouped by destination rank ascending,
 * within a destination by global plan index ascending. */
p2p_status p2p_halo_pack(p2p_plan plan, const void *d_q_owned, void *d_send, void *stream);

/* Release all host and device memory of the plan.  NULL is a no-op. */
p2p_status p2p_destroy(p2p_plan plan);

typedef struct {
    uint32_t struct_size;
    int32_t level, tile_log2, layout, precision, device, part_world, part_rank;
    int64_t side;                /* 2^(L-1) */
    int64_t boxes;               /* 4^(L-1) */
    int64_t n_src, n_tgt;        /* global */
    int64_t n_src_local;         /* sources the kernel reads (owned + halo) */
    int64_t n_tgt_local;         /* targets owned by this partition */
    int64_t n_src_owned, src_owned_begin, tgt_begin; /* global plan index ranges */
    int64_t n_halo, n_send;      /* per-apply exchange sizes (elements) */
    int64_t occupied_src_boxes, occupied_tgt_boxes;
    int64_t t_max;               /* max over boxes of max(#src, #tgt) ("t") */
    double density;              /* D = N_tgt / 4^(L-1) */
    double density_occupied;     /* N_tgt / occupied target boxes */
    int64_t pairs;               /* pair-interactions of this partition (int64, exact) */
    int64_t pairs_global;        /* pair-interactions of the whole problem */
    int64_t tiles;               /* CTAs per apply (non-empty tiles of this partition) */
    int64_t smem_bytes;          /* dynamic shared memory per CTA */
    int64_t halo_entries;        /* R layout: packed halo entries (incl. padding) */
    int64_t alg_bytes_kernel;    /* algorithmic HBM bytes per apply, independent of the layout:
                                    each target's coordinates read + potential written, each source's
                                    coordinates + weight read once, 8 B of CSR offsets per box of the
                                    launched tiles */
    int64_t layout_bytes_apply;  /* bytes the plan's layout moves per apply (model): NR = alg;
                                    R = packed halo + pack_r; TILED = packed regions (+ring
                                    redundancy), index, tables, packed targets, weight gather */
    int64_t device_bytes;        /* device memory held by the plan */
    double build_seconds;        /* host plan build */
    double upload_seconds;       /* host -> device upload */
    int32_t cta_threads;         /* threads per CTA of the P2P kernel */
    int32_t slots_per_unit;      /* TILED: target slots per work unit (2: dense fp32 pairs of one box) */
    int32_t items_per_unit;      /* TILED: 3 = one item per row-run (sorted item list), 1 = whole unit */
    int32_t flags;               /* TILED: bit 0 n9-ordered boxes, bit 1 flattened row-runs */
    int64_t interior_launches;   /* TILED: queue entries run by p2p_apply_dist_interior */
    int64_t paper_model_bytes;   /* PAPER_INDEXING: Eq. 3 (40N + 4^L(2 + 10t)); PAPER_REPETITION: Eq. 8
                                    (8N(3 + 27 ct)); else 0 */
    int64_t record_stride;       /* PAPER_REPETITION: doubles per record (3 + 27 C); else 0 */
    int64_t launches;            /* queue entries of a full apply (tiles, tail tiles split) */
    int32_t kernel;              /* p2p_kernel */
    int32_t components;          /* values per weight / result: 1 (real), 2 (complex) */
    double wavenumber;           /* HELMHOLTZ_2D: kappa */
} p2p_plan_info;

/* Plan statistics.  Versioning: a caller compiled against an older (smaller)
 * p2p_plan_info sets info->struct_size = sizeof(its struct) and receives that
 * prefix only; struct_size = 0 (or >= the current size) means the current
 * layout.  On return struct_size holds the number of bytes written. */
p2p_status p2p_plan_get_info(p2p_plan plan, p2p_plan_info *info);

typedef enum {
    P2P_EXPORT_SRC_PERM = 0,        /* int64[n_src_local]: original (user) index of each local source, plan order */
    P2P_EXPORT_TGT_PERM = 1,        /* int64[n_tgt_local]: original index of each owned target, plan order */
    P2P_EXPORT_SRC_BOX_OFFSETS = 2, /* int64[boxes+1]: global CSR offsets of sources per Morton box */
    P2P_EXPORT_TGT_BOX_OFFSETS = 3, /* int64[boxes+1]: global CSR offsets of targets per Morton box */
    P2P_EXPORT_NEIGHBORS = 4,       /* int64[boxes*9]: E1 list per box, ascending Morton, -1 padded */
    P2P_EXPORT_PARTITION = 5,       /* int64[2*(part_world+1)]: src_begin[0..W], tgt_begin[0..W] (global plan idx) */
    P2P_EXPORT_SRC_GLOBAL = 6,      /* int64[n_src_local]: global plan index of each local source */
    P2P_EXPORT_HALO_COUNTS = 7,     /* int64[2*part_world]: recv count per owner rank, send count per dest rank */
    P2P_EXPORT_TILES = 8,           /* int64[tiles]: Morton index of each CTA tile (launch order) */
    P2P_EXPORT_HALO_INDEX = 9,      /* int64[halo_entries]: R layout, local source of each packed entry (-1 = pad) */
    P2P_EXPORT_SEND_INDEX = 10,     /* int64[n_send]: owned-local index of each sent weight */
    P2P_EXPORT_HALO_OFFSETS = 11,   /* int64[boxes+1]: R layout, packed-halo offsets per Morton box */
    P2P_EXPORT_REGION_OFFSETS = 12, /* int64[tiles+1]: TILED layout, packed-region offsets per tile (Morton tile order) */
    P2P_EXPORT_REGION_INDEX = 13,   /* int64[entries]: TILED layout, local source of each packed entry (-1 = pad) */
    P2P_EXPORT_REGION_TABLE = 14,   /* int64[tiles*stride]: TILED, per tile its region box starts then its slot count */
    P2P_EXPORT_SLOT_OFFSETS = 15,   /* int64[tiles+1]: TILED, target-slot offsets per tile (Morton tile order) */
    P2P_EXPORT_SLOT_BASE = 16,      /* int64[slots]: TILED, row-run base j0 = by*(W+2) + bx of each slot */
    P2P_EXPORT_SLOT_OUTPUT = 17,    /* int64[slots]: TILED, tile-local output index of each slot (-1 = duplicate) */
    P2P_EXPORT_ITEM_OFFSETS = 18,   /* int64[tiles+1]: TILED NS = 3 plans, item-list offsets per tile */
    P2P_EXPORT_ITEMS = 19,          /* int64[items]: TILED NS = 3 plans, unit << 2 | row in kernel order */
    P2P_EXPORT_LAUNCH = 20,         /* int64[2*launches]: TILED, Morton-order slot of each queue entry, then its
                                       part | nparts << 16 */
    P2P_EXPORT_PAPER_NEI_OFFSETS = 21, /* int64[boxes+1]: PAPER_INDEXING, offsets into the E1 source lists */
    P2P_EXPORT_PAPER_NEI_INDEX = 22,   /* int64[entries]: PAPER_INDEXING, original index of each E1 source */
    P2P_EXPORT_PAPER_RECORDS = 23,     /* int64[n_tgt*stride]: PAPER_REPETITION, the raw 8-byte record words
                                          (bit patterns of the doubles; q slots as of the last apply) */
    P2P_EXPORT_LEAVES = 24,            /* int64[3*leaves]: ADAPTIVE, (level, ix, iy) per leaf, Morton order */
    P2P_EXPORT_ULIST_OFFSETS = 25,     /* int64[leaves+1]: ADAPTIVE, U-list offsets per leaf (Morton order) */
    P2P_EXPORT_ULIST = 26              /* int64[entries]: ADAPTIVE, U-list leaf indices (ascending) */
} p2p_export_kind;

/* Copy a plan array to host memory.  If host_dst is NULL, *bytes receives the
 * required size; otherwise *bytes must be >= that size.  Arrays are computed
 * by the host builder and are bit-exact functions of the inputs. */
p2p_status p2p_plan_export(p2p_plan plan, int32_t kind, void *host_dst, size_t *bytes);

const char *p2p_status_string(p2p_status status);
const char *p2p_last_error(void); /* thread-local detail of the last failure ("" if none) */
int32_t p2p_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* P2P_B200_H */
