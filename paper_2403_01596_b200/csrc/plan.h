// plan.h -- internal plan representation shared by the host builder
// (plan_builder.cpp), the C ABI (p2p_capi.cpp) and the kernel launchers
// (p2p_kernels.cu).  Not part of the public ABI (include/p2p.h).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "p2p.h"

#if defined(__CUDACC__)
#define P2P_HD __host__ __device__
#else
#define P2P_HD
#endif

namespace p2p {

// ---- shared-memory layouts of the P2P kernels (byte offsets), used by the
// plan builder (sizing), the launcher and the kernels (carving).
P2P_HD inline int align16(int x) { return (x + 15) & ~15; }
#ifndef P2P_LOG256
#define P2P_LOG256 1  // fp64 log: 256-entry table + degree-5 log1p (0: round 1's 128 entries + degree 6)
#endif
// fp64 log: table of (1/c_k rounded, -log of it), c_k = 1 + (k + 1/2) / kLogTab
constexpr int kLogTab = P2P_LOG256 ? 256 : 128;
constexpr int kLogTab32 = 32;  // fp64 log, warp-register table (log_shfl): one entry per lane
constexpr int kLogTab8 = 64;   // fp64 log, dense TILED: 64 entries replicated 8x (log_tab8, no bank conflicts)

struct NrCarve {
    int sstart, gstart, cnt, toff, pstart, uj0, ut, tslot, tu, tv, part, src, ltab, total, ucap;
};
// NR layout.  src_cap: max padded region sources of a tile (multiple of 4);
// tgt_cap: max targets of a tile (multiple of 4); tpi: targets per work unit
// (1, or 2 = pairs of targets of the same box).
P2P_HD inline int nr_unit_cap(int k, int tgt_cap, int tpi) {
    const int WW = 1 << (2 * k);
    return tpi > 1 ? (((tgt_cap + (tpi - 1) * WW) / tpi + 4) & ~3) : tgt_cap;
}
P2P_HD inline NrCarve nr_carve(int k, int src_cap, int tgt_cap, int e, int tpi) {
    const int W = 1 << k, R = W + 2, RR = R * R, WW = W * W;
    NrCarve c;
    c.ucap = nr_unit_cap(k, tgt_cap, tpi);
    c.sstart = 0;
    c.gstart = c.sstart + 4 * (RR + 1);
    c.cnt = c.gstart + 4 * RR;
    c.toff = c.cnt + 4 * RR;
    c.pstart = c.toff + 4 * (WW + 1);
    c.uj0 = c.pstart + 4 * (WW + 1);
    c.ut = c.uj0 + 4 * c.ucap;                      // unit -> its tpi targets
    c.tslot = c.ut + 4 * tpi * c.ucap;              // target -> slot of its partials
    c.tu = align16(c.tslot + 4 * tgt_cap);
    c.tv = align16(c.tu + e * tgt_cap);
    c.part = align16(c.tv + e * tgt_cap);
    c.src = align16(c.part + 3 * e * tpi * c.ucap);
    c.ltab = align16(c.src + 3 * e * src_cap);  // fp64: the log table
    c.total = c.ltab + (e == 8 ? 16 * kLogTab : 0);
    return c;
}

struct RCarve {
    int toff, hoff, tbx, tu, tv, part, bar, src, ltab, total;
};
// src_cap: max packed-halo entries of a tile (multiple of 4).
P2P_HD inline RCarve r_carve(int k, int src_cap, int tgt_cap, int e) {
    const int W = 1 << k, WW = W * W;
    RCarve c;
    c.toff = 0;
    c.hoff = c.toff + 4 * (WW + 1);
    c.tbx = c.hoff + 4 * (WW + 1);
    c.tu = align16(c.tbx + 4 * tgt_cap);
    c.tv = align16(c.tu + e * tgt_cap);
    c.part = align16(c.tv + e * tgt_cap);
    c.bar = align16(c.part + 3 * e * tgt_cap);
    c.src = align16(c.bar + 16);
    c.ltab = align16(c.src + 3 * e * src_cap);  // fp64: the log table
    c.total = c.ltab + (e == 8 ? 16 * kLogTab : 0);
    return c;
}

struct TCarve {
    int buf0, bufsz;                            // NBUF bulk-copied buffers of bufsz bytes from buf0
    int table, uv, idx, tuv, tbl, oix, items;   // offsets inside one buffer
    int q, part, ltab, bar, total, tstride, icap;
};
// TILED layout.  Per tile record: table (region box starts + slot count), region
// entries (coordinates, source index), target slots (coordinates, row-run base,
// output index) and, for NS = 3 plans, the item list.  src_cap: max region
// entries of a tile (multiple of 4); slot_cap: max target slots of a tile
// (multiple of 8); tpi: slots per unit; ns: items per unit (1, or 3 row-runs).
P2P_HD inline int tiled_table_stride(int k) {
    const int W = 1 << k, R = W + 2;
    return (R * R + 2 + 7) & ~7;  // uint16: region box starts [R*R + 1], then the tile's slot count
}
P2P_HD inline int tiled_item_cap(int slot_cap, int tpi, int ns) {
    return ns == 3 ? (3 * (slot_cap / tpi) + 7) & ~7 : 0;
}
P2P_HD inline TCarve tiled_carve(int k, int src_cap, int slot_cap, int e, int tpi, int ns, int nbuf, int lt8 = 0) {
    TCarve c;
    c.tstride = tiled_table_stride(k);
    c.icap = tiled_item_cap(slot_cap, tpi, ns);
    c.table = 0;
    c.uv = align16(2 * c.tstride);
    c.idx = c.uv + 2 * e * src_cap;
    c.tuv = align16(c.idx + 4 * src_cap);
    c.tbl = c.tuv + 2 * e * slot_cap;
    c.oix = c.tbl + 2 * slot_cap;
    c.items = c.oix + 2 * slot_cap;
    c.bufsz = align16(c.items + 2 * c.icap);
    c.buf0 = 0;
    // weights: fp32 single-buffered records gather q in place over the entry indices (each entry's
    // index is read and its weight written by the same thread; the indices are dead afterwards)
    const bool q_alias = e == 4 && nbuf == 1;
    c.q = q_alias ? c.idx : nbuf * c.bufsz;
    c.part = align16(q_alias ? nbuf * c.bufsz : c.q + e * src_cap);  // NS = 3: three partial sums per slot
    // ns = 1, tpi = 1 (lean): `part` stages the tile's results in output order (coalesced stores)
    // fp64 dense (ns = 3): the log table -- kLogTab entries, or (lt8) 8 x kLogTab8; lean: none (log_shfl)
    c.ltab = align16(c.part + (ns == 3 ? 3 * e * slot_cap : tpi == 1 ? e * slot_cap : 0));
    c.bar = align16(c.ltab + (e == 8 && ns == 3 ? 16 * (lt8 ? 8 * kLogTab8 : kLogTab) : 0));
    c.total = c.bar + 16;
    return c;
}

// TILED Helmholtz kernel: the TILED record buffer, then complex weights (2 values per region
// entry), the fp64 log table and the mbarrier.
struct HCarve {
    TCarve t;
    int q, ltab, bar, total;
};
P2P_HD inline HCarve helm_carve(int k, int src_cap, int slot_cap, int e) {
    HCarve h;
    h.t = tiled_carve(k, src_cap, slot_cap, e, 1, 1, 1);
    h.q = h.t.bufsz;  // complex weights (2 e bytes) after the record buffer (not over the indices)
    h.ltab = align16(h.q + 2 * e * src_cap);
    h.bar = align16(h.ltab + (e == 8 ? 16 * kLogTab : 0));
    h.total = h.bar + 16;
    return h;
}

struct Error : std::runtime_error {
    p2p_status code;
    Error(p2p_status c, const std::string &m) : std::runtime_error(m), code(c) {}
};

constexpr int kMaxLevel = 15;          // full-grid CSR offsets: 4^(L-1) <= 2^28 boxes
constexpr int kMaxLevel3 = 9;          // 3D: 8^(L-1) <= 2^24 boxes
// 3D: threads per CTA (one target box per CTA): 64 for Laplace, 128 for Helmholtz (measured,
// tools/gpu/gpu_ab16.sh)
inline int box3d_threads(int kernel) { return kernel == P2P_KERNEL_HELMHOLTZ_3D ? 128 : 64; }
P2P_HD inline int kernel_dim(int kernel) { return kernel >= P2P_KERNEL_LAPLACE_3D ? 3 : 2; }
// 3D box kernel shared memory: staged sources (x, y, z, q_re) and q_im (complex), per-thread
// partial sums (comps values), and per neighbour box its source start, prefix and shift code.
#ifndef P2P_BOX3_HELM_PAIR
#define P2P_BOX3_HELM_PAIR 1
#endif
// partial sums per thread of the 3D box kernel: fp32 Laplace 2 (two targets), complex 2 (re, im),
// fp32 Helmholtz with two targets per thread 4
P2P_HD inline int box3d_parts(bool helm, int e) {
    return helm ? ((e == 4 && P2P_BOX3_HELM_PAIR) ? 4 : 2) : (e == 4 ? 2 : 1);
}
struct B3Carve {
    int p, qi, part, nbs, pre, nbd, total;
};
// comps: values per weight (2: complex, staged q_im); parts: partial sums per thread
P2P_HD inline B3Carve box3d_carve(int src_cap, int e, int comps, int nt, int parts) {
    B3Carve c;
    c.p = 0;
    c.qi = c.p + 4 * e * src_cap;
    c.part = align16(c.qi + (comps == 2 ? e * src_cap : 0));
    c.nbs = align16(c.part + nt * parts * e);
    c.pre = c.nbs + 4 * 28;
    c.nbd = c.pre + 4 * 28;
    c.total = c.nbd + 4 * 28;
    return c;
}
inline int64_t box3d_smem(int64_t src_cap, int e, int comps, int nt, int parts) {
    if (src_cap > (1 << 20)) return int64_t(1) << 40;
    return box3d_carve((int)src_cap, e, comps, nt, parts).total;
}
constexpr int kThreads = 256;          // CTA size of the P2P kernels
constexpr int kMaxTileLog2 = 6;
constexpr int64_t kSmemLimit = 200 * 1024;
#ifndef P2P_SPLIT_SHARE
#define P2P_SPLIT_SHARE (148 * 8)
#endif
constexpr int64_t kSplitShare = P2P_SPLIT_SHARE;  // TILED: a tile above 1/1184 of the pairs is split (heavy tiles)
constexpr int64_t kSplitMax = 32;         // at most 32 launch entries per tile
// Launch entries of a tile with `tile_pairs` pairs: ceil(tile_pairs / share) (<= 32), at least `base`.
P2P_HD inline int64_t split_parts(int64_t tile_pairs, int64_t share, int64_t base) {
    int64_t p = (tile_pairs + share - 1) / share;
    p = p > kSplitMax ? kSplitMax : p;
    return p > base ? p : base;
}

// ---- Morton (Z-order) codes: x in the even bits, y in the odd bits
// ("the order of the boxes' morton index").
inline uint32_t spread16(uint32_t v) {
    v &= 0x0000FFFFu;
    v = (v | (v << 8)) & 0x00FF00FFu;
    v = (v | (v << 4)) & 0x0F0F0F0Fu;
    v = (v | (v << 2)) & 0x33333333u;
    v = (v | (v << 1)) & 0x55555555u;
    return v;
}
inline uint32_t compact16(uint32_t v) {
    v &= 0x55555555u;
    v = (v | (v >> 1)) & 0x33333333u;
    v = (v | (v >> 2)) & 0x0F0F0F0Fu;
    v = (v | (v >> 4)) & 0x00FF00FFu;
    v = (v | (v >> 8)) & 0x0000FFFFu;
    return v;
}
inline uint32_t morton_encode(uint32_t ix, uint32_t iy) { return spread16(ix) | (spread16(iy) << 1); }
inline void morton_decode(uint32_t m, uint32_t &ix, uint32_t &iy) {
    ix = compact16(m);
    iy = compact16(m >> 1);
}

// Precision-specific device layout, built on the host.
template <typename T>
struct Layout {
    std::vector<T> src_uv;   // [n_src_local][2] box-local coordinates (x - ix*h, y - iy*h)
    std::vector<T> tgt_uv;   // [n_tgt_local][2]
    std::vector<T> halo_uv;  // R: fp32 -> per source pair (u0,u1,v0,v1); fp64 -> (u,v) per entry
    std::vector<T> reg_uv;   // TILED: region-relative, same pair packing as halo_uv
    std::vector<T> tgt_ruv;  // TILED: per-tile packed targets, coordinates relative to the region origin
};

struct HostPlan {
    // ---- parameters
    int L = 0, k = 0, layout = 0, precision = 0, device = -1;
    int kernel = P2P_KERNEL_LAPLACE_2D;          // p2p_kernel
    int dim = 2;                                 // 3 for the 3D kernels (octree leaf grid)
    bool warp_leaf = false;                      // ADAPTIVE: one warp per target leaf (small leaves)
    double kappa = 0.0;                          // HELMHOLTZ_2D wavenumber
    int part_world = 1, part_rank = 0;
    int64_t S = 0, B = 0;        // grid side, number of leaf boxes
    double h = 0.0, eps = 1e-12;
    int64_t n_src = 0, n_tgt = 0;

    // ---- global indexing (bit-exact exports)
    std::vector<int32_t> src_off_g, tgt_off_g;    // [B+1] CSR offsets in Morton order
    std::vector<int32_t> src_perm_g, tgt_perm_g;  // global plan index -> user index

    // ---- tiles and partition
    std::vector<int32_t> tiles_g;                 // non-empty tiles (Morton tile index), ascending
    std::vector<int64_t> tile_pairs_g;            // pairs per non-empty tile
    std::vector<int64_t> part_tile;               // [W+1] cut indices into tiles_g
    std::vector<int64_t> part_src, part_tgt;      // [W+1] global plan index cuts
    std::vector<int32_t> tiles;                   // this partition's tiles (launch order)

    // ---- local (this partition) indexing
    std::vector<int32_t> src_off, tgt_off;        // [B+1] local CSR offsets
    std::vector<int32_t> src_gidx;                // local source -> global plan index
    std::vector<int32_t> src_uidx;                // local source -> user index
    std::vector<int32_t> tgt_uidx;                // local target -> user index
    std::vector<int32_t> src_qidx;                // local source -> index into [owned | halo]
    std::vector<int32_t> halo_lidx;               // local index of each halo source, in halo-slot order
    int64_t owned_local_begin = 0;                // owned sources = local indices [begin, begin + n_src_owned)
    int64_t n_interior = 0;                       // TILED: launch entries [0, n_interior) read owned sources only
    int64_t n_src_local = 0, n_tgt_local = 0, n_src_owned = 0, n_halo = 0, n_send = 0;
    int64_t src_owned_begin = 0, tgt_begin = 0;
    std::vector<int64_t> recv_counts, send_counts;  // [W]
    std::vector<int32_t> send_idx;                  // owned-local index per sent weight

    // ---- R layout
    std::vector<uint32_t> halo_off;               // [B+1]
    std::vector<int32_t> halo_idx;                // local source index, -1 = pad
    int64_t halo_entries = 0;

    // ---- TILED layout (per tile in Morton order = "slot")
    std::vector<uint32_t> reg_off;                // [tiles+1] packed-region offsets
    std::vector<int32_t> reg_idx;                 // local source index, -1 = pad
    std::vector<int32_t> reg_uidx;                // user (original) source index, -1 = pad: ORDER_USER applies
    std::vector<uint16_t> reg_table;              // [tiles][tstride] region box starts, then the slot count
    std::vector<uint16_t> tgt_bl;                 // per target slot: row-run base j0 = by * R + bx
    std::vector<uint16_t> tgt_oix;                // per target slot: tile-local output index (0xFFFF: duplicate)
    std::vector<uint32_t> tgt_pack_off;           // [tiles+1] target-slot offsets (multiples of 8)
    std::vector<uint32_t> item_off;               // NS = 3: [tiles+1] item-list offsets (multiples of 8)
    std::vector<uint16_t> items;                  // NS = 3: unit << 2 | row, sorted by row-run length per part
    std::vector<int32_t> tile_tgt_base;           // [tiles] plan index of each tile's first target
    int ns = 3;                                   // TILED work segments per target
    int nbuf = 1;                                 // TILED record buffers (2 = prefetch next tile)
    bool pad = true;                              // TILED: boxes padded to even counts (packed f32x2 loops)
    int nt = 256;                                 // threads per CTA (TILED: 128 or 256)
    bool lean = false;                            // TILED lean kernel path (tpi 1, ns 1, unpadded)
    bool tsort = false;                           // ns 1: target boxes of a tile ordered by n9 (descending)
    bool flat = false;                            // lean path: row-runs swept as one sequence (sparse)
    bool lt8 = false;                             // dense fp64: the 8-fold 64-entry log table (log_tab8)
    std::vector<double> log_tab;                  // fp64: kLogTab x (c_inv, -log c_inv) for the table-driven log

    // ---- the paper's layouts (PAPER_INDEXING / PAPER_REPETITION)
    std::vector<int32_t> pi_nei_off, pi_nei_idx;  // per box (Morton): its E1 sources' original indices
    std::vector<double> pi_src_xy, pi_tgt_xy;     // coordinates in the caller's order
    std::vector<double> pr_records;               // n_tgt x pr_stride doubles, caller's target order
    std::vector<int32_t> pr_slot;                 // n_tgt x pr_maxn: original source index per triple, -1 = none
    int64_t pr_stride = 0, pr_maxn = 0, paper_model_bytes = 0;
    // ---- ADAPTIVE (NEXT-4): leaves in Morton order, U-lists over leaves (CSR)
    std::vector<int32_t> leaf_lvl, leaf_ix, leaf_iy;   // per leaf
    std::vector<int32_t> leaf_s0, leaf_s1, leaf_t0, leaf_t1;  // source / target ranges (plan order)
    std::vector<int32_t> ul_off, ul_leaf;              // [leaves+1], U-list leaf indices (ascending)
    std::vector<int32_t> pt_cell_s, pt_cell_t;         // per point: finest-grid cell (x, y) pairs
    std::vector<int32_t> tile_slot;               // launch order -> slot
    std::vector<int32_t> tile_part;               // launch order -> part | nparts << 16 (tail splitting)
    int64_t reg_entries = 0;
    int64_t table_entries = 0;                    // TILED: uint16 entries of the region tables (tiles x stride)
    bool device_built = false;                    // built by the device builder (p2p_plan_create_device)
    bool local_input = false;                     // built from this rank's points only (p2p_plan_create_local)

    Layout<float> f32;
    Layout<double> f64;

    // ---- statistics
    int64_t pairs = 0, pairs_global = 0, t_max = 0, occ_src = 0, occ_tgt = 0;
    int64_t boxes_in_tiles = 0, max_region = 0, max_tile_halo = 0, smem_bytes = 0;
    int64_t src_cap = 0, tgt_cap = 0;            // kernel smem capacities (multiples of 4)
    int group_log2 = 0;                          // NR staging lanes per region box (log2)
    int tpi = 1;                                 // targets per work unit (2 for dense fp32 NR)
    bool lpt = false;                            // tiles queued by decreasing pairs (working set fits L2)
    double density = 0.0, density_occ = 0.0, build_seconds = 0.0;
};

// Per-tile maxima at a candidate tile size (the inputs of the kernel-option choice).
struct TileStats {
    int64_t ntiles = 0;          // non-empty tiles
    int64_t max_region_pad = 0;  // region (tile + ring) sources, boxes padded to even counts
    int64_t max_region = 0;      // region sources, unpadded
    int64_t max_tile_halo = 0;   // R layout: packed halo entries of a tile
    int64_t max_tcount = 0;      // targets of a tile
    int64_t max_tcount2 = 0;     // target slots of a tile with 2-slot units (odd boxes padded)
};
// Kernel options (tpi, pad, ns, nt, lean, tsort, flat, caps) and shared memory per CTA at tile
// size k; used by both builders so they take the same decisions.  Returns hp.smem_bytes.
int64_t choose_tile_params(const p2p_plan_desc &d, HostPlan &hp, int k, const TileStats &st);
void check_kernel(const p2p_plan_desc &d);  // kernel function + envelope (throws Error)

// Local-input partitioned plans (p2p_plan_create_local / p2p_partition_route): this rank passes
// only the points it holds (with their global ids) and the GLOBAL per-box point counts; the
// partition, tile choice and global plan indices follow from the counts alone, so the plan is
// the one the global-input builder makes for this rank (bit-identical applies).
struct LocalInput {
    const int64_t *src_ids = nullptr, *tgt_ids = nullptr;        // global ids of the passed points
    const int32_t *src_counts = nullptr, *tgt_counts = nullptr;  // [4^(L-1)] global counts, Morton order
    int64_t n_src_global = 0, n_tgt_global = 0;
    // route-only mode: stop after the partition and write, per passed point, the bit mask of the
    // ranks that need it (sources: the owner of its box + every rank with an owned tile whose
    // region holds the box; targets: the owner of its box)
    uint32_t *src_mask = nullptr, *tgt_mask = nullptr;
};
void build_host_plan(const p2p_plan_desc &desc, HostPlan &hp, const LocalInput *li = nullptr);
void box_counts(int level, int64_t n, const double *xy, int32_t *counts);  // [4^(L-1)] per-box counts
void build_host_plan_3d(const p2p_plan_desc &desc, HostPlan &hp);
void build_host_plan_adaptive(const p2p_plan_desc &desc, HostPlan &hp);
// ADAPTIVE kernel shared memory: staged sources (x, y, q) relative to the target leaf, the
// U-list source starts and prefix (up to kMaxUlist leaves), partial sums per thread.
constexpr int kMaxUlist = 256;
constexpr int kAdaptiveThreads = 64;
// ADAPTIVE warp-per-leaf kernel: one slice per warp (staged sources, U-list starts / prefix, partials)
P2P_HD inline int adaptive_warp_slice(int src_cap, int e) {
    return align16(src_cap * 4 * e) + 8 * kMaxUlist + 16 + align16(32 * e);
}
inline int64_t adaptive_smem(int64_t src_cap, int e) {
    return ((src_cap * 4 * e + 15) & ~int64_t(15)) + 8 * kMaxUlist + 16 + kAdaptiveThreads * e + 16;
}
void build_log_table(HostPlan &hp);
std::vector<int64_t> neighbors_export(const HostPlan &hp);

}  // namespace p2p
