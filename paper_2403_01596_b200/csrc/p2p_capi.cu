// p2p_capi.cu -- implementation of include/p2p.h: plan lifecycle, device
// upload, apply dispatch, introspection and export.
#include <algorithm>
#include <chrono>
#include <cstddef>
#include <cmath>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges cost nothing unless a profiler attaches

#include "p2p.h"
#include "p2p_kernels.cuh"
#include "plan.h"
#include "plan_device.cuh"

namespace {

thread_local std::string g_last_error;

p2p_status set_error(p2p_status s, const std::string &msg) {
    g_last_error = msg;
    return s;
}

struct CudaError : p2p::Error {
    CudaError(const std::string &m) : p2p::Error(P2P_ERROR_CUDA, m) {}
};

void ck(cudaError_t e, const char *what) {
    if (e != cudaSuccess) {
        if (e == cudaErrorMemoryAllocation) throw p2p::Error(P2P_ERROR_OUT_OF_MEMORY, std::string(what) + ": out of device memory");
        throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
    }
}

struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
};

// NVTX range over one ABI call / phase (nsys and ncu timelines: plan, exchange, interior,
// boundary, gather)
struct Nvtx {
    explicit Nvtx(const char *name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
};

}  // namespace

struct p2p_plan_s {
    p2p::HostPlan hp;
    int device = -1;
    cudaStream_t stream = nullptr;
    // device arrays
    DevBuf pi_src_xy, pi_tgt_xy, pi_nei_off, pi_nei_idx, pr_records, pr_slot, phi_user, paper_q, halo_lidx, tiles, src_off, tgt_off, src_uv, tgt_uv, src_gidx, src_uidx, tgt_uidx, send_idx;
    DevBuf halo_off, halo_idx, halo_uv, halo_q;
    DevBuf tile_slot, tile_part, reg_off, reg_idx, reg_uidx, reg_uv, reg_table, tgt_bl, tgt_oix, item_off, items, log_tab, tgt_ruv, tgt_pack_off, tile_tgt_base;
    DevBuf q_local, phi, io_q, io_out, queue;  // workspace (the active slot's buffers)
    // p2p_plan_set_workspaces: n workspace slots rotated over p2p_apply / p2p_apply_host* so up
    // to n applies of one plan can be in flight on different streams; each apply waits (device
    // side, an event) for the apply that last used its slot.  Empty = one slot, the fields above.
    struct Workspace {
        DevBuf q_local, phi, io_q, io_out, queue;
        cudaEvent_t done = nullptr;
    };
    std::vector<Workspace> ws;
    size_t ws_next = 0;
    DevBuf leaf_rng, leaf_org, ul_off, ul_leaf, src_cell, tgt_cell;  // ADAPTIVE (NEXT-4)
    DevBuf halo_owner, halo_oidx;                // peer-memory halo: owner rank, owner-local index per halo slot
    struct PeerSync {                            // device-synchronised peer exchange (p2p_apply_peer_sync, p2p_gather)
        DevBuf pub_w, pub_o, sig, ctr, err, oidx_w, seg_o;
        void *pub_w_peer[16] = {}, *pub_o_peer[16] = {}, *sig_peer[16] = {};
        unsigned readers_w = 0, owners_w = 0, all = 0;
        bool connected = false;
        cudaStream_t side = nullptr;
        cudaEvent_t ev_pub = nullptr, ev_pull = nullptr;
    } peer;
    int grid = 0;                                // persistent CTAs per launch
    int64_t occ_sms = 1;                         // resident CTAs per SM x SMs (grid cap of a launch)
    unsigned long long *trace = nullptr;         // diagnostics: per-tile timeline buffer (device)
    int64_t device_bytes = 0;
    double upload_seconds = 0.0;
    bool paper_kernel_only = false;              // diagnostics: PAPER_REPETITION applies skip the weight pack
    int elem = 4;
    int comps = 1;                               // values per weight / result (2: complex, HELMHOLTZ_2D)

    template <typename V>
    void upload(DevBuf &b, const std::vector<V> &v) {
        b.bytes = v.size() * sizeof(V);
        if (!b.bytes) return;
        ck(cudaMalloc(&b.p, b.bytes), "cudaMalloc");
        device_bytes += (int64_t)b.bytes;
        ck(cudaMemcpyAsync(b.p, v.data(), b.bytes, cudaMemcpyHostToDevice, stream), "cudaMemcpyAsync H2D");
    }
    void alloc(DevBuf &b, size_t bytes) {
        b.bytes = bytes;
        if (!bytes) return;
        ck(cudaMalloc(&b.p, bytes), "cudaMalloc");
        device_bytes += (int64_t)bytes;
    }
    void release() {
        if (!ws.empty()) {  // the fields alias one slot: free the slots, then forget the aliases
            for (Workspace &w : ws) {
                for (DevBuf *b : {&w.q_local, &w.phi, &w.io_q, &w.io_out, &w.queue})
                    if (b->p) cudaFree(b->p);
                if (w.done) cudaEventDestroy(w.done);
            }
            ws.clear();
            q_local = phi = io_q = io_out = queue = DevBuf{};
        }
        DevBuf *all[] = {&pi_src_xy, &pi_tgt_xy, &pi_nei_off, &pi_nei_idx, &pr_records, &pr_slot, &phi_user, &paper_q, &halo_lidx, &tiles, &src_off, &tgt_off, &src_uv, &tgt_uv, &src_gidx, &src_uidx, &tgt_uidx,
                         &send_idx, &halo_off, &halo_idx, &halo_uv, &halo_q,
                         &tile_slot, &tile_part, &reg_off, &reg_idx, &reg_uidx, &reg_uv, &reg_table, &tgt_bl, &tgt_oix, &item_off, &items, &log_tab, &tgt_ruv,
                         &tgt_pack_off, &tile_tgt_base, &q_local, &phi, &leaf_rng, &leaf_org, &ul_off, &ul_leaf,
                         &src_cell, &tgt_cell, &halo_owner, &halo_oidx,
                         &io_q, &io_out, &queue, &peer.pub_w, &peer.pub_o, &peer.sig, &peer.ctr, &peer.err,
                         &peer.oidx_w, &peer.seg_o};
        if (peer.ev_pub) cudaEventDestroy(peer.ev_pub);
        if (peer.ev_pull) cudaEventDestroy(peer.ev_pull);
        if (peer.side) cudaStreamDestroy(peer.side);
        peer.ev_pub = peer.ev_pull = nullptr;
        peer.side = nullptr;
        peer.connected = false;
        for (DevBuf *b : all) {
            if (b->p) cudaFree(b->p);
            b->p = nullptr;
            b->bytes = 0;
        }
    }
};

namespace {

template <typename T>
const p2p::Layout<T> &layout_of(const p2p::HostPlan &hp);
template <>
const p2p::Layout<float> &layout_of<float>(const p2p::HostPlan &hp) { return hp.f32; }
template <>
const p2p::Layout<double> &layout_of<double>(const p2p::HostPlan &hp) { return hp.f64; }

// TILED kernel instance for the plan's options (element type, targets per unit, CTA size, padding).
template <typename T, int TPI, bool PAD, int NS>
const void *tiled_fn_nt(int nt) {
    using namespace p2p::dev;
    if constexpr (TPI == 1 && !PAD && NS == 1)  // lean path: one-warp CTAs as well
        if (nt == 32) return (const void *)p2p_tiled_kernel<T, TPI, 32, PAD, NS>;
    switch (nt) {
    case 64: return (const void *)p2p_tiled_kernel<T, TPI, 64, PAD, NS>;
    case 128: return (const void *)p2p_tiled_kernel<T, TPI, 128, PAD, NS>;
    default: return (const void *)p2p_tiled_kernel<T, TPI, 256, PAD, NS>;
    }
}

// TILED kernel instance for the plan's options (element type, slots per unit, CTA size, padding,
// items per unit).  Defaults: dense fp32 (2 slots/unit, padded, 3 row items), sparse fp32 and
// fp64 (1 slot/unit, unpadded, whole-unit items = the lean path); the rest are tuning variants.
template <typename T>
const void *tiled_fn(int tpi, int nt, bool pad, int ns) {
    if constexpr (sizeof(T) == 4) {
        if (tpi == 2) return ns == 3 ? tiled_fn_nt<float, 2, true, 3>(nt) : tiled_fn_nt<float, 2, true, 1>(nt);
        if (pad) return ns == 3 ? tiled_fn_nt<float, 1, true, 3>(nt) : tiled_fn_nt<float, 1, true, 1>(nt);
        return ns == 3 ? tiled_fn_nt<float, 1, false, 3>(nt) : tiled_fn_nt<float, 1, false, 1>(nt);
    } else {
        if (tpi == 2) return tiled_fn_nt<double, 2, false, 3>(nt);  // dense fp64, two targets per unit
        return ns == 3 ? tiled_fn_nt<double, 1, false, 3>(nt) : tiled_fn_nt<double, 1, false, 1>(nt);
    }
}

template <typename T>
void finalize_plan(p2p_plan_s &P);

template <typename T>
const void *box3d_fn(bool helm) {  // CTA sizes of p2p::box3d_threads
    return helm ? (const void *)p2p::dev::p2p_box3d_kernel<T, true, 128>
                : (const void *)p2p::dev::p2p_box3d_kernel<T, false, 64>;
}

template <typename T>
const void *helm_fn(int nt) {
    using namespace p2p::dev;
    switch (nt) {
    case 32: return (const void *)p2p_tiled_helm_kernel<T, 32>;
    case 64: return (const void *)p2p_tiled_helm_kernel<T, 64>;
    case 256: return (const void *)p2p_tiled_helm_kernel<T, 256>;
    default: return (const void *)p2p_tiled_helm_kernel<T, 128>;
    }
}

template <typename T>
void upload_plan(p2p_plan_s &P) {
    const p2p::HostPlan &hp = P.hp;
    const p2p::Layout<T> &lay = layout_of<T>(hp);
    P.upload(P.tiles, hp.tiles);
    P.upload(P.tgt_off, hp.tgt_off);
    P.upload(P.tgt_uv, lay.tgt_uv);
    P.upload(P.tgt_uidx, hp.tgt_uidx);
    P.upload(P.src_uidx, hp.src_uidx);
    P.upload(P.log_tab, hp.log_tab);  // fp64 plans
    if (hp.part_world > 1) {
        P.upload(P.src_gidx, hp.src_gidx);
        P.upload(P.halo_lidx, hp.halo_lidx);
        P.upload(P.send_idx, hp.send_idx);
        // peer-memory halo: owner rank and owner-local index of each halo slot (the owner of a
        // global plan index is the last rank whose source range starts at or before it)
        std::vector<int32_t> own(hp.halo_lidx.size()), oix(hp.halo_lidx.size());
        for (size_t h = 0; h < hp.halo_lidx.size(); ++h) {
            const int64_t g = hp.src_gidx[hp.halo_lidx[h]];
            const int r = (int)(std::upper_bound(hp.part_src.begin(), hp.part_src.end(), g) - hp.part_src.begin()) - 1;
            own[h] = r;
            oix[h] = (int32_t)(g - hp.part_src[r]);
        }
        P.upload(P.halo_owner, own);
        P.upload(P.halo_oidx, oix);
    }
    if (hp.layout == P2P_LAYOUT_PAPER_INDEXING) {
        P.upload(P.pi_src_xy, hp.pi_src_xy);
        P.upload(P.pi_tgt_xy, hp.pi_tgt_xy);
        P.upload(P.pi_nei_off, hp.pi_nei_off);
        P.upload(P.pi_nei_idx, hp.pi_nei_idx);
    } else if (hp.layout == P2P_LAYOUT_PAPER_REPETITION) {
        P.upload(P.pr_records, hp.pr_records);
        P.upload(P.pr_slot, hp.pr_slot);
    } else if (hp.layout == P2P_LAYOUT_ADAPTIVE) {
        const size_t nl = hp.leaf_lvl.size();
        std::vector<int32_t> rng(4 * nl), org(2 * nl);
        for (size_t i = 0; i < nl; ++i) {
            rng[4 * i] = hp.leaf_s0[i];
            rng[4 * i + 1] = hp.leaf_s1[i];
            rng[4 * i + 2] = hp.leaf_t0[i];
            rng[4 * i + 3] = hp.leaf_t1[i];
            const int sz = 1 << (hp.L - hp.leaf_lvl[i]);
            org[2 * i] = hp.leaf_ix[i] * sz;
            org[2 * i + 1] = hp.leaf_iy[i] * sz;
        }
        P.upload(P.leaf_rng, rng);
        P.upload(P.leaf_org, org);
        P.upload(P.ul_off, hp.ul_off);
        P.upload(P.ul_leaf, hp.ul_leaf);
        P.upload(P.src_cell, hp.pt_cell_s);
        P.upload(P.tgt_cell, hp.pt_cell_t);
        P.upload(P.src_uv, lay.src_uv);
    } else if (hp.layout == P2P_LAYOUT_NONREDUNDANT) {
        P.upload(P.src_off, hp.src_off);
        P.upload(P.src_uv, lay.src_uv);
    } else if (hp.layout == P2P_LAYOUT_TILED) {
        P.upload(P.tile_slot, hp.tile_slot);
        P.upload(P.tile_part, hp.tile_part);
        P.upload(P.reg_off, hp.reg_off);
        P.upload(P.reg_idx, hp.reg_idx);
        P.upload(P.reg_uidx, hp.reg_uidx);
        P.upload(P.reg_uv, lay.reg_uv);
        P.upload(P.reg_table, hp.reg_table);
        P.upload(P.tgt_bl, hp.tgt_bl);
        P.upload(P.tgt_oix, hp.tgt_oix);
        P.upload(P.item_off, hp.item_off);
        P.upload(P.items, hp.items);
        P.upload(P.tgt_ruv, lay.tgt_ruv);
        P.upload(P.tgt_pack_off, hp.tgt_pack_off);
        P.upload(P.tile_tgt_base, hp.tile_tgt_base);
    } else {
        P.upload(P.halo_off, hp.halo_off);
        P.upload(P.halo_idx, hp.halo_idx);
        P.upload(P.halo_uv, lay.halo_uv);
        P.alloc(P.halo_q, (size_t)hp.halo_entries * sizeof(T));
    }
    finalize_plan<T>(P);
}

// Kernel attributes, persistent grid size and apply workspace of a plan whose layout is on the device.
template <typename T>
void finalize_plan(p2p_plan_s &P) {
    const p2p::HostPlan &hp = P.hp;
    // Dynamic shared memory is fixed per plan: opt in once (a permission, not a
    // reservation, so one value serves all plans), then size the persistent grid.
    const bool two = hp.tpi == 2;
    const void *kfn = hp.layout == P2P_LAYOUT_ADAPTIVE
                          ? (hp.warp_leaf ? (const void *)p2p::dev::p2p_adaptive_warp_kernel<T, 128>
                                          : (const void *)p2p::dev::p2p_adaptive_kernel<T, p2p::kAdaptiveThreads>)
                      : hp.dim == 3 ? box3d_fn<T>(hp.kernel == P2P_KERNEL_HELMHOLTZ_3D)
                      : hp.kernel == P2P_KERNEL_HELMHOLTZ_2D ? helm_fn<T>(hp.nt)
                      : hp.layout == P2P_LAYOUT_REDUNDANT ? (const void *)p2p::dev::p2p_r_kernel<T>
                      : hp.layout == P2P_LAYOUT_TILED
                          ? tiled_fn<T>(hp.tpi, hp.nt, hp.pad, hp.ns)
                          : (two ? (const void *)p2p::dev::p2p_nr_kernel<T, sizeof(T) == 4 ? 2 : 1>
                                 : (const void *)p2p::dev::p2p_nr_kernel<T, 1>);
    ck(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p2p::kSmemLimit), "smem attr");
    int occ = 0, dev = 0, sms = 0;
    const int block = hp.nt;
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, block, (size_t)hp.smem_bytes), "occupancy");
    ck(cudaGetDevice(&dev), "cudaGetDevice");
    ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "SM count");
    P.occ_sms = (int64_t)std::max(occ, 1) * sms;
    P.grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)hp.tiles.size(), P.occ_sms));
    P.alloc(P.queue, 16);
    ck(cudaMemsetAsync(P.queue.p, 0, 16, P.stream), "queue init");  // kernels reset it on exit
    ck(cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared),
       "carveout");
    const size_t cs = (size_t)P.comps * sizeof(T);  // bytes per weight / result
    P.alloc(P.q_local, (size_t)std::max<int64_t>(hp.n_src_local, 1) * cs);
    P.alloc(P.phi, (size_t)std::max<int64_t>(hp.n_tgt_local, 1) * cs);
    P.alloc(P.io_q, (size_t)std::max<int64_t>(hp.n_src, 1) * cs);
    P.alloc(P.io_out, (size_t)std::max<int64_t>(hp.n_tgt, 1) * cs);
}

int grid_for(int64_t n) {
    int64_t g = (n + 255) / 256;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16));
}

// The P2P kernel proper on q_local (local plan order) -> out (local plan order).
template <typename T>
void launch_p2p(p2p_plan_s &P, const T *q_local, T *out, int accumulate, cudaStream_t s, bool user = false,
                int64_t e0 = 0, int64_t e1 = -1) {
    const p2p::HostPlan &hp = P.hp;
    // TILED: launch entries [e0, e1) of the queue (interior / boundary phases); NR, R: all tiles
    if (e1 < 0 || hp.layout != P2P_LAYOUT_TILED) {
        e0 = 0;
        e1 = (int64_t)hp.tiles.size();
    }
    const int ntiles = (int)(e1 - e0);
    if (ntiles <= 0) return;
    p2p::dev::P2PArgs<T> a{};
    a.tiles = (const int32_t *)P.tiles.p;
    a.ntiles = ntiles;
    a.queue = (int *)P.queue.p;
    a.k = hp.k;
    a.S = hp.S;
    a.h = (T)hp.h;
    a.eps2 = (T)(hp.eps * hp.eps);
    a.log_tab = (const double2 *)P.log_tab.p;
    a.src_cap = (int)hp.src_cap;
    a.tgt_cap = (int)hp.tgt_cap;
    a.group_log2 = hp.group_log2;
    a.tgt_off = (const int32_t *)P.tgt_off.p;
    a.tgt_uv = (const typename p2p::dev::V2<T>::type *)P.tgt_uv.p;
    a.out = out;
    a.accumulate = accumulate;
    a.trace = P.trace;
    if (hp.layout == P2P_LAYOUT_NONREDUNDANT) {
        a.src_off = (const int32_t *)P.src_off.p;
        a.src_uv = (const typename p2p::dev::V2<T>::type *)P.src_uv.p;
        a.q = q_local;
        if (hp.tpi == 2)
            p2p::dev::p2p_nr_kernel<T, sizeof(T) == 4 ? 2 : 1><<<P.grid, p2p::kThreads, hp.smem_bytes, s>>>(a);
        else
            p2p::dev::p2p_nr_kernel<T, 1><<<P.grid, p2p::kThreads, hp.smem_bytes, s>>>(a);
    } else if (hp.layout == P2P_LAYOUT_TILED) {
        a.q = q_local;
        a.tile_slot = (const int32_t *)P.tile_slot.p + e0;
        a.tile_part = (const int32_t *)P.tile_part.p + e0;
        a.trace = P.trace ? P.trace + 8 * e0 : nullptr;
        a.reg_off = (const uint32_t *)P.reg_off.p;
        // ORDER_USER (TILED): weights gathered through the entries' user indices and results written
        // through the targets' user indices, inside the kernel (no permutation kernels)
        a.reg_idx = (const int32_t *)(user ? P.reg_uidx.p : P.reg_idx.p);
        a.out_idx = user ? (const int32_t *)P.tgt_uidx.p : nullptr;
        a.reg_uv = (const T *)P.reg_uv.p;
        a.reg_table = (const uint16_t *)P.reg_table.p;
        a.tgt_bl = (const uint16_t *)P.tgt_bl.p;
        a.tgt_oix = (const uint16_t *)P.tgt_oix.p;
        a.item_off = (const uint32_t *)P.item_off.p;
        a.items = (const uint16_t *)P.items.p;
        a.tgt_ruv = (const T *)P.tgt_ruv.p;
        a.tgt_pack_off = (const uint32_t *)P.tgt_pack_off.p;
        a.tile_tgt_base = (const int32_t *)P.tile_tgt_base.p;
        a.ns = hp.ns;
        a.flat = hp.flat ? 1 : 0;
        a.lt8 = hp.lt8 ? 1 : 0;
        a.nbuf = hp.nbuf;
        a.kappa = (T)hp.kappa;
        void *args[] = {&a};
        const int grid = (int)std::min<int64_t>(ntiles, P.occ_sms);
        const void *fn = hp.kernel == P2P_KERNEL_HELMHOLTZ_2D ? helm_fn<T>(hp.nt)
                                                              : tiled_fn<T>(hp.tpi, hp.nt, hp.pad, hp.ns);
        ck(cudaLaunchKernel(fn, dim3(grid), dim3(hp.nt), args, (size_t)hp.smem_bytes, s), "tiled launch");
    } else {
        if (hp.halo_entries > 0)
            p2p::dev::pack_r_kernel<T><<<grid_for(hp.halo_entries), 256, 0, s>>>(
                (const int32_t *)P.halo_idx.p, q_local, (T *)P.halo_q.p, hp.halo_entries);
        a.halo_off = (const uint32_t *)P.halo_off.p;
        a.halo_uv = (const T *)P.halo_uv.p;
        a.q = (const T *)P.halo_q.p;
        p2p::dev::p2p_r_kernel<T><<<P.grid, p2p::kThreads, hp.smem_bytes, s>>>(a);
    }
    ck(cudaGetLastError(), "kernel launch");
}

// The paper's kernels (NEXT-1): native order is the caller's (their arrays index original
// points); plan-order weights are scattered to caller's order first and the potentials gathered
// back (no accumulate then).
void apply_paper(p2p_plan_s &P, const void *d_q, void *d_out, int order, int accumulate, cudaStream_t s) {
    const p2p::HostPlan &hp = P.hp;
    if (order == P2P_ORDER_PLAN && accumulate)
        throw p2p::Error(P2P_ERROR_NOT_SUPPORTED, "the paper's layouts: accumulate needs P2P_ORDER_USER");
    const double *q = (const double *)d_q;
    double *out = (double *)d_out;
    if (order == P2P_ORDER_PLAN) {
        // scatter into a buffer of its own: d_q may be io_q itself (p2p_apply_host, plan order)
        if (!P.paper_q.p) P.alloc(P.paper_q, (size_t)std::max<int64_t>(hp.n_src, 1) * sizeof(double));
        if (hp.n_src)
            p2p::dev::scatter_kernel<double><<<grid_for(hp.n_src), 256, 0, s>>>(
                (const int32_t *)P.src_uidx.p, (const double *)d_q, (double *)P.paper_q.p, hp.n_src, 0);
        if (!P.phi_user.p) P.alloc(P.phi_user, (size_t)std::max<int64_t>(hp.n_tgt, 1) * sizeof(double));
        q = (const double *)P.paper_q.p;
        out = (double *)P.phi_user.p;
    }
    const double eps2 = hp.eps * hp.eps;
    if (hp.layout == P2P_LAYOUT_PAPER_INDEXING) {
        if (hp.B)
            p2p::dev::paper_indexing_kernel<<<(unsigned)((hp.B + 255) / 256), 256, 0, s>>>(
                hp.B, (const int32_t *)P.tgt_off.p, (const int32_t *)P.tgt_uidx.p, (const int32_t *)P.pi_nei_off.p,
                (const int32_t *)P.pi_nei_idx.p, (const double2 *)P.pi_src_xy.p, (const double2 *)P.pi_tgt_xy.p, q,
                out, eps2, accumulate);
    } else {
        if (!P.paper_kernel_only && hp.n_tgt)
            p2p::dev::paper_rep_pack_kernel<<<grid_for(hp.n_tgt * hp.pr_maxn), 256, 0, s>>>(
                hp.n_tgt, hp.pr_maxn, hp.pr_stride, (const int32_t *)P.pr_slot.p, q, (double *)P.pr_records.p);
        if (hp.n_tgt)
            p2p::dev::paper_repetition_kernel<<<(unsigned)((hp.n_tgt + 255) / 256), 256, 0, s>>>(
                hp.n_tgt, hp.pr_stride, (const double *)P.pr_records.p, out, eps2, accumulate);
    }
    if (order == P2P_ORDER_PLAN && hp.n_tgt)
        p2p::dev::gather_kernel<double><<<grid_for(hp.n_tgt), 256, 0, s>>>(
            (const int32_t *)P.tgt_uidx.p, (const double *)P.phi_user.p, (double *)d_out, hp.n_tgt);
    ck(cudaGetLastError(), "paper apply launch");
}

// 3D kernels (NEXT-3): one CTA per target box; user order fused (weights gathered through the
// sources' user indices while staging, results written through the targets' user indices).
template <typename T>
void launch_box3d(p2p_plan_s &P, const T *q, T *out, bool user, int accumulate, cudaStream_t s) {
    const p2p::HostPlan &hp = P.hp;
    const int ntiles = (int)hp.tiles.size();
    if (ntiles <= 0) return;
    p2p::dev::P2PArgs<T> a{};
    a.tiles = (const int32_t *)P.tiles.p;
    a.ntiles = ntiles;
    a.queue = (int *)P.queue.p;
    a.S = hp.S;
    a.src_cap = (int)hp.src_cap;
    a.src_off = (const int32_t *)P.src_off.p;
    a.tgt_off = (const int32_t *)P.tgt_off.p;
    a.src_p4 = (const T *)P.src_uv.p;
    a.tgt_p4 = (const T *)P.tgt_uv.p;
    a.src_idx = user ? (const int32_t *)P.src_uidx.p : nullptr;
    a.out_idx = user ? (const int32_t *)P.tgt_uidx.p : nullptr;
    a.q = q;
    a.out = out;
    a.accumulate = accumulate;
    const double eh = hp.eps * (double)hp.S;  // eps in units of h
    a.eps2 = (T)(eh * eh);
    a.scale = (T)(1.0 / (4.0 * 3.14159265358979323846 * hp.h));
    a.kh = (T)(hp.kappa * hp.h);
    void *args[] = {&a};
    const int grid = (int)std::min<int64_t>(ntiles, P.occ_sms);
    ck(cudaLaunchKernel(box3d_fn<T>(hp.kernel == P2P_KERNEL_HELMHOLTZ_3D), dim3(grid), dim3(hp.nt), args,
                        (size_t)hp.smem_bytes, s),
       "box3d launch");
}

// ADAPTIVE (NEXT-4): one CTA per target leaf over its U-list; user order fused.
template <typename T>
void launch_adaptive(p2p_plan_s &P, const T *q, T *out, bool user, int accumulate, cudaStream_t s) {
    const p2p::HostPlan &hp = P.hp;
    const int ntiles = (int)hp.tiles.size();
    if (ntiles <= 0) return;
    p2p::dev::P2PArgs<T> a{};
    a.tiles = (const int32_t *)P.tiles.p;
    a.ntiles = ntiles;
    a.queue = (int *)P.queue.p;
    a.src_cap = (int)hp.src_cap;
    a.h = (T)hp.h;
    a.eps2 = (T)(hp.eps * hp.eps);
    a.leaf_rng = (const int4 *)P.leaf_rng.p;
    a.leaf_org = (const int2 *)P.leaf_org.p;
    a.ul_off = (const int32_t *)P.ul_off.p;
    a.ul_leaf = (const int32_t *)P.ul_leaf.p;
    a.src_cell = (const int2 *)P.src_cell.p;
    a.tgt_cell = (const int2 *)P.tgt_cell.p;
    a.src_uv = (const typename p2p::dev::V2<T>::type *)P.src_uv.p;
    a.tgt_uv = (const typename p2p::dev::V2<T>::type *)P.tgt_uv.p;
    a.src_idx = user ? (const int32_t *)P.src_uidx.p : nullptr;
    a.out_idx = user ? (const int32_t *)P.tgt_uidx.p : nullptr;
    a.q = q;
    a.out = out;
    a.accumulate = accumulate;
    void *args[] = {&a};
    const int grid = (int)std::min<int64_t>(ntiles, P.occ_sms);
    if (hp.warp_leaf) {
        const int g = (int)std::min<int64_t>((ntiles + 3) / 4, P.occ_sms);
        ck(cudaLaunchKernel((const void *)p2p::dev::p2p_adaptive_warp_kernel<T, 128>, dim3(g), dim3(128), args,
                            (size_t)hp.smem_bytes, s),
           "adaptive launch");
        return;
    }
    ck(cudaLaunchKernel((const void *)p2p::dev::p2p_adaptive_kernel<T, p2p::kAdaptiveThreads>, dim3(grid),
                        dim3(p2p::kAdaptiveThreads), args, (size_t)hp.smem_bytes, s),
       "adaptive launch");
}

template <typename T>
void apply_impl(p2p_plan_s &P, const void *d_q, void *d_out, int order, int accumulate, cudaStream_t s) {
    const p2p::HostPlan &hp = P.hp;
    if (hp.layout == P2P_LAYOUT_ADAPTIVE) {
        launch_adaptive<T>(P, (const T *)d_q, (T *)d_out, order == P2P_ORDER_USER, accumulate, s);
        return;
    }
    if (hp.dim == 3) {
        launch_box3d<T>(P, (const T *)d_q, (T *)d_out, order == P2P_ORDER_USER, accumulate, s);
        return;
    }
    if (hp.layout == P2P_LAYOUT_PAPER_INDEXING || hp.layout == P2P_LAYOUT_PAPER_REPETITION) {
        if constexpr (sizeof(T) == 8) apply_paper(P, d_q, d_out, order, accumulate, s);
        return;
    }
    const T *q_local = (const T *)d_q;
    if (order == P2P_ORDER_USER && hp.layout == P2P_LAYOUT_TILED) {  // permutations fused into the kernel
        launch_p2p<T>(P, (const T *)d_q, (T *)d_out, accumulate, s, true);
        ck(cudaGetLastError(), "apply launch");
        return;
    }
    if (order == P2P_ORDER_USER) {
        if (hp.n_src_local)
            p2p::dev::gather_kernel<T><<<grid_for(hp.n_src_local), 256, 0, s>>>(
                (const int32_t *)P.src_uidx.p, (const T *)d_q, (T *)P.q_local.p, hp.n_src_local);
        q_local = (const T *)P.q_local.p;
    } else if (hp.part_world > 1) {  // replicated weights in global plan order
        using V = typename p2p::dev::V2<T>::type;
        if (hp.n_src_local && P.comps == 2)
            p2p::dev::gather_kernel<V><<<grid_for(hp.n_src_local), 256, 0, s>>>(
                (const int32_t *)P.src_gidx.p, (const V *)d_q, (V *)P.q_local.p, hp.n_src_local);
        else if (hp.n_src_local)
            p2p::dev::gather_kernel<T><<<grid_for(hp.n_src_local), 256, 0, s>>>(
                (const int32_t *)P.src_gidx.p, (const T *)d_q, (T *)P.q_local.p, hp.n_src_local);
        q_local = (const T *)P.q_local.p;
    }
    if (order == P2P_ORDER_USER) {
        launch_p2p<T>(P, q_local, (T *)P.phi.p, 0, s);
        if (hp.n_tgt_local)
            p2p::dev::scatter_kernel<T><<<grid_for(hp.n_tgt_local), 256, 0, s>>>(
                (const int32_t *)P.tgt_uidx.p, (const T *)P.phi.p, (T *)d_out, hp.n_tgt_local, accumulate);
    } else {
        launch_p2p<T>(P, q_local, (T *)d_out, accumulate, s);
    }
    ck(cudaGetLastError(), "apply launch");
}

// Distributed apply in two phases on one stream: the interior phase needs
// only the owned weights (copied into the local set's owned range) and runs the TILED tiles
// whose regions hold owned sources only; the boundary phase scatters the received halo
// weights into the local set and runs the remaining tiles (NR, R: everything).
template <typename T>
void apply_dist_interior_impl(p2p_plan_s &P, const void *d_q_owned, void *d_out, int accumulate, cudaStream_t s) {
    const p2p::HostPlan &hp = P.hp;
    if (hp.n_src_owned)
        ck(cudaMemcpyAsync((T *)P.q_local.p + hp.owned_local_begin * P.comps, d_q_owned,
                           (size_t)hp.n_src_owned * sizeof(T) * P.comps, cudaMemcpyDeviceToDevice, s),
           "owned weights");
    if (hp.layout == P2P_LAYOUT_TILED)
        launch_p2p<T>(P, (const T *)P.q_local.p, (T *)d_out, accumulate, s, false, 0, hp.n_interior);
    ck(cudaGetLastError(), "apply_dist interior launch");
}

template <typename T>
void apply_dist_boundary_impl(p2p_plan_s &P, const void *d_q_halo, void *d_out, int accumulate, cudaStream_t s) {
    const p2p::HostPlan &hp = P.hp;
    if (hp.n_halo) {
        using V = typename p2p::dev::V2<T>::type;  // complex weights: (re, im) moved as one element
        if (P.comps == 2)
            p2p::dev::copy_scatter_kernel<V><<<grid_for(hp.n_halo), 256, 0, s>>>(
                (const int32_t *)P.halo_lidx.p, (const V *)d_q_halo, (V *)P.q_local.p, hp.n_halo);
        else
            p2p::dev::copy_scatter_kernel<T><<<grid_for(hp.n_halo), 256, 0, s>>>(
                (const int32_t *)P.halo_lidx.p, (const T *)d_q_halo, (T *)P.q_local.p, hp.n_halo);
    }
    if (hp.layout == P2P_LAYOUT_TILED)
        launch_p2p<T>(P, (const T *)P.q_local.p, (T *)d_out, accumulate, s, false, hp.n_interior,
                      (int64_t)hp.tiles.size());
    else
        launch_p2p<T>(P, (const T *)P.q_local.p, (T *)d_out, accumulate, s);
    ck(cudaGetLastError(), "apply_dist boundary launch");
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (dev >= 0 && dev != prev) ck(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

template <typename F>
p2p_status guarded(F f) {
    try {
        f();
        g_last_error.clear();
        return P2P_SUCCESS;
    } catch (const p2p::Error &e) {
        return set_error(e.code, e.what());
    } catch (const std::bad_alloc &) {
        return set_error(P2P_ERROR_OUT_OF_MEMORY, "host allocation failed");
    } catch (const std::exception &e) {
        return set_error(P2P_ERROR_CUDA, e.what());
    }
}

void require_device(const p2p_plan_s *P) {
    if (P->device < 0) throw p2p::Error(P2P_ERROR_NO_DEVICE, "host-only plan (device < 0): no apply; there is no CPU fallback");
}


// ---- the plan build on the device (plan_device.cuh) ----

// Stream-ordered temporaries of a device build, released on exit.
struct DevTmp {
    cudaStream_t s;
    std::vector<void *> held;
    explicit DevTmp(cudaStream_t st) : s(st) {}
    template <typename V>
    V *get(int64_t n) {
        void *p = nullptr;
        ck(cudaMallocAsync(&p, (size_t)std::max<int64_t>(n, 1) * sizeof(V), s), "cudaMallocAsync (build temporaries)");
        held.push_back(p);
        return (V *)p;
    }
    ~DevTmp() {
        for (void *p : held) cudaFreeAsync(p, s);
    }
};

template <typename V>
void d2h(V *dst, const void *src, int64_t n, cudaStream_t s) {
    if (n <= 0) return;
    ck(cudaMemcpyAsync(dst, src, (size_t)n * sizeof(V), cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync D2H");
    ck(cudaStreamSynchronize(s), "device build sync");
}

// Exclusive scan of n uint32 counts into off[0..n] (off[0] = 0); returns off[n].
int64_t scan_offsets(DevTmp &tmp, const uint32_t *cnt, uint32_t *off, int64_t n, cudaStream_t s) {
    ck(cudaMemsetAsync(off, 0, sizeof(uint32_t), s), "memset");
    if (n > 0) {
        size_t tb = 0;
        ck(cub::DeviceScan::InclusiveSum(nullptr, tb, cnt, off + 1, (int)n, s), "cub scan");
        void *t = tmp.get<char>((int64_t)tb);
        ck(cub::DeviceScan::InclusiveSum(t, tb, cnt, off + 1, (int)n, s), "cub scan");
    }
    uint32_t last = 0;
    d2h(&last, off + n, 1, s);
    return last;
}

// a2 + a3 on the device: codes at grid side S, stable radix sort of (code, index), CSR offsets.
void device_csr(DevTmp &tmp, const double *xy, int64_t n, int L, int64_t S, int64_t B, int32_t *perm, int32_t *off,
                cudaStream_t s) {
    using namespace p2p::dbuild;
    uint32_t *code = tmp.get<uint32_t>(n), *code_s = tmp.get<uint32_t>(n);
    int32_t *idx = tmp.get<int32_t>(n);
    codes_kernel<<<nblocks(n), kB, 0, s>>>((const double2 *)xy, n, S, code, idx);
    const int bits = 2 * (L - 1);
    if (bits > 0) {
        size_t tb = 0;
        ck(cub::DeviceRadixSort::SortPairs(nullptr, tb, code, code_s, idx, perm, (int)n, 0, bits, s), "cub sort");
        void *t = tmp.get<char>((int64_t)tb);
        ck(cub::DeviceRadixSort::SortPairs(t, tb, code, code_s, idx, perm, (int)n, 0, bits, s), "cub sort");
    } else {  // one box: the identity
        ck(cudaMemcpyAsync(code_s, code, (size_t)n * 4, cudaMemcpyDeviceToDevice, s), "copy");
        ck(cudaMemcpyAsync(perm, idx, (size_t)n * 4, cudaMemcpyDeviceToDevice, s), "copy");
    }
    offsets_kernel<<<nblocks(B + 1), kB, 0, s>>>(code_s, n, B, off);
}

// a1 CT loop on the device: codes at l_max sorted once; the most points in a box at each level
// is the longest run of equal code prefixes (§3.1; the host's ct_loop_level).
int device_ct_level(DevTmp &tmp, const p2p_plan_desc &d, const double *dsrc, const double *dtgt, cudaStream_t s) {
    using namespace p2p::dbuild;
    const int lmax = std::min(d.l_max, p2p::kMaxLevel);
    if (d.l_start < 1) throw p2p::Error(P2P_ERROR_INVALID_ARGUMENT, "l_start must be >= 1");
    if (d.ct < 1) throw p2p::Error(P2P_ERROR_INVALID_ARGUMENT, "ct must be >= 1");
    const int64_t Sref = int64_t(1) << (lmax - 1);
    const int l0 = std::max(1, d.l_start);
    int64_t *mr = tmp.get<int64_t>(32);
    ck(cudaMemsetAsync(mr, 0, 32 * sizeof(int64_t), s), "memset");
    const double *xy[2] = {dsrc, dtgt};
    const int64_t nn[2] = {d.n_src, d.n_tgt};
    for (int w = 0; w < 2; ++w) {
        const int64_t n = nn[w];
        uint32_t *code = tmp.get<uint32_t>(n), *code_s = tmp.get<uint32_t>(n);
        codes_kernel<<<nblocks(n), kB, 0, s>>>((const double2 *)xy[w], n, Sref, code, nullptr);
        const int bits = 2 * (lmax - 1);
        if (bits > 0) {
            size_t tb = 0;
            ck(cub::DeviceRadixSort::SortKeys(nullptr, tb, code, code_s, (int)n, 0, bits, s), "cub sort");
            void *t = tmp.get<char>((int64_t)tb);
            ck(cub::DeviceRadixSort::SortKeys(t, tb, code, code_s, (int)n, 0, bits, s), "cub sort");
        } else {
            ck(cudaMemcpyAsync(code_s, code, (size_t)n * 4, cudaMemcpyDeviceToDevice, s), "copy");
        }
        if (l0 <= lmax) maxrun_kernel<<<nblocks(n), kB, 0, s>>>(code_s, n, l0, lmax, lmax, mr + 16 * w);
    }
    int64_t h[32];
    d2h(h, mr, 32, s);
    for (int L = l0; L <= lmax; ++L)
        if (h[L] <= d.ct && h[16 + L] <= d.ct) return L;
    throw p2p::Error(P2P_ERROR_CONSTRUCTION_FAILURE,
                     "CT loop: some leaf box still holds more than CT points at L = " + std::to_string(lmax) +
                         " (cap; SPEC.md L75)");
}

// The whole plan on the device, bit-identical to build_host_plan for one partition and the NR /
// TILED layouts.  Device arrays go straight into P's buffers; hp gets the scalars and the launch
// list (host arrays for export are mirrored on demand, mirror_device_plan).
template <typename T>
void build_device_plan(p2p_plan_s &P, const p2p_plan_desc &d, const double *dsrc, const double *dtgt) {
    using namespace p2p::dbuild;
    p2p::HostPlan &hp = P.hp;
    cudaStream_t s = P.stream;
    const auto t0 = std::chrono::steady_clock::now();
    DevTmp tmp(s);
    hp.device_built = true;
    hp.kernel = d.kernel;
    hp.kappa = d.kernel == P2P_KERNEL_HELMHOLTZ_2D ? d.wavenumber : 0.0;
    hp.layout = d.layout;
    hp.precision = d.precision;
    hp.device = d.device;
    hp.eps = d.epsilon;
    hp.part_world = 1;
    hp.part_rank = 0;
    hp.n_src = d.n_src;
    hp.n_tgt = d.n_tgt;
    const int e = sizeof(T);

    {   // coordinates inside the unit square, NaN rejected
        unsigned long long *bad = tmp.get<unsigned long long>(2), hb[2];
        ck(cudaMemsetAsync(bad, 0xFF, 2 * sizeof(unsigned long long), s), "memset");
        validate_kernel<<<nblocks(2 * d.n_src), kB, 0, s>>>(dsrc, 2 * d.n_src, bad);
        validate_kernel<<<nblocks(2 * d.n_tgt), kB, 0, s>>>(dtgt, 2 * d.n_tgt, bad + 1);
        d2h(hb, bad, 2, s);
        for (int w = 0; w < 2; ++w)
            if (hb[w] != ~0ull)
                throw p2p::Error(P2P_ERROR_INVALID_ARGUMENT, std::string(w ? "targets" : "sources") + ": coordinate " +
                                                                 std::to_string(hb[w] / 2) +
                                                                 " outside the unit square [0,1]^2 (SPEC.md L119)");
    }
    // ---- a1 level
    int L = d.level > 0 ? d.level : device_ct_level(tmp, d, dsrc, dtgt, s);
    L += d.level_delta;
    if (L < 1) throw p2p::Error(P2P_ERROR_INVALID_ARGUMENT, "L + level_delta < 1 (SPEC.md L85)");
    if (L > p2p::kMaxLevel) throw p2p::Error(P2P_ERROR_NOT_SUPPORTED, "L > 15 (full-grid CSR offsets; see DESIGN.md)");
    hp.L = L;
    hp.S = int64_t(1) << (L - 1);
    hp.B = hp.S * hp.S;
    hp.h = 1.0 / (double)hp.S;
    const int64_t S = hp.S, B = hp.B;

    // ---- a2, a3 (P = 1: the local sets are the global ones)
    P.alloc(P.src_uidx, (size_t)d.n_src * 4);
    P.alloc(P.tgt_uidx, (size_t)d.n_tgt * 4);
    P.alloc(P.src_off, (size_t)(B + 1) * 4);
    P.alloc(P.tgt_off, (size_t)(B + 1) * 4);
    int32_t *sperm = (int32_t *)P.src_uidx.p, *tperm = (int32_t *)P.tgt_uidx.p;
    int32_t *so = (int32_t *)P.src_off.p, *to = (int32_t *)P.tgt_off.p;
    device_csr(tmp, dsrc, d.n_src, L, S, B, sperm, so, s);
    device_csr(tmp, dtgt, d.n_tgt, L, S, B, tperm, to, s);

    // ---- box statistics and E1 source counts
    int32_t *n9 = tmp.get<int32_t>(B);
    {
        unsigned long long *acc = tmp.get<unsigned long long>(3), ha[3];
        ck(cudaMemsetAsync(acc, 0, 3 * sizeof(unsigned long long), s), "memset");
        box_stats_kernel<<<nblocks(B), kB, 0, s>>>(so, to, B, S, n9, acc);
        d2h(ha, acc, 3, s);
        hp.occ_src = (int64_t)ha[0];
        hp.occ_tgt = (int64_t)ha[1];
        hp.t_max = (int64_t)ha[2];
    }
    hp.density = (double)hp.n_tgt / (double)hp.B;
    hp.density_occ = hp.occ_tgt ? (double)hp.n_tgt / (double)hp.occ_tgt : 0.0;

    // ---- CTA tile size (the host builder's rule: smallest k whose non-empty tiles hold >= 115 targets)
    const int kmax = std::min(L - 1, p2p::kMaxTileLog2);
    int k;
    if (d.tile_log2 >= 0) {
        k = std::min(d.tile_log2, kmax);
    } else {
        unsigned long long *ne = tmp.get<unsigned long long>(8), hn[8];
        ck(cudaMemsetAsync(ne, 0, 8 * sizeof(unsigned long long), s), "memset");
        tile_count_kernel<<<nblocks(B), kB, 0, s>>>(to, B, kmax, ne);
        d2h(hn, ne, kmax + 1, s);
        k = kmax;
        for (int kk = 0; kk <= kmax; ++kk)
            if ((double)hp.n_tgt / (double)std::max<int64_t>((int64_t)hn[kk], 1) >= 115.0) {
                k = kk;
                break;
            }
    }
    int32_t *tiles_m = nullptr;  // non-empty tiles, Morton order (= TILED slot order)
    int64_t *tile_pairs = nullptr;
    int64_t nt = 0;
    unsigned long long hs[6];
    for (;; --k) {
        const int64_t WW = int64_t(1) << (2 * k), ntile_all = B / WW;
        int32_t *flag = tmp.get<int32_t>(ntile_all), *pos = tmp.get<int32_t>(ntile_all);
        tile_flag_kernel<<<nblocks(ntile_all), kB, 0, s>>>(to, ntile_all, WW, flag);
        size_t tb = 0;
        ck(cub::DeviceScan::ExclusiveSum(nullptr, tb, flag, pos, (int)ntile_all, s), "cub scan");
        void *t = tmp.get<char>((int64_t)tb);
        ck(cub::DeviceScan::ExclusiveSum(t, tb, flag, pos, (int)ntile_all, s), "cub scan");
        int32_t lastp[2];
        ck(cudaMemcpyAsync(&lastp[0], pos + ntile_all - 1, 4, cudaMemcpyDeviceToHost, s), "D2H");
        d2h(&lastp[1], flag + ntile_all - 1, 1, s);
        nt = (int64_t)lastp[0] + lastp[1];
        tiles_m = tmp.get<int32_t>(nt);
        tile_pairs = tmp.get<int64_t>(nt);
        compact_kernel<<<nblocks(ntile_all), kB, 0, s>>>(flag, pos, ntile_all, tiles_m);
        unsigned long long *st = tmp.get<unsigned long long>(6);
        ck(cudaMemsetAsync(st, 0, 6 * sizeof(unsigned long long), s), "memset");
        if (nt) tile_stats_kernel<<<nblocks(nt, 64), 64, 0, s>>>(tiles_m, nt, k, S, so, to, n9, tile_pairs, st);
        d2h(hs, st, 6, s);
        p2p::TileStats ts;
        ts.ntiles = nt;
        ts.max_region_pad = (int64_t)hs[0];
        ts.max_region = (int64_t)hs[1];
        ts.max_tcount = (int64_t)hs[2];
        ts.max_tcount2 = (int64_t)hs[3];
        const int64_t smem = p2p::choose_tile_params(d, hp, k, ts);
        if (smem <= p2p::kSmemLimit) break;
        if (k == 0 || d.tile_log2 >= 0)
            throw p2p::Error(P2P_ERROR_NOT_SUPPORTED, "a tile's near-field sources need " + std::to_string(smem) +
                                                          " B of shared memory (> 200 KB); use a deeper level (CT loop) -- see DESIGN.md");
    }
    hp.k = k;
    {
        int g = 1;
        while (g < 5 && (double)(1 << g) < hp.density_occ) ++g;
        hp.group_log2 = g;
    }
    const int64_t W = int64_t(1) << k, WW = W * W, R = W + 2;
    hp.pairs_global = hp.pairs = (int64_t)hs[5];
    hp.part_tile = {0, nt};
    hp.part_src = {0, hp.n_src};
    hp.part_tgt = {0, hp.n_tgt};
    hp.boxes_in_tiles = nt * WW;
    hp.src_owned_begin = 0;
    hp.n_src_owned = hp.n_src_local = hp.n_src;
    hp.tgt_begin = 0;
    hp.n_tgt_local = hp.n_tgt;
    hp.owned_local_begin = 0;
    hp.n_halo = hp.n_send = 0;
    hp.recv_counts.assign(1, 0);
    hp.send_counts.assign(1, 0);

    // ---- a5 point coordinates: box-local (NR sources; targets for every layout)
    P.alloc(P.tgt_uv, (size_t)hp.n_tgt * 2 * e);
    uv_kernel<T><<<nblocks(hp.n_tgt), kB, 0, s>>>((const double2 *)dtgt, tperm, hp.n_tgt, S, hp.h, (T *)P.tgt_uv.p);
    if (d.layout == P2P_LAYOUT_NONREDUNDANT) {
        P.alloc(P.src_uv, (size_t)hp.n_src * 2 * e);
        uv_kernel<T><<<nblocks(hp.n_src), kB, 0, s>>>((const double2 *)dsrc, sperm, hp.n_src, S, hp.h, (T *)P.src_uv.p);
    }

    // ---- TILED layout (per Morton-order tile = slot)
    int32_t *nparts = tmp.get<int32_t>(nt);
    if (d.layout == P2P_LAYOUT_TILED) {
        const int ts = p2p::tiled_table_stride(k);
        hp.table_entries = nt * ts;
        P.alloc(P.reg_table, (size_t)hp.table_entries * 2);
        if (hp.table_entries) ck(cudaMemsetAsync(P.reg_table.p, 0, P.reg_table.bytes, s), "memset");
        uint32_t *reg_sz = tmp.get<uint32_t>(nt), *slot_sz = tmp.get<uint32_t>(nt), *item_sz = tmp.get<uint32_t>(nt);
        int *err = tmp.get<int>(1);
        ck(cudaMemsetAsync(err, 0, sizeof(int), s), "memset");
        P.alloc(P.tile_tgt_base, (size_t)nt * 4);
        if (nt)
            tiled_table_kernel<<<nblocks(nt, 64), 64, 0, s>>>(tiles_m, nt, k, S, ts, hp.pad, hp.tpi, hp.ns, so, to,
                                                             (uint16_t *)P.reg_table.p, reg_sz, slot_sz, item_sz,
                                                             (int32_t *)P.tile_tgt_base.p, err);
        int herr = 0;
        d2h(&herr, err, 1, s);
        if (herr & 1) throw p2p::Error(P2P_ERROR_NOT_SUPPORTED, "TILED region exceeds 65535 entries; use NR");
        if (herr & 2)
            throw p2p::Error(P2P_ERROR_NOT_SUPPORTED, "TILED tile exceeds its target-slot limit; use a deeper level or NR");
        P.alloc(P.reg_off, (size_t)(nt + 1) * 4);
        P.alloc(P.tgt_pack_off, (size_t)(nt + 1) * 4);
        hp.reg_entries = scan_offsets(tmp, reg_sz, (uint32_t *)P.reg_off.p, nt, s);
        const int64_t np = scan_offsets(tmp, slot_sz, (uint32_t *)P.tgt_pack_off.p, nt, s);
        // packed regions: pads keep index -1 and coordinate 1e4
        P.alloc(P.reg_idx, (size_t)hp.reg_entries * 4);
        P.alloc(P.reg_uidx, (size_t)hp.reg_entries * 4);
        P.alloc(P.reg_uv, (size_t)hp.reg_entries * 2 * e);
        fill_kernel<int32_t><<<nblocks(hp.reg_entries), kB, 0, s>>>((int32_t *)P.reg_idx.p, hp.reg_entries, -1);
        fill_kernel<int32_t><<<nblocks(hp.reg_entries), kB, 0, s>>>((int32_t *)P.reg_uidx.p, hp.reg_entries, -1);
        fill_kernel<T><<<nblocks(2 * hp.reg_entries), kB, 0, s>>>((T *)P.reg_uv.p, 2 * hp.reg_entries, (T)1.0e4);
        if (nt)
            tiled_region_kernel<T><<<nblocks(nt, 1), 128, 0, s>>>(tiles_m, nt, k, S, hp.h, ts, hp.pad, so, sperm,
                                                                  (const double2 *)dsrc, (const uint16_t *)P.reg_table.p,
                                                                  (const uint32_t *)P.reg_off.p, (int32_t *)P.reg_idx.p,
                                                                  (int32_t *)P.reg_uidx.p, (T *)P.reg_uv.p);
        // target slots
        P.alloc(P.tgt_bl, (size_t)np * 2);
        P.alloc(P.tgt_oix, (size_t)np * 2);
        P.alloc(P.tgt_ruv, (size_t)np * 2 * e);
        if (np) {
            ck(cudaMemsetAsync(P.tgt_bl.p, 0, P.tgt_bl.bytes, s), "memset");
            ck(cudaMemsetAsync(P.tgt_oix.p, 0xFF, P.tgt_oix.bytes, s), "memset");
            ck(cudaMemsetAsync(P.tgt_ruv.p, 0, P.tgt_ruv.bytes, s), "memset");
        }
        const size_t slot_smem = (size_t)3 * WW * 4;
        ck(cudaFuncSetAttribute(tiled_slots_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024),
           "smem attr");
        if (nt)
            tiled_slots_kernel<T><<<nblocks(nt, 1), 128, slot_smem, s>>>(
                tiles_m, nt, k, hp.h, hp.tpi, hp.tsort ? 1 : 0, to, n9, tperm, (const double2 *)dtgt,
                (const uint32_t *)P.tgt_pack_off.p, (uint16_t *)P.tgt_bl.p, (uint16_t *)P.tgt_oix.p, (T *)P.tgt_ruv.p);
        // ---- queue order: longest first when the working set fits L2, else Morton with the tail split
        if (hp.ns == 3) {
            P.alloc(P.item_off, (size_t)(nt + 1) * 4);
            const int64_t ni = scan_offsets(tmp, item_sz, (uint32_t *)P.item_off.p, nt, s);
            P.alloc(P.items, (size_t)ni * 2);
            if (ni) ck(cudaMemsetAsync(P.items.p, 0, P.items.bytes, s), "memset");
        }
    }
    const int64_t ws = (hp.n_src_local + hp.n_tgt_local) * 3 * (int64_t)e + 8 * hp.boxes_in_tiles +
                       (hp.halo_entries + hp.reg_entries) * 3 * (int64_t)e;
    hp.lpt = ws < (int64_t)100 << 20;
    if (const char *v = std::getenv("P2P_LPT")) hp.lpt = std::atoi(v) != 0;
    int32_t *order = nullptr;
    if (hp.lpt && nt > 1) {  // stable sort by descending pair count (CUB's radix sort is stable)
        uint64_t *ks = tmp.get<uint64_t>(nt);
        int32_t *iot = tmp.get<int32_t>(nt);
        order = tmp.get<int32_t>(nt);
        iota_kernel<<<nblocks(nt), kB, 0, s>>>(iot, nt);
        size_t tb = 0;
        ck(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, (const uint64_t *)tile_pairs, ks, iot, order, (int)nt,
                                                      0, 64, s),
           "cub sort");
        void *t = tmp.get<char>((int64_t)tb);
        ck(cub::DeviceRadixSort::SortPairsDescending(t, tb, (const uint64_t *)tile_pairs, ks, iot, order, (int)nt, 0, 64,
                                                      s),
           "cub sort");
    }
    int64_t keep = nt;
    int parts = 1;
    if (d.layout == P2P_LAYOUT_TILED) {
        int64_t tail = hp.lpt ? 0 : 148 * 4;
        int pp = 4;
        if (const char *v = std::getenv("P2P_TAIL_TILES")) tail = std::atoll(v);
        if (const char *v = std::getenv("P2P_TAIL_PARTS")) pp = std::max(1, std::min(16, std::atoi(v)));
        tail = std::min<int64_t>(tail, nt / 2);
        if (pp > 1 && tail > 0) {
            keep = nt - tail;
            parts = pp;
        }
    }
    // entries per queue position (tail and heavy-tile splits, TILED only), then their offsets
    uint32_t *cnt = tmp.get<uint32_t>(nt), *eoff = tmp.get<uint32_t>(nt + 1);
    const int64_t share = d.layout == P2P_LAYOUT_TILED
                              ? std::max<int64_t>(1, (hp.pairs + p2p::kSplitShare - 1) / p2p::kSplitShare) : 0;
    if (nt) split_count_kernel<<<nblocks(nt), kB, 0, s>>>(order, tile_pairs, nt, keep, parts, share, cnt);
    const int64_t nent = scan_offsets(tmp, cnt, eoff, nt, s);
    P.alloc(P.tiles, (size_t)nent * 4);
    P.alloc(P.tile_slot, (size_t)nent * 4);
    P.alloc(P.tile_part, (size_t)nent * 4);
    if (nt)
        queue_kernel<<<nblocks(nt), kB, 0, s>>>(order, tiles_m, nt, cnt, eoff, (int32_t *)P.tiles.p,
                                                (int32_t *)P.tile_slot.p, (int32_t *)P.tile_part.p, nparts);
    hp.n_interior = nent;
    hp.tiles.resize((size_t)nent);
    d2h(hp.tiles.data(), P.tiles.p, nent, s);
    // ---- NS = 3 item lists (TILED)
    if (d.layout == P2P_LAYOUT_TILED && hp.ns == 3 && nt) {
        const int64_t maxitems = 3 * (hp.tgt_cap / hp.tpi) + 8;
        const size_t ism = (size_t)maxitems * 3 * 4;
        if (ism > 160 * 1024) throw p2p::Error(P2P_ERROR_NOT_SUPPORTED, "device build: tile item list too large");
        ck(cudaFuncSetAttribute(tiled_items_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024),
           "smem attr");
        tiled_items_kernel<<<nblocks(nt, 1), 128, ism, s>>>(nt, k, p2p::tiled_table_stride(k), hp.tpi, hp.nt,
                                                           (const uint16_t *)P.reg_table.p,
                                                           (const uint32_t *)P.tgt_pack_off.p,
                                                           (const uint16_t *)P.tgt_bl.p, nparts,
                                                           (const uint32_t *)P.item_off.p, (uint16_t *)P.items.p);
    }
    (void)R;
    if (d.precision == P2P_FP64) {
        p2p::build_log_table(hp);
        P.upload(P.log_tab, hp.log_tab);
    }
    ck(cudaGetLastError(), "device build launch");
    finalize_plan<T>(P);
    ck(cudaStreamSynchronize(s), "device build sync");
    hp.build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// Host copies of a device-built plan's arrays, for p2p_plan_export (on first use).
void mirror_device_plan(p2p_plan_s &P) {
    p2p::HostPlan &hp = P.hp;
    if (!hp.device_built || !hp.src_off_g.empty()) return;
    DeviceGuard g(P.device);
    cudaStream_t s = P.stream;
    auto get = [&](auto &vec, const DevBuf &b) {
        using V = typename std::decay_t<decltype(vec)>::value_type;
        vec.resize(b.bytes / sizeof(V));
        d2h(vec.data(), b.p, (int64_t)vec.size(), s);
    };
    get(hp.src_uidx, P.src_uidx);
    get(hp.tgt_uidx, P.tgt_uidx);
    hp.src_perm_g = hp.src_uidx;
    hp.tgt_perm_g = hp.tgt_uidx;
    get(hp.src_off_g, P.src_off);
    get(hp.tgt_off_g, P.tgt_off);
    hp.src_off = hp.src_off_g;
    hp.tgt_off = hp.tgt_off_g;
    hp.src_gidx.resize((size_t)hp.n_src);
    std::iota(hp.src_gidx.begin(), hp.src_gidx.end(), 0);
    get(hp.tile_slot, P.tile_slot);
    get(hp.tile_part, P.tile_part);
    if (hp.layout == P2P_LAYOUT_TILED) {
        get(hp.reg_off, P.reg_off);
        get(hp.reg_idx, P.reg_idx);
        get(hp.reg_uidx, P.reg_uidx);
        get(hp.reg_table, P.reg_table);
        get(hp.tgt_pack_off, P.tgt_pack_off);
        get(hp.tgt_bl, P.tgt_bl);
        get(hp.tgt_oix, P.tgt_oix);
        get(hp.tile_tgt_base, P.tile_tgt_base);
        get(hp.item_off, P.item_off);
        get(hp.items, P.items);
    }
}

}  // namespace

extern "C" {

void p2p_plan_desc_init(p2p_plan_desc *d) {
    if (!d) return;
    std::memset(d, 0, sizeof(*d));
    d->struct_size = sizeof(p2p_plan_desc);
    d->abi_version = P2P_ABI_VERSION;
    d->level = 0;
    d->ct = 15;
    d->l_start = 3;
    d->l_max = p2p::kMaxLevel;
    d->level_delta = 0;
    d->kernel = P2P_KERNEL_LAPLACE_2D;
    d->epsilon = 1e-12;
    d->layout = P2P_LAYOUT_NONREDUNDANT;
    d->precision = P2P_FP32;
    d->device = 0;
    d->tile_log2 = -1;
    d->stream = nullptr;
    d->part_world = 1;
    d->part_rank = 0;
}

static p2p_status plan_create_common(const p2p_plan_desc *desc, const p2p::LocalInput *li, p2p_plan *out) {
    Nvtx nvtx_("p2p_plan_create");
    if (out) *out = nullptr;
    if (!desc || !out) return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL desc or out");
    std::unique_ptr<p2p_plan_s> P(new (std::nothrow) p2p_plan_s());
    if (!P) return set_error(P2P_ERROR_OUT_OF_MEMORY, "host allocation failed");
    p2p_status st = guarded([&] {
        p2p::build_host_plan(*desc, P->hp, li);
        P->device = desc->device;
        P->elem = desc->precision == P2P_FP32 ? 4 : 8;
        P->comps = (desc->kernel == P2P_KERNEL_HELMHOLTZ_2D || desc->kernel == P2P_KERNEL_HELMHOLTZ_3D) ? 2 : 1;
        if (desc->device >= 0) {
            int ndev = 0;
            if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
                throw p2p::Error(P2P_ERROR_NO_DEVICE, "no CUDA device visible");
            if (desc->device >= ndev) throw p2p::Error(P2P_ERROR_INVALID_ARGUMENT, "device ordinal out of range");
            DeviceGuard g(desc->device);
            P->stream = (cudaStream_t)desc->stream;
            auto t0 = std::chrono::steady_clock::now();
            try {
                if (desc->precision == P2P_FP32) upload_plan<float>(*P);
                else upload_plan<double>(*P);
                ck(cudaStreamSynchronize(P->stream), "upload sync");
            } catch (...) {
                P->release();
                throw;
            }
            P->upload_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
    });
    if (st == P2P_SUCCESS) *out = P.release();
    return st;
}

p2p_status p2p_plan_create(const p2p_plan_desc *desc, p2p_plan *out) { return plan_create_common(desc, nullptr, out); }

p2p_status p2p_plan_create_local(const p2p_plan_desc *desc, const int64_t *src_ids, const int64_t *tgt_ids,
                                 const int32_t *src_counts, const int32_t *tgt_counts, int64_t n_src_global,
                                 int64_t n_tgt_global, p2p_plan *out) {
    p2p::LocalInput li;
    li.src_ids = src_ids;
    li.tgt_ids = tgt_ids;
    li.src_counts = src_counts;
    li.tgt_counts = tgt_counts;
    li.n_src_global = n_src_global;
    li.n_tgt_global = n_tgt_global;
    return plan_create_common(desc, &li, out);
}

p2p_status p2p_box_counts(int32_t level, int64_t n, const double *xy, int32_t *counts) {
    if (level < 1 || level > 15) return set_error(P2P_ERROR_INVALID_ARGUMENT, "level outside 1..15");
    if (n < 0 || (n && !xy) || !counts) return set_error(P2P_ERROR_INVALID_ARGUMENT, "bad arguments");
    return guarded([&] { p2p::box_counts(level, n, xy, counts); });
}

p2p_status p2p_partition_route(const p2p_plan_desc *desc, const int64_t *src_ids, const int64_t *tgt_ids,
                               const int32_t *src_counts, const int32_t *tgt_counts, int64_t n_src_global,
                               int64_t n_tgt_global, uint32_t *src_mask, uint32_t *tgt_mask) {
    if (!desc || (desc->n_src && !src_mask) || (desc->n_tgt && !tgt_mask))
        return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL desc or mask");
    p2p::LocalInput li;
    li.src_ids = src_ids;
    li.tgt_ids = tgt_ids;
    li.src_counts = src_counts;
    li.tgt_counts = tgt_counts;
    li.n_src_global = n_src_global;
    li.n_tgt_global = n_tgt_global;
    li.src_mask = src_mask;
    li.tgt_mask = tgt_mask;
    return guarded([&] {
        p2p::HostPlan hp;
        p2p::build_host_plan(*desc, hp, &li);
    });
}

p2p_status p2p_plan_create_device(const p2p_plan_desc *desc, const double *d_src_xy, const double *d_tgt_xy,
                                  p2p_plan *out) {
    Nvtx nvtx_("p2p_plan_create_device");
    if (out) *out = nullptr;
    if (!desc || !out) return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL desc or out");
    std::unique_ptr<p2p_plan_s> P(new (std::nothrow) p2p_plan_s());
    if (!P) return set_error(P2P_ERROR_OUT_OF_MEMORY, "host allocation failed");
    p2p_status st = guarded([&] {
        const p2p_plan_desc &d = *desc;
        if (d.struct_size != sizeof(p2p_plan_desc)) throw p2p::Error(P2P_ERROR_INVALID_ARGUMENT, "desc.struct_size mismatch");
        p2p::check_kernel(d);
        if (p2p::kernel_dim(d.kernel) == 3) throw p2p::Error(P2P_ERROR_NOT_SUPPORTED, "device build: 2D kernels");
        if (d.precision != P2P_FP32 && d.precision != P2P_FP64) throw p2p::Error(P2P_ERROR_INVALID_ARGUMENT, "bad precision");
        if (d.layout != P2P_LAYOUT_NONREDUNDANT && d.layout != P2P_LAYOUT_TILED)
            throw p2p::Error(P2P_ERROR_NOT_SUPPORTED, "device build: NR and TILED layouts only (others: p2p_plan_create)");
        if (d.part_world != 1 || d.part_rank != 0)
            throw p2p::Error(P2P_ERROR_NOT_SUPPORTED, "device build: one partition only (part_world = 1)");
        if (!(d.epsilon > 0.0) || !std::isfinite(d.epsilon)) throw p2p::Error(P2P_ERROR_INVALID_ARGUMENT, "epsilon must be > 0");
        if (d.n_src < 1 || d.n_tgt < 1) throw p2p::Error(P2P_ERROR_INVALID_ARGUMENT, "n must be >= 1 (SPEC.md L55)");
        if (!d_src_xy || !d_tgt_xy) throw p2p::Error(P2P_ERROR_INVALID_ARGUMENT, "NULL device coordinates");
        if (d.n_src > INT32_MAX - 8 || d.n_tgt > INT32_MAX - 8)
            throw p2p::Error(P2P_ERROR_NOT_SUPPORTED, "more than 2^31 points per set");
        if (d.device < 0) throw p2p::Error(P2P_ERROR_NO_DEVICE, "device build needs a CUDA device (device >= 0)");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw p2p::Error(P2P_ERROR_NO_DEVICE, "no CUDA device visible");
        if (d.device >= ndev) throw p2p::Error(P2P_ERROR_INVALID_ARGUMENT, "device ordinal out of range");
        DeviceGuard g(d.device);
        P->device = d.device;
        P->elem = d.precision == P2P_FP32 ? 4 : 8;
        P->comps = d.kernel == P2P_KERNEL_HELMHOLTZ_2D ? 2 : 1;
        P->stream = (cudaStream_t)d.stream;
        try {
            if (d.precision == P2P_FP32) build_device_plan<float>(*P, d, d_src_xy, d_tgt_xy);
            else build_device_plan<double>(*P, d, d_src_xy, d_tgt_xy);
        } catch (...) {
            cudaStreamSynchronize(P->stream);
            P->release();
            throw;
        }
    });
    if (st == P2P_SUCCESS) *out = P.release();
    return st;
}

namespace {
// Selects the next workspace slot for one apply (stream-ordered wait on its last user) and
// records the slot's event when the apply's work is enqueued.
struct WsSlot {
    p2p_plan_s &P;
    cudaStream_t s;
    p2p_plan_s::Workspace *w = nullptr;
    WsSlot(p2p_plan_s &P_, cudaStream_t s_) : P(P_), s(s_) {
        if (P.ws.size() < 2) return;
        w = &P.ws[P.ws_next++ % P.ws.size()];
        ck(cudaStreamWaitEvent(s, w->done, 0), "workspace wait");
        P.q_local = w->q_local;
        P.phi = w->phi;
        P.io_q = w->io_q;
        P.io_out = w->io_out;
        P.queue = w->queue;
    }
    ~WsSlot() {
        if (w) cudaEventRecord(w->done, s);
    }
};
}  // namespace

p2p_status p2p_plan_set_workspaces(p2p_plan P, int32_t n) {
    if (!P || n < 1 || n > 8) return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL plan or n outside 1..8");
    if (P->hp.part_world > 1) return set_error(P2P_ERROR_NOT_SUPPORTED, "workspace slots: single-partition plans");
    if (P->hp.layout == P2P_LAYOUT_PAPER_INDEXING || P->hp.layout == P2P_LAYOUT_PAPER_REPETITION)
        return set_error(P2P_ERROR_NOT_SUPPORTED, "workspace slots: not for the paper's layouts");
    return guarded([&] {
        require_device(P);
        DeviceGuard g(P->device);
        auto &ws = P->ws;
        if (ws.empty()) {  // slot 0 = the plan's own buffers
            ws.resize(1);
            ws[0].q_local = P->q_local;
            ws[0].phi = P->phi;
            ws[0].io_q = P->io_q;
            ws[0].io_out = P->io_out;
            ws[0].queue = P->queue;
            ck(cudaEventCreateWithFlags(&ws[0].done, cudaEventDisableTiming), "workspace event");
            ck(cudaEventRecord(ws[0].done, P->stream), "workspace event");
        }
        while ((int)ws.size() < n) {
            p2p_plan_s::Workspace w;
            auto mk = [&](DevBuf &b, size_t bytes) {
                b.bytes = bytes;
                ck(cudaMalloc(&b.p, std::max<size_t>(bytes, 16)), "cudaMalloc workspace");
                P->device_bytes += (int64_t)bytes;
            };
            mk(w.q_local, ws[0].q_local.bytes);
            mk(w.phi, ws[0].phi.bytes);
            mk(w.io_q, ws[0].io_q.bytes);
            mk(w.io_out, ws[0].io_out.bytes);
            mk(w.queue, 16);
            ck(cudaMemset(w.queue.p, 0, 16), "queue init");  // kernels reset it on exit
            ck(cudaEventCreateWithFlags(&w.done, cudaEventDisableTiming), "workspace event");
            ck(cudaEventRecord(w.done, P->stream), "workspace event");
            ws.push_back(w);
        }
        ck(cudaDeviceSynchronize(), "workspace init");
    });
}

p2p_status p2p_apply(p2p_plan P, const void *d_q, void *d_out, int32_t order, int32_t accumulate, void *stream) {
    Nvtx nvtx_("p2p_apply");
    if (!P || !d_q || !d_out) return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL plan or buffer");
    if (order != P2P_ORDER_PLAN && order != P2P_ORDER_USER) return set_error(P2P_ERROR_INVALID_ARGUMENT, "bad order");
    if (P->hp.local_input && order == P2P_ORDER_USER)
        return set_error(P2P_ERROR_NOT_SUPPORTED, "local-input plans: plan order only (no global user order here)");
    return guarded([&] {
        require_device(P);
        DeviceGuard g(P->device);
        cudaStream_t s = (cudaStream_t)stream;
        WsSlot slot(*P, s);
        if (P->elem == 4) apply_impl<float>(*P, d_q, d_out, order, accumulate ? 1 : 0, s);
        else apply_impl<double>(*P, d_q, d_out, order, accumulate ? 1 : 0, s);
    });
}

static p2p_status apply_host_common(p2p_plan P, const void *h_q, void *h_out, int32_t order, int32_t accumulate,
                                    void *stream, bool sync) {
    if (!P || !h_q || !h_out) return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL plan or buffer");
    if (order != P2P_ORDER_PLAN && order != P2P_ORDER_USER) return set_error(P2P_ERROR_INVALID_ARGUMENT, "bad order");
    if (P->hp.local_input) return set_error(P2P_ERROR_NOT_SUPPORTED, "local-input plans: p2p_apply_dist*");
    return guarded([&] {
        require_device(P);
        DeviceGuard g(P->device);
        cudaStream_t s = (cudaStream_t)stream;
        const p2p::HostPlan &hp = P->hp;
        WsSlot slot(*P, s);
        const size_t qb = (size_t)hp.n_src * P->elem * P->comps;
        const size_t ob = (size_t)(order == P2P_ORDER_USER ? hp.n_tgt : hp.n_tgt_local) * P->elem * P->comps;
        ck(cudaMemcpyAsync(P->io_q.p, h_q, qb, cudaMemcpyHostToDevice, s), "H2D q");
        if (accumulate) ck(cudaMemcpyAsync(P->io_out.p, h_out, ob, cudaMemcpyHostToDevice, s), "H2D out");
        if (P->elem == 4) apply_impl<float>(*P, P->io_q.p, P->io_out.p, order, accumulate ? 1 : 0, s);
        else apply_impl<double>(*P, P->io_q.p, P->io_out.p, order, accumulate ? 1 : 0, s);
        ck(cudaMemcpyAsync(h_out, P->io_out.p, ob, cudaMemcpyDeviceToHost, s), "D2H out");
        if (sync) ck(cudaStreamSynchronize(s), "apply_host sync");
    });
}

p2p_status p2p_apply_host(p2p_plan P, const void *h_q, void *h_out, int32_t order, int32_t accumulate,
                          void *stream) {
    return apply_host_common(P, h_q, h_out, order, accumulate, stream, true);
}

p2p_status p2p_apply_host_async(p2p_plan P, const void *h_q, void *h_out, int32_t order, int32_t accumulate,
                                void *stream) {
    return apply_host_common(P, h_q, h_out, order, accumulate, stream, false);
}

p2p_status p2p_apply_dist(p2p_plan P, const void *d_q_owned, const void *d_q_halo, void *d_out, int32_t accumulate,
                          void *stream) {
    p2p_status st = p2p_apply_dist_interior(P, d_q_owned, d_out, accumulate, stream);
    return st == P2P_SUCCESS ? p2p_apply_dist_boundary(P, d_q_halo, d_out, accumulate, stream) : st;
}

p2p_status p2p_apply_dist_interior(p2p_plan P, const void *d_q_owned, void *d_out, int32_t accumulate,
                                   void *stream) {
    Nvtx nvtx_("p2p_apply_dist interior");
    if (!P || !d_out) return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL plan or output");
    if (P->hp.n_src_owned && !d_q_owned) return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL d_q_owned");
    return guarded([&] {
        require_device(P);
        DeviceGuard g(P->device);
        cudaStream_t s = (cudaStream_t)stream;
        if (P->elem == 4) apply_dist_interior_impl<float>(*P, d_q_owned, d_out, accumulate ? 1 : 0, s);
        else apply_dist_interior_impl<double>(*P, d_q_owned, d_out, accumulate ? 1 : 0, s);
    });
}

p2p_status p2p_apply_dist_boundary(p2p_plan P, const void *d_q_halo, void *d_out, int32_t accumulate,
                                   void *stream) {
    Nvtx nvtx_("p2p_apply_dist boundary");
    if (!P || !d_out) return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL plan or output");
    if (P->hp.n_halo && !d_q_halo) return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL d_q_halo");
    return guarded([&] {
        require_device(P);
        DeviceGuard g(P->device);
        cudaStream_t s = (cudaStream_t)stream;
        if (P->elem == 4) apply_dist_boundary_impl<float>(*P, d_q_halo, d_out, accumulate ? 1 : 0, s);
        else apply_dist_boundary_impl<double>(*P, d_q_halo, d_out, accumulate ? 1 : 0, s);
    });
}

p2p_status p2p_apply_dist_peer(p2p_plan P, const void *d_q_owned, const void *const *d_peer_q, void *d_out,
                               int32_t accumulate, void *stream) {
    if (!P || !d_out || !d_peer_q) return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL plan, output or peer array");
    if (P->hp.n_src_owned && !d_q_owned) return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL d_q_owned");
    if (P->hp.part_world > 16) return set_error(P2P_ERROR_INVALID_ARGUMENT, "part_world > 16");
    return guarded([&] {
        require_device(P);
        DeviceGuard g(P->device);
        cudaStream_t s = (cudaStream_t)stream;
        const p2p::HostPlan &hp = P->hp;
        auto run = [&](auto tag, auto vtag) {
            using T = decltype(tag);     // plan precision
            using V = decltype(vtag);    // one weight: T, or (re, im) for complex kernels
            p2p::dev::PeerPtrs<V> pp{};
            for (int r = 0; r < hp.part_world; ++r) {
                pp.p[r] = r == hp.part_rank ? (const V *)d_q_owned : (const V *)d_peer_q[r];
                if (!pp.p[r] && r != hp.part_rank) throw p2p::Error(P2P_ERROR_INVALID_ARGUMENT, "NULL peer pointer");
            }
            if (hp.n_src_owned)
                ck(cudaMemcpyAsync((V *)P->q_local.p + hp.owned_local_begin, d_q_owned,
                                   (size_t)hp.n_src_owned * sizeof(V), cudaMemcpyDeviceToDevice, s),
                   "owned weights");
            if (hp.n_halo)
                p2p::dev::halo_peer_kernel<V><<<grid_for(hp.n_halo), 256, 0, s>>>(
                    pp, (const int32_t *)P->halo_owner.p, (const int32_t *)P->halo_oidx.p,
                    (const int32_t *)P->halo_lidx.p, (V *)P->q_local.p, hp.n_halo);
            launch_p2p<T>(*P, (const T *)P->q_local.p, (T *)d_out, accumulate ? 1 : 0, s);
            ck(cudaGetLastError(), "apply_dist_peer launch");
        };
        if (P->elem == 4 && P->comps == 1) run(float{}, float{});
        else if (P->elem == 4) run(float{}, float2{});
        else if (P->comps == 1) run(double{}, double{});
        else run(double{}, double2{});
    });
}

p2p_status p2p_gather_peer(p2p_plan P, const void *const *d_peer_out, void *d_global, void *stream) {
    if (!P || !d_peer_out || !d_global) return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL plan or buffer");
    return guarded([&] {
        require_device(P);
        DeviceGuard g(P->device);
        const p2p::HostPlan &hp = P->hp;
        const size_t el = (size_t)P->elem * P->comps;
        for (int r = 0; r < hp.part_world; ++r) {
            const int64_t n = hp.part_tgt[r + 1] - hp.part_tgt[r];
            if (!n) continue;
            if (!d_peer_out[r]) throw p2p::Error(P2P_ERROR_INVALID_ARGUMENT, "NULL peer output");
            ck(cudaMemcpyAsync((char *)d_global + (size_t)hp.part_tgt[r] * el, d_peer_out[r], (size_t)n * el,
                               cudaMemcpyDeviceToDevice, (cudaStream_t)stream),
               "gather_peer copy");
        }
    });
}

// ---- device-synchronised peer exchange (include/p2p.h p2p_peer_buffers .. p2p_gather)
p2p_status p2p_peer_buffers(p2p_plan P, void **d_pub_w, void **d_pub_o, void **d_sig) {
    if (!P || !d_pub_w || !d_pub_o || !d_sig) return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL pointer");
    if (P->hp.part_world > 16) return set_error(P2P_ERROR_INVALID_ARGUMENT, "part_world > 16");
    if (P->hp.layout == P2P_LAYOUT_ADAPTIVE || P->hp.layout == P2P_LAYOUT_PAPER_INDEXING ||
        P->hp.layout == P2P_LAYOUT_PAPER_REPETITION || P->hp.kernel == P2P_KERNEL_LAPLACE_3D ||
        P->hp.kernel == P2P_KERNEL_HELMHOLTZ_3D)
        return set_error(P2P_ERROR_NOT_SUPPORTED, "peer exchange: NR, R and TILED 2D plans");
    return guarded([&] {
        require_device(P);
        DeviceGuard g(P->device);
        auto &ps = P->peer;
        const p2p::HostPlan &hp = P->hp;
        const size_t el = (size_t)P->elem * P->comps;
        if (!ps.sig.p) {
            P->alloc(ps.pub_w, (size_t)std::max<int64_t>(hp.n_send, 1) * el);
            P->alloc(ps.pub_o, (size_t)std::max<int64_t>(hp.n_tgt_local, 1) * el);
            P->alloc(ps.sig, p2p::dev::kSigWords * sizeof(unsigned long long));
            P->alloc(ps.ctr, 4 * sizeof(unsigned));
            P->alloc(ps.err, sizeof(int));
            ck(cudaMemset(ps.sig.p, 0, ps.sig.bytes), "peer signal init");
            ck(cudaMemset(ps.ctr.p, 0, ps.ctr.bytes), "peer counter init");
            ck(cudaMemset(ps.err.p, 0, ps.err.bytes), "peer error init");
            ck(cudaDeviceSynchronize(), "peer buffers");  // zeroed before any peer can map them
        }
        *d_pub_w = ps.pub_w.p;
        *d_pub_o = ps.pub_o.p;
        *d_sig = ps.sig.p;
    });
}

p2p_status p2p_peer_connect(p2p_plan P, const void *const *peer_pub_w, const void *const *peer_pub_o,
                            const void *const *peer_sig, const int64_t *displ) {
    if (!P || !peer_pub_w || !peer_pub_o || !peer_sig || !displ)
        return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL pointer");
    if (!P->peer.sig.p) return set_error(P2P_ERROR_INVALID_ARGUMENT, "p2p_peer_buffers first");
    return guarded([&] {
        DeviceGuard g(P->device);
        auto &ps = P->peer;
        const p2p::HostPlan &hp = P->hp;
        const int W = hp.part_world, me = hp.part_rank;
        ps.readers_w = ps.owners_w = 0;
        ps.all = W >= 32 ? ~0u : (1u << W) - 1u;
        std::vector<int64_t> base((size_t)W + 1, 0);
        for (int r = 0; r < W; ++r) {
            if (!peer_pub_w[r] || !peer_pub_o[r] || !peer_sig[r])
                throw p2p::Error(P2P_ERROR_INVALID_ARGUMENT, "NULL peer pointer");
            ps.pub_w_peer[r] = const_cast<void *>(peer_pub_w[r]);
            ps.pub_o_peer[r] = const_cast<void *>(peer_pub_o[r]);
            ps.sig_peer[r] = const_cast<void *>(peer_sig[r]);
            if (r != me && hp.send_counts[r] > 0) ps.readers_w |= 1u << r;
            if (r != me && hp.recv_counts[r] > 0) ps.owners_w |= 1u << r;
            base[r + 1] = base[r] + hp.recv_counts[r];
        }
        // per halo slot: its index in the owner's published send buffer (the owner packs, per
        // reader, that reader's halo in the reader's order -- the all-to-all layout)
        std::vector<int32_t> oidx((size_t)hp.n_halo);
        for (int o = 0, h = 0; o < W; ++o)
            for (int64_t k = 0; k < hp.recv_counts[o]; ++k, ++h) oidx[h] = (int32_t)(displ[o] + k);
        if (ps.oidx_w.p) cudaFree(ps.oidx_w.p), ps.oidx_w = DevBuf{};
        if (ps.seg_o.p) cudaFree(ps.seg_o.p), ps.seg_o = DevBuf{};
        P->upload(ps.oidx_w, oidx);
        P->upload(ps.seg_o, hp.part_tgt);
        ck(cudaStreamSynchronize(P->stream), "peer connect upload");
        if (!ps.side) ck(cudaStreamCreateWithFlags(&ps.side, cudaStreamNonBlocking), "peer side stream");
        if (!ps.ev_pub) ck(cudaEventCreateWithFlags(&ps.ev_pub, cudaEventDisableTiming), "peer event");
        if (!ps.ev_pull) ck(cudaEventCreateWithFlags(&ps.ev_pull, cudaEventDisableTiming), "peer event");
        ps.connected = true;
    });
}

extern "C++" {
namespace {
template <typename T, typename V>
void apply_peer_sync_impl(p2p_plan_s &P, const void *d_q_owned, void *d_out, int accumulate, cudaStream_t s) {
    namespace D = p2p::dev;
    auto &ps = P.peer;
    const p2p::HostPlan &hp = P.hp;
    unsigned *ctr = (unsigned *)ps.ctr.p;
    unsigned long long *sig = (unsigned long long *)ps.sig.p;
    D::PeerPtrs<V> pub{};
    D::SigPtrs sp{};
    for (int r = 0; r < hp.part_world; ++r) {
        pub.p[r] = (const V *)ps.pub_w_peer[r];
        sp.p[r] = (unsigned long long *)ps.sig_peer[r];
    }
    // 1. publish this epoch's send buffer (after every reader is done with the previous one)
    Nvtx n1("publish + pull halo (exchange)");
    D::peer_publish_kernel<V><<<grid_for(std::max<int64_t>(hp.n_send, 1)), 256, 0, s>>>(
        (const int32_t *)P.send_idx.p, (const V *)d_q_owned, (V *)ps.pub_w.p, hp.n_send, sig, 0, ps.readers_w, ctr,
        (int *)ps.err.p);
    ck(cudaEventRecord(ps.ev_pub, s), "peer event");
    // 2. side stream: pull the halo straight from the owners' published buffers
    ck(cudaStreamWaitEvent(ps.side, ps.ev_pub, 0), "peer fork");
    D::peer_pull_kernel<V><<<grid_for(std::max<int64_t>(hp.n_halo, 1)), 256, 0, ps.side>>>(
        pub, sp, sig, 0, hp.part_rank, ps.owners_w, (const int32_t *)P.halo_owner.p, (const int32_t *)ps.oidx_w.p,
        nullptr, 0, (const int32_t *)P.halo_lidx.p, (V *)P.q_local.p, hp.n_halo, ctr + 1, (int *)ps.err.p);
    ck(cudaEventRecord(ps.ev_pull, ps.side), "peer event");
    // 3. interior tiles meanwhile; 4. boundary tiles once the halo is in
    { Nvtx n2("interior tiles"); apply_dist_interior_impl<T>(P, d_q_owned, d_out, accumulate, s); }
    Nvtx n3("boundary tiles");
    ck(cudaStreamWaitEvent(s, ps.ev_pull, 0), "peer join");
    if (hp.layout == P2P_LAYOUT_TILED)
        launch_p2p<T>(P, (const T *)P.q_local.p, (T *)d_out, accumulate, s, false, hp.n_interior,
                      (int64_t)hp.tiles.size());
    else
        launch_p2p<T>(P, (const T *)P.q_local.p, (T *)d_out, accumulate, s);
    ck(cudaGetLastError(), "apply_peer_sync launch");
}

template <typename V>
void gather_sync_impl(p2p_plan_s &P, const void *d_local, void *d_global, cudaStream_t s) {
    namespace D = p2p::dev;
    auto &ps = P.peer;
    const p2p::HostPlan &hp = P.hp;
    unsigned *ctr = (unsigned *)ps.ctr.p;
    unsigned long long *sig = (unsigned long long *)ps.sig.p;
    D::PeerPtrs<V> pub{};
    D::SigPtrs sp{};
    for (int r = 0; r < hp.part_world; ++r) {
        pub.p[r] = (const V *)ps.pub_o_peer[r];
        sp.p[r] = (unsigned long long *)ps.sig_peer[r];
    }
    D::peer_publish_kernel<V><<<grid_for(std::max<int64_t>(hp.n_tgt_local, 1)), 256, 0, s>>>(
        nullptr, (const V *)d_local, (V *)ps.pub_o.p, hp.n_tgt_local, sig, 1, ps.all, ctr + 2, (int *)ps.err.p);
    D::peer_pull_kernel<V><<<grid_for(std::max<int64_t>(hp.n_tgt, 1)), 256, 0, s>>>(
        pub, sp, sig, 1, hp.part_rank, ps.all, nullptr, nullptr, (const int64_t *)ps.seg_o.p, hp.part_world, nullptr,
        (V *)d_global, hp.n_tgt, ctr + 3, (int *)ps.err.p);
    ck(cudaGetLastError(), "gather launch");
}
}  // namespace
}  // extern "C++"

p2p_status p2p_apply_peer_sync(p2p_plan P, const void *d_q_owned, void *d_out, int32_t accumulate, void *stream) {
    Nvtx nvtx_("p2p_apply_peer_sync");
    if (!P || !d_out) return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL plan or output");
    if (P->hp.n_src_owned && !d_q_owned) return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL d_q_owned");
    if (!P->peer.connected) return set_error(P2P_ERROR_INVALID_ARGUMENT, "p2p_peer_connect first");
    return guarded([&] {
        require_device(P);
        DeviceGuard g(P->device);
        cudaStream_t s = (cudaStream_t)stream;
        const int a = accumulate ? 1 : 0;
        if (P->elem == 4 && P->comps == 1) apply_peer_sync_impl<float, float>(*P, d_q_owned, d_out, a, s);
        else if (P->elem == 4) apply_peer_sync_impl<float, float2>(*P, d_q_owned, d_out, a, s);
        else if (P->comps == 1) apply_peer_sync_impl<double, double>(*P, d_q_owned, d_out, a, s);
        else apply_peer_sync_impl<double, double2>(*P, d_q_owned, d_out, a, s);
    });
}

p2p_status p2p_gather(p2p_plan P, const void *d_local, void *d_global, void *stream) {
    Nvtx nvtx_("p2p_gather (allgatherv)");
    if (!P || !d_global) return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL plan or output");
    if (P->hp.n_tgt_local && !d_local) return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL d_local");
    if (!P->peer.connected) return set_error(P2P_ERROR_INVALID_ARGUMENT, "p2p_peer_connect first");
    return guarded([&] {
        require_device(P);
        DeviceGuard g(P->device);
        cudaStream_t s = (cudaStream_t)stream;
        if (P->elem == 4 && P->comps == 1) gather_sync_impl<float>(*P, d_local, d_global, s);
        else if (P->elem == 4) gather_sync_impl<float2>(*P, d_local, d_global, s);
        else if (P->comps == 1) gather_sync_impl<double>(*P, d_local, d_global, s);
        else gather_sync_impl<double2>(*P, d_local, d_global, s);
    });
}

p2p_status p2p_peer_check(p2p_plan P) {
    if (!P) return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL plan");
    if (!P->peer.err.p) return P2P_SUCCESS;
    int e = 0;
    p2p_status st = guarded([&] {
        DeviceGuard g(P->device);
        ck(cudaMemcpy(&e, P->peer.err.p, sizeof(int), cudaMemcpyDeviceToHost), "peer error word");
    });
    if (st != P2P_SUCCESS) return st;
    return e ? set_error(P2P_ERROR_CUDA, "peer exchange: a wait for a peer's signal timed out") : P2P_SUCCESS;
}

p2p_status p2p_ipc_export(const void *d_ptr, void *handle64, int64_t *offset) {
    if (!d_ptr || !handle64 || !offset) return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL pointer");
    return guarded([&] {
        // base of the allocation holding d_ptr (driver cuMemGetAddressRange through the runtime)
        typedef int (*range_fn)(unsigned long long *, size_t *, unsigned long long);
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        ck(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q), "driver entry point");
        if (!fn || q != cudaDriverEntryPointSuccess) throw p2p::Error(P2P_ERROR_CUDA, "cuMemGetAddressRange unavailable");
        unsigned long long base = 0;
        size_t size = 0;
        if (((range_fn)fn)(&base, &size, (unsigned long long)(uintptr_t)d_ptr) != 0)
            throw p2p::Error(P2P_ERROR_CUDA, "cuMemGetAddressRange failed");
        cudaIpcMemHandle_t h;
        ck(cudaIpcGetMemHandle(&h, (void *)(uintptr_t)base), "cudaIpcGetMemHandle");
        static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
        std::memcpy(handle64, &h, sizeof(h));
        *offset = (int64_t)((uintptr_t)d_ptr - base);
    });
}

p2p_status p2p_ipc_open(const void *handle64, int64_t offset, int32_t device, void **d_ptr) {
    if (!handle64 || !d_ptr) return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL pointer");
    *d_ptr = nullptr;
    return guarded([&] {
        DeviceGuard g(device);
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle64, sizeof(h));
        void *base = nullptr;
        ck(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
        *d_ptr = (char *)base + offset;
    });
}

p2p_status p2p_ipc_close(void *d_ptr, int64_t offset) {
    if (!d_ptr) return P2P_SUCCESS;
    return guarded([&] { ck(cudaIpcCloseMemHandle((char *)d_ptr - offset), "cudaIpcCloseMemHandle"); });
}

p2p_status p2p_halo_pack(p2p_plan P, const void *d_q_owned, void *d_send, void *stream) {
    Nvtx nvtx_("p2p_halo_pack (exchange)");
    if (!P) return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL plan");
    if (P->hp.n_send && (!d_q_owned || !d_send)) return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL buffer");
    return guarded([&] {
        require_device(P);
        DeviceGuard g(P->device);
        cudaStream_t s = (cudaStream_t)stream;
        const int64_t n = P->hp.n_send;
        if (!n) return;
        const int32_t *ix = (const int32_t *)P->send_idx.p;
        if (P->elem == 4 && P->comps == 1)
            p2p::dev::gather_kernel<float><<<grid_for(n), 256, 0, s>>>(ix, (const float *)d_q_owned, (float *)d_send, n);
        else if (P->elem == 4)
            p2p::dev::gather_kernel<float2><<<grid_for(n), 256, 0, s>>>(ix, (const float2 *)d_q_owned, (float2 *)d_send, n);
        else if (P->comps == 1)
            p2p::dev::gather_kernel<double><<<grid_for(n), 256, 0, s>>>(ix, (const double *)d_q_owned, (double *)d_send, n);
        else
            p2p::dev::gather_kernel<double2><<<grid_for(n), 256, 0, s>>>(ix, (const double2 *)d_q_owned, (double2 *)d_send,
                                                                         n);
        ck(cudaGetLastError(), "halo_pack launch");
    });
}

p2p_status p2p_destroy(p2p_plan P) {
    if (!P) return P2P_SUCCESS;
    if (P->device >= 0) {
        int prev = -1;
        cudaGetDevice(&prev);
        cudaSetDevice(P->device);
        P->release();
        if (prev >= 0) cudaSetDevice(prev);
    }
    delete P;
    return P2P_SUCCESS;
}

p2p_status p2p_plan_get_info(p2p_plan P, p2p_plan_info *out) {
    if (!P || !out) return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL plan or info");
    const uint32_t want = out->struct_size;
    if (want && want < offsetof(p2p_plan_info, level))
        return set_error(P2P_ERROR_INVALID_ARGUMENT, "p2p_plan_info.struct_size too small");
    const size_t n = want && want < sizeof(p2p_plan_info) ? want : sizeof(p2p_plan_info);
    const p2p::HostPlan &hp = P->hp;
    p2p_plan_info full;
    p2p_plan_info *info = &full;
    std::memset(info, 0, sizeof(*info));
    info->struct_size = (uint32_t)n;
    info->level = hp.L;
    info->tile_log2 = hp.k;
    info->layout = hp.layout;
    info->precision = hp.precision;
    info->device = P->device;
    info->part_world = hp.part_world;
    info->part_rank = hp.part_rank;
    info->side = hp.S;
    info->boxes = hp.B;
    info->n_src = hp.n_src;
    info->n_tgt = hp.n_tgt;
    info->n_src_local = hp.n_src_local;
    info->n_tgt_local = hp.n_tgt_local;
    info->n_src_owned = hp.n_src_owned;
    info->src_owned_begin = hp.src_owned_begin;
    info->tgt_begin = hp.tgt_begin;
    info->n_halo = hp.n_halo;
    info->n_send = hp.n_send;
    info->occupied_src_boxes = hp.occ_src;
    info->occupied_tgt_boxes = hp.occ_tgt;
    info->t_max = hp.t_max;
    info->density = hp.density;
    info->density_occupied = hp.density_occ;
    info->pairs = hp.pairs;
    info->pairs_global = hp.pairs_global;
    info->tiles = (int64_t)hp.tiles.size();
    info->smem_bytes = hp.smem_bytes;
    info->halo_entries = hp.halo_entries;
    const int64_t e = (hp.precision == P2P_FP32 ? 4 : 8) * (int64_t)P->comps;  // bytes per weight / result
    const int64_t offs = 8 * hp.boxes_in_tiles;  // tgt + src CSR offsets of the tiles' boxes
    info->alg_bytes_kernel = hp.n_tgt_local * 3 * e + hp.n_src_local * 3 * e + offs;
    if (hp.layout == P2P_LAYOUT_NONREDUNDANT) {
        info->layout_bytes_apply = info->alg_bytes_kernel;
    } else if (hp.layout == P2P_LAYOUT_TILED) {
        // targets: region-relative coords + row-run base (+ output index) + out; region: coords +
        // index; tables; weights gathered once from plan order
        info->layout_bytes_apply = hp.n_tgt_local * (3 * e + 2 + (hp.lean ? 2 : 0)) +
                                   hp.reg_entries * (2 * e + 4) + hp.table_entries * 2 +
                                   hp.n_src_local * e;
    } else {
        info->layout_bytes_apply = hp.n_tgt_local * 3 * e + hp.halo_entries * 3 * e + offs +
                                   hp.halo_entries * (4 + e) + hp.n_src_local * e;
    }
    info->device_bytes = P->device_bytes;
    info->build_seconds = hp.build_seconds;
    info->upload_seconds = P->upload_seconds;
    info->cta_threads = hp.layout == P2P_LAYOUT_TILED ? hp.nt : p2p::kThreads;
    info->slots_per_unit = hp.tpi;
    info->items_per_unit = hp.layout == P2P_LAYOUT_TILED ? hp.ns : 3;
    info->flags = (hp.tsort ? 1 : 0) | (hp.flat ? 2 : 0);
    info->interior_launches = hp.layout == P2P_LAYOUT_TILED ? hp.n_interior : 0;
    info->paper_model_bytes = hp.paper_model_bytes;
    info->record_stride = hp.pr_stride;
    info->launches = (int64_t)hp.tiles.size();
    info->kernel = hp.kernel;
    info->components = P->comps;
    info->wavenumber = hp.kappa;
    std::memcpy(out, info, n);
    return P2P_SUCCESS;
}

p2p_status p2p_plan_export(p2p_plan P, int32_t kind, void *host_dst, size_t *bytes) {
    if (!P || !bytes) return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL plan or bytes");
    return guarded([&] {
        mirror_device_plan(*P);
        const p2p::HostPlan &hp = P->hp;
        std::vector<int64_t> v;
        auto take = [&](const auto &src) { v.assign(src.begin(), src.end()); };
        switch (kind) {
        case P2P_EXPORT_SRC_PERM: take(hp.src_uidx); break;
        case P2P_EXPORT_TGT_PERM: take(hp.tgt_uidx); break;
        case P2P_EXPORT_SRC_BOX_OFFSETS: take(hp.src_off_g); break;
        case P2P_EXPORT_TGT_BOX_OFFSETS: take(hp.tgt_off_g); break;
        case P2P_EXPORT_NEIGHBORS: v = p2p::neighbors_export(hp); break;
        case P2P_EXPORT_PARTITION:
            v.assign(hp.part_src.begin(), hp.part_src.end());
            v.insert(v.end(), hp.part_tgt.begin(), hp.part_tgt.end());
            break;
        case P2P_EXPORT_SRC_GLOBAL: take(hp.src_gidx); break;
        case P2P_EXPORT_HALO_COUNTS:
            v.assign(hp.recv_counts.begin(), hp.recv_counts.end());
            v.insert(v.end(), hp.send_counts.begin(), hp.send_counts.end());
            break;
        case P2P_EXPORT_TILES: take(hp.tiles); break;
        case P2P_EXPORT_HALO_INDEX: take(hp.halo_idx); break;
        case P2P_EXPORT_SEND_INDEX: take(hp.send_idx); break;
        case P2P_EXPORT_HALO_OFFSETS: take(hp.halo_off); break;
        case P2P_EXPORT_REGION_OFFSETS: take(hp.reg_off); break;
        case P2P_EXPORT_REGION_INDEX: take(hp.reg_idx); break;
        case P2P_EXPORT_REGION_TABLE: take(hp.reg_table); break;
        case P2P_EXPORT_SLOT_OFFSETS: take(hp.tgt_pack_off); break;
        case P2P_EXPORT_SLOT_BASE: take(hp.tgt_bl); break;
        case P2P_EXPORT_SLOT_OUTPUT:
            take(hp.tgt_oix);
            for (int64_t &x : v) x = x == 0xFFFF ? -1 : x;
            break;
        case P2P_EXPORT_ITEM_OFFSETS: take(hp.item_off); break;
        case P2P_EXPORT_ITEMS: take(hp.items); break;
        case P2P_EXPORT_PAPER_NEI_OFFSETS: take(hp.pi_nei_off); break;
        case P2P_EXPORT_PAPER_NEI_INDEX: take(hp.pi_nei_idx); break;
        case P2P_EXPORT_PAPER_RECORDS: {
            std::vector<double> rec = hp.pr_records;
            if (P->pr_records.p && P->device >= 0) {  // as of the last apply (q slots filled)
                DeviceGuard g(P->device);
                ck(cudaMemcpy(rec.data(), P->pr_records.p, rec.size() * 8, cudaMemcpyDeviceToHost), "records D2H");
            }
            v.resize(rec.size());
            std::memcpy(v.data(), rec.data(), rec.size() * 8);
            break;
        }
        case P2P_EXPORT_LEAVES:
            for (size_t i = 0; i < hp.leaf_lvl.size(); ++i) {
                v.push_back(hp.leaf_lvl[i]);
                v.push_back(hp.leaf_ix[i]);
                v.push_back(hp.leaf_iy[i]);
            }
            break;
        case P2P_EXPORT_ULIST_OFFSETS: take(hp.ul_off); break;
        case P2P_EXPORT_ULIST: take(hp.ul_leaf); break;
        case P2P_EXPORT_LAUNCH:
            take(hp.tile_slot);
            v.insert(v.end(), hp.tile_part.begin(), hp.tile_part.end());
            break;
        default: throw p2p::Error(P2P_ERROR_INVALID_ARGUMENT, "unknown export kind");
        }
        const size_t need = v.size() * sizeof(int64_t);
        if (!host_dst) {
            *bytes = need;
            return;
        }
        if (*bytes < need) throw p2p::Error(P2P_ERROR_INVALID_ARGUMENT, "export buffer too small");
        if (need) std::memcpy(host_dst, v.data(), need);
        *bytes = need;
    });
}

const char *p2p_status_string(p2p_status s) {
    switch (s) {
    case P2P_SUCCESS: return "P2P_SUCCESS";
    case P2P_ERROR_INVALID_ARGUMENT: return "P2P_ERROR_INVALID_ARGUMENT";
    case P2P_ERROR_CONSTRUCTION_FAILURE: return "P2P_ERROR_CONSTRUCTION_FAILURE";
    case P2P_ERROR_LAYOUT_CORRUPT: return "P2P_ERROR_LAYOUT_CORRUPT";
    case P2P_ERROR_OUT_OF_MEMORY: return "P2P_ERROR_OUT_OF_MEMORY";
    case P2P_ERROR_CUDA: return "P2P_ERROR_CUDA";
    case P2P_ERROR_NOT_SUPPORTED: return "P2P_ERROR_NOT_SUPPORTED";
    case P2P_ERROR_NO_DEVICE: return "P2P_ERROR_NO_DEVICE";
    }
    return "P2P_ERROR_UNKNOWN";
}

const char *p2p_last_error(void) { return g_last_error.c_str(); }

int32_t p2p_abi_version(void) { return P2P_ABI_VERSION; }

// Diagnostics only (not part of include/p2p.h): per-tile timeline of the TILED
// kernel -- d_trace = device buffer of 8 x uint64 per tile (queue position):
// {smid << 32 | cta, t_claim, t_data, t_units, -, t_end, units, entries}
// in %globaltimer ns; NULL disables.
// Undeclared diagnostics hook: PAPER_REPETITION applies skip the weight pack (the records keep the
// weights of the last full apply), so the repetition kernel can be timed alone.
p2p_status p2p_internal_paper_kernel_only(p2p_plan P, int on) {
    if (!P) return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL plan");
    P->paper_kernel_only = on != 0;
    return P2P_SUCCESS;
}

p2p_status p2p_internal_set_trace(p2p_plan P, void *d_trace) {
    if (!P) return set_error(P2P_ERROR_INVALID_ARGUMENT, "NULL plan");
    P->trace = (unsigned long long *)d_trace;
    return P2P_SUCCESS;
}

}  // extern "C"
