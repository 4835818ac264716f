// plan_builder.cpp -- host-side plan builder ("data collection", PAPER.md
// §3.2 L79 and §3.3, re-derived for B200).
//
// Steps:
//   a1 level selection: explicit L, or the CT loop of PAPER.md §3.1
//      (start at l_start, L += 1 until no leaf holds more than CT sources or
//      CT targets), then L += level_delta (§4.6 Eq. 37).
//   a2 box assignment: ix = min(floor(x*S), S-1) -> Morton code.
//   a3 stable counting sort by Morton code -> permutation + CSR box offsets
//      (the paper's "second order index").
//   a4 E1 neighbourhoods are implicit (3x3 block, clipped); an
//      explicit list is only materialised for export.
//   a5 NR layout (Morton-sorted box-local coordinates) and R layout (per
//      target box, the packed halo of its E1 sources; §3.3).
// Plus CTA tiling, exact int64 pair counts and the Morton-range partition
// across ranks.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <numeric>
#include <thread>

#include "plan.h"

#include <cstdlib>

namespace p2p {

namespace {

[[noreturn]] void fail(p2p_status c, const std::string &m) { throw Error(c, m); }

template <typename F>
void parallel_for(int64_t n, F f, int64_t grain = 1 << 15) {
    unsigned hw = std::thread::hardware_concurrency();
    unsigned nt = std::max(1u, std::min(hw ? hw : 1u, 64u));
    if (n <= grain || nt == 1) {
        f(int64_t(0), n);
        return;
    }
    nt = (unsigned)std::min<int64_t>(nt, (n + grain - 1) / grain);
    std::vector<std::thread> th;
    int64_t chunk = (n + nt - 1) / nt;
    for (unsigned t = 0; t < nt; ++t) {
        int64_t a = (int64_t)t * chunk, b = std::min(n, a + chunk);
        if (a >= b) break;
        th.emplace_back([=] { f(a, b); });
    }
    for (auto &x : th) x.join();
}

inline uint32_t cell_of(double x, int64_t S) {
    // floor(x*S) is exact: S is a power of two.  Closed at the upper edge.
    int64_t c = (int64_t)std::floor(x * (double)S);
    if (c > S - 1) c = S - 1;
    if (c < 0) c = 0;
    return (uint32_t)c;
}

inline int64_t pad2(int64_t n) { return (n + 1) & ~int64_t(1); }
inline int64_t pad4(int64_t n) { return (n + 3) & ~int64_t(3); }
inline int64_t pad8(int64_t n) { return (n + 7) & ~int64_t(7); }

void validate_points(const double *xy, int64_t n, const char *what) {
    if (n < 1) fail(P2P_ERROR_INVALID_ARGUMENT, std::string(what) + ": n must be >= 1 (SPEC.md L55)");
    if (!xy) fail(P2P_ERROR_INVALID_ARGUMENT, std::string(what) + ": NULL coordinates");
    for (int64_t i = 0; i < 2 * n; ++i) {
        double v = xy[i];
        if (!(v >= 0.0 && v <= 1.0))  // also rejects NaN
            fail(P2P_ERROR_INVALID_ARGUMENT, std::string(what) + ": coordinate " + std::to_string(i / 2) +
                                                 " outside the unit square [0,1]^2 (SPEC.md L119)");
    }
}

// Max number of points sharing one cell at level L, from codes sorted at
// level lref >= L (a Morton code's prefix is the parent box: code_L = code >> 2(lref-L)).
int64_t max_run(const std::vector<uint32_t> &sorted, int shift) {
    int64_t best = 0, run = 0;
    uint32_t prev = 0;
    for (size_t i = 0; i < sorted.size(); ++i) {
        uint32_t c = sorted[i] >> shift;
        run = (i && c == prev) ? run + 1 : 1;
        prev = c;
        best = std::max(best, run);
    }
    return best;
}

// a1: PAPER.md §3.1 L67-69 tree-construction loop.
int ct_loop_level(const p2p_plan_desc &d) {
    int lmax = std::min(d.l_max, kMaxLevel);
    if (d.l_start < 1) fail(P2P_ERROR_INVALID_ARGUMENT, "l_start must be >= 1");
    if (d.ct < 1) fail(P2P_ERROR_INVALID_ARGUMENT, "ct must be >= 1");
    int64_t Sref = int64_t(1) << (lmax - 1);
    auto codes = [&](const double *xy, int64_t n) {
        std::vector<uint32_t> c((size_t)n);
        parallel_for(n, [&](int64_t a, int64_t b) {
            for (int64_t i = a; i < b; ++i)
                c[i] = morton_encode(cell_of(xy[2 * i], Sref), cell_of(xy[2 * i + 1], Sref));
        });
        std::sort(c.begin(), c.end());
        return c;
    };
    std::vector<uint32_t> cs = codes(d.src_xy, d.n_src), ct = codes(d.tgt_xy, d.n_tgt);
    for (int L = std::max(1, d.l_start); L <= lmax; ++L) {
        int shift = 2 * (lmax - L);
        if (max_run(cs, shift) <= d.ct && max_run(ct, shift) <= d.ct) return L;
    }
    fail(P2P_ERROR_CONSTRUCTION_FAILURE,
         "CT loop: some leaf box still holds more than CT points at L = " + std::to_string(lmax) +
             " (cap; SPEC.md L75)");
}

// a2 + a3: stable counting sort of points by Morton code of their leaf box.
void csr_sort(const double *xy, int64_t n, const HostPlan &hp, std::vector<int32_t> &off,
              std::vector<int32_t> &perm) {
    std::vector<uint32_t> code((size_t)n);
    parallel_for(n, [&](int64_t a, int64_t b) {
        for (int64_t i = a; i < b; ++i)
            code[i] = morton_encode(cell_of(xy[2 * i], hp.S), cell_of(xy[2 * i + 1], hp.S));
    });
    off.assign((size_t)hp.B + 1, 0);
    for (int64_t i = 0; i < n; ++i) off[code[i] + 1] += 1;
    for (int64_t b = 0; b < hp.B; ++b) off[b + 1] += off[b];
    std::vector<int32_t> pos(off.begin(), off.end() - 1);
    perm.resize((size_t)n);
    for (int64_t i = 0; i < n; ++i) perm[pos[code[i]]++] = (int32_t)i;
}

// Item layout for the kernel's mapping (position p -> round p / nt, warp (p % nt) / 32,
// lane p % 32) from items sorted by descending length: 32-item batches (sorted, so the
// lanes of a batch sweep near-equal runs) are dealt to warps longest-processing-time
// first, so every warp of the CTA reaches the tile's barrier at about the same time.
// The partial batch (if any) takes the one partial slot, which the mapping gives to
// the last position's warp.
void balance_batches(const std::vector<int32_t> &ord, const std::vector<int32_t> &len, int nt,
                     std::vector<int32_t> &lay) {
    const int64_t n = (int64_t)ord.size(), nw = nt / 32;
    lay.assign(ord.begin(), ord.end());
    if (n <= 32 || nw <= 1) return;
    const int64_t nb = (n + 31) / 32;  // batches; the last one may be partial
    // slots: position blocks of 32 in kernel order; slot s covers positions [32 s, 32 s + 32)
    std::vector<int64_t> load((size_t)nw, 0);
    std::vector<std::vector<int64_t>> slots((size_t)nw);
    for (int64_t sl = 0; sl < nb; ++sl) slots[(size_t)((sl * 32 % nt) / 32)].push_back(sl);
    std::vector<int64_t> free_full((size_t)nw, 0);
    const bool partial = n % 32 != 0;
    for (int64_t w = 0; w < nw; ++w)
        for (int64_t sl : slots[(size_t)w]) free_full[(size_t)w] += !(partial && sl == nb - 1);
    std::vector<int64_t> slot_of_batch((size_t)nb, -1);
    if (partial) {  // the partial batch (the shortest items) fills the partial slot
        const int64_t w = ((nb - 1) * 32 % nt) / 32;
        slot_of_batch[(size_t)(nb - 1)] = nb - 1;
        load[(size_t)w] += len[(size_t)ord[(size_t)((nb - 1) * 32)]];
    }
    std::vector<size_t> next((size_t)nw, 0);
    for (int64_t b = 0; b < nb - (partial ? 1 : 0); ++b) {  // batch b: items [32 b, 32 b + 32), longest first
        int64_t best = -1;
        for (int64_t w = 0; w < nw; ++w)
            if (free_full[(size_t)w] > 0 && (best < 0 || load[(size_t)w] < load[(size_t)best])) best = w;
        // the batch's duration ~ its longest item (lanes run in lockstep)
        load[(size_t)best] += len[(size_t)ord[(size_t)(32 * b)]];
        --free_full[(size_t)best];
        while (partial && slots[(size_t)best][next[(size_t)best]] == nb - 1) ++next[(size_t)best];
        slot_of_batch[(size_t)b] = slots[(size_t)best][next[(size_t)best]++];
    }
    for (int64_t b = 0; b < nb; ++b) {
        const int64_t sl = slot_of_batch[(size_t)b];
        for (int64_t x = 0; x < 32 && 32 * b + x < n; ++x) lay[(size_t)(32 * sl + x)] = ord[(size_t)(32 * b + x)];
    }
}

}  // namespace

// fp64 log tables, the log from the 64-bit-mantissa long double logl:
//   [0, kLogTab): (c_inv_k, -log c_inv_k), c_inv_k = 1 / (1 + (k + 1/2) / kLogTab) rounded to
//     double -- the shared-memory table of the kernels' `log_tab`;
//   then kLogTab32 entries (c_k, -log c_k), c_k = 1 / (1 + (k + 1/2) / 32) rounded to FLOAT (held
//     exactly in the double) -- the warp-register table of `log_shfl` (lane k holds entry k);
//   then kLogTab8 entries (c_inv_k, -log c_inv_k), c_inv_k = 1 / (1 + (k + 1/2) / 64) -- staged
//     8-fold in shared memory by the dense fp64 TILED kernel (`log_tab8`).
void build_log_table(HostPlan &hp) {
    hp.log_tab.resize(2 * (kLogTab + kLogTab32 + kLogTab8));
    for (int kk = 0; kk < kLogTab; ++kk) {
        const double c = 1.0 + (kk + 0.5) / kLogTab;
        const double cinv = 1.0 / c;
        hp.log_tab[2 * kk] = cinv;
        hp.log_tab[2 * kk + 1] = (double)(-logl((long double)cinv));
    }
    for (int kk = 0; kk < kLogTab32; ++kk) {
        const float cinv = (float)(1.0 / (1.0 + (kk + 0.5) / kLogTab32));
        hp.log_tab[2 * (kLogTab + kk)] = (double)cinv;
        hp.log_tab[2 * (kLogTab + kk) + 1] = (double)(-logl((long double)cinv));
    }
    for (int kk = 0; kk < kLogTab8; ++kk) {  // then kLogTab8 entries (c_inv_k, -log c_inv_k) for log_tab8
        const double cinv = 1.0 / (1.0 + (kk + 0.5) / kLogTab8);
        hp.log_tab[2 * (kLogTab + kLogTab32 + kk)] = cinv;
        hp.log_tab[2 * (kLogTab + kLogTab32 + kk) + 1] = (double)(-logl((long double)cinv));
    }
}

// Kernel function and its envelope (include/p2p.h p2p_kernel): Helmholtz runs on the TILED
// layout, one partition.
void check_kernel(const p2p_plan_desc &d) {
    if (d.kernel == P2P_KERNEL_LAPLACE_2D) return;
    if (d.kernel < P2P_KERNEL_HELMHOLTZ_2D || d.kernel > P2P_KERNEL_HELMHOLTZ_3D)
        fail(P2P_ERROR_INVALID_ARGUMENT, "bad kernel");
    if (d.kernel != P2P_KERNEL_LAPLACE_3D && (!(d.wavenumber > 0.0) || !std::isfinite(d.wavenumber)))
        fail(P2P_ERROR_INVALID_ARGUMENT, "Helmholtz kernels need wavenumber > 0");
    if (d.kernel == P2P_KERNEL_HELMHOLTZ_2D && d.layout != P2P_LAYOUT_TILED)
        fail(P2P_ERROR_NOT_SUPPORTED, "HELMHOLTZ_2D runs on the TILED layout");
    if (kernel_dim(d.kernel) == 3 && d.layout != P2P_LAYOUT_NONREDUNDANT)
        fail(P2P_ERROR_NOT_SUPPORTED, "3D kernels run on the NONREDUNDANT (box-per-CTA) layout");
    if (d.part_world != 1 && d.kernel != P2P_KERNEL_HELMHOLTZ_2D)
        fail(P2P_ERROR_NOT_SUPPORTED, "3D kernels: one partition");
}

// ---- ADAPTIVE: the CT-driven quadtree, per box (§3.1
// applied locally), and U-lists of touching leaves.
void build_host_plan_adaptive(const p2p_plan_desc &d, HostPlan &hp) {
    auto t0 = std::chrono::steady_clock::now();
    if (d.kernel != P2P_KERNEL_LAPLACE_2D) fail(P2P_ERROR_NOT_SUPPORTED, "ADAPTIVE: LAPLACE_2D");
    if (d.precision != P2P_FP32 && d.precision != P2P_FP64) fail(P2P_ERROR_INVALID_ARGUMENT, "bad precision");
    if (!(d.epsilon > 0.0) || !std::isfinite(d.epsilon)) fail(P2P_ERROR_INVALID_ARGUMENT, "epsilon must be > 0");
    if (d.part_world != 1 || d.part_rank != 0) fail(P2P_ERROR_NOT_SUPPORTED, "ADAPTIVE: one partition");
    if (d.ct < 1) fail(P2P_ERROR_INVALID_ARGUMENT, "ct must be >= 1");
    validate_points(d.src_xy, d.n_src, "sources");
    validate_points(d.tgt_xy, d.n_tgt, "targets");
    if (d.n_src > INT32_MAX - 8 || d.n_tgt > INT32_MAX - 8) fail(P2P_ERROR_NOT_SUPPORTED, "more than 2^31 points per set");
    const int lmax = std::min(d.l_max, kMaxLevel);
    if (lmax < 1) fail(P2P_ERROR_INVALID_ARGUMENT, "l_max must be >= 1");
    hp.layout = d.layout;
    hp.precision = d.precision;
    hp.device = d.device;
    hp.eps = d.epsilon;
    hp.kernel = d.kernel;
    hp.n_src = d.n_src;
    hp.n_tgt = d.n_tgt;
    hp.L = lmax;
    hp.S = int64_t(1) << (lmax - 1);
    hp.h = 1.0 / (double)hp.S;
    const int64_t Sf = hp.S;
    // finest-grid codes, stable sort (plan order = Morton order of the finest cell, then index)
    auto sortf = [&](const double *xy, int64_t n, std::vector<uint32_t> &codes, std::vector<int32_t> &perm,
                     std::vector<int32_t> &cells) {
        std::vector<uint32_t> c((size_t)n);
        parallel_for(n, [&](int64_t a, int64_t b) {
            for (int64_t i = a; i < b; ++i)
                c[i] = morton_encode(cell_of(xy[2 * i], Sf), cell_of(xy[2 * i + 1], Sf));
        });
        perm.resize((size_t)n);
        std::iota(perm.begin(), perm.end(), 0);
        std::stable_sort(perm.begin(), perm.end(), [&](int32_t x, int32_t y) { return c[x] < c[y]; });
        codes.resize((size_t)n);
        cells.resize((size_t)(2 * n));
        for (int64_t i = 0; i < n; ++i) {
            codes[i] = c[perm[i]];
            cells[2 * i] = (int32_t)cell_of(xy[2 * (int64_t)perm[i]], Sf);
            cells[2 * i + 1] = (int32_t)cell_of(xy[2 * (int64_t)perm[i] + 1], Sf);
        }
    };
    std::vector<uint32_t> cs, ctg;
    sortf(d.src_xy, d.n_src, cs, hp.src_perm_g, hp.pt_cell_s);
    sortf(d.tgt_xy, d.n_tgt, ctg, hp.tgt_perm_g, hp.pt_cell_t);
    auto range = [](const std::vector<uint32_t> &c, uint64_t lo, uint64_t hi) {  // [lo, hi) finest codes
        const int64_t a = std::lower_bound(c.begin(), c.end(), (uint32_t)std::min<uint64_t>(lo, UINT32_MAX)) - c.begin();
        const int64_t b = hi > UINT32_MAX ? (int64_t)c.size()
                                          : std::lower_bound(c.begin(), c.end(), (uint32_t)hi) - c.begin();
        return std::make_pair(a, b);
    };
    // depth-first split, children in Morton order
    std::vector<std::pair<int32_t, uint32_t>> stack{{1, 0u}};  // (level, Morton code at that level)
    while (!stack.empty()) {
        const auto [L, P] = stack.back();
        stack.pop_back();
        const int sh = 2 * (lmax - L);
        const uint64_t lo = (uint64_t)P << sh, hi = ((uint64_t)P + 1) << sh;
        const auto rs = range(cs, lo, hi), rt = range(ctg, lo, hi);
        if ((rs.second - rs.first > d.ct || rt.second - rt.first > d.ct) && L < lmax) {
            for (int c = 3; c >= 0; --c) stack.push_back({L + 1, (P << 2) | (uint32_t)c});
            continue;
        }
        uint32_t ix, iy;
        morton_decode(P, ix, iy);
        hp.leaf_lvl.push_back(L);
        hp.leaf_ix.push_back((int32_t)ix);
        hp.leaf_iy.push_back((int32_t)iy);
        hp.leaf_s0.push_back((int32_t)rs.first);
        hp.leaf_s1.push_back((int32_t)rs.second);
        hp.leaf_t0.push_back((int32_t)rt.first);
        hp.leaf_t1.push_back((int32_t)rt.second);
    }
    const int64_t nl = (int64_t)hp.leaf_lvl.size();
    hp.B = nl;
    std::vector<uint64_t> lstart((size_t)nl);  // first finest code of each leaf (ascending: Morton DFS)
    for (int64_t i = 0; i < nl; ++i) {
        const uint32_t P = morton_encode((uint32_t)hp.leaf_ix[i], (uint32_t)hp.leaf_iy[i]);
        lstart[i] = (uint64_t)P << (2 * (lmax - hp.leaf_lvl[i]));
    }
    auto lookup = [&](int64_t cx, int64_t cy) -> int64_t {  // the leaf holding finest cell (cx, cy)
        const uint64_t m = morton_encode((uint32_t)cx, (uint32_t)cy);
        return (std::upper_bound(lstart.begin(), lstart.end(), m) - lstart.begin()) - 1;
    };
    // U-lists: the leaf itself + every leaf met walking just outside its four sides and corners
    hp.ul_off.assign((size_t)nl + 1, 0);
    std::vector<int64_t> lp((size_t)nl, 0);
    int64_t max_src = 0, max_ul = 0;
    std::vector<int32_t> u;
    for (int64_t i = 0; i < nl; ++i) {
        u.clear();
        if (hp.leaf_t1[i] > hp.leaf_t0[i]) {
            const int64_t sz = int64_t(1) << (lmax - hp.leaf_lvl[i]);
            const int64_t x0 = hp.leaf_ix[i] * sz, y0 = hp.leaf_iy[i] * sz, x1 = x0 + sz, y1 = y0 + sz;
            u.push_back((int32_t)i);
            auto extent = [&](int64_t j, int64_t &ex0, int64_t &ex1, int64_t &ey0, int64_t &ey1) {
                const int64_t s2 = int64_t(1) << (lmax - hp.leaf_lvl[j]);
                ex0 = hp.leaf_ix[j] * s2;
                ex1 = ex0 + s2;
                ey0 = hp.leaf_iy[j] * s2;
                ey1 = ey0 + s2;
            };
            for (int side = 0; side < 2; ++side) {  // rows below / above
                const int64_t y = side ? y1 : y0 - 1;
                if (y < 0 || y >= Sf) continue;
                for (int64_t x = x0; x < x1;) {
                    const int64_t j = lookup(x, y);
                    u.push_back((int32_t)j);
                    int64_t ex0, ex1, ey0, ey1;
                    extent(j, ex0, ex1, ey0, ey1);
                    x = ex1;
                }
            }
            for (int side = 0; side < 2; ++side) {  // columns left / right
                const int64_t x = side ? x1 : x0 - 1;
                if (x < 0 || x >= Sf) continue;
                for (int64_t y = y0; y < y1;) {
                    const int64_t j = lookup(x, y);
                    u.push_back((int32_t)j);
                    int64_t ex0, ex1, ey0, ey1;
                    extent(j, ex0, ex1, ey0, ey1);
                    y = ey1;
                }
            }
            const int64_t cx[2] = {x0 - 1, x1}, cy[2] = {y0 - 1, y1};
            for (int a = 0; a < 2; ++a)
                for (int b = 0; b < 2; ++b)
                    if (cx[a] >= 0 && cx[a] < Sf && cy[b] >= 0 && cy[b] < Sf) u.push_back((int32_t)lookup(cx[a], cy[b]));
            std::sort(u.begin(), u.end());
            u.erase(std::unique(u.begin(), u.end()), u.end());
        }
        int64_t ns_u = 0;
        for (int32_t j : u) ns_u += hp.leaf_s1[j] - hp.leaf_s0[j];
        hp.ul_leaf.insert(hp.ul_leaf.end(), u.begin(), u.end());
        hp.ul_off[i + 1] = (int32_t)hp.ul_leaf.size();
        const int64_t ntl = hp.leaf_t1[i] - hp.leaf_t0[i];
        lp[i] = ntl * ns_u;
        hp.pairs += lp[i];
        if (ntl) {
            max_src = std::max(max_src, ns_u);
            max_ul = std::max<int64_t>(max_ul, (int64_t)u.size());
            hp.tgt_cap = std::max(hp.tgt_cap, ntl);
            hp.occ_tgt += 1;
        }
        if (hp.leaf_s1[i] > hp.leaf_s0[i]) hp.occ_src += 1;
        hp.t_max = std::max<int64_t>(hp.t_max, std::max<int64_t>(hp.leaf_s1[i] - hp.leaf_s0[i], ntl));
    }
    if (max_ul > kMaxUlist) fail(P2P_ERROR_NOT_SUPPORTED, "ADAPTIVE: a U-list exceeds 256 leaves");
    hp.pairs_global = hp.pairs;
    hp.density = (double)hp.n_tgt / (double)std::max<int64_t>(nl, 1);
    hp.density_occ = hp.occ_tgt ? (double)hp.n_tgt / (double)hp.occ_tgt : 0.0;
    // queue: target leaves by decreasing pairs (stable)
    std::vector<int32_t> tl;
    for (int64_t i = 0; i < nl; ++i)
        if (hp.leaf_t1[i] > hp.leaf_t0[i]) tl.push_back((int32_t)i);
    std::stable_sort(tl.begin(), tl.end(), [&](int32_t x, int32_t y) { return lp[x] > lp[y]; });
    hp.tiles = tl;
    hp.tile_slot.resize(tl.size());
    std::iota(hp.tile_slot.begin(), hp.tile_slot.end(), 0);
    hp.tile_part.assign(tl.size(), 1 << 16);
    hp.n_interior = (int64_t)tl.size();
    hp.boxes_in_tiles = (int64_t)tl.size();
    hp.src_cap = max_src;
    hp.nt = kAdaptiveThreads;
    const int e = d.precision == P2P_FP32 ? 4 : 8;
    hp.smem_bytes = adaptive_smem(hp.src_cap, e);
    // fp32 leaves of <= 32 targets: one warp per leaf, 4 warps per CTA (measured: +38 % at CT = 16,
    // +12 % at CT = 32; slower for larger leaves and for fp64, tools/gpu/gpu_ab20.sh); P2P_ADAPTIVE_WARP=0: off
    hp.warp_leaf = e == 4 && hp.tgt_cap <= 32;
    if (const char *v = std::getenv("P2P_ADAPTIVE_WARP")) hp.warp_leaf = hp.warp_leaf && std::atoi(v) != 0;
    if (hp.warp_leaf) {
        hp.nt = 128;
        hp.smem_bytes = 4 * (int64_t)adaptive_warp_slice((int)std::min<int64_t>(hp.src_cap, 1 << 20), e);
    }
    if (hp.smem_bytes > kSmemLimit)
        fail(P2P_ERROR_NOT_SUPPORTED, "ADAPTIVE: a U-list holds " + std::to_string(max_src) +
                                          " sources (> shared memory); lower ct");
    // one partition, local = global
    hp.part_tile = {0, (int64_t)tl.size()};
    hp.part_src = {0, hp.n_src};
    hp.part_tgt = {0, hp.n_tgt};
    hp.n_src_local = hp.n_src_owned = hp.n_src;
    hp.n_tgt_local = hp.n_tgt;
    hp.src_gidx.resize((size_t)hp.n_src);
    std::iota(hp.src_gidx.begin(), hp.src_gidx.end(), 0);
    hp.src_uidx = hp.src_perm_g;
    hp.tgt_uidx = hp.tgt_perm_g;
    hp.recv_counts.assign(1, 0);
    hp.send_counts.assign(1, 0);
    // per point: offset within its finest cell (x - cx hf), plan order; cells in pt_cell_*
    auto fillc = [&](auto &vec, const double *xy, const std::vector<int32_t> &perm) {
        using V = typename std::decay_t<decltype(vec)>::value_type;
        const int64_t n = (int64_t)perm.size();
        vec.resize((size_t)(2 * n));
        for (int64_t i = 0; i < n; ++i)
            for (int c = 0; c < 2; ++c) {
                const double x = xy[2 * (int64_t)perm[i] + c];
                vec[2 * i + c] = (V)(x - (double)cell_of(x, Sf) * hp.h);
            }
    };
    if (d.precision == P2P_FP32) {
        fillc(hp.f32.src_uv, d.src_xy, hp.src_uidx);
        fillc(hp.f32.tgt_uv, d.tgt_xy, hp.tgt_uidx);
    } else {
        fillc(hp.f64.src_uv, d.src_xy, hp.src_uidx);
        fillc(hp.f64.tgt_uv, d.tgt_xy, hp.tgt_uidx);
    }
    hp.build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// ---- 3D: octree leaf grid, 3D Morton order (x bit 3i, y 3i+1, z 3i+2),
// E1 = the 3x3x3 block clipped at the faces; one CTA per target box stages its <= 27 neighbour
// boxes (p2p_box3d_kernel).
namespace {
inline uint32_t spread3(uint32_t v) {
    uint32_t r = 0;
    for (int b = 0; b < 10; ++b) r |= ((v >> b) & 1u) << (3 * b);
    return r;
}
inline uint32_t morton3(uint32_t x, uint32_t y, uint32_t z) { return spread3(x) | spread3(y) << 1 | spread3(z) << 2; }
}  // namespace

void build_host_plan_3d(const p2p_plan_desc &d, HostPlan &hp) {
    auto t0 = std::chrono::steady_clock::now();
    if (d.layout != P2P_LAYOUT_NONREDUNDANT) fail(P2P_ERROR_NOT_SUPPORTED, "3D: NONREDUNDANT layout");
    if (d.precision != P2P_FP32 && d.precision != P2P_FP64) fail(P2P_ERROR_INVALID_ARGUMENT, "bad precision");
    if (!(d.epsilon > 0.0) || !std::isfinite(d.epsilon)) fail(P2P_ERROR_INVALID_ARGUMENT, "epsilon must be > 0");
    if (d.part_world != 1 || d.part_rank != 0) fail(P2P_ERROR_NOT_SUPPORTED, "3D: one partition");
    auto validate3 = [&](const double *xyz, int64_t n, const char *what) {
        if (n < 1) fail(P2P_ERROR_INVALID_ARGUMENT, std::string(what) + ": n must be >= 1 (SPEC.md L55)");
        if (!xyz) fail(P2P_ERROR_INVALID_ARGUMENT, std::string(what) + ": NULL coordinates");
        for (int64_t i = 0; i < 3 * n; ++i)
            if (!(xyz[i] >= 0.0 && xyz[i] <= 1.0))
                fail(P2P_ERROR_INVALID_ARGUMENT, std::string(what) + ": coordinate " + std::to_string(i / 3) +
                                                     " outside the unit cube [0,1]^3");
    };
    validate3(d.src_xy, d.n_src, "sources");
    validate3(d.tgt_xy, d.n_tgt, "targets");
    if (d.n_src > INT32_MAX - 8 || d.n_tgt > INT32_MAX - 8) fail(P2P_ERROR_NOT_SUPPORTED, "more than 2^31 points per set");
    if (d.level < 1) fail(P2P_ERROR_NOT_SUPPORTED, "3D: give the leaf level (no CT loop)");
    const int L = d.level + d.level_delta;
    if (L < 1) fail(P2P_ERROR_INVALID_ARGUMENT, "L + level_delta < 1 (SPEC.md L85)");
    if (L > kMaxLevel3) fail(P2P_ERROR_NOT_SUPPORTED, "3D: L > 9 (8^(L-1) <= 2^24 boxes)");
    hp.dim = 3;
    hp.kernel = d.kernel;
    hp.kappa = d.kernel == P2P_KERNEL_HELMHOLTZ_3D ? d.wavenumber : 0.0;
    hp.layout = d.layout;
    hp.precision = d.precision;
    hp.device = d.device;
    hp.eps = d.epsilon;
    hp.n_src = d.n_src;
    hp.n_tgt = d.n_tgt;
    hp.L = L;
    hp.S = int64_t(1) << (L - 1);
    hp.B = hp.S * hp.S * hp.S;
    hp.h = 1.0 / (double)hp.S;
    const int64_t S = hp.S, B = hp.B;
    auto sort3 = [&](const double *xyz, int64_t n, std::vector<int32_t> &off, std::vector<int32_t> &perm) {
        std::vector<uint32_t> code((size_t)n);
        parallel_for(n, [&](int64_t a, int64_t b) {
            for (int64_t i = a; i < b; ++i)
                code[i] = morton3(cell_of(xyz[3 * i], S), cell_of(xyz[3 * i + 1], S), cell_of(xyz[3 * i + 2], S));
        });
        off.assign((size_t)B + 1, 0);
        for (int64_t i = 0; i < n; ++i) off[code[i] + 1] += 1;
        for (int64_t b = 0; b < B; ++b) off[b + 1] += off[b];
        std::vector<int32_t> pos(off.begin(), off.end() - 1);
        perm.resize((size_t)n);
        for (int64_t i = 0; i < n; ++i) perm[pos[code[i]]++] = (int32_t)i;
    };
    sort3(d.src_xy, d.n_src, hp.src_off_g, hp.src_perm_g);
    sort3(d.tgt_xy, d.n_tgt, hp.tgt_off_g, hp.tgt_perm_g);
    const int32_t *so = hp.src_off_g.data(), *to = hp.tgt_off_g.data();
    // occupied target boxes, their E1 source counts and pairs
    std::vector<int32_t> boxes;
    std::vector<int64_t> bpairs;
    int64_t max27 = 0;
    for (int64_t b = 0; b < B; ++b) {
        const int64_t a = so[b + 1] - so[b], t = to[b + 1] - to[b];
        hp.occ_src += a > 0;
        hp.occ_tgt += t > 0;
        hp.t_max = std::max(hp.t_max, std::max(a, t));
        if (!t) continue;
        uint32_t ix = 0, iy = 0, iz = 0;
        for (int bit = 0; bit < 10; ++bit) {
            ix |= ((uint32_t)(b >> (3 * bit)) & 1u) << bit;
            iy |= ((uint32_t)(b >> (3 * bit + 1)) & 1u) << bit;
            iz |= ((uint32_t)(b >> (3 * bit + 2)) & 1u) << bit;
        }
        int64_t c = 0;
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const int64_t x = (int64_t)ix + dx, y = (int64_t)iy + dy, z = (int64_t)iz + dz;
                    if (x < 0 || y < 0 || z < 0 || x >= S || y >= S || z >= S) continue;
                    const uint32_t m = morton3((uint32_t)x, (uint32_t)y, (uint32_t)z);
                    c += so[m + 1] - so[m];
                }
        boxes.push_back((int32_t)b);
        bpairs.push_back(t * c);
        max27 = std::max(max27, c);
        hp.pairs += t * c;
        hp.tgt_cap = std::max(hp.tgt_cap, t);
    }
    hp.pairs_global = hp.pairs;
    hp.density = (double)hp.n_tgt / (double)B;
    hp.density_occ = hp.occ_tgt ? (double)hp.n_tgt / (double)hp.occ_tgt : 0.0;
    // queue: boxes by decreasing pair count (stable), so the last wave holds the short boxes
    std::vector<int64_t> ord(boxes.size());
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int64_t x, int64_t y) { return bpairs[x] > bpairs[y]; });
    hp.tiles.resize(boxes.size());
    for (size_t i = 0; i < ord.size(); ++i) hp.tiles[i] = boxes[ord[i]];
    hp.tile_slot.assign(hp.tiles.size(), 0);
    std::iota(hp.tile_slot.begin(), hp.tile_slot.end(), 0);
    hp.tile_part.assign(hp.tiles.size(), 1 << 16);
    hp.n_interior = (int64_t)hp.tiles.size();
    hp.k = 0;
    hp.boxes_in_tiles = (int64_t)hp.tiles.size();
    hp.src_cap = max27;
    hp.nt = box3d_threads(d.kernel);
    const int e = d.precision == P2P_FP32 ? 4 : 8, comps = d.kernel == P2P_KERNEL_HELMHOLTZ_3D ? 2 : 1;
    hp.smem_bytes = box3d_smem(hp.src_cap, e, comps, hp.nt, box3d_parts(comps == 2, e));
    if (hp.smem_bytes > kSmemLimit)
        fail(P2P_ERROR_NOT_SUPPORTED, "3D: a box's 27 neighbours hold " + std::to_string(max27) +
                                          " sources (> shared memory); use a deeper level");
    // partition / local sets (one partition)
    hp.part_tile = {0, (int64_t)hp.tiles.size()};
    hp.part_src = {0, hp.n_src};
    hp.part_tgt = {0, hp.n_tgt};
    hp.src_off = hp.src_off_g;
    hp.tgt_off = hp.tgt_off_g;
    hp.n_src_local = hp.n_src_owned = hp.n_src;
    hp.n_tgt_local = hp.n_tgt;
    hp.src_gidx.resize((size_t)hp.n_src);
    std::iota(hp.src_gidx.begin(), hp.src_gidx.end(), 0);
    hp.src_uidx = hp.src_perm_g;
    hp.tgt_uidx = hp.tgt_perm_g;
    hp.recv_counts.assign(1, 0);
    hp.send_counts.assign(1, 0);
    // box-local coordinates in units of h: u = (x - ix h) S (exact in fp64), 4 per point
    auto fill4 = [&](auto &vec, const double *xyz, const std::vector<int32_t> &perm) {
        using V = typename std::decay_t<decltype(vec)>::value_type;
        const int64_t n = (int64_t)perm.size();
        vec.assign((size_t)(4 * n), (V)0);
        parallel_for(n, [&](int64_t a, int64_t b) {
            for (int64_t i = a; i < b; ++i)
                for (int c = 0; c < 3; ++c) {
                    const double x = xyz[3 * (int64_t)perm[i] + c];
                    vec[4 * i + c] = (V)((x - (double)cell_of(x, S) * hp.h) * (double)S);
                }
        });
    };
    if (d.precision == P2P_FP32) {
        fill4(hp.f32.src_uv, d.src_xy, hp.src_uidx);
        fill4(hp.f32.tgt_uv, d.tgt_xy, hp.tgt_uidx);
    } else {
        fill4(hp.f64.src_uv, d.src_xy, hp.src_uidx);
        fill4(hp.f64.tgt_uv, d.tgt_xy, hp.tgt_uidx);
    }
    hp.build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// Kernel options and shared-memory size of a plan at tile size k, from its tile statistics
// (shared by the host and the device builders, so both make the same decisions).
int64_t choose_tile_params(const p2p_plan_desc &d, HostPlan &hp, int k, const TileStats &st) {
    const int e = d.precision == P2P_FP32 ? 4 : 8;
    hp.max_region = st.max_region_pad;
    hp.max_tile_halo = st.max_tile_halo;
    hp.src_cap = d.layout == P2P_LAYOUT_REDUNDANT ? hp.max_tile_halo : pad4(hp.max_region);
    // fp32 two-target units: from 8 points per occupied box (NR), from 3 (TILED: measured against the
    // lean path on 1e7-point plates, tools/gpu/gpu_dense_threshold.sh: D_occ 2.3 lean 191 / dense 207 us,
    // 3.2 dense 203 / items 219, 4.1 dense 215 / lean 273, 6.0 dense 229 / items 336)
    // fp64 TILED two-target units with (unit, row) items from 4 points per occupied box (same plates,
    // tools/gpu/gpu_f64_ab.sh: D_occ 3.2 lean 714 / dense 790 us, 4.1 847 / 769, 6.0 1225 / 920)
    double dense_from = d.layout == P2P_LAYOUT_TILED ? 3.0 : 8.0, dense64_from = d.layout == P2P_LAYOUT_TILED ? 4.0 : 8.0;
    if (const char *v = std::getenv("P2P_DENSE_FROM")) dense_from = dense64_from = std::atof(v);  // tuning hook
    hp.tpi = (d.precision == P2P_FP32 && hp.density_occ >= dense_from && k <= 3 && d.layout != P2P_LAYOUT_REDUNDANT)
                 ? 2 : 1;
    // dense fp64 TILED: two targets per unit as well (each source load serves both; P2P_TPI64=0: one)
    if (d.precision == P2P_FP64 && d.layout == P2P_LAYOUT_TILED && hp.density_occ >= dense64_from && k <= 3) {
        hp.tpi = 2;
        if (const char *v = std::getenv("P2P_TPI64")) hp.tpi = std::atoi(v) == 1 ? 1 : 2;
    }
    // TILED defaults: dense fp32 -> padded pairs, 2 targets per unit, (unit, row) items;
    // sparse or fp64 -> unpadded, one item per target; 128-thread CTAs.
    hp.pad = d.layout == P2P_LAYOUT_TILED ? (hp.tpi == 2) : true;
    // fp64 dense boxes: (target, row-run) items too (sorted), 256-thread CTAs (tools/gpu/gpu_ab11.sh)
    const bool dense64 = d.precision == P2P_FP64 && hp.density_occ >= dense64_from;
    hp.ns = hp.tpi > 1 || dense64 ? 3 : 1;
    hp.nbuf = 1;
    // measured best (tools/gpu/gpu_ab*.sh): 128 threads for dense fp32 units and sparse fp64,
    // 256 for dense fp64, 64 (or 32, below) for sparse fp32
    hp.nt = d.layout == P2P_LAYOUT_TILED
                ? (dense64 ? 256 : hp.tpi > 1 || d.precision == P2P_FP64 ? 128 : 64) : kThreads;
    // dense fp32 TILED below 5 points per occupied box: 64-thread CTAs (same sweep: D_occ 3.2 64 203 /
    // 128 227 us, 4.1 215 / 217; 6.0 272 / 229)
    if (d.layout == P2P_LAYOUT_TILED && d.precision == P2P_FP32 && hp.tpi > 1 && hp.density_occ < 5.0) hp.nt = 64;
    // tuning hooks (experiments only): P2P_TPI, P2P_NS, P2P_NBUF, P2P_PAD, P2P_NT
    if (const char *v = std::getenv("P2P_TPI"))
        if (d.precision == P2P_FP32 && d.layout != P2P_LAYOUT_REDUNDANT) {
            const int x = std::atoi(v);
            hp.tpi = x == 2 ? 2 : 1;
        }
    if (const char *v = std::getenv("P2P_PAD"))
        if (d.layout == P2P_LAYOUT_TILED && d.precision == P2P_FP32) hp.pad = std::atoi(v) != 0;
    if (hp.tpi > 1) hp.pad = true;
    if (d.precision == P2P_FP64 && d.layout == P2P_LAYOUT_TILED) hp.pad = false;
    if (const char *v = std::getenv("P2P_NS")) hp.ns = std::atoi(v) == 3 ? 3 : 1;
    if (const char *v = std::getenv("P2P_NBUF")) hp.nbuf = std::atoi(v) == 2 ? 2 : 1;
    if (const char *v = std::getenv("P2P_NT"))
        if (d.layout == P2P_LAYOUT_TILED) {
            const int x = std::atoi(v);
            hp.nt = x <= 32 ? 32 : x <= 64 ? 64 : x <= 128 ? 128 : 256;
        }
    // lean sparse path: targets of a tile sorted by neighbourhood size (n9), so the
    // lanes of a warp sweep near-equal pair counts (P2P_TSORT=0 disables)
    hp.lean = d.layout == P2P_LAYOUT_TILED && hp.tpi == 1 && hp.ns == 1 && !hp.pad;
    hp.tsort = hp.lean;
    if (hp.nt == 32 && !hp.lean) hp.nt = 64;  // one-warp CTAs: lean instances only
    // lean fp32: ~4 targets per thread measured best (tools/gpu/gpu_prof5.sh): one-warp CTAs for small tiles
    if (hp.lean && d.precision == P2P_FP32 && !std::getenv("P2P_NT") &&
        (double)hp.n_tgt / (double)std::max<int64_t>(st.ntiles, 1) < 192.0)
        hp.nt = 32;
    if (const char *v = std::getenv("P2P_TSORT")) hp.tsort = hp.ns == 1 && std::atoi(v) != 0;
    // flattened row-runs pay below ~3 sources per box (more index work per pair,
    // fewer idle lanes) and always in fp64 (the log dwarfs the index work); above,
    // row loops (P2P_FLAT overrides)
    // dense fp64: the conflict-free replicated log table (one more DP op per pair, no bank
    // conflicts) pays below ~24 sources per box; denser boxes keep the 256-entry table (measured,
    // tools/gpu/gpu_f64_ab2.sh: surf_2e7 / d16 -3..-4 %, d32 / d64 +5..+10 % with it)
    hp.lt8 = d.layout == P2P_LAYOUT_TILED && dense64 && hp.density_occ < 24.0;
    if (const char *v = std::getenv("P2P_LT8")) hp.lt8 = d.layout == P2P_LAYOUT_TILED && dense64 && std::atoi(v) != 0;
    hp.flat = hp.lean && (hp.density_occ < 3.0 || d.precision == P2P_FP64);
    if (const char *v = std::getenv("P2P_FLAT")) hp.flat = hp.lean && std::atoi(v) != 0;
    if (d.kernel == P2P_KERNEL_HELMHOLTZ_2D) {  // one thread per target, n9-sorted, flattened runs
        hp.tpi = 1;
        hp.pad = false;
        hp.ns = 1;
        hp.nbuf = 1;
        hp.lean = hp.tsort = hp.flat = true;
        hp.nt = 128;
        if (const char *v = std::getenv("P2P_NT")) {
            const int x = std::atoi(v);
            hp.nt = x <= 32 ? 32 : x <= 64 ? 64 : x <= 128 ? 128 : 256;
        }
    }
    hp.tgt_cap = pad8(d.layout == P2P_LAYOUT_TILED && hp.tpi == 2 ? st.max_tcount2 : st.max_tcount);
    if (d.layout == P2P_LAYOUT_TILED && !hp.pad) hp.src_cap = pad4(st.max_region);  // unpadded region sizes
    if (d.layout == P2P_LAYOUT_PAPER_INDEXING || d.layout == P2P_LAYOUT_PAPER_REPETITION) {
        hp.smem_bytes = 0;  // global-memory kernels: no tiles to size
        return 0;
    }
    const int sc = (int)std::min<int64_t>(hp.src_cap, 1 << 24), tc = (int)std::min<int64_t>(hp.tgt_cap, 1 << 24);
    if (d.kernel == P2P_KERNEL_HELMHOLTZ_2D) {
        hp.smem_bytes = helm_carve(k, sc, tc, e).total;
        return hp.smem_bytes;
    }
    int64_t smem = d.layout == P2P_LAYOUT_NONREDUNDANT ? (int64_t)nr_carve(k, sc, tc, e, hp.tpi).total
                   : d.layout == P2P_LAYOUT_TILED
                       ? (int64_t)tiled_carve(k, sc, tc, e, hp.tpi, hp.ns, hp.nbuf, hp.lt8).total
                                                       : (int64_t)r_carve(k, sc, tc, e).total;
    hp.smem_bytes = smem;
    return smem;
}

// Local input: global CSR offsets from the global per-box counts, and the passed points sorted
// by (box, global id) -- the global plan's order restricted to them.
void local_sort(const double *xy, const int64_t *ids, int64_t n, const HostPlan &hp, std::vector<uint32_t> &code,
                std::vector<int32_t> &order) {
    code.resize((size_t)n);
    parallel_for(n, [&](int64_t a, int64_t b) {
        for (int64_t i = a; i < b; ++i)
            code[i] = morton_encode(cell_of(xy[2 * i], hp.S), cell_of(xy[2 * i + 1], hp.S));
    });
    order.resize((size_t)n);
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
        return code[a] != code[b] ? code[a] < code[b] : ids[a] < ids[b];
    });
    for (int64_t i = 1; i < n; ++i)
        if (code[order[i]] == code[order[i - 1]] && ids[order[i]] == ids[order[i - 1]])
            fail(P2P_ERROR_INVALID_ARGUMENT, "duplicate global id among the passed points");
}

void box_counts(int level, int64_t n, const double *xy, int32_t *counts) {
    const int64_t S = int64_t(1) << (level - 1), B = S * S;
    if (n) validate_points(xy, n, "points");
    std::fill(counts, counts + B, 0);
    for (int64_t i = 0; i < n; ++i) counts[morton_encode(cell_of(xy[2 * i], S), cell_of(xy[2 * i + 1], S))] += 1;
}

std::vector<int32_t> offsets_from_counts(const int32_t *counts, int64_t B, int64_t n_global, const char *what) {
    std::vector<int32_t> off((size_t)B + 1, 0);
    int64_t acc = 0;
    for (int64_t b = 0; b < B; ++b) {
        if (counts[b] < 0) fail(P2P_ERROR_INVALID_ARGUMENT, std::string("negative ") + what + " box count");
        acc += counts[b];
        if (acc > INT32_MAX - 8) fail(P2P_ERROR_NOT_SUPPORTED, "more than 2^31 points per set");
        off[b + 1] = (int32_t)acc;
    }
    if (acc != n_global) fail(P2P_ERROR_INVALID_ARGUMENT, std::string(what) + " box counts do not sum to n_global");
    return off;
}

void build_host_plan(const p2p_plan_desc &d, HostPlan &hp, const LocalInput *li) {
    auto t0 = std::chrono::steady_clock::now();
    if (li) {
        if (d.level <= 0) fail(P2P_ERROR_NOT_SUPPORTED, "local-input plans need an explicit level");
        if (d.layout != P2P_LAYOUT_NONREDUNDANT && d.layout != P2P_LAYOUT_REDUNDANT && d.layout != P2P_LAYOUT_TILED)
            fail(P2P_ERROR_NOT_SUPPORTED, "local-input plans: NR, R and TILED layouts");
        if (d.part_world > 32) fail(P2P_ERROR_NOT_SUPPORTED, "local-input plans: part_world <= 32");
        if ((d.n_src && !li->src_ids) || (d.n_tgt && !li->tgt_ids) || !li->src_counts || !li->tgt_counts)
            fail(P2P_ERROR_INVALID_ARGUMENT, "NULL ids or box counts");
    }
    if (d.struct_size != sizeof(p2p_plan_desc)) fail(P2P_ERROR_INVALID_ARGUMENT, "desc.struct_size mismatch");
    check_kernel(d);
    if (kernel_dim(d.kernel) == 3) {
        if (li) fail(P2P_ERROR_NOT_SUPPORTED, "local-input plans: 2D kernels");
        build_host_plan_3d(d, hp);
        return;
    }
    if (d.layout == P2P_LAYOUT_ADAPTIVE) {
        build_host_plan_adaptive(d, hp);
        return;
    }
    if (d.layout < P2P_LAYOUT_NONREDUNDANT || d.layout > P2P_LAYOUT_ADAPTIVE)
        fail(P2P_ERROR_INVALID_ARGUMENT, "bad layout");
    const bool paper = d.layout == P2P_LAYOUT_PAPER_INDEXING || d.layout == P2P_LAYOUT_PAPER_REPETITION;
    if (paper && d.precision != P2P_FP64)
        fail(P2P_ERROR_NOT_SUPPORTED, "the paper's layouts are fp64 (PAPER.md L98: stored as Double)");
    if (paper && d.part_world != 1) fail(P2P_ERROR_NOT_SUPPORTED, "the paper's layouts are single-partition");
    if (d.precision != P2P_FP32 && d.precision != P2P_FP64) fail(P2P_ERROR_INVALID_ARGUMENT, "bad precision");
    if (!(d.epsilon > 0.0) || !std::isfinite(d.epsilon)) fail(P2P_ERROR_INVALID_ARGUMENT, "epsilon must be > 0");
    if (d.part_world < 1 || d.part_rank < 0 || d.part_rank >= d.part_world)
        fail(P2P_ERROR_INVALID_ARGUMENT, "bad part_world / part_rank");
    if (!li) {
        validate_points(d.src_xy, d.n_src, "sources");
        validate_points(d.tgt_xy, d.n_tgt, "targets");
    } else {  // zero passed points is fine (a rank may hold none); the global sets may not be empty
        if (d.n_src < 0 || d.n_tgt < 0 || (d.n_src && !d.src_xy) || (d.n_tgt && !d.tgt_xy))
            fail(P2P_ERROR_INVALID_ARGUMENT, "bad local point arrays");
        if (d.n_src) validate_points(d.src_xy, d.n_src, "sources");
        if (d.n_tgt) validate_points(d.tgt_xy, d.n_tgt, "targets");
        if (li->n_src_global < 1 || li->n_tgt_global < 1)
            fail(P2P_ERROR_INVALID_ARGUMENT, "n = 0 (SPEC.md L55)");
    }
    if (d.n_src > INT32_MAX - 8 || d.n_tgt > INT32_MAX - 8)
        fail(P2P_ERROR_NOT_SUPPORTED, "more than 2^31 points per set");

    hp.layout = d.layout;
    hp.precision = d.precision;
    hp.device = d.device;
    hp.eps = d.epsilon;
    hp.kernel = d.kernel;
    hp.kappa = d.kernel == P2P_KERNEL_HELMHOLTZ_2D ? d.wavenumber : 0.0;
    hp.part_world = d.part_world;
    hp.part_rank = d.part_rank;
    hp.n_src = li ? li->n_src_global : d.n_src;
    hp.n_tgt = li ? li->n_tgt_global : d.n_tgt;
    hp.local_input = li != nullptr;

    // ---- a1 level
    int L = d.level > 0 ? d.level : ct_loop_level(d);
    L += d.level_delta;
    if (L < 1) fail(P2P_ERROR_INVALID_ARGUMENT, "L + level_delta < 1 (SPEC.md L85)");
    if (L > kMaxLevel) fail(P2P_ERROR_NOT_SUPPORTED, "L > 15 (full-grid CSR offsets; see DESIGN.md)");
    hp.L = L;
    hp.S = int64_t(1) << (L - 1);
    hp.B = hp.S * hp.S;
    hp.h = 1.0 / (double)hp.S;

    // ---- a2, a3
    std::vector<uint32_t> lcode_s, lcode_t;  // local input: passed points' box codes ...
    std::vector<int32_t> lord_s, lord_t;      // ... and their (box, global id) order
    if (!li) {
        csr_sort(d.src_xy, d.n_src, hp, hp.src_off_g, hp.src_perm_g);
        csr_sort(d.tgt_xy, d.n_tgt, hp, hp.tgt_off_g, hp.tgt_perm_g);
    } else {
        hp.src_off_g = offsets_from_counts(li->src_counts, hp.B, hp.n_src, "source");
        hp.tgt_off_g = offsets_from_counts(li->tgt_counts, hp.B, hp.n_tgt, "target");
        local_sort(d.src_xy, li->src_ids, d.n_src, hp, lcode_s, lord_s);
        local_sort(d.tgt_xy, li->tgt_ids, d.n_tgt, hp, lcode_t, lord_t);
    }
    const int32_t *so = hp.src_off_g.data(), *to = hp.tgt_off_g.data();
    auto ns = [&](int64_t b) -> int64_t { return so[b + 1] - so[b]; };
    auto ntg = [&](int64_t b) -> int64_t { return to[b + 1] - to[b]; };

    for (int64_t b = 0; b < hp.B; ++b) {
        int64_t a = ns(b), t = ntg(b);
        hp.occ_src += a > 0;
        hp.occ_tgt += t > 0;
        hp.t_max = std::max(hp.t_max, std::max(a, t));
    }
    hp.density = (double)hp.n_tgt / (double)hp.B;
    hp.density_occ = hp.occ_tgt ? (double)hp.n_tgt / (double)hp.occ_tgt : 0.0;

    // E1 source count of every target-occupied box (3x3, clipped).
    std::vector<int32_t> n9((size_t)hp.B, 0);
    const int64_t S = hp.S;
    parallel_for(hp.B, [&](int64_t a, int64_t bnd) {
        for (int64_t b = a; b < bnd; ++b) {
            if (ntg(b) == 0) continue;
            uint32_t ix, iy;
            morton_decode((uint32_t)b, ix, iy);
            int64_t c = 0;
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    int64_t x = (int64_t)ix + dx, y = (int64_t)iy + dy;
                    if (x < 0 || y < 0 || x >= S || y >= S) continue;
                    c += ns(morton_encode((uint32_t)x, (uint32_t)y));
                }
            n9[b] = (int32_t)c;
        }
    });

    // ---- CTA tiles: Morton-aligned 2^k x 2^k blocks = contiguous Morton ranges.
    const int e = d.precision == P2P_FP32 ? 4 : 8;
    int kmax = std::min(L - 1, kMaxTileLog2);
    int k;
    if (d.tile_log2 >= 0) {
        k = std::min(d.tile_log2, kmax);
    } else {
        // smallest k whose non-empty tiles hold >= ~256 targets on average (256 = CTA size)
        k = kmax;
        for (int kk = 0; kk <= kmax; ++kk) {
            const int64_t WWk = int64_t(1) << (2 * kk);
            int64_t ne = 0;
            for (int64_t t = 0; t < hp.B / WWk; ++t) ne += to[(t + 1) * WWk] > to[t * WWk];
            if ((double)hp.n_tgt / (double)std::max<int64_t>(ne, 1) >= 115.0) {  // measured best (tools/sweep.py)
                k = kk;
                break;
            }
        }
        // the R layout stages 9x the sources: keep its tile halo modest so >= 4 CTAs fit per SM
        if (d.layout == P2P_LAYOUT_REDUNDANT)
            while (k > 0 && 9.0 * hp.density_occ * (double)(int64_t(1) << (2 * k)) * 3 * e > 48.0 * 1024) --k;
    }
    for (;; --k) {
        const int64_t W = int64_t(1) << k, WW = W * W, R = W + 2;
        const int64_t ntile_all = hp.B / WW;
        const int64_t side_t = S / W;
        (void)side_t;
        hp.tiles_g.clear();
        for (int64_t t = 0; t < ntile_all; ++t)
            if (to[(t + 1) * WW] > to[t * WW]) hp.tiles_g.push_back((int32_t)t);
        const int64_t nt = (int64_t)hp.tiles_g.size();
        hp.tile_pairs_g.assign((size_t)nt, 0);
        std::vector<int64_t> region((size_t)nt, 0), region_u((size_t)nt, 0), halo((size_t)nt, 0), tcount((size_t)nt, 0),
            tcount2((size_t)nt, 0);
        parallel_for(nt, [&](int64_t a, int64_t bnd) {
            for (int64_t i = a; i < bnd; ++i) {
                int64_t t = hp.tiles_g[i];
                int64_t pr = 0, hl = 0, sl2 = 0;
                for (int64_t b = t * WW; b < (t + 1) * WW; ++b) {
                    int64_t c = ntg(b);
                    if (!c) continue;
                    sl2 += c + (c & 1);  // target slots of 2-target units (odd boxes: one duplicate)
                    pr += c * (int64_t)n9[b];
                    hl += pad2(n9[b]);
                }
                uint32_t tx, ty;
                morton_decode((uint32_t)t, tx, ty);
                int64_t X0 = (int64_t)tx * W - 1, Y0 = (int64_t)ty * W - 1, rg = 0, rgu = 0;
                for (int64_t ly = 0; ly < R; ++ly)
                    for (int64_t lx = 0; lx < R; ++lx) {
                        int64_t x = X0 + lx, y = Y0 + ly;
                        if (x < 0 || y < 0 || x >= S || y >= S) continue;
                        const int64_t c = ns(morton_encode((uint32_t)x, (uint32_t)y));
                        rg += pad2(c);
                        rgu += c;
                    }
                region_u[i] = rgu;
                hp.tile_pairs_g[i] = pr;
                tcount[i] = to[(t + 1) * WW] - to[t * WW];
                tcount2[i] = sl2;
                region[i] = rg;
                halo[i] = pad4(hl);
            }
        }, 256);
        auto vmax = [](const std::vector<int64_t> &v) { return v.empty() ? int64_t(0) : *std::max_element(v.begin(), v.end()); };
        TileStats st;
        st.ntiles = nt;
        st.max_region_pad = vmax(region);
        st.max_region = vmax(region_u);
        st.max_tile_halo = vmax(halo);
        st.max_tcount = vmax(tcount);
        st.max_tcount2 = vmax(tcount2);
        const int64_t smem = choose_tile_params(d, hp, k, st);
        if (paper) break;
        if (smem <= kSmemLimit) break;
        if (k == 0 || d.tile_log2 >= 0)
            fail(P2P_ERROR_NOT_SUPPORTED,
                 "a tile's near-field sources need " + std::to_string(smem) +
                     " B of shared memory (> 200 KB); use a deeper level (CT loop) -- see DESIGN.md");
    }
    hp.k = k;
    {   // NR staging: 2^g lanes per region box, g = ceil(log2(D_occ)) clamped to [1, 5]
        int g = 1;
        while (g < 5 && (double)(1 << g) < hp.density_occ) ++g;
        hp.group_log2 = g;
    }
    const int64_t W = int64_t(1) << k, WW = W * W, R = W + 2;
    const int64_t ntiles = (int64_t)hp.tiles_g.size();
    hp.pairs_global = 0;
    for (int64_t p : hp.tile_pairs_g) hp.pairs_global += p;

    // ---- partition: contiguous Morton ranges of tiles balanced by pair count.
    const int P = d.part_world, r = d.part_rank;
    std::vector<int64_t> box_begin((size_t)P + 1);  // first box of each rank's Morton range
    {
        std::vector<int64_t> prefix((size_t)ntiles + 1, 0);
        for (int64_t i = 0; i < ntiles; ++i) prefix[i + 1] = prefix[i] + hp.tile_pairs_g[i];
        hp.part_tile.assign((size_t)P + 1, 0);
        hp.part_tile[P] = ntiles;
        for (int q = 1; q < P; ++q) {
            // first tile index j with prefix[j] * P >= q * total
            int64_t lo = 0, hi = ntiles;
            while (lo < hi) {
                int64_t mid = (lo + hi) / 2;
                if ((__int128)prefix[mid] * P >= (__int128)q * hp.pairs_global) hi = mid;
                else lo = mid + 1;
            }
            hp.part_tile[q] = std::max<int64_t>(lo, hp.part_tile[q - 1]);
        }
        for (int q = 0; q <= P; ++q) {
            if (q == 0) box_begin[q] = 0;
            else if (q == P || hp.part_tile[q] >= ntiles) box_begin[q] = hp.B;
            else box_begin[q] = (int64_t)hp.tiles_g[hp.part_tile[q]] * WW;
        }
        hp.part_src.resize((size_t)P + 1);
        hp.part_tgt.resize((size_t)P + 1);
        for (int q = 0; q <= P; ++q) {
            hp.part_src[q] = so[box_begin[q]];
            hp.part_tgt[q] = to[box_begin[q]];
        }
        hp.tiles.assign(hp.tiles_g.begin() + hp.part_tile[r], hp.tiles_g.begin() + hp.part_tile[r + 1]);
        hp.pairs = prefix[hp.part_tile[r + 1]] - prefix[hp.part_tile[r]];
    }
    hp.boxes_in_tiles = (int64_t)hp.tiles.size() * WW;

    // Region boxes (tile + ring) of a tile, as Morton codes inside the grid.
    auto region_boxes = [&](int64_t t, std::vector<uint32_t> &out) {
        uint32_t tx, ty;
        morton_decode((uint32_t)t, tx, ty);
        int64_t X0 = (int64_t)tx * W - 1, Y0 = (int64_t)ty * W - 1;
        for (int64_t ly = 0; ly < R; ++ly)
            for (int64_t lx = 0; lx < R; ++lx) {
                int64_t x = X0 + lx, y = Y0 + ly;
                if (x < 0 || y < 0 || x >= S || y >= S) continue;
                out.push_back(morton_encode((uint32_t)x, (uint32_t)y));
            }
    };

    // ---- local input, route-only (p2p_partition_route): which ranks need each passed point
    auto owner_of_box = [&](int64_t b) -> int {
        return (int)(std::upper_bound(box_begin.begin(), box_begin.end(), b) - box_begin.begin()) - 1;
    };
    if (li && (li->src_mask || li->tgt_mask)) {
        const int64_t S2 = hp.S;
        auto tile_nonempty = [&](int64_t t) { return to[(t + 1) * WW] > to[t * WW]; };
        if (li->src_mask)
            parallel_for(d.n_src, [&](int64_t a, int64_t bnd) {
                for (int64_t i = a; i < bnd; ++i) {
                    const uint32_t b = lcode_s[i];
                    uint32_t m = 1u << std::min(owner_of_box(b), 31);
                    uint32_t ix, iy;
                    morton_decode(b, ix, iy);
                    for (int dy = -1; dy <= 1; ++dy)
                        for (int dx = -1; dx <= 1; ++dx) {
                            const int64_t x = (int64_t)ix + dx, y = (int64_t)iy + dy;
                            if (x < 0 || y < 0 || x >= S2 || y >= S2) continue;
                            const int64_t t = (int64_t)morton_encode((uint32_t)x, (uint32_t)y) >> (2 * k);
                            if (tile_nonempty(t)) m |= 1u << owner_of_box(t * WW);
                        }
                    li->src_mask[i] = m;
                }
            });
        if (li->tgt_mask)
            for (int64_t i = 0; i < d.n_tgt; ++i) li->tgt_mask[i] = 1u << owner_of_box(lcode_t[i]);
        return;
    }

    // ---- local source set: all sources (P = 1), or those in the regions of the owned tiles
    // plus every box of the owned Morton range, so that the owned sources -- the global plan
    // range [part_src[r], part_src[r+1]) -- are one contiguous block of the local set (local
    // order = global order) even where an owned box lies outside every owned tile region.
    hp.src_owned_begin = hp.part_src[r];
    hp.n_src_owned = hp.part_src[r + 1] - hp.part_src[r];
    hp.tgt_begin = hp.part_tgt[r];
    hp.n_tgt_local = hp.part_tgt[r + 1] - hp.part_tgt[r];
    if (li) {
        // the marked boxes: (P = 1) every box; else the regions of the owned tiles and the owned
        // box range.  Each must arrive whole: all of its sources, in (box, global id) order.
        std::vector<uint8_t> mark((size_t)hp.B, P == 1 ? 1 : 0);
        if (P > 1) {
            std::vector<uint32_t> boxes;
            for (int32_t t : hp.tiles) {
                boxes.clear();
                region_boxes(t, boxes);
                for (uint32_t m : boxes) mark[m] = 1;
            }
            for (int64_t b = box_begin[r]; b < box_begin[r + 1]; ++b) mark[b] = 1;
        }
        hp.src_off.assign((size_t)hp.B + 1, 0);
        hp.src_gidx.clear();
        hp.src_uidx.clear();
        const int64_t nl = d.n_src;
        int64_t p = 0;
        for (int64_t b = 0; b < hp.B; ++b) {
            const int64_t lo = p;
            while (p < nl && lcode_s[lord_s[p]] == (uint32_t)b) ++p;
            if (mark[b] && ns(b)) {
                if (p - lo != ns(b))
                    fail(P2P_ERROR_INVALID_ARGUMENT, "local input: box " + std::to_string(b) + " needs " +
                                                         std::to_string(ns(b)) + " sources, " +
                                                         std::to_string(p - lo) + " passed");
                for (int64_t j = 0; j < ns(b); ++j) {
                    hp.src_gidx.push_back((int32_t)(so[b] + j));
                    hp.src_uidx.push_back(lord_s[lo + j]);
                }
            }
            hp.src_off[b + 1] = (int32_t)hp.src_gidx.size();
        }
        hp.n_src_local = (int64_t)hp.src_gidx.size();
        // targets: exactly those of the owned box range
        if (d.n_tgt != hp.n_tgt_local)
            fail(P2P_ERROR_INVALID_ARGUMENT, "local input: " + std::to_string(hp.n_tgt_local) + " owned targets, " +
                                                 std::to_string(d.n_tgt) + " passed");
        for (int64_t i = 0; i < d.n_tgt; ++i) {
            const int64_t b = lcode_t[lord_t[i]];
            if (b < box_begin[r] || b >= box_begin[r + 1])
                fail(P2P_ERROR_INVALID_ARGUMENT, "local input: a passed target lies outside this rank's boxes");
        }
    } else if (P == 1) {
        hp.src_off = hp.src_off_g;
        hp.n_src_local = hp.n_src;
        hp.src_gidx.resize((size_t)hp.n_src);
        std::iota(hp.src_gidx.begin(), hp.src_gidx.end(), 0);
    } else {
        std::vector<uint8_t> mark((size_t)hp.B, 0);
        std::vector<uint32_t> boxes;
        for (int32_t t : hp.tiles) {
            boxes.clear();
            region_boxes(t, boxes);
            for (uint32_t m : boxes) mark[m] = 1;
        }
        for (int64_t b = box_begin[r]; b < box_begin[r + 1]; ++b)
            if (so[b + 1] > so[b]) mark[b] = 1;
        hp.src_off.assign((size_t)hp.B + 1, 0);
        hp.src_gidx.clear();
        for (int64_t b = 0; b < hp.B; ++b) {
            if (mark[b])
                for (int32_t g = so[b]; g < so[b + 1]; ++g) hp.src_gidx.push_back(g);
            hp.src_off[b + 1] = (int32_t)hp.src_gidx.size();
        }
        hp.n_src_local = (int64_t)hp.src_gidx.size();
    }
    if (!li) {
        hp.src_uidx.resize((size_t)hp.n_src_local);
        for (int64_t i = 0; i < hp.n_src_local; ++i) hp.src_uidx[i] = hp.src_perm_g[hp.src_gidx[i]];
    }

    hp.tgt_off.resize((size_t)hp.B + 1);
    for (int64_t b = 0; b <= hp.B; ++b)
        hp.tgt_off[b] = (int32_t)std::min<int64_t>(std::max<int64_t>(to[b] - hp.tgt_begin, 0), hp.n_tgt_local);
    if (li) hp.tgt_uidx.assign(lord_t.begin(), lord_t.end());
    else hp.tgt_uidx.assign(hp.tgt_perm_g.begin() + hp.tgt_begin, hp.tgt_perm_g.begin() + hp.tgt_begin + hp.n_tgt_local);

    // ---- halo bookkeeping for the per-apply weight exchange (P > 1).
    hp.recv_counts.assign((size_t)P, 0);
    hp.send_counts.assign((size_t)P, 0);
    hp.src_qidx.resize((size_t)hp.n_src_local);
    {
        int64_t halo = 0;
        hp.halo_lidx.clear();
        hp.owned_local_begin = std::lower_bound(hp.src_gidx.begin(), hp.src_gidx.end(), (int32_t)hp.part_src[r]) -
                               hp.src_gidx.begin();  // local order = global order: owned is contiguous
        for (int64_t i = 0; i < hp.n_src_local; ++i) {
            int64_t g = hp.src_gidx[i];
            if (g >= hp.part_src[r] && g < hp.part_src[r + 1]) {
                hp.src_qidx[i] = (int32_t)(g - hp.part_src[r]);
            } else {
                hp.halo_lidx.push_back((int32_t)i);
                int owner = (int)(std::upper_bound(hp.part_src.begin(), hp.part_src.end(), g) - hp.part_src.begin()) - 1;
                // empty partitions share a begin index; the owner is the last rank starting at or before g
                hp.recv_counts[owner] += 1;
                hp.src_qidx[i] = (int32_t)(hp.n_src_owned + halo++);
            }
        }
        hp.n_halo = halo;
        if (hp.n_src_local - halo != hp.n_src_owned)  // the dist applies copy owned weights as one block
            fail(P2P_ERROR_LAYOUT_CORRUPT, "owned sources are not one contiguous block of the local set");
    }
    if (P > 1) {
        std::vector<uint32_t> boxes;
        const int64_t bb_lo = hp.part_src[r], bb_hi = hp.part_src[r + 1];
        for (int q = 0; q < P; ++q) {
            if (q == r) continue;
            boxes.clear();
            for (int64_t i = hp.part_tile[q]; i < hp.part_tile[q + 1]; ++i) region_boxes(hp.tiles_g[i], boxes);
            std::sort(boxes.begin(), boxes.end());
            boxes.erase(std::unique(boxes.begin(), boxes.end()), boxes.end());
            for (uint32_t m : boxes)
                for (int32_t g = so[m]; g < so[m + 1]; ++g)
                    if (g >= bb_lo && g < bb_hi) {
                        hp.send_idx.push_back((int32_t)(g - bb_lo));
                        hp.send_counts[q] += 1;
                    }
        }
        hp.n_send = (int64_t)hp.send_idx.size();
    }

    // ---- a5 NR layout: box-local coordinates u = x - ix*h (exact in fp64 by Sterbenz).
    // (fp32 R targets: relative to the corner of their 3x3 block, (ix - 1) h -- the R halo's frame,
    // computed in fp64 and rounded once like the halo's sources, so a collocated pair is exactly 0)
    auto fill_points = [&](auto &vec, const double *xy, const std::vector<int32_t> &uidx, int shift = 0) {
        int64_t n = (int64_t)uidx.size();
        vec.resize((size_t)(2 * n));
        parallel_for(n, [&](int64_t a, int64_t bnd) {
            for (int64_t i = a; i < bnd; ++i) {
                double x = xy[2 * (int64_t)uidx[i]], y = xy[2 * (int64_t)uidx[i] + 1];
                vec[2 * i] = (typename std::decay_t<decltype(vec)>::value_type)(x - ((double)cell_of(x, S) - shift) * hp.h);
                vec[2 * i + 1] = (typename std::decay_t<decltype(vec)>::value_type)(y - ((double)cell_of(y, S) - shift) * hp.h);
            }
        });
    };
    if (d.precision == P2P_FP32) {
        fill_points(hp.f32.src_uv, d.src_xy, hp.src_uidx);
        fill_points(hp.f32.tgt_uv, d.tgt_xy, hp.tgt_uidx, d.layout == P2P_LAYOUT_REDUNDANT ? 1 : 0);
    } else {
        fill_points(hp.f64.src_uv, d.src_xy, hp.src_uidx);
        fill_points(hp.f64.tgt_uv, d.tgt_xy, hp.tgt_uidx);
    }

    // ---- a5 R layout: per target box, its E1 sources packed contiguously in
    // the 3x3 row order (dy outer, dx inner), each box padded to an even count,
    // each tile to 4.  Coordinates are relative to the target box origin (fp64),
    // or in fp32 to the corner of its 3x3 block, (ix - 1, iy - 1) h: every target
    // then sits >= h from the frame origin, so two fp32 coordinates either
    // coincide or differ by >= ulp(h/2) >= 2^-38 > eps, and the fast loop's
    // r^2 = 0 check is the whole guard (R17).
    if (d.layout == P2P_LAYOUT_REDUNDANT) {
        const int64_t nlt = (int64_t)hp.tiles.size();
        std::vector<uint32_t> len((size_t)hp.B + 1, 0);
        for (int64_t i = 0; i < nlt; ++i) {
            int64_t t = hp.tiles[i], tot = 0;
            for (int64_t b = t * WW; b < (t + 1) * WW; ++b)
                if (ntg(b)) {
                    len[b] = (uint32_t)pad2(n9[b]);
                    tot += len[b];
                }
            len[(t + 1) * WW - 1] += (uint32_t)(pad4(tot) - tot);
        }
        hp.halo_off.assign((size_t)hp.B + 1, 0);
        for (int64_t b = 0; b < hp.B; ++b) hp.halo_off[b + 1] = hp.halo_off[b] + len[b];
        hp.halo_entries = hp.halo_off[hp.B];
        if (hp.halo_entries > (int64_t)UINT32_MAX - 8) fail(P2P_ERROR_NOT_SUPPORTED, "R halo exceeds 2^32 entries");
        hp.halo_idx.assign((size_t)hp.halo_entries, -1);
        const double PADC = 1.0e4;
        const bool f32 = d.precision == P2P_FP32;
        if (f32) hp.f32.halo_uv.assign((size_t)hp.halo_entries * 2, (float)PADC);
        else hp.f64.halo_uv.assign((size_t)hp.halo_entries * 2, PADC);
        const double *sxy = d.src_xy;
        parallel_for(nlt, [&](int64_t a, int64_t bnd) {
            for (int64_t i = a; i < bnd; ++i) {
                int64_t t = hp.tiles[i];
                for (int64_t b = t * WW; b < (t + 1) * WW; ++b) {
                    if (!ntg(b)) continue;
                    uint32_t ix, iy;
                    morton_decode((uint32_t)b, ix, iy);
                    double ox = ix * hp.h, oy = iy * hp.h;
                    if (f32) {
                        ox -= hp.h;
                        oy -= hp.h;
                    }
                    int64_t ent = hp.halo_off[b];
                    for (int dy = -1; dy <= 1; ++dy)
                        for (int dx = -1; dx <= 1; ++dx) {
                            int64_t x = (int64_t)ix + dx, y = (int64_t)iy + dy;
                            if (x < 0 || y < 0 || x >= S || y >= S) continue;
                            uint32_t m = morton_encode((uint32_t)x, (uint32_t)y);
                            for (int32_t j = hp.src_off[m]; j < hp.src_off[m + 1]; ++j, ++ent) {
                                int64_t u = hp.src_uidx[j];
                                double rx = sxy[2 * u] - ox, ry = sxy[2 * u + 1] - oy;
                                hp.halo_idx[ent] = j;
                                if (f32) {  // (u0,u1,v0,v1) per source pair
                                    int64_t p = ent >> 1, s = ent & 1;
                                    hp.f32.halo_uv[4 * p + s] = (float)rx;
                                    hp.f32.halo_uv[4 * p + 2 + s] = (float)ry;
                                } else {
                                    hp.f64.halo_uv[2 * ent] = rx;
                                    hp.f64.halo_uv[2 * ent + 1] = ry;
                                }
                            }
                        }
                }
            }
        }, 64);
    }
    // ---- TILED layout: per local tile (Morton order = slot), its region (tile +
    // one-box ring) in row-major box order, each box padded to an even count,
    // each tile to 4 entries; coordinates relative to the region origin
    // ((tx*W - 1) h, (ty*W - 1) h), computed in fp64 and rounded once.
    const int64_t nlt = (int64_t)hp.tiles.size();
    hp.tile_slot.resize((size_t)nlt);
    std::iota(hp.tile_slot.begin(), hp.tile_slot.end(), 0);
    if (d.layout == P2P_LAYOUT_TILED) {
        const int ts = tiled_table_stride(k);
        hp.reg_off.assign((size_t)nlt + 1, 0);
        hp.reg_table.assign((size_t)nlt * ts, 0);
        for (int64_t i = 0; i < nlt; ++i) {  // sizes and tables
            uint32_t tx, ty;
            morton_decode((uint32_t)hp.tiles[i], tx, ty);
            const int64_t X0 = (int64_t)tx * W - 1, Y0 = (int64_t)ty * W - 1;
            int64_t run = 0;
            for (int64_t j = 0; j < R * R; ++j) {
                hp.reg_table[i * ts + j] = (uint16_t)run;
                const int64_t x = X0 + j % R, y = Y0 + j / R;
                if (x < 0 || y < 0 || x >= S || y >= S) continue;
                const uint32_t m = morton_encode((uint32_t)x, (uint32_t)y);
                const int64_t cnt = hp.src_off[m + 1] - hp.src_off[m];
                run += hp.pad ? pad2(cnt) : cnt;
            }
            if (run > 65535) fail(P2P_ERROR_NOT_SUPPORTED, "TILED region exceeds 65535 entries; use NR");
            hp.reg_table[i * ts + R * R] = (uint16_t)run;
            hp.reg_off[i + 1] = hp.reg_off[i] + (uint32_t)pad4(run);
        }
        hp.reg_entries = hp.reg_off[nlt];
        hp.table_entries = (int64_t)hp.reg_table.size();
        hp.reg_idx.assign((size_t)hp.reg_entries, -1);
        hp.reg_uidx.assign((size_t)hp.reg_entries, -1);
        const double PADC = 1.0e4;
        const bool f32 = d.precision == P2P_FP32;
        if (f32) hp.f32.reg_uv.assign((size_t)hp.reg_entries * 2, (float)PADC);
        else hp.f64.reg_uv.assign((size_t)hp.reg_entries * 2, PADC);
        const double *sxy = d.src_xy;
        parallel_for(nlt, [&](int64_t a, int64_t bnd) {
            for (int64_t i = a; i < bnd; ++i) {
                uint32_t tx, ty;
                morton_decode((uint32_t)hp.tiles[i], tx, ty);
                const int64_t X0 = (int64_t)tx * W - 1, Y0 = (int64_t)ty * W - 1;
                const double ox = X0 * hp.h, oy = Y0 * hp.h;
                for (int64_t j = 0; j < R * R; ++j) {
                    const int64_t x = X0 + j % R, y = Y0 + j / R;
                    if (x < 0 || y < 0 || x >= S || y >= S) continue;
                    const uint32_t m = morton_encode((uint32_t)x, (uint32_t)y);
                    int64_t ent = hp.reg_off[i] + hp.reg_table[i * ts + j];
                    for (int32_t sj = hp.src_off[m]; sj < hp.src_off[m + 1]; ++sj, ++ent) {
                        const int64_t u = hp.src_uidx[sj];
                        const double rx = sxy[2 * u] - ox, ry = sxy[2 * u + 1] - oy;
                        hp.reg_idx[ent] = sj;
                        hp.reg_uidx[ent] = (int32_t)u;
                        if (f32 && hp.pad) {  // (u0,u1,v0,v1) per source pair
                            const int64_t p = ent >> 1, sl = ent & 1;
                            hp.f32.reg_uv[4 * p + sl] = (float)rx;
                            hp.f32.reg_uv[4 * p + 2 + sl] = (float)ry;
                        } else if (f32) {     // (u, v) per entry
                            hp.f32.reg_uv[2 * ent] = (float)rx;
                            hp.f32.reg_uv[2 * ent + 1] = (float)ry;
                        } else {
                            hp.f64.reg_uv[2 * ent] = rx;
                            hp.f64.reg_uv[2 * ent + 1] = ry;
                        }
                    }
                }
            }
        }, 64);
        // target slots, packed per tile (8-entry aligned for the bulk copy): the
        // tile's target boxes in Morton order (NS = 1 plans: by descending n9, so
        // the lanes of a warp sweep near-equal pair counts), each box's targets in
        // plan order; TPI = 2: units = consecutive slot pairs of one box, odd boxes
        // end with a duplicate slot (output index 0xFFFF).  Per slot: coordinates
        // relative to the region origin, row-run base j0 = by*R + bx, output index.
        const int tpi = hp.tpi;
        auto box_slots = [&](int64_t b) {
            const int64_t c = hp.tgt_off[b + 1] - hp.tgt_off[b];
            return tpi == 2 ? c + (c & 1) : c;
        };
        hp.tgt_pack_off.assign((size_t)nlt + 1, 0);
        hp.tile_tgt_base.assign((size_t)nlt, 0);
        for (int64_t i = 0; i < nlt; ++i) {
            const int64_t m0 = (int64_t)hp.tiles[i] * WW;
            int64_t n = 0;
            for (int64_t bl = 0; bl < WW; ++bl) n += box_slots(m0 + bl);
            if (n > (hp.ns == 3 ? 16383 * tpi : 65534))
                fail(P2P_ERROR_NOT_SUPPORTED, "TILED tile exceeds its target-slot limit; use a deeper level or NR");
            hp.tile_tgt_base[i] = hp.tgt_off[m0];
            hp.tgt_pack_off[i + 1] = hp.tgt_pack_off[i] + (uint32_t)pad8(n);
            hp.reg_table[i * ts + R * R + 1] = (uint16_t)n;
        }
        const int64_t np = hp.tgt_pack_off[nlt];
        hp.tgt_bl.assign((size_t)np, 0);
        hp.tgt_oix.assign((size_t)np, 0xFFFF);
        if (f32) hp.f32.tgt_ruv.assign((size_t)np * 2, 0.f);
        else hp.f64.tgt_ruv.assign((size_t)np * 2, 0.0);
        const double *txy = d.tgt_xy;
        parallel_for(nlt, [&](int64_t a, int64_t bnd) {
            std::vector<int32_t> order;
            for (int64_t i = a; i < bnd; ++i) {
                const uint32_t t = (uint32_t)hp.tiles[i];
                uint32_t tx, ty;
                morton_decode(t, tx, ty);
                const double ox = ((int64_t)tx * W - 1) * hp.h, oy = ((int64_t)ty * W - 1) * hp.h;
                const int64_t m0 = (int64_t)t * WW, g0 = hp.tgt_off[m0];
                order.resize((size_t)WW);
                std::iota(order.begin(), order.end(), 0);
                if (hp.tsort)
                    std::stable_sort(order.begin(), order.end(),
                                     [&](int32_t x, int32_t y) { return n9[(size_t)(m0 + x)] > n9[(size_t)(m0 + y)]; });
                int64_t j = hp.tgt_pack_off[i];
                for (int32_t bl : order) {
                    const int64_t b = m0 + bl, ns_b = box_slots(b);
                    uint32_t bx, by;
                    morton_decode((uint32_t)bl, bx, by);
                    for (int64_t x = 0; x < ns_b; ++x, ++j) {
                        const int64_t g = std::min<int64_t>(hp.tgt_off[b] + x, hp.tgt_off[b + 1] - 1);
                        const int64_t u = hp.tgt_uidx[g];
                        hp.tgt_bl[j] = (uint16_t)(by * R + bx);
                        if (hp.tgt_off[b] + x < hp.tgt_off[b + 1]) hp.tgt_oix[j] = (uint16_t)(g - g0);
                        if (f32) {
                            hp.f32.tgt_ruv[2 * j] = (float)(txy[2 * u] - ox);
                            hp.f32.tgt_ruv[2 * j + 1] = (float)(txy[2 * u + 1] - oy);
                        } else {
                            hp.f64.tgt_ruv[2 * j] = txy[2 * u] - ox;
                            hp.f64.tgt_ruv[2 * j + 1] = txy[2 * u + 1] - oy;
                        }
                    }
                }
            }
        }, 64);
    }

    // ---- queue order of this partition's tiles: when the working set fits
    // comfortably in L2, longest tiles first (LPT) to shorten the tail; else
    // Morton order, so concurrently running CTAs share their halo rings in L2
    // (and the tail is split instead, below).
    {
        const int64_t ws = (hp.n_src_local + hp.n_tgt_local) * 3 * (int64_t)e + 8 * hp.boxes_in_tiles +
                           (hp.halo_entries + hp.reg_entries) * 3 * (int64_t)e;
        hp.lpt = ws < (int64_t)100 << 20;  // L2 = 126 MB; measured (tools/gpu/gpu_ab12.sh)
        if (const char *v = std::getenv("P2P_LPT")) hp.lpt = std::atoi(v) != 0;  // tuning hook
        if (hp.lpt) {
            const int64_t base = hp.part_tile[r];
            std::vector<int64_t> order(hp.tiles.size());
            std::iota(order.begin(), order.end(), 0);
            std::stable_sort(order.begin(), order.end(), [&](int64_t x, int64_t y) {
                return hp.tile_pairs_g[base + x] > hp.tile_pairs_g[base + y];
            });
            std::vector<int32_t> t2(hp.tiles.size()), s2(hp.tiles.size());
            for (size_t i = 0; i < order.size(); ++i) {
                t2[i] = hp.tiles[order[i]];
                s2[i] = hp.tile_slot[order[i]];
            }
            hp.tiles.swap(t2);
            hp.tile_slot.swap(s2);
        }
    }
    // ---- interior tiles first (TILED, P > 1): tiles whose regions hold owned sources only can
    // run before the halo weights arrive (p2p_apply_dist_interior), overlapping the exchange;
    // the boundary tiles follow (p2p_apply_dist_boundary).  Relative order kept in each class.
    hp.n_interior = (int64_t)hp.tiles.size();
    if (d.layout == P2P_LAYOUT_TILED && P > 1) {
        const int64_t lo = hp.owned_local_begin, hi = hp.owned_local_begin + hp.n_src_owned;
        std::vector<uint8_t> interior(hp.tiles.size(), 1);
        for (size_t li = 0; li < hp.tiles.size(); ++li) {
            const int32_t slot = hp.tile_slot[li];
            for (uint32_t e = hp.reg_off[slot]; e < hp.reg_off[slot + 1]; ++e) {
                const int32_t x = hp.reg_idx[e];
                if (x >= 0 && (x < lo || x >= hi)) {
                    interior[li] = 0;
                    break;
                }
            }
        }
        std::vector<size_t> ord(hp.tiles.size());
        std::iota(ord.begin(), ord.end(), 0);
        std::stable_partition(ord.begin(), ord.end(), [&](size_t x) { return interior[x] != 0; });
        std::vector<int32_t> t2(ord.size()), s2(ord.size());
        for (size_t i = 0; i < ord.size(); ++i) {
            t2[i] = hp.tiles[ord[i]];
            s2[i] = hp.tile_slot[ord[i]];
        }
        hp.tiles.swap(t2);
        hp.tile_slot.swap(s2);
        hp.n_interior = std::count(interior.begin(), interior.end(), (uint8_t)1);
    }
    // ---- tile splitting (TILED): a queue entry may run a unit range of its tile (each target is
    // still computed whole by one thread: results do not depend on the split).
    //   tail: without LPT, the last 592 queue entries are split in 4 so the final wave is
    //         fine-grained (LPT already ends on the short tiles);
    //   heavy: a tile holding more than 1/1184 of the partition's pairs is split into
    //         ceil(pairs / that share) parts (<= 32) -- clustered clouds (a curve, NEXT-4) put
    //         a large share of the work in a few tiles, and one CTA per tile would serialise it.
    hp.tile_part.assign(hp.tiles.size(), 1 << 16);
    if (d.layout == P2P_LAYOUT_TILED) {
        int64_t tail = hp.lpt ? 0 : 148 * 4, parts = 4;
        if (const char *v = std::getenv("P2P_TAIL_TILES")) tail = std::atoll(v);
        if (const char *v = std::getenv("P2P_TAIL_PARTS")) parts = std::max(1, std::min(16, std::atoi(v)));
        tail = std::min<int64_t>(tail, (int64_t)hp.tiles.size() / 2);
        const int64_t keep = parts > 1 && tail > 0 ? (int64_t)hp.tiles.size() - tail : (int64_t)hp.tiles.size();
        const int64_t share = std::max<int64_t>(1, (hp.pairs + kSplitShare - 1) / kSplitShare);
        std::vector<int32_t> t2, s2, p2;
        int64_t n_int = 0;
        for (int64_t i = 0; i < (int64_t)hp.tiles.size(); ++i) {
            const int64_t tp = hp.tile_pairs_g[hp.part_tile[r] + hp.tile_slot[i]];
            const int64_t np_ = split_parts(tp, share, i >= keep ? parts : 1);
            for (int64_t q = 0; q < np_; ++q) {
                t2.push_back(hp.tiles[i]);
                s2.push_back(hp.tile_slot[i]);
                p2.push_back((int32_t)(q | (np_ << 16)));
            }
            if (i < hp.n_interior) n_int += np_;
        }
        hp.tiles.swap(t2);
        hp.tile_slot.swap(s2);
        hp.tile_part.swap(p2);
        hp.n_interior = n_int;
    }
    // ---- fp64 log table: log x = e ln2 + L_k + log1p(t), t = m c_inv_k - 1, |t| < 2^-8, with
    // c_inv_k = 1 / (1 + (k + 1/2) / 128) rounded to double and L_k = -log(c_inv_k) from the
    // 64-bit-mantissa long double log (the kernel's `log_tab`)
    if (d.precision == P2P_FP64) build_log_table(hp);
    // ---- NS = 3 item lists (TILED): per tile, the (unit, row-run) items of each
    // part's unit range [nu*ip/np, nu*(ip+1)/np) sorted by row-run length
    // (descending, stable), so the lanes of a warp sweep near-equal runs.
    if (d.layout == P2P_LAYOUT_TILED && hp.ns == 3) {
        const int ts = tiled_table_stride(k), tpi = hp.tpi;
        std::vector<int32_t> nparts((size_t)nlt, 1);
        for (size_t li = 0; li < hp.tile_slot.size(); ++li) nparts[hp.tile_slot[li]] = hp.tile_part[li] >> 16;
        hp.item_off.assign((size_t)nlt + 1, 0);
        for (int64_t i = 0; i < nlt; ++i)
            hp.item_off[i + 1] = hp.item_off[i] + (uint32_t)pad8(3 * (hp.reg_table[i * ts + R * R + 1] / tpi));
        hp.items.assign(hp.item_off[nlt], 0);
        const int nt = hp.nt;
        bool balance = true;  // P2P_BALANCE=0: items in plain length order (A/B)
        if (const char *v = std::getenv("P2P_BALANCE")) balance = std::atoi(v) != 0;
        parallel_for(nlt, [&](int64_t a, int64_t bnd) {
            std::vector<int32_t> len, ord, lay;
            for (int64_t i = a; i < bnd; ++i) {
                const uint16_t *tab = &hp.reg_table[i * ts];
                const int64_t nu = tab[R * R + 1] / tpi, tb = hp.tgt_pack_off[i], np_ = nparts[i];
                len.assign((size_t)(3 * nu), 0);
                for (int64_t u = 0; u < nu; ++u)
                    for (int row = 0; row < 3; ++row) {
                        const int64_t j0 = hp.tgt_bl[tb + tpi * u] + row * R;
                        len[3 * u + row] = tab[j0 + 3] - tab[j0];
                    }
                for (int64_t ip = 0; ip < np_; ++ip) {
                    const int64_t ub = nu * ip / np_, ue = nu * (ip + 1) / np_;
                    ord.resize((size_t)(3 * (ue - ub)));
                    std::iota(ord.begin(), ord.end(), (int32_t)(3 * ub));
                    std::stable_sort(ord.begin(), ord.end(), [&](int32_t x, int32_t y) { return len[x] > len[y]; });
                    if (balance) balance_batches(ord, len, nt, lay);
                    else lay = ord;
                    for (size_t q = 0; q < lay.size(); ++q)
                        hp.items[hp.item_off[i] + 3 * ub + q] = (uint16_t)((lay[q] / 3) << 2 | (lay[q] % 3));
                }
            }
        }, 64);
    }
    // ---- the paper's layouts, as written (§3.2-3.3; SPEC.md layouts)
    if (paper) {
        const std::vector<int64_t> nb = neighbors_export(hp);  // E1 per box, ascending Morton
        if (d.layout == P2P_LAYOUT_PAPER_INDEXING) {
            // per box, the original indices of its E1 sources: neighbour boxes ascending Morton,
            // sources in per-box (original index) order; boxes in Morton order
            hp.pi_nei_off.assign((size_t)hp.B + 1, 0);
            int64_t tot = 0;
            for (int64_t b = 0; b < hp.B; ++b) {
                for (int c = 0; c < 9 && nb[9 * b + c] >= 0; ++c)
                    tot += hp.src_off_g[nb[9 * b + c] + 1] - hp.src_off_g[nb[9 * b + c]];
                if (tot > INT32_MAX) fail(P2P_ERROR_NOT_SUPPORTED, "PAPER_INDEXING: > 2^31 neighbour entries");
                hp.pi_nei_off[b + 1] = (int32_t)tot;
            }
            hp.pi_nei_idx.resize((size_t)tot);
            hp.pi_src_xy.assign(d.src_xy, d.src_xy + 2 * hp.n_src);
            hp.pi_tgt_xy.assign(d.tgt_xy, d.tgt_xy + 2 * hp.n_tgt);
            parallel_for(hp.B, [&](int64_t a, int64_t bnd) {
                for (int64_t b = a; b < bnd; ++b) {
                    int64_t e = hp.pi_nei_off[b];
                    for (int c = 0; c < 9 && nb[9 * b + c] >= 0; ++c)
                        for (int32_t g = hp.src_off_g[nb[9 * b + c]]; g < hp.src_off_g[nb[9 * b + c] + 1]; ++g)
                            hp.pi_nei_idx[e++] = hp.src_perm_g[g];
                }
            }, 4096);
            // Eq. 3: 5N Double + 4^(L-1)(2 + t + 9t) Integer (source/target counts may differ)
            int64_t four_L = 1;
            for (int i = 0; i < L; ++i) four_L *= 4;
            hp.paper_model_bytes = 8 * (3 * hp.n_src + 2 * hp.n_tgt) + four_L * (2 + 10 * hp.t_max);
        } else {
            // one record per target (caller's order): [x_t, y_t, count, (x_s, y_s, q_s) x count],
            // stride 3 + 27 C with C = max(ct, t): a record must hold 9t sources (levels below the
            // CT loop's choice, level_delta < 0, exceed ct) -- DESIGN.md R20
            const int64_t C = std::max<int64_t>(d.ct, hp.t_max);
            hp.pr_maxn = 9 * C;
            hp.pr_stride = 3 + 27 * C;
            const double bytes = 8.0 * (double)hp.n_tgt * (double)hp.pr_stride;
            if (bytes > 16.0e9) fail(P2P_ERROR_NOT_SUPPORTED, "PAPER_REPETITION records would exceed 16 GB");
            hp.pr_records.assign((size_t)(hp.n_tgt * hp.pr_stride), 0.0);
            hp.pr_slot.assign((size_t)(hp.n_tgt * hp.pr_maxn), -1);
            const double *sxy = d.src_xy, *txy = d.tgt_xy;
            parallel_for(hp.B, [&](int64_t a, int64_t bnd) {
                for (int64_t b = a; b < bnd; ++b)
                    for (int32_t i = hp.tgt_off_g[b]; i < hp.tgt_off_g[b + 1]; ++i) {
                        const int64_t r = hp.tgt_perm_g[i];
                        double *rec = &hp.pr_records[(size_t)(r * hp.pr_stride)];
                        int32_t *sl = &hp.pr_slot[(size_t)(r * hp.pr_maxn)];
                        rec[0] = txy[2 * r];
                        rec[1] = txy[2 * r + 1];
                        int64_t cnt = 0;
                        for (int c = 0; c < 9 && nb[9 * b + c] >= 0; ++c)
                            for (int32_t g = hp.src_off_g[nb[9 * b + c]]; g < hp.src_off_g[nb[9 * b + c] + 1]; ++g) {
                                const int64_t s = hp.src_perm_g[g];
                                rec[3 + 3 * cnt] = sxy[2 * s];
                                rec[3 + 3 * cnt + 1] = sxy[2 * s + 1];
                                sl[cnt++] = (int32_t)s;
                            }
                        // the count: an integer in the low 4 bytes of a double slot (SPEC.md layouts)
                        const uint64_t bits = (uint64_t)(uint32_t)cnt;
                        std::memcpy(&rec[2], &bits, 8);
                    }
            }, 1024);
            hp.paper_model_bytes = 8 * hp.n_tgt * (3 + 27 * (int64_t)d.ct);  // Eq. 8
        }
    }
    hp.build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

std::vector<int64_t> neighbors_export(const HostPlan &hp) {
    if (hp.dim == 3 || hp.layout == P2P_LAYOUT_ADAPTIVE) fail(P2P_ERROR_NOT_SUPPORTED, "neighbour export: uniform 2D plans");
    std::vector<int64_t> nb((size_t)hp.B * 9, -1);
    for (int64_t b = 0; b < hp.B; ++b) {
        uint32_t ix, iy;
        morton_decode((uint32_t)b, ix, iy);
        int64_t list[9];
        int c = 0;
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                int64_t x = (int64_t)ix + dx, y = (int64_t)iy + dy;
                if (x < 0 || y < 0 || x >= hp.S || y >= hp.S) continue;
                list[c++] = morton_encode((uint32_t)x, (uint32_t)y);
            }
        std::sort(list, list + c);
        std::copy(list, list + c, nb.begin() + 9 * b);
    }
    return nb;
}

}  // namespace p2p
