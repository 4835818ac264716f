// plan_device.cuh -- the plan build on the GPU: the paper's "collection" (§3.2,
// §3.3; its dominant cost, alpha ~ 0.82 of the total) moved onto the
// B200.  Included by p2p_capi.cu (it fills a p2p_plan_s).
//
// Steps, each a device pass over device-resident coordinates:
//   a1 level: explicit, or the CT loop (§3.1) from codes sorted once at l_max
//      (max run of a Morton prefix = max points in a box of that level);
//   a2 box assignment + Morton code;
//   a3 stable radix sort (CUB) of (code, index) -> permutation; CSR offsets by lower_bound
//      over the sorted codes (the paper's "second order index");
//   box statistics (occupancy, t, E1 source counts n9: PAPER.md L88 3x3 clipped);
//   CTA tiles (non-empty Morton-aligned 2^k x 2^k blocks), per-tile statistics, then the
//   same kernel-option choice as the host builder (choose_tile_params);
//   a5 layouts: NR (box-local coordinates) or TILED (per tile: region table, packed region,
//   target slots, item lists), queue order (longest first when the working set fits L2,
//   else Morton with a split tail).
// The result is bit-identical to the host builder's plan (tests/test_device_plan.py compares
// every exported array).  Scope: one partition (part_world = 1), NR and TILED layouts, the
// default kernel options (the P2P_* tuning hooks are honoured where they only change the
// option choice; P2P_LPT / P2P_TAIL_* likewise).
#pragma once

#include <cub/cub.cuh>

namespace p2p {
namespace dbuild {

constexpr int kB = 256;  // threads per block of the build kernels

inline unsigned nblocks(int64_t n, int per = kB) {
    int64_t g = (n + per - 1) / per;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(g, 148LL * 64));
}

__device__ __forceinline__ uint32_t spread(uint32_t v) {
    v &= 0x0000FFFFu;
    v = (v | (v << 8)) & 0x00FF00FFu;
    v = (v | (v << 4)) & 0x0F0F0F0Fu;
    v = (v | (v << 2)) & 0x33333333u;
    v = (v | (v << 1)) & 0x55555555u;
    return v;
}
__device__ __forceinline__ uint32_t compact(uint32_t v) {
    v &= 0x55555555u;
    v = (v | (v >> 1)) & 0x33333333u;
    v = (v | (v >> 2)) & 0x0F0F0F0Fu;
    v = (v | (v >> 4)) & 0x00FF00FFu;
    v = (v | (v >> 8)) & 0x0000FFFFu;
    return v;
}
__device__ __forceinline__ uint32_t menc(uint32_t x, uint32_t y) { return spread(x) | (spread(y) << 1); }
// floor(x S) is exact (S a power of two); closed at the upper edge
__device__ __forceinline__ uint32_t cell(double x, int64_t S) {
    int64_t c = (int64_t)floor(x * (double)S);
    c = c > S - 1 ? S - 1 : c;
    return (uint32_t)(c < 0 ? 0 : c);
}
__device__ __forceinline__ int64_t p2(int64_t n) { return (n + 1) & ~int64_t(1); }
__device__ __forceinline__ int64_t p4(int64_t n) { return (n + 3) & ~int64_t(3); }
__device__ __forceinline__ int64_t p8(int64_t n) { return (n + 7) & ~int64_t(7); }

// first coordinate outside [0,1] (or NaN): min flat index into *bad (init UINT64_MAX)
__global__ void validate_kernel(const double *__restrict__ xy, int64_t n2, unsigned long long *bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = xy[i];
        if (!(v >= 0.0 && v <= 1.0)) atomicMin(bad, (unsigned long long)i);
    }
}

// a2: Morton code of each point's leaf box at grid side S; idx = iota (sort values)
__global__ void codes_kernel(const double2 *__restrict__ xy, int64_t n, int64_t S, uint32_t *__restrict__ code,
                             int32_t *__restrict__ idx) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double2 p = xy[i];
        code[i] = menc(cell(p.x, S), cell(p.y, S));
        if (idx) idx[i] = (int32_t)i;
    }
}

// a1 (CT loop): for every level L in [l0, l1], the longest run of equal code prefixes
// (code >> 2(lmax - L)) in the sorted codes = the most points in one box at level L.
__global__ void maxrun_kernel(const uint32_t *__restrict__ c, int64_t n, int l0, int l1, int lmax,
                              int64_t *__restrict__ mr) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        for (int L = l0; L <= l1; ++L) {
            const int sh = 2 * (lmax - L);
            const uint32_t key = c[i] >> sh;
            if (i > 0 && (c[i - 1] >> sh) == key) continue;  // not the start of a run
            int64_t lo = i, step = 1, hi;                     // gallop, then bisect: end of the run
            for (;;) {
                hi = i + step;
                if (hi >= n || (c[hi] >> sh) != key) break;
                lo = hi;
                step <<= 1;
            }
            if (hi > n) hi = n;
            while (hi - lo > 1) {  // c[lo] in the run; hi is past it (or n)
                const int64_t mid = (lo + hi) / 2;
                if ((c[mid] >> sh) == key) lo = mid;
                else hi = mid;
            }
            atomicMax((unsigned long long *)&mr[L], (unsigned long long)(lo + 1 - i));
        }
    }
}

// a3: CSR offsets off[b] = #points with code < b, b in [0, B]
__global__ void offsets_kernel(const uint32_t *__restrict__ c, int64_t n, int64_t B, int32_t *__restrict__ off) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b <= B; b += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            const int64_t mid = (lo + hi) / 2;
            if ((int64_t)c[mid] < b) lo = mid + 1;
            else hi = mid;
        }
        off[b] = (int32_t)lo;
    }
}

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
    for (int o = 16; o; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ long long warp_max(long long v) {
    for (int o = 16; o; o >>= 1) v = max(v, __shfl_down_sync(0xffffffffu, v, o));
    return v;
}

// Box statistics: acc[0] += occupied source boxes, acc[1] += occupied target boxes,
// acc[2] = max(#src, #tgt) over boxes (t); n9[b] = E1 sources of every target-occupied box.
__global__ void box_stats_kernel(const int32_t *__restrict__ so, const int32_t *__restrict__ to, int64_t B,
                                 int64_t S, int32_t *__restrict__ n9, unsigned long long *acc) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t nround = (B + stride - 1) / stride;
    for (int64_t r = 0; r < nround; ++r) {  // uniform trip count: whole warps reach the shuffles
        const int64_t b = r * stride + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
        unsigned long long os = 0, ot = 0;
        long long tm = 0;
        if (b < B) {
            const int64_t a = so[b + 1] - so[b], t = to[b + 1] - to[b];
            os = a > 0;
            ot = t > 0;
            tm = max(a, t);
            int32_t c = 0;
            if (t) {
                const uint32_t ix = compact((uint32_t)b), iy = compact((uint32_t)b >> 1);
                for (int dy = -1; dy <= 1; ++dy)
                    for (int dx = -1; dx <= 1; ++dx) {
                        const int64_t x = (int64_t)ix + dx, y = (int64_t)iy + dy;
                        if (x < 0 || y < 0 || x >= S || y >= S) continue;
                        const uint32_t m = menc((uint32_t)x, (uint32_t)y);
                        c += so[m + 1] - so[m];
                    }
            }
            n9[b] = c;
        }
        os = warp_sum(os);
        ot = warp_sum(ot);
        tm = warp_max(tm);
        if ((threadIdx.x & 31) == 0) {
            if (os) atomicAdd(&acc[0], os);
            if (ot) atomicAdd(&acc[1], ot);
            atomicMax((unsigned long long *)&acc[2], (unsigned long long)tm);
        }
    }
}

// Non-empty tiles at every tile size kk <= kmax (the auto tile-size choice): ne[kk] += 1 for
// each Morton-aligned block of 4^kk boxes holding a target.
__global__ void tile_count_kernel(const int32_t *__restrict__ to, int64_t B, int kmax, unsigned long long *ne) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t nround = (B + stride - 1) / stride;
    for (int64_t r = 0; r < nround; ++r) {
        const int64_t b = r * stride + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
        for (int kk = 0; kk <= kmax; ++kk) {
            const int64_t WW = int64_t(1) << (2 * kk);
            unsigned long long f = 0;
            if (b < B && (b & (WW - 1)) == 0) f = to[b + WW] > to[b];
            f = warp_sum(f);
            if ((threadIdx.x & 31) == 0 && f) atomicAdd(&ne[kk], f);
        }
    }
}

__global__ void tile_flag_kernel(const int32_t *__restrict__ to, int64_t ntile_all, int64_t WW,
                                 int32_t *__restrict__ flag) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ntile_all; t += (int64_t)gridDim.x * blockDim.x)
        flag[t] = to[(t + 1) * WW] > to[t * WW];
}

__global__ void compact_kernel(const int32_t *__restrict__ flag, const int32_t *__restrict__ pos, int64_t n,
                               int32_t *__restrict__ out) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        if (flag[t]) out[pos[t]] = (int32_t)t;
}

// Per non-empty tile: pairs (sum over its target boxes of #targets x n9), region sizes (tile +
// one-box ring; padded and unpadded), target counts; maxima into st[0..4] and the pair total
// into st[5]: {region_pad, region, tcount, tcount2, unused, pairs}.
__global__ void tile_stats_kernel(const int32_t *__restrict__ tiles, int64_t nt, int k, int64_t S,
                                  const int32_t *__restrict__ so, const int32_t *__restrict__ to,
                                  const int32_t *__restrict__ n9, int64_t *__restrict__ tile_pairs,
                                  unsigned long long *st) {
    const int64_t W = int64_t(1) << k, WW = W * W, R = W + 2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nt; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = tiles[i];
        int64_t pr = 0, sl2 = 0;
        for (int64_t b = t * WW; b < (t + 1) * WW; ++b) {
            const int64_t c = to[b + 1] - to[b];
            if (!c) continue;
            sl2 += c + (c & 1);
            pr += c * (int64_t)n9[b];
        }
        const int64_t X0 = (int64_t)compact((uint32_t)t) * W - 1, Y0 = (int64_t)compact((uint32_t)t >> 1) * W - 1;
        int64_t rg = 0, rgu = 0;
        for (int64_t ly = 0; ly < R; ++ly)
            for (int64_t lx = 0; lx < R; ++lx) {
                const int64_t x = X0 + lx, y = Y0 + ly;
                if (x < 0 || y < 0 || x >= S || y >= S) continue;
                const uint32_t m = menc((uint32_t)x, (uint32_t)y);
                const int64_t c = so[m + 1] - so[m];
                rg += p2(c);
                rgu += c;
            }
        tile_pairs[i] = pr;
        atomicMax(&st[0], (unsigned long long)rg);
        atomicMax(&st[1], (unsigned long long)rgu);
        atomicMax(&st[2], (unsigned long long)(to[(t + 1) * WW] - to[t * WW]));
        atomicMax(&st[3], (unsigned long long)sl2);
        atomicAdd(&st[5], (unsigned long long)pr);
    }
}

// NR layout: box-local coordinates of the points in plan order, u = x - ix h (exact in fp64).
template <typename T>
__global__ void uv_kernel(const double2 *__restrict__ xy, const int32_t *__restrict__ perm, int64_t n, int64_t S,
                          double h, T *__restrict__ uv) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double2 p = xy[perm[i]];
        uv[2 * i] = (T)(p.x - (double)cell(p.x, S) * h);
        uv[2 * i + 1] = (T)(p.y - (double)cell(p.y, S) * h);
    }
}

template <typename V>
__global__ void fill_kernel(V *__restrict__ p, int64_t n, V v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

__global__ void iota_kernel(int32_t *__restrict__ p, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = (int32_t)i;
}

// TILED, per tile (one thread): the region table (start of every box of the (W+2)^2 region in
// row-major order, then the region size and the slot count), the region's padded size and the
// tile's slot and item counts.  err[0] |= 1: region > 65535 entries; |= 2: slot limit exceeded.
__global__ void tiled_table_kernel(const int32_t *__restrict__ tiles, int64_t nt, int k, int64_t S, int ts, int pad,
                                   int tpi, int ns, const int32_t *__restrict__ so, const int32_t *__restrict__ to,
                                   uint16_t *__restrict__ table, uint32_t *__restrict__ reg_sz,
                                   uint32_t *__restrict__ slot_sz, uint32_t *__restrict__ item_sz,
                                   int32_t *__restrict__ tgt_base, int *err) {
    const int64_t W = int64_t(1) << k, WW = W * W, R = W + 2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nt; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = tiles[i];
        const int64_t X0 = (int64_t)compact((uint32_t)t) * W - 1, Y0 = (int64_t)compact((uint32_t)t >> 1) * W - 1;
        uint16_t *tab = table + i * ts;
        int64_t run = 0;
        for (int64_t j = 0; j < R * R; ++j) {
            tab[j] = (uint16_t)run;
            const int64_t x = X0 + j % R, y = Y0 + j / R;
            if (x < 0 || y < 0 || x >= S || y >= S) continue;
            const uint32_t m = menc((uint32_t)x, (uint32_t)y);
            const int64_t cnt = so[m + 1] - so[m];
            run += pad ? p2(cnt) : cnt;
        }
        if (run > 65535) atomicOr(err, 1);
        tab[R * R] = (uint16_t)run;
        reg_sz[i] = (uint32_t)p4(run);
        const int64_t m0 = t * WW;
        int64_t n = 0;
        for (int64_t bl = 0; bl < WW; ++bl) {
            const int64_t c = to[m0 + bl + 1] - to[m0 + bl];
            n += tpi == 2 ? c + (c & 1) : c;
        }
        if (n > (ns == 3 ? 16383 * tpi : 65534)) atomicOr(err, 2);
        tab[R * R + 1] = (uint16_t)n;
        slot_sz[i] = (uint32_t)p8(n);
        item_sz[i] = ns == 3 ? (uint32_t)p8(3 * (n / tpi)) : 0u;  // NS = 3: (unit, row-run) items
        tgt_base[i] = to[m0];
    }
}

// TILED, one CTA per tile: the packed region -- per region box (row-major) its sources in plan
// order, coordinates relative to the region origin ((tx W - 1) h, (ty W - 1) h) computed in fp64
// and rounded once; per entry the local and the user source index.  Pads keep the fill values.
template <typename T>
__global__ void tiled_region_kernel(const int32_t *__restrict__ tiles, int64_t nt, int k, int64_t S, double h,
                                    int ts, int pad, const int32_t *__restrict__ so,
                                    const int32_t *__restrict__ perm, const double2 *__restrict__ sxy,
                                    const uint16_t *__restrict__ table, const uint32_t *__restrict__ reg_off,
                                    int32_t *__restrict__ reg_idx, int32_t *__restrict__ reg_uidx, T *__restrict__ uv) {
    const int64_t W = int64_t(1) << k, R = W + 2;
    for (int64_t i = blockIdx.x; i < nt; i += gridDim.x) {
        const int64_t t = tiles[i];
        const int64_t X0 = (int64_t)compact((uint32_t)t) * W - 1, Y0 = (int64_t)compact((uint32_t)t >> 1) * W - 1;
        const double ox = X0 * h, oy = Y0 * h;
        for (int64_t j = threadIdx.x; j < R * R; j += blockDim.x) {
            const int64_t x = X0 + j % R, y = Y0 + j / R;
            if (x < 0 || y < 0 || x >= S || y >= S) continue;
            const uint32_t m = menc((uint32_t)x, (uint32_t)y);
            int64_t ent = (int64_t)reg_off[i] + table[i * ts + j];
            for (int32_t sj = so[m]; sj < so[m + 1]; ++sj, ++ent) {
                const int64_t u = perm[sj];
                const double2 p = sxy[u];
                const double rx = p.x - ox, ry = p.y - oy;
                reg_idx[ent] = sj;
                reg_uidx[ent] = (int32_t)u;
                if (sizeof(T) == 4 && pad) {  // (u0,u1,v0,v1) per source pair
                    const int64_t pp = ent >> 1, sl = ent & 1;
                    uv[4 * pp + sl] = (T)rx;
                    uv[4 * pp + 2 + sl] = (T)ry;
                } else {
                    uv[2 * ent] = (T)rx;
                    uv[2 * ent + 1] = (T)ry;
                }
            }
        }
    }
}

// TILED, one CTA per tile: target slots.  The tile's target boxes in Morton order, or (tsort) by
// descending n9 (stable), each box's targets in plan order; tpi = 2: an odd box ends with a
// duplicate of its last target (output index 0xFFFF).  Per slot: coordinates relative to the
// region origin, row-run base j0 = by R + bx, tile-local output index.
// Dynamic smem: 3 int32 per box of the tile (WW <= 4096).
template <typename T>
__global__ void tiled_slots_kernel(const int32_t *__restrict__ tiles, int64_t nt, int k, double h, int tpi, int tsort,
                                   const int32_t *__restrict__ to, const int32_t *__restrict__ n9,
                                   const int32_t *__restrict__ tperm, const double2 *__restrict__ txy,
                                   const uint32_t *__restrict__ pack_off, uint16_t *__restrict__ bl_out,
                                   uint16_t *__restrict__ oix_out, T *__restrict__ ruv) {
    extern __shared__ int32_t sm[];
    const int WW = 1 << (2 * k), W = 1 << k, R = W + 2;
    int32_t *box = sm, *key = sm + WW, *start = sm + 2 * WW;  // nonempty boxes (Morton order), n9, slot start
    __shared__ int nbox;
    for (int64_t i = blockIdx.x; i < nt; i += gridDim.x) {
        const int64_t t = tiles[i], m0 = t * WW;
        const int32_t g0 = to[m0];
        if (threadIdx.x == 0) {
            int m = 0;
            for (int bl = 0; bl < WW; ++bl)
                if (to[m0 + bl + 1] > to[m0 + bl]) {
                    box[m] = bl;
                    key[m] = n9[m0 + bl];
                    ++m;
                }
            nbox = m;
        }
        __syncthreads();
        const int m = nbox;
        // rank of each box in the (stable) order: by descending n9 when tsort, else Morton
        for (int a = threadIdx.x; a < m; a += blockDim.x) {
            int r = a;
            if (tsort) {
                r = 0;
                const int ka = key[a];
                for (int b = 0; b < m; ++b) r += key[b] > ka || (key[b] == ka && b < a);
            }
            start[a] = r;  // rank for now
        }
        __syncthreads();
        if (threadIdx.x == 0) {  // slot start of each box = sum of the slots of the boxes ranked before it
            // invert the ranks through key[] (free now), then scan in rank order
            for (int a = 0; a < m; ++a) key[start[a]] = a;
            int s = 0;
            for (int r = 0; r < m; ++r) {
                const int a = key[r];
                const int64_t b = m0 + box[a];
                const int c = to[b + 1] - to[b];
                start[a] = s;
                s += tpi == 2 ? c + (c & 1) : c;
            }
        }
        __syncthreads();
        const int64_t tx = compact((uint32_t)t), ty = compact((uint32_t)t >> 1);
        const double ox = (tx * W - 1) * h, oy = (ty * W - 1) * h;
        for (int a = threadIdx.x; a < m; a += blockDim.x) {
            const int bl = box[a];
            const int64_t b = m0 + bl;
            const int c = to[b + 1] - to[b], nsl = tpi == 2 ? c + (c & 1) : c;
            const uint32_t bx = compact((uint32_t)bl), by = compact((uint32_t)bl >> 1);
            int64_t j = (int64_t)pack_off[i] + start[a];
            for (int x = 0; x < nsl; ++x, ++j) {
                const int64_t g = min((int64_t)to[b] + x, (int64_t)to[b + 1] - 1);
                const double2 p = txy[tperm[g]];
                bl_out[j] = (uint16_t)(by * R + bx);
                if (x < c) oix_out[j] = (uint16_t)(g - g0);
                ruv[2 * j] = (T)(p.x - ox);
                ruv[2 * j + 1] = (T)(p.y - oy);
            }
        }
        __syncthreads();
    }
}

// Queue order, step 1: launch entries of queue position li (tile order[li]): the tail split
// (li >= keep: `parts`) and the heavy-tile split (split_parts, plan.h), as the host builder.
__global__ void split_count_kernel(const int32_t *__restrict__ order, const int64_t *__restrict__ tile_pairs,
                                   int64_t nt, int64_t keep, int parts, int64_t share, uint32_t *__restrict__ cnt) {
    for (int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; li < nt; li += (int64_t)gridDim.x * blockDim.x) {
        const int32_t s = order ? order[li] : (int32_t)li;
        cnt[li] = share > 0 ? (uint32_t)split_parts(tile_pairs[s], share, li >= keep ? parts : 1) : 1u;
    }
}

// Step 2: launch entry off[li] + q -> tile, slot (Morton-order tile index), q | nparts << 16.
__global__ void queue_kernel(const int32_t *__restrict__ order, const int32_t *__restrict__ tiles_m, int64_t nt,
                             const uint32_t *__restrict__ cnt, const uint32_t *__restrict__ off,
                             int32_t *__restrict__ tiles_out, int32_t *__restrict__ slot_out,
                             int32_t *__restrict__ part_out, int32_t *__restrict__ nparts) {
    for (int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; li < nt; li += (int64_t)gridDim.x * blockDim.x) {
        const int32_t s = order ? order[li] : (int32_t)li;
        const int np = (int)cnt[li];
        for (int q = 0; q < np; ++q) {
            const int64_t e = (int64_t)off[li] + q;
            tiles_out[e] = tiles_m[s];
            slot_out[e] = s;
            part_out[e] = (int32_t)(q | (np << 16));
        }
        if (nparts) nparts[s] = np;
    }
}

// NS = 3 item lists, one CTA per tile: per part's unit range [nu ip / np, nu (ip+1) / np), the
// (unit, row-run) items sorted by row-run length (descending, stable), then 32-item batches
// dealt to warps longest-processing-time first (the host builder's balance_batches, same
// arithmetic).  Dynamic smem: 3 int32 per item of the largest tile.
__global__ void tiled_items_kernel(int64_t nt, int k, int ts, int tpi, int nthreads_kernel,
                                   const uint16_t *__restrict__ table, const uint32_t *__restrict__ pack_off,
                                   const uint16_t *__restrict__ tgt_bl, const int32_t *__restrict__ nparts_of,
                                   const uint32_t *__restrict__ item_off, uint16_t *__restrict__ items) {
    extern __shared__ int32_t sm[];
    const int R = (1 << k) + 2;
    for (int64_t i = blockIdx.x; i < nt; i += gridDim.x) {
        const uint16_t *tab = table + i * ts;
        const int nu = tab[R * R + 1] / tpi, np_ = nparts_of[i];
        const int64_t tb = pack_off[i];
        const int nitem = 3 * nu;
        int32_t *len = sm, *ord = sm + nitem, *lay = sm + 2 * nitem;
        for (int x = threadIdx.x; x < nitem; x += blockDim.x) {
            const int u = x / 3, row = x % 3;
            const int j0 = tgt_bl[tb + (int64_t)tpi * u] + row * R;
            len[x] = tab[j0 + 3] - tab[j0];
        }
        __syncthreads();
        for (int ip = 0; ip < np_; ++ip) {
            const int ub = (int)((int64_t)nu * ip / np_), ue = (int)((int64_t)nu * (ip + 1) / np_);
            const int lo = 3 * ub, n = 3 * (ue - ub);
            for (int a = threadIdx.x; a < n; a += blockDim.x) {  // stable rank by descending length
                const int la = len[lo + a];
                int r = 0;
                for (int b = 0; b < n; ++b) {
                    const int lb = len[lo + b];
                    r += lb > la || (lb == la && b < a);
                }
                ord[lo + r] = lo + a;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                const int32_t *o = ord + lo;
                int32_t *ly = lay + lo;
                const int nw = nthreads_kernel / 32;
                for (int x = 0; x < n; ++x) ly[x] = o[x];
                if (n > 32 && nw > 1) {
                    const int nb = (n + 31) / 32;
                    const bool partial = n % 32 != 0;
                    long long load[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                    int free_full[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                    for (int sl = 0; sl < nb; ++sl) {
                        const int w = (sl * 32 % nthreads_kernel) / 32;
                        free_full[w] += !(partial && sl == nb - 1);
                    }
                    // slots of warp w, in ascending order: sl = w + nw * c (sl * 32 % nt / 32 = sl % nw)
                    int next[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                    if (partial) {  // the partial batch (the shortest items) fills the partial slot
                        const int w = ((nb - 1) * 32 % nthreads_kernel) / 32;
                        load[w] += len[o[(nb - 1) * 32]];
                        for (int x = 0; x < 32 && 32 * (nb - 1) + x < n; ++x) ly[32 * (nb - 1) + x] = o[32 * (nb - 1) + x];
                    }
                    for (int b = 0; b < nb - (partial ? 1 : 0); ++b) {
                        int best = -1;
                        for (int w = 0; w < nw; ++w)
                            if (free_full[w] > 0 && (best < 0 || load[w] < load[best])) best = w;
                        load[best] += len[o[32 * b]];
                        --free_full[best];
                        // the next slot of warp `best` (skipping the partial slot)
                        int sl;
                        for (;;) {
                            sl = best + nw * next[best];
                            if (!(partial && sl == nb - 1)) break;
                            ++next[best];
                        }
                        ++next[best];
                        for (int x = 0; x < 32; ++x) ly[32 * sl + x] = o[32 * b + x];
                    }
                }
            }
            __syncthreads();
        }
        const int64_t io = item_off[i];
        for (int x = threadIdx.x; x < nitem; x += blockDim.x)
            items[io + x] = (uint16_t)((lay[x] / 3) << 2 | (lay[x] % 3));
        __syncthreads();
    }
}

}  // namespace dbuild
}  // namespace p2p
