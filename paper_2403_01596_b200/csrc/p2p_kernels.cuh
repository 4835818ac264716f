// p2p_kernels.cuh -- sm_100a kernels of the near-field P2P operator.
//
//   phi_t = sum_{s : box(s) in E1(box(t)), r >= eps} q_s ln(1/r)
//
// One CTA per non-empty Morton-aligned tile of 2^k x 2^k leaf boxes.  The
// tile's targets are one contiguous Morton range; each thread owns one target
// (held in registers) and sweeps the sources of its 3x3 box neighbourhood
// from shared memory.  The neighbourhood is walked as three row-runs (boxes
// x-1..x+1 of rows y-1, y, y+1): in the NR kernel the tile's region (tile +
// one-box ring) is staged in row-major box order, so each row-run is one
// contiguous shared-memory span; in the R kernel the halo of each target box
// is one contiguous span already (packed at plan time, §3.3).
//
// fp32 pair evaluation: coordinates are relative to the CTA
// region (NR) or the target box (R) in global units, so
//     ln(1/r) = -1/2 ln2 * lg2(r^2)
// with one MUFU.LG2 per pair and packed f32x2 FADD2/FMUL2/FFMA2 for two
// sources per step.  The eps guard is taken off the hot loop: an r^2 that
// underflows to 0 gives lg2 = -inf, which makes the target's sum non-finite,
// and only those (rare) targets are recomputed with the explicit guard.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace p2p {
namespace dev {

constexpr int kThreads = 256;
constexpr float kLn2 = 0.69314718055994530942f;

// ---------------------------------------------------------------- Morton
__device__ __forceinline__ uint32_t spread16(uint32_t v) {
    v &= 0x0000FFFFu;
    v = (v | (v << 8)) & 0x00FF00FFu;
    v = (v | (v << 4)) & 0x0F0F0F0Fu;
    v = (v | (v << 2)) & 0x33333333u;
    v = (v | (v << 1)) & 0x55555555u;
    return v;
}
__device__ __forceinline__ uint32_t compact16(uint32_t v) {
    v &= 0x55555555u;
    v = (v | (v >> 1)) & 0x33333333u;
    v = (v | (v >> 2)) & 0x0F0F0F0Fu;
    v = (v | (v >> 4)) & 0x00FF00FFu;
    v = (v | (v >> 8)) & 0x0000FFFFu;
    return v;
}

// ---------------------------------------------------------------- f32x2 (sm_100a)
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t f2_pack(float a, float b) {
    f2_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void f2_unpack(f2_t r, float &a, float &b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ f2_t f2_sub(f2_t a, f2_t b) {
    f2_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2_t f2_mul(f2_t a, f2_t b) {
    f2_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2_t f2_fma(f2_t a, f2_t b, f2_t c) {
    f2_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ float lg2_approx(float x) {
    float r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// ---------------------------------------------------------------- block scan
// In-place exclusive scan of a[0..n) (n <= ~64 per thread), returns the total.
__device__ __forceinline__ int block_exclusive_scan(int *a, int n, int *warp_tot) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int per = (n + kThreads - 1) / kThreads;
    const int lo = min(n, tid * per), hi = min(n, lo + per);
    int s = 0;
    for (int i = lo; i < hi; ++i) s += a[i];
    int incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        int v = lane < kThreads / 32 ? warp_tot[lane] : 0;
        int w = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int x = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += x;
        }
        if (lane < kThreads / 32) warp_tot[lane] = w - v;  // exclusive warp prefix
        if (lane == kThreads / 32 - 1) warp_tot[32] = w;   // grand total
    }
    __syncthreads();
    int run = warp_tot[wid] + incl - s;
    for (int i = lo; i < hi; ++i) {
        int v = a[i];
        a[i] = run;
        run += v;
    }
    int total = warp_tot[32];
    __syncthreads();
    return total;
}

// Last index j in [0, n) with a[j] <= x (a non-decreasing, a[0] <= x < a[n]).
__device__ __forceinline__ int seg_search(const int *a, int n, int x) {
    int lo = 0, hi = n;
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (a[mid] <= x) lo = mid;
        else hi = mid;
    }
    return lo;
}

// ---------------------------------------------------------------- pair loops
// fp32: sources stored per pair as float4 (u0,u1,v0,v1) + float2 (q0,q1);
// the span [p0, p1) counts source pairs.  Returns sum q * lg2(r^2).
__device__ __forceinline__ float span_f32(const float4 *__restrict__ A, const float2 *__restrict__ Q,
                                          int p0, int p1, float ut, float vt) {
    const f2_t U = f2_pack(ut, ut), V = f2_pack(vt, vt);
    f2_t acc = 0ull;
#pragma unroll 4
    for (int p = p0; p < p1; ++p) {
        const float4 s = A[p];
        const float2 q = Q[p];
        const f2_t du = f2_sub(U, f2_pack(s.x, s.y));
        const f2_t dv = f2_sub(V, f2_pack(s.z, s.w));
        const f2_t r2 = f2_fma(dv, dv, f2_mul(du, du));
        float r0, r1;
        f2_unpack(r2, r0, r1);
        acc = f2_fma(f2_pack(q.x, q.y), f2_pack(lg2_approx(r0), lg2_approx(r1)), acc);
    }
    float a0, a1;
    f2_unpack(acc, a0, a1);
    return a0 + a1;
}

// Explicitly guarded fp32 sweep (slow path for targets whose fast sum is not finite).
__device__ __noinline__ float span_f32_guarded(const float4 *__restrict__ A, const float2 *__restrict__ Q,
                                               int p0, int p1, float ut, float vt, float eps2) {
    const float *Af = reinterpret_cast<const float *>(A);
    const float *Qf = reinterpret_cast<const float *>(Q);
    float acc = 0.f;
    for (int j = 2 * p0; j < 2 * p1; ++j) {
        const int p = j >> 1, s = j & 1;
        const float du = ut - Af[4 * p + s], dv = vt - Af[4 * p + 2 + s];
        const float r2 = fmaf(dv, dv, du * du);
        if (r2 >= eps2) acc = fmaf(Qf[j], lg2_approx(r2), acc);
    }
    return acc;
}

// fp64: SoA u, v, q; returns sum q * log(r^2) over non-guarded pairs.
__device__ __forceinline__ double span_f64(const double *__restrict__ su, const double *__restrict__ sv,
                                           const double *__restrict__ sq, int j0, int j1, double ut,
                                           double vt, double eps2) {
    double acc = 0.0;
#pragma unroll 2
    for (int j = j0; j < j1; ++j) {
        const double du = ut - su[j], dv = vt - sv[j];
        const double r2 = fma(dv, dv, du * du);
        if (r2 >= eps2) acc = fma(sq[j], log(r2), acc);
    }
    return acc;
}

template <typename T> struct V2;
template <> struct V2<float> { using type = float2; };
template <> struct V2<double> { using type = double2; };

// ---------------------------------------------------------------- NR kernel
// Shared memory: int sstart[RR+1], gstart[RR], cnt[RR], toff[WW+1], then the
// staged region sources (fp32: float4 A[npair], float2 Q[npair];
// fp64: double u[n], v[n], q[n]).  npair_max / n_max from the plan.
template <typename T>
__global__ void __launch_bounds__(kThreads)
p2p_nr_kernel(const int32_t *__restrict__ tiles, int k, int64_t S, T h, T eps2, int max_region,
              const int32_t *__restrict__ src_off, const int32_t *__restrict__ tgt_off,
              const typename V2<T>::type *__restrict__ src_uv, const T *__restrict__ q,
              const typename V2<T>::type *__restrict__ tgt_uv, T *__restrict__ out, int accumulate) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ int warp_tot[33];
    const int W = 1 << k, R = W + 2, RR = R * R, WW = W * W;
    int *sstart = reinterpret_cast<int *>(smem);
    int *gstart = sstart + RR + 1;
    int *cnt = gstart + RR;
    int *toff = cnt + RR;
    const int tbytes = ((4 * (3 * RR + WW + 2)) + 15) & ~15;
    unsigned char *data = smem + tbytes;

    const uint32_t tile = (uint32_t)tiles[blockIdx.x];
    const uint32_t m0 = tile << (2 * k);
    const int64_t X0 = (int64_t)compact16(tile) * W - 1, Y0 = (int64_t)compact16(tile >> 1) * W - 1;
    const int tid = threadIdx.x;

    // 1. region box table (row-major over the (W+2)^2 region) + tile target offsets
    for (int j = tid; j < RR; j += kThreads) {
        const int lx = j % R, ly = j / R;
        const int64_t gx = X0 + lx, gy = Y0 + ly;
        int a = 0, c = 0;
        if (gx >= 0 && gy >= 0 && gx < S && gy < S) {
            const uint32_t m = spread16((uint32_t)gx) | (spread16((uint32_t)gy) << 1);
            a = src_off[m];
            c = src_off[m + 1] - a;
        }
        gstart[j] = a;
        cnt[j] = c;
        sstart[j] = (c + 1) & ~1;  // each box padded to an even count
    }
    for (int i = tid; i <= WW; i += kThreads) toff[i] = tgt_off[m0 + i];
    __syncthreads();
    const int total = block_exclusive_scan(sstart, RR, warp_tot);
    if (tid == 0) sstart[RR] = total;
    __syncthreads();

    // 2. stage the region's sources, rebased to the region origin (global units)
    if constexpr (sizeof(T) == 4) {
        float *Af = reinterpret_cast<float *>(data);
        float *Qf = Af + 2 * max_region;
        for (int i = tid; i < total; i += kThreads) {
            const int j = seg_search(sstart, RR, i);
            const int e = i - sstart[j];
            float u = 1.0e4f, v = 1.0e4f, qq = 0.f;  // pad: far away, zero weight
            if (e < cnt[j]) {
                const int s = gstart[j] + e;
                const float2 uv = src_uv[s];
                u = uv.x + (float)(j % R) * h;
                v = uv.y + (float)(j / R) * h;
                qq = q[s];
            }
            const int p = i >> 1, sl = i & 1;
            Af[4 * p + sl] = u;
            Af[4 * p + 2 + sl] = v;
            Qf[i] = qq;
        }
    } else {
        double *su = reinterpret_cast<double *>(data);
        double *sv = su + max_region;
        double *sq = sv + max_region;
        for (int i = tid; i < total; i += kThreads) {
            const int j = seg_search(sstart, RR, i);
            const int e = i - sstart[j];
            double u = 1.0e4, v = 1.0e4, qq = 0.0;
            if (e < cnt[j]) {
                const int s = gstart[j] + e;
                const double2 uv = src_uv[s];
                u = uv.x + (double)(j % R) * h;
                v = uv.y + (double)(j / R) * h;
                qq = q[s];
            }
            su[i] = u;
            sv[i] = v;
            sq[i] = qq;
        }
    }
    __syncthreads();

    // 3. one target per thread: three row-runs of its 3x3 neighbourhood
    const int tb = toff[0], nt = toff[WW] - tb;
    for (int it = tid; it < nt; it += kThreads) {
        const int gi = tb + it;
        const int bl = seg_search(toff, WW, gi);
        const int bx = (int)compact16((uint32_t)bl), by = (int)compact16((uint32_t)bl >> 1);
        const typename V2<T>::type uv = tgt_uv[gi];
        const T ut = uv.x + (T)(bx + 1) * h, vt = uv.y + (T)(by + 1) * h;
        T phi;
        if constexpr (sizeof(T) == 4) {
            const float4 *A = reinterpret_cast<const float4 *>(data);
            const float2 *Q = reinterpret_cast<const float2 *>(reinterpret_cast<const float *>(data) + 2 * max_region);
            float acc = 0.f;
#pragma unroll 1
            for (int row = 0; row < 3; ++row) {
                const int j0 = (by + row) * R + bx;
                acc += span_f32(A, Q, sstart[j0] >> 1, sstart[j0 + 3] >> 1, ut, vt);
            }
            if (!isfinite(acc)) {  // a guarded pair (r < eps) is present: explicit guard
                acc = 0.f;
                for (int row = 0; row < 3; ++row) {
                    const int j0 = (by + row) * R + bx;
                    acc += span_f32_guarded(A, Q, sstart[j0] >> 1, sstart[j0 + 3] >> 1, ut, vt, eps2);
                }
            }
            phi = (-0.5f * kLn2) * acc;
        } else {
            const double *su = reinterpret_cast<const double *>(data);
            const double *sv = su + max_region;
            const double *sq = sv + max_region;
            double acc = 0.0;
#pragma unroll 1
            for (int row = 0; row < 3; ++row) {
                const int j0 = (by + row) * R + bx;
                acc += span_f64(su, sv, sq, sstart[j0], sstart[j0 + 3], ut, vt, eps2);
            }
            phi = -0.5 * acc;
        }
        out[gi] = accumulate ? out[gi] + phi : phi;
    }
}

// ---------------------------------------------------------------- R kernel
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
p2p_r_kernel(const int32_t *__restrict__ tiles, int k, T eps2, const int32_t *__restrict__ tgt_off,
             const uint32_t *__restrict__ halo_off, const T *__restrict__ halo_uv,
             const T *__restrict__ halo_q, const typename V2<T>::type *__restrict__ tgt_uv,
             T *__restrict__ out, int accumulate) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int W = 1 << k, WW = W * W;
    int *toff = reinterpret_cast<int *>(smem);
    int *hoff = toff + WW + 1;
    const int tbytes = (8 * (WW + 1) + 16 + 31) & ~31;
    uint64_t *mbar = reinterpret_cast<uint64_t *>(smem + tbytes - 16);
    unsigned char *data = smem + tbytes;

    const uint32_t tile = (uint32_t)tiles[blockIdx.x];
    const uint32_t m0 = tile << (2 * k);
    const uint32_t hb = halo_off[m0], he = halo_off[m0 + WW];
    const uint32_t nent = he - hb;  // multiple of 4 (plan pads each tile)
    const int tid = threadIdx.x;

    // TMA bulk copy of the tile's packed halo (one contiguous span per array).
    const uint32_t bar = smem_addr(mbar);
    T *s_uv = reinterpret_cast<T *>(data);
    T *s_q = s_uv + 2 * (size_t)nent;
    if (tid == 0 && nent > 0) {
        const uint32_t b_uv = nent * 2 * sizeof(T), b_q = nent * sizeof(T);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(b_uv + b_q) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_addr(s_uv)),
            "l"(halo_uv + 2 * (size_t)hb), "r"(b_uv), "r"(bar)
            : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_addr(s_q)),
            "l"(halo_q + hb), "r"(b_q), "r"(bar)
            : "memory");
    }
    for (int i = tid; i <= WW; i += kThreads) {
        toff[i] = tgt_off[m0 + i];
        hoff[i] = (int)(halo_off[m0 + i] - hb);
    }
    __syncthreads();
    if (nent > 0) {
        asm volatile(
            "{\n\t.reg .pred P;\n"
            "WAIT_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t"
            "@!P bra WAIT_%=;\n}" ::"r"(bar)
            : "memory");
    }

    const int tb = toff[0], nt = toff[WW] - tb;
    for (int it = tid; it < nt; it += kThreads) {
        const int gi = tb + it;
        const int bl = seg_search(toff, WW, gi);
        const int j0 = hoff[bl], j1 = hoff[bl + 1];
        const typename V2<T>::type uv = tgt_uv[gi];
        T phi;
        if constexpr (sizeof(T) == 4) {
            const float4 *A = reinterpret_cast<const float4 *>(s_uv);
            const float2 *Q = reinterpret_cast<const float2 *>(s_q);
            float acc = span_f32(A, Q, j0 >> 1, j1 >> 1, uv.x, uv.y);
            if (!isfinite(acc)) acc = span_f32_guarded(A, Q, j0 >> 1, j1 >> 1, uv.x, uv.y, eps2);
            phi = (-0.5f * kLn2) * acc;
        } else {
            const double *su = s_uv;
            double acc = 0.0;
            for (int j = j0; j < j1; ++j) {
                const double du = uv.x - su[2 * j], dv = uv.y - su[2 * j + 1];
                const double r2 = fma(dv, dv, du * du);
                if (r2 >= eps2) acc = fma(s_q[j], log(r2), acc);
            }
            phi = -0.5 * acc;
        }
        out[gi] = accumulate ? out[gi] + phi : phi;
    }
}

// ---------------------------------------------------------------- data movement
// R pack: q_halo[e] = q_local[halo_idx[e]] (0 for pads).
template <typename T>
__global__ void pack_r_kernel(const int32_t *__restrict__ idx, const T *__restrict__ q, T *__restrict__ qh,
                              int64_t n) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = idx[e];
        qh[e] = i >= 0 ? q[i] : T(0);
    }
}

// dst[i] = src[idx[i]]  (ORDER_USER import / replicated-weight gather)
template <typename T>
__global__ void gather_kernel(const int32_t *__restrict__ idx, const T *__restrict__ src, T *__restrict__ dst,
                              int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[idx[i]];
}

// dst[i] = i2 < n_owned ? owned[i2] : halo[i2 - n_owned], i2 = qidx[i]  (distributed import)
template <typename T>
__global__ void gather2_kernel(const int32_t *__restrict__ qidx, const T *__restrict__ owned,
                               const T *__restrict__ halo, int64_t n_owned, T *__restrict__ dst, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = qidx[i];
        dst[i] = j < n_owned ? owned[j] : halo[j - n_owned];
    }
}

// out[idx[i]] (+)= phi[i]  (ORDER_USER export)
template <typename T>
__global__ void scatter_kernel(const int32_t *__restrict__ idx, const T *__restrict__ phi, T *__restrict__ out,
                               int64_t n, int accumulate) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t o = idx[i];
        out[o] = accumulate ? out[o] + phi[i] : phi[i];
    }
}

}  // namespace dev
}  // namespace p2p
