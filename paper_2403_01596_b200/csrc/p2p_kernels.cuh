// p2p_kernels.cuh -- sm_100a kernels of the near-field P2P operator.
//
//   phi_t = sum_{s : box(s) in E1(box(t)), r >= eps} q_s ln(1/r)
//
// Work unit: a non-empty Morton-aligned tile of 2^k x 2^k leaf boxes (one
// contiguous Morton range of targets).  Persistent CTAs pull tiles from a
// queue.  The sources a tile needs are staged in shared memory; targets are
// held in registers and sweep contiguous shared-memory spans.  The 3x3
// neighbourhood is walked as three row-runs (boxes x-1..x+1 of rows y-1, y,
// y+1): the NR kernel stages the tile's region (tile + one-box ring) in
// row-major box order so each row-run is one contiguous span; the R kernel's
// halo of each target box is one contiguous span already (packed at plan
// time, §3.3).
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

#include "plan.h"

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

// Two targets sharing one span x two sources per step: 4 pairs per LDS.128 + LDS.64,
// ~3 non-MUFU issue slots per pair (FADD2 x4, FMUL2 x2, FFMA2 x4 per 4 pairs).
#ifndef P2P_SPAN2_UNROLL
#define P2P_SPAN2_UNROLL 4
#endif
#define P2P_PRAGMA(x) _Pragma(#x)
#define P2P_UNROLL(n) P2P_PRAGMA(unroll n)
__device__ __forceinline__ void span2_f32(const float4 *__restrict__ A, const float2 *__restrict__ Q, int p0,
                                          int p1, float ut0, float vt0, float ut1, float vt1, float &r0,
                                          float &r1) {
    const f2_t U0 = f2_pack(ut0, ut0), V0 = f2_pack(vt0, vt0);
    const f2_t U1 = f2_pack(ut1, ut1), V1 = f2_pack(vt1, vt1);
    f2_t a0 = 0ull, a1 = 0ull;
    P2P_UNROLL(P2P_SPAN2_UNROLL)
    for (int p = p0; p < p1; ++p) {
        const float4 s = A[p];
        const float2 q = Q[p];
        const f2_t su = f2_pack(s.x, s.y), sv = f2_pack(s.z, s.w), qq = f2_pack(q.x, q.y);
        const f2_t d0u = f2_sub(U0, su), d0v = f2_sub(V0, sv);
        const f2_t d1u = f2_sub(U1, su), d1v = f2_sub(V1, sv);
        const f2_t w0 = f2_fma(d0v, d0v, f2_mul(d0u, d0u));
        const f2_t w1 = f2_fma(d1v, d1v, f2_mul(d1u, d1u));
        float x0, x1, y0, y1;
        f2_unpack(w0, x0, x1);
        f2_unpack(w1, y0, y1);
        a0 = f2_fma(qq, f2_pack(lg2_approx(x0), lg2_approx(x1)), a0);
        a1 = f2_fma(qq, f2_pack(lg2_approx(y0), lg2_approx(y1)), a1);
    }
    float c0, c1;
    f2_unpack(a0, c0, c1);
    r0 = c0 + c1;
    f2_unpack(a1, c0, c1);
    r1 = c0 + c1;
}

// Unpadded fp32 layout (sparse tiles): (u, v) per entry + q per entry, one
// pair per step.  Returns sum q * lg2(r^2) (non-finite if some r^2 underflows).
__device__ __forceinline__ float span1_f32(const float2 *__restrict__ UV, const float *__restrict__ Q, int j0, int j1,
                                           float ut, float vt) {
    float acc = 0.f;
#pragma unroll 2
    for (int j = j0; j < j1; ++j) {
        const float2 s = UV[j];
        const float du = ut - s.x, dv = vt - s.y;
        acc = fmaf(Q[j], lg2_approx(fmaf(dv, dv, du * du)), acc);
    }
    return acc;
}
__device__ __noinline__ float span1_f32_guarded(const float2 *__restrict__ UV, const float *__restrict__ Q, int j0,
                                                int j1, float ut, float vt, float eps2) {
    float acc = 0.f;
    for (int j = j0; j < j1; ++j) {
        const float du = ut - UV[j].x, dv = vt - UV[j].y;
        const float r2 = fmaf(dv, dv, du * du);
        if (r2 >= eps2) acc = fmaf(Q[j], lg2_approx(r2), acc);
    }
    return acc;
}
// fp64 log, table-driven (libdevice's log is ~30 DP ops; this is 8): x = m 2^e, m in [1, 2);
// k = top 8 mantissa bits; LT[k] = (c_inv, -log c_inv) with c_inv ~ 1 / (1 + (k + 1/2)/256) (host,
// plan_builder.cpp); t = m c_inv - 1 (one fma, |t| < 2^-9); log1p(t) to degree 5 (truncation
// < 1e-17); log x = e ln2 + (-log c_inv + log1p(t)), e ln2 in one fma (|e| <= 80 for r^2 >= eps^2:
// the rounding of ln2 adds < 2e-15 to a result of that size).  x must be a positive normal double.
// (P2P_LOG256 = 0: round 1's 128-entry table, degree 6, ln2 split hi / lo: 11 DP ops.)
constexpr double kLn2d = 6.93147180559945309417e-01;
// the log polynomials' coefficients that are not short immediates, in the constant bank: DFMA
// reads them as c[][] operands (as immediates each costs a UMOV pair per use)
__constant__ double kLogK[6] = {1.0 / 7.0, -1.0 / 6.0, 0.2, 1.0 / 3.0, 6.93147180559945309417e-01, -0.125};
constexpr double kLn2Hi = 6.93147180369123816490e-01, kLn2Lo = 1.90821492927058770002e-10;
__device__ __forceinline__ double log_tab(double x, const double2 *__restrict__ LT) {
    const long long b = __double_as_longlong(x);
    const int e = (int)(b >> 52) - 1023;
    const double m = __longlong_as_double((b & 0x000FFFFFFFFFFFFFLL) | 0x3FF0000000000000LL);
#if P2P_LOG256
    const double2 c = LT[(int)(b >> 44) & 255];
    const double t = fma(m, c.x, -1.0);
    double q = fma(t, kLogK[2], -0.25);
    q = fma(t, q, kLogK[3]);
    q = fma(t, q, -0.5);
    const double p = fma(t * t, q, t);
    return fma((double)e, kLogK[4], c.y + p);
#else
    const double2 c = LT[(int)(b >> 45) & 127];
    const double t = fma(m, c.x, -1.0);
    double q = fma(t, -1.0 / 6.0, 0.2);
    q = fma(t, q, -0.25);
    q = fma(t, q, 1.0 / 3.0);
    q = fma(t, q, -0.5);
    const double p = fma(t * t, q, t);
    const double de = (double)e;
    return fma(de, kLn2Hi, c.y) + fma(de, kLn2Lo, p);
#endif
}

// fp64 log for the dense TILED path: a 64-entry table replicated 8 times in shared memory, entry k
// of copy c at 16-byte slot 8 k + c, and lane l reads copy l & 7 -- the 8 lanes of each quarter-
// warp phase of an LDS.128 always hit 8 distinct bank groups (no conflicts; the 256-entry table's
// random lookups cost 2.5x the ideal wavefronts).  k = top 6 mantissa bits, |t| < 2^-7, log1p
// to degree 7 (truncation < 1e-17): 10 DP operations.
__device__ __forceinline__ double log_tab8(double x, const double2 *__restrict__ LT8, int l8) {
    const long long b = __double_as_longlong(x);
    const int e = (int)(b >> 52) - 1023;
    const double2 c = LT8[(((int)(b >> 46) & 63) << 3) + l8];
    const double m = __longlong_as_double((b & 0x000FFFFFFFFFFFFFLL) | 0x3FF0000000000000LL);
    const double t = fma(m, c.x, -1.0);
    double q = fma(t, kLogK[0], kLogK[1]);
    q = fma(t, q, kLogK[2]);
    q = fma(t, q, -0.25);
    q = fma(t, q, kLogK[3]);
    q = fma(t, q, -0.5);
    const double p = fma(t * t, q, t);
    return fma((double)e, kLogK[4], c.y + p);
}
__device__ __forceinline__ double span1_f64r(const double2 *__restrict__ UV, const double *__restrict__ Q, int j0,
                                             int j1, double ut, double vt, double eps2,
                                             const double2 *__restrict__ LT8, int l8) {
    double acc = 0.0;
#pragma unroll 4
    for (int j = j0; j < j1; ++j) {  // guard by selection, no branch (a guarded pair's log is of 1.0)
        const double2 s = UV[j];
        const double du = ut - s.x, dv = vt - s.y;
        const double r2 = fma(dv, dv, du * du);
        const bool ok = r2 >= eps2;
        const double lg = log_tab8(ok ? r2 : 1.0, LT8, l8);
        const double qj = Q[j];
        acc = ok ? fma(qj, lg, acc) : acc;
    }
    return acc;
}

// Dense fp64, two targets (a, b) of one box per source load, the log from the replicated 64-entry
// table (lt8) or the 256-entry one.  The eps guard is off the loop: each target keeps the minimum
// high word of its r^2 (one integer min per pair; high words of non-negative doubles order like
// the values), and a target whose minimum does not exceed the high word of eps^2 -- a superset of
// the targets with a pair closer than eps -- returns NaN, so finish() recomputes it with the
// explicit guard (same logs, same order: the results equal the guarded loop's).
__device__ __forceinline__ void span1x2_f64(const double2 *__restrict__ UV, const double *__restrict__ Q, int j0,
                                            int j1, double ua, double va, double ub, double vb, double eps2,
                                            const double2 *__restrict__ LT, int l8, int lt8, double &ra,
                                            double &rb) {
    double a0 = 0.0, a1 = 0.0;
    int ma = 0x7fffffff, mb = 0x7fffffff;
#pragma unroll 2
    for (int j = j0; j < j1; ++j) {
        const double2 s = UV[j];
        const double qj = Q[j];
        const double dua = ua - s.x, dva = va - s.y, dub = ub - s.x, dvb = vb - s.y;
        const double r2a = fma(dva, dva, dua * dua), r2b = fma(dvb, dvb, dub * dub);
        ma = min(ma, __double2hiint(r2a));
        mb = min(mb, __double2hiint(r2b));
        const double la = lt8 ? log_tab8(r2a, LT, l8) : log_tab(r2a, LT);
        const double lb = lt8 ? log_tab8(r2b, LT, l8) : log_tab(r2b, LT);
        a0 = fma(qj, la, a0);
        a1 = fma(qj, lb, a1);
    }
    const int he = __double2hiint(eps2);
    ra = ma <= he ? __longlong_as_double(0x7ff8000000000000LL) : a0;
    rb = mb <= he ? __longlong_as_double(0x7ff8000000000000LL) : a1;
}

// fp64 log without the shared-memory table (the TILED lean fp64 path, sparse tiles): a 32-entry
// table held one entry per lane in registers (c_k rounded to float, L_k = -log c_k;
// plan_builder.cpp build_log_table) and fetched with warp shuffles.  The 256-entry table's random
// LDS.128 are 2.5x bank-conflicted (69 % of the dense fp64 kernel's shared wavefronts, ncu
// surf_2e7); without them the sparse fp64 path runs 13 % faster, while the dense path (long
// runs, 44 instructions per pair with the shuffles and masks) turns issue-bound and keeps
// log_tab (profiles/r02_ncu_fp64.txt).
// k = top 5 mantissa bits, t = m c_k - 1 (|t| < 2^-6 + 2^-23), log1p(t) to degree 8 (truncation
// < 1e-17), log x = fma(e, ln2, L_k + log1p(t)): 11 DP operations.  All 32 lanes of the warp must
// call it together (converged); x must be a positive normal double.
__device__ __forceinline__ double log_shfl(double x, float lc, double lL) {
    const long long b = __double_as_longlong(x);
    const int e = (int)(b >> 52) - 1023;
    const int kk = (int)(b >> 47) & 31;
    const double m = __longlong_as_double((b & 0x000FFFFFFFFFFFFFLL) | 0x3FF0000000000000LL);
    const float c = __shfl_sync(0xffffffffu, lc, kk);
    const double L = __shfl_sync(0xffffffffu, lL, kk);
    const double t = fma(m, (double)c, -1.0);
    double q = fma(t, kLogK[5], kLogK[0]);
    q = fma(t, q, kLogK[1]);
    q = fma(t, q, kLogK[2]);
    q = fma(t, q, -0.25);
    q = fma(t, q, kLogK[3]);
    q = fma(t, q, -0.5);
    const double p = fma(t * t, q, t);
    return fma((double)e, kLogK[4], L + p);
}

// fp64, one target's sources j(v), v < n, with the explicit guard, for log_shfl: every lane of the
// warp runs the warp's longest count (lanes past their own n -- or with no target: n = 0 --
// evaluate a masked pair), so the shuffles always see the whole warp.
template <typename J>
__device__ __forceinline__ double sweep_f64w(const double2 *__restrict__ UV, const double *__restrict__ Q, int n,
                                             J jof, double ut, double vt, double eps2, float lc, double lL) {
    const int nmax = __reduce_max_sync(0xffffffffu, n);
    double acc = 0.0;
#pragma unroll 2
    for (int v = 0; v < nmax; ++v) {
        const bool live = v < n;
        const int j = live ? jof(v) : 0;
        const double2 s = UV[j];
        const double du = ut - s.x, dv = vt - s.y;
        const double r2 = fma(dv, dv, du * du);
        const bool use = live && r2 >= eps2;
        const double lg = log_shfl(use ? r2 : 1.0, lc, lL);
        const double qj = Q[j];
        acc = use ? fma(qj, lg, acc) : acc;
    }
    return acc;
}

// fp64, (u, v) per entry, explicit guard.
__device__ __forceinline__ double span1_f64(const double2 *__restrict__ UV, const double *__restrict__ Q, int j0,
                                            int j1, double ut, double vt, double eps2,
                                            const double2 *__restrict__ LT) {
    double acc = 0.0;
    for (int j = j0; j < j1; ++j) {
        const double2 s = UV[j];
        const double du = ut - s.x, dv = vt - s.y;
        const double r2 = fma(dv, dv, du * du);
        if (r2 >= eps2) acc = fma(Q[j], log_tab(r2, LT), acc);
    }
    return acc;
}

// The three row-runs [s_r, e_r) of a target as ONE index sequence v = s0 .. s0+n-1
// mapped to j = v + (v >= b1 ? d1 : 0) + (v >= b2 ? d2 : 0): lanes whose targets
// have equal totals (tsort plans) stay converged across row boundaries.  One
// accumulator, sources in row order (a fixed order per target).
#ifndef P2P_SPAN3_UNROLL
#define P2P_SPAN3_UNROLL 2  // the sparse flattened loop (tools/gpu/gpu_ab_variants.sh: 1, 2, 4)
#endif
struct Runs3 {
    int v0, n, b1, d1, b2, d2;
    __device__ __forceinline__ Runs3(int s0, int e0, int s1, int e1, int s2, int e2)
        : v0(s0), n((e0 - s0) + (e1 - s1) + (e2 - s2)), b1(e0), d1(s1 - e0), b2(e0 + (e1 - s1)), d2(s2 - e1) {}
    __device__ __forceinline__ int at(int v) const { return v + (v >= b1 ? d1 : 0) + (v >= b2 ? d2 : 0); }
};
__device__ __forceinline__ float span3_f32(const float2 *__restrict__ UV, const float *__restrict__ Q, const Runs3 &r,
                                           float ut, float vt) {
    float acc = 0.f;
    const int v1 = r.v0 + r.n;
    P2P_UNROLL(P2P_SPAN3_UNROLL)
    for (int v = r.v0; v < v1; ++v) {
        const int j = r.at(v);
        const float2 s = UV[j];
        const float du = ut - s.x, dv = vt - s.y;
        acc = fmaf(Q[j], lg2_approx(fmaf(dv, dv, du * du)), acc);
    }
    return acc;
}
__device__ __forceinline__ double span3_f64(const double2 *__restrict__ UV, const double *__restrict__ Q,
                                            const Runs3 &r, double ut, double vt, double eps2,
                                            const double2 *__restrict__ LT) {
    double acc = 0.0;
    const int v1 = r.v0 + r.n;
    for (int v = r.v0; v < v1; ++v) {
        const int j = r.at(v);
        const double2 s = UV[j];
        const double du = ut - s.x, dv = vt - s.y;
        const double r2 = fma(dv, dv, du * du);
        if (r2 >= eps2) acc = fma(Q[j], log_tab(r2, LT), acc);
    }
    return acc;
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
                                           double vt, double eps2, const double2 *__restrict__ LT) {
    double acc = 0.0;
#pragma unroll 2
    for (int j = j0; j < j1; ++j) {
        const double du = ut - su[j], dv = vt - sv[j];
        const double r2 = fma(dv, dv, du * du);
        if (r2 >= eps2) acc = fma(sq[j], log_tab(r2, LT), acc);
    }
    return acc;
}

template <typename T> struct V2;
template <> struct V2<float> { using type = float2; };
template <> struct V2<double> { using type = double2; };

// ---------------------------------------------------------------- launch arguments
template <typename T>
struct P2PArgs {
    const int32_t *tiles;  // Morton tile indices in queue order (LPT or Morton, chosen by the plan)
    int ntiles;
    int *queue;            // [0] dynamic tile counter, [1] exited CTAs; the last CTA out resets both
    int k;                 // tile side = 2^k leaf boxes
    int64_t S;             // grid side 2^(L-1)
    T h, eps2;
    int src_cap;           // NR: max padded region sources of a tile; R: max packed-halo entries of a tile
    int tgt_cap;           // max targets of a tile (multiple of 4)
    int group_log2;        // NR source staging: 2^group_log2 lanes per region box
    const int32_t *src_off, *tgt_off;  // [B+1] CSR offsets (local plan order)
    const typename V2<T>::type *src_uv, *tgt_uv;  // box-local coordinates
    const T *q;            // NR: q in local plan order; R: packed halo q (from pack_r)
    const uint32_t *halo_off;  // R: [B+1] packed-halo offsets
    const T *halo_uv;      // R: packed-halo coordinates relative to the target box origin
    const int32_t *tile_slot;   // TILED: launch order -> Morton slot of the per-tile arrays
    const int32_t *tile_part;   // TILED: launch order -> part | nparts << 16 (unit range of the tile)
    const uint32_t *reg_off;    // TILED: [slots+1] packed-region offsets
    const int32_t *reg_idx;     // TILED: local source index per packed entry (-1 = pad)
    const T *reg_uv;            // TILED: region-relative coordinates (fp32: (u0,u1,v0,v1) per pair)
    const uint16_t *reg_table;  // TILED: [slots][tstride] region box starts, then target box starts
    const uint16_t *tgt_bl;     // TILED: packed targets' row-run base j0 = by*R + bx in the region
    const uint16_t *tgt_oix;    // TILED: per target slot, tile-local output index (0xFFFF: duplicate slot)
    const uint32_t *item_off;   // TILED NS = 3: [slots+1] item-list offsets
    const uint16_t *items;      // TILED NS = 3: unit << 2 | row, length-sorted per part
    const double2 *log_tab;     // fp64: kLogTab x (c_inv, -log c_inv) for log_tab()
    const int32_t *out_idx;     // TILED: output position of each local target (ORDER_USER), or nullptr
    const T *tgt_ruv;           // TILED: packed targets' coordinates relative to the region origin
    const uint32_t *tgt_pack_off;   // TILED: [slots+1] packed-target offsets (multiples of 8)
    const int32_t *tile_tgt_base;   // TILED: plan index of each tile's first target
    int ns;                     // TILED: work items per target (1 = whole target, 3 = one per row-run)
    int flat;                   // TILED lean path: sweep the three row-runs as one sequence
    int lt8;                    // TILED dense fp64: log_tab8 (8-fold 64-entry table) instead of log_tab
    int nbuf;                   // TILED: 2 = prefetch the next tile's record during this tile
    unsigned long long *trace;  // optional per-tile timeline (diagnostics; nullptr = off)
    T *out;
    int accumulate;
    T kappa;                    // HELMHOLTZ_2D wavenumber
    // 3D box kernel (NEXT-3)
    const T *src_p4, *tgt_p4;   // box-local coordinates in units of h, 4 per point (x, y, z, 0), plan order
    const int32_t *src_idx;     // ORDER_USER: user index of each plan-order source (weights gathered through it)
    T scale;                    // 1 / (4 pi h)
    T kh;                       // kappa h (HELMHOLTZ_3D)
    // ADAPTIVE (NEXT-4)
    const int4 *leaf_rng;       // per leaf: source range, target range (plan order)
    const int2 *leaf_org;       // per leaf: origin in finest-grid cells
    const int32_t *ul_off, *ul_leaf;  // U-lists (CSR over leaves)
    const int2 *src_cell, *tgt_cell;  // per point: finest cell (plan order); src_uv / tgt_uv: offsets in the cell
};

__device__ __forceinline__ int warp_incl_scan(int v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += x;
    }
    return v;
}

// s_q[i] = q[s_idx[i]] (0 for pads) for i = first, first + stride, ... < n, with
// up to 8 independent L2 loads in flight per thread.
// q[j] if j >= 0, else 0: one predicated ld.global.nc (no branch, no load for j < 0)
__device__ __forceinline__ float ldg_pred(const float *q, int j) {
    float w;
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ge.s32 p, %2, 0;\n\tmov.b32 %0, 0;\n\t"
                 "@p ld.global.nc.f32 %0, [%1];\n\t}"
                 : "=f"(w) : "l"(q + (j < 0 ? 0 : j)), "r"(j));
    return w;
}
__device__ __forceinline__ double ldg_pred(const double *q, int j) {
    double w;
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ge.s32 p, %2, 0;\n\tmov.b64 %0, 0;\n\t"
                 "@p ld.global.nc.f64 %0, [%1];\n\t}"
                 : "=d"(w) : "l"(q + (j < 0 ? 0 : j)), "r"(j));
    return w;
}
template <typename T>
__device__ __forceinline__ void gather_weights(const int32_t *__restrict__ s_idx, const T *__restrict__ q,
                                               T *__restrict__ s_q, int n, int first, int stride) {
    for (int base = first; base < n; base += 8 * stride) {
        T v[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) {  // predicated loads, no branches: pads (-1) and i >= n give 0
            const int i = base + x * stride;
            const int32_t j = i < n ? s_idx[i] : -1;
            v[x] = ldg_pred(q, j);
        }
#pragma unroll
        for (int x = 0; x < 8; ++x) {
            const int i = base + x * stride;
            if (i < n) s_q[i] = v[x];
        }
    }
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

// Called once per CTA by one thread after its last tile: the last CTA to leave
// resets the queue for the next launch (no per-apply memset node).
__device__ __forceinline__ void queue_exit(int *queue) {
    __threadfence();
    if (atomicAdd(queue + 1, 1) == (int)gridDim.x - 1) {
        queue[0] = 0;
        queue[1] = 0;
        __threadfence();
    }
}

// Next tile from the dynamic queue (one atomic per CTA per tile).
__device__ __forceinline__ int next_tile(int *queue, int *s_tile) {
    if (threadIdx.x == 0) *s_tile = atomicAdd(queue, 1);
    __syncthreads();
    return *s_tile;
}

// ---------------------------------------------------------------- NR kernel
// Persistent CTAs pull Morton-aligned 2^k x 2^k tiles from a queue.  Per tile:
//  A1 all threads: region box table (source CSR segments of the (W+2)^2
//     region, row-major) and the tile's target offsets;
//  A2 warp 0: prefix of the even-padded box counts (warp shuffles) ->
//     shared-memory start of every region box; warp 1 (TPI = 2): prefix of
//     the per-box number of target pairs;
//  A3 targets of each tile box, rebased to the region origin, grouped into
//     work units of TPI targets of the same box (same row-runs);
//  B  2^g lanes per region box copy its sources into shared memory, rebased
//     to the region origin (global units), padded to an even count;
//  C  work items (unit, row): TPI targets sweep one contiguous row-run;
//  D  fixed-order sum of the 3 row partials of each target (deterministic).
template <typename T, int TPI>
__global__ void __launch_bounds__(kThreads)
p2p_nr_kernel(const P2PArgs<T> a) {
    static_assert(TPI == 1 || (TPI == 2 && sizeof(T) == 4), "TPI = 2 is the fp32 path");
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ int s_tile, s_units;
    const int k = a.k, W = 1 << k, R = W + 2, RR = R * R, WW = W * W;
    const NrCarve c = nr_carve(k, a.src_cap, a.tgt_cap, (int)sizeof(T), TPI);
    double2 *s_lt = reinterpret_cast<double2 *>(smem + c.ltab);
    if constexpr (sizeof(T) == 8)  // visible after next_tile()'s barrier
        for (int i = threadIdx.x; i < kLogTab; i += blockDim.x) s_lt[i] = a.log_tab[i];
    int *sstart = reinterpret_cast<int *>(smem + c.sstart);
    int *gstart = reinterpret_cast<int *>(smem + c.gstart);
    int *cnt = reinterpret_cast<int *>(smem + c.cnt);
    int *toff = reinterpret_cast<int *>(smem + c.toff);
    int *pstart = reinterpret_cast<int *>(smem + c.pstart);
    int *uj0 = reinterpret_cast<int *>(smem + c.uj0);
    int *ut = reinterpret_cast<int *>(smem + c.ut);
    int *tslot = reinterpret_cast<int *>(smem + c.tslot);
    T *tu = reinterpret_cast<T *>(smem + c.tu);
    T *tv = reinterpret_cast<T *>(smem + c.tv);
    T *part = reinterpret_cast<T *>(smem + c.part);
    unsigned char *src = smem + c.src;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const T h = a.h;

    for (int ti = next_tile(a.queue, &s_tile); ti < a.ntiles; ti = next_tile(a.queue, &s_tile)) {
        const uint32_t tile = (uint32_t)a.tiles[ti];
        const uint32_t m0 = tile << (2 * k);
        const int64_t X0 = (int64_t)compact16(tile) * W - 1, Y0 = (int64_t)compact16(tile >> 1) * W - 1;
        const int tb = a.tgt_off[m0];

        // A1: tables
        for (int j = tid; j < RR; j += kThreads) {
            const int lx = j % R, ly = j / R;
            const int64_t gx = X0 + lx, gy = Y0 + ly;
            int st = 0, cn = 0;
            if (gx >= 0 && gy >= 0 && gx < a.S && gy < a.S) {
                const uint32_t m = spread16((uint32_t)gx) | (spread16((uint32_t)gy) << 1);
                st = a.src_off[m];
                cn = a.src_off[m + 1] - st;
            }
            gstart[j] = st;
            cnt[j] = cn;
        }
        for (int i = tid; i <= WW; i += kThreads) toff[i] = a.tgt_off[m0 + i] - tb;
        __syncthreads();

        // A2: prefixes
        if (wid == 0) {
            int carry = 0;
            for (int base = 0; base < RR; base += 32) {
                const int j = base + lane;
                const int pc = j < RR ? ((cnt[j] + 1) & ~1) : 0;
                const int incl = warp_incl_scan(pc);
                if (j < RR) sstart[j] = carry + incl - pc;
                carry += __shfl_sync(0xffffffffu, incl, 31);
            }
            if (lane == 0) sstart[RR] = carry;
        } else if (wid == 1) {
            int carry = 0;
            for (int base = 0; base < WW; base += 32) {
                const int bl = base + lane;
                const int n = bl < WW ? toff[bl + 1] - toff[bl] : 0;
                const int np = TPI == 2 ? (n + 1) >> 1 : n;
                const int incl = warp_incl_scan(np);
                if (bl < WW) pstart[bl] = carry + incl - np;
                carry += __shfl_sync(0xffffffffu, incl, 31);
            }
            if (lane == 0) s_units = carry;
        }
        __syncthreads();

        // A3: targets -> units (flat over targets; box by binary search over the tile's offsets)
        const int nt = toff[WW];
        for (int t = tid; t < nt; t += kThreads) {
            int lo = 0, hi = WW;  // last box bl with toff[bl] <= t
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (toff[mid] <= t) lo = mid;
                else hi = mid;
            }
            const int bl = lo, t0 = toff[bl], t1 = toff[bl + 1];
            const int bx = (int)compact16((uint32_t)bl), by = (int)compact16((uint32_t)bl >> 1);
            const typename V2<T>::type uv = a.tgt_uv[tb + t];
            tu[t] = uv.x + (T)(bx + 1) * h;
            tv[t] = uv.y + (T)(by + 1) * h;
            const int r = t - t0, u = pstart[bl] + r / TPI, sl = r % TPI;
            ut[TPI * u + sl] = t;
            tslot[t] = TPI * u + sl;
            if (sl == 0) {
                uj0[u] = by * R + bx;
                if (TPI == 2 && t + 1 == t1) ut[TPI * u + 1] = t;  // odd box: duplicate, result unused
            }
        }

        // B: sources, 2^g lanes per region box
        {
            const int G = 1 << a.group_log2, gl = tid & (G - 1), ngrp = kThreads >> a.group_log2;
            for (int j = tid >> a.group_log2; j < RR; j += ngrp) {
                const int cn = cnt[j], s0 = sstart[j], g0 = gstart[j], pc = (cn + 1) & ~1;
                const T ox = (T)(j % R) * h, oy = (T)(j / R) * h;
                for (int e = gl; e < pc; e += G) {
                    T u = (T)1.0e4, v = (T)1.0e4, qq = (T)0;  // pad: far away, zero weight
                    if (e < cn) {
                        const typename V2<T>::type uv = a.src_uv[g0 + e];
                        u = uv.x + ox;
                        v = uv.y + oy;
                        qq = a.q[g0 + e];
                    }
                    const int i = s0 + e;
                    if constexpr (sizeof(T) == 4) {
                        float *Af = reinterpret_cast<float *>(src);
                        float *Qf = Af + 2 * a.src_cap;
                        const int p = i >> 1, sl = i & 1;
                        Af[4 * p + sl] = u;
                        Af[4 * p + 2 + sl] = v;
                        Qf[i] = qq;
                    } else {
                        double *su = reinterpret_cast<double *>(src);
                        su[i] = u;
                        su[a.src_cap + i] = v;
                        su[2 * a.src_cap + i] = qq;
                    }
                }
            }
        }
        __syncthreads();

        // C: (unit, row-run) work items
        const int nu = s_units;
        for (int it = tid; it < 3 * nu; it += kThreads) {
            const int row = (it >= nu) + (it >= 2 * nu);
            const int u = it - row * nu;
            const int j0 = uj0[u] + row * R;
            const int i0 = sstart[j0], i1 = sstart[j0 + 3];
            T *pp = part + row * TPI * nu + TPI * u;
            if constexpr (sizeof(T) == 4) {
                const float4 *A = reinterpret_cast<const float4 *>(src);
                const float2 *Q = reinterpret_cast<const float2 *>(reinterpret_cast<const float *>(src) + 2 * a.src_cap);
                if constexpr (TPI == 2) {
                    const int t0 = ut[2 * u], t1 = ut[2 * u + 1];
                    span2_f32(A, Q, i0 >> 1, i1 >> 1, tu[t0], tv[t0], tu[t1], tv[t1], pp[0], pp[1]);
                } else {
                    const int t = ut[u];
                    pp[0] = span_f32(A, Q, i0 >> 1, i1 >> 1, tu[t], tv[t]);
                }
            } else {
                const int t = ut[u];
                const double *su = reinterpret_cast<const double *>(src);
                pp[0] = span_f64(su, su + a.src_cap, su + 2 * a.src_cap, i0, i1, tu[t], tv[t], a.eps2, s_lt);
            }
        }
        __syncthreads();

        // D: fixed-order reduction of the three row partials, write
        const int rs = TPI * nu;
        for (int t = tid; t < nt; t += kThreads) {
            const int sl = tslot[t];
            T acc = part[sl] + part[rs + sl] + part[2 * rs + sl];
            T phi;
            if constexpr (sizeof(T) == 4) {
                if (!isfinite(acc)) {  // a pair closer than eps: redo this target with the explicit guard
                    const float4 *A = reinterpret_cast<const float4 *>(src);
                    const float2 *Q = reinterpret_cast<const float2 *>(reinterpret_cast<const float *>(src) + 2 * a.src_cap);
                    acc = 0.f;
                    const int jb = uj0[sl / TPI];
                    for (int row = 0; row < 3; ++row) {
                        const int j0 = jb + row * R;
                        acc += span_f32_guarded(A, Q, sstart[j0] >> 1, sstart[j0 + 3] >> 1, tu[t], tv[t], a.eps2);
                    }
                }
                phi = (-0.5f * kLn2) * acc;
            } else {
                phi = -0.5 * acc;
            }
            a.out[tb + t] = a.accumulate ? a.out[tb + t] + phi : phi;
        }
        // the next_tile() barrier orders this tile's shared-memory reads before the next tile's writes
    }
    if (tid == 0) queue_exit(a.queue);
}

// ---------------------------------------------------------------- R kernel
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// Persistent CTAs; per tile one TMA bulk copy (cp.async.bulk) per array brings
// the tile's packed halo (contiguous in HBM, 16-B aligned) into shared memory
// while the threads stage the tile's targets.  Work items (target, third of
// its halo) balance the CTA; fixed-order reduction keeps results deterministic.
template <typename T>
__global__ void __launch_bounds__(kThreads)
p2p_r_kernel(const P2PArgs<T> a) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ int s_tile;
    const int k = a.k, W = 1 << k, WW = W * W;
    const RCarve c = r_carve(k, a.src_cap, a.tgt_cap, (int)sizeof(T));
    double2 *s_lt = reinterpret_cast<double2 *>(smem + c.ltab);
    if constexpr (sizeof(T) == 8)  // visible after the first tile's barrier
        for (int i = threadIdx.x; i < kLogTab; i += blockDim.x) s_lt[i] = a.log_tab[i];
    int *toff = reinterpret_cast<int *>(smem + c.toff);
    int *hoff = reinterpret_cast<int *>(smem + c.hoff);
    int *tbx = reinterpret_cast<int *>(smem + c.tbx);
    T *tu = reinterpret_cast<T *>(smem + c.tu);
    T *tv = reinterpret_cast<T *>(smem + c.tv);
    T *part = reinterpret_cast<T *>(smem + c.part);
    uint64_t *mbar = reinterpret_cast<uint64_t *>(smem + c.bar);
    T *s_uv = reinterpret_cast<T *>(smem + c.src);
    T *s_q = s_uv + 2 * (size_t)a.src_cap;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t bar = smem_addr(mbar);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    uint32_t parity = 0;

    for (int ti = next_tile(a.queue, &s_tile); ti < a.ntiles; ti = next_tile(a.queue, &s_tile)) {
        const uint32_t m0 = (uint32_t)a.tiles[ti] << (2 * k);
        const int tb = a.tgt_off[m0];
        const uint32_t hb = a.halo_off[m0], nent = a.halo_off[m0 + WW] - hb;  // multiple of 4
        if (tid == 0) {
            const uint32_t b_uv = nent * 2 * (uint32_t)sizeof(T), b_q = nent * (uint32_t)sizeof(T);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(b_uv + b_q)
                         : "memory");
            if (nent) {
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_addr(s_uv)),
                    "l"(a.halo_uv + 2 * (size_t)hb), "r"(b_uv), "r"(bar)
                    : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_addr(s_q)),
                    "l"(a.q + hb), "r"(b_q), "r"(bar)
                    : "memory");
            }
        }
        for (int i = tid; i <= WW; i += kThreads) {
            toff[i] = a.tgt_off[m0 + i] - tb;
            hoff[i] = (int)(a.halo_off[m0 + i] - hb);
        }
        __syncthreads();
        for (int t = tid; t < toff[WW]; t += kThreads) {
            int lo = 0, hi = WW;  // last box bl with toff[bl] <= t
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (toff[mid] <= t) lo = mid;
                else hi = mid;
            }
            const typename V2<T>::type uv = a.tgt_uv[tb + t];
            tu[t] = uv.x;  // fp32: relative to the 3x3 block's corner, like the halo (R17)
            tv[t] = uv.y;
            tbx[t] = lo;
        }
        asm volatile(
            "{\n\t.reg .pred P;\n"
            "WAIT_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
            "@!P bra WAIT_%=;\n}" ::"r"(bar),
            "r"(parity)
            : "memory");
        parity ^= 1u;
        __syncthreads();

        const int nt = toff[WW];
        for (int it = tid; it < 3 * nt; it += kThreads) {
            const int part3 = (it >= nt) + (it >= 2 * nt);
            const int t = it - part3 * nt;
            const int bl = tbx[t];
            const int p0 = hoff[bl] >> 1, np = (hoff[bl + 1] >> 1) - p0;  // source pairs of this box's halo
            const int q0 = p0 + (np * part3) / 3, q1 = p0 + (np * (part3 + 1)) / 3;
            if constexpr (sizeof(T) == 4) {
                part[it] = span_f32(reinterpret_cast<const float4 *>(s_uv), reinterpret_cast<const float2 *>(s_q), q0,
                                    q1, tu[t], tv[t]);
            } else {
                const double *su = s_uv;
                double acc = 0.0;
                for (int j = 2 * q0; j < 2 * q1; ++j) {
                    const double du = tu[t] - su[2 * j], dv = tv[t] - su[2 * j + 1];
                    const double r2 = fma(dv, dv, du * du);
                    if (r2 >= a.eps2) acc = fma(s_q[j], log_tab(r2, s_lt), acc);
                }
                part[it] = acc;
            }
        }
        __syncthreads();
        for (int t = tid; t < nt; t += kThreads) {
            T acc = part[t] + part[nt + t] + part[2 * nt + t];
            T phi;
            if constexpr (sizeof(T) == 4) {
                if (!isfinite(acc)) {
                    const int bl = tbx[t];
                    acc = span_f32_guarded(reinterpret_cast<const float4 *>(s_uv),
                                           reinterpret_cast<const float2 *>(s_q), hoff[bl] >> 1, hoff[bl + 1] >> 1,
                                           tu[t], tv[t], a.eps2);
                }
                phi = (-0.5f * kLn2) * acc;
            } else {
                phi = -0.5 * acc;
            }
            a.out[tb + t] = a.accumulate ? a.out[tb + t] + phi : phi;
        }
    }
    if (tid == 0) queue_exit(a.queue);
}

// ---------------------------------------------------------------- TILED kernel
// The TILED layout packs, per tile, everything the CTA needs contiguously at
// plan time: a table record (region box starts + slot count), the region's
// sources (tile + one-box ring, rebased to the region origin, in row-run order)
// with a per-entry source index, the tile's target slots (coordinates, row-run
// base, output index) and, for NS = 3, the item list.  One elected thread
// bulk-copies a tile's record with TMA (cp.async.bulk, mbarrier completion),
// optionally one tile ahead (NBUF = 2).  Weights are gathered through the
// per-entry index (q stays in plan order).
//   PAD  (dense fp32): boxes padded to even counts, sources packed per pair,
//        packed f32x2 loops; TPI = 2 slots per unit share each LDS.
//   !PAD (sparse, fp64): no padding, one pair per step.
//   NS = 3: items (unit, row-run) in the plan's length-sorted order, then the
//   fixed-order reduction of the three partials; NS = 1: one item per unit
//   sweeps its three row-runs in order (LEAN: TPI = 1 unpadded, boxes ordered
//   by n9, the three runs optionally flattened into one sequence).
// Every target's sum has a fixed order independent of the launch, the tile
// split and the partition: results are bit-reproducible.
#ifndef P2P_HELM_PAIR
#define P2P_HELM_PAIR 1  // fp32 Helmholtz: two sources per step, series packed in f32x2
#endif
#ifndef P2P_BOX3_HELM_PAIR
#define P2P_BOX3_HELM_PAIR 1  // 3D Helmholtz fp32: two targets per thread
#endif
#ifndef P2P_LEAN_MINB
#define P2P_LEAN_MINB 0  // > 0: register cap via min resident CTAs for the 64-thread lean instances
#endif
#ifndef P2P_DENSE_MINB
#define P2P_DENSE_MINB 0  // > 0: register cap via min resident CTAs for the TPI = 2 instances (experiments)
#endif
template <typename T, int TPI, int NT, bool PAD, int NS>
__global__ void __launch_bounds__(NT, (TPI == 2 && P2P_DENSE_MINB > 0)                          ? P2P_DENSE_MINB
                                      : (TPI == 1 && !PAD && NS == 1 && NT == 64 && P2P_LEAN_MINB > 0) ? P2P_LEAN_MINB
                                                                                                  : 0)
p2p_tiled_kernel(const P2PArgs<T> a) {
    static_assert(TPI == 1 || (TPI == 2 && PAD && sizeof(T) == 4) || (TPI == 2 && !PAD && sizeof(T) == 8 && NS == 3),
                  "TPI = 2: the padded fp32 path, or dense fp64 (unpadded, row items)");
    static_assert(!PAD || sizeof(T) == 4, "the padded layout is fp32");
    static_assert(NS == 1 || NS == 3, "one item per unit, or one per row-run");
    constexpr bool LEAN = NS == 1 && TPI == 1 && !PAD;
    extern __shared__ __align__(128) unsigned char smem[];
    // next tile + its first target, double-buffered by iteration parity: thread 0 writes slot
    // (it + 1) & 1 during iteration it while the others may still read slot it & 1
    __shared__ int s_next[2], s_base_next[2], s_part_next[2];
    const int k = a.k, W = 1 << k, R = W + 2, RR = R * R;
    const TCarve c = tiled_carve(k, a.src_cap, a.tgt_cap, (int)sizeof(T), TPI, NS, a.nbuf, a.lt8);
    const bool db = a.nbuf == 2;
    T *s_q = reinterpret_cast<T *>(smem + c.q);
    T *part = reinterpret_cast<T *>(smem + c.part);
    double2 *s_lt = reinterpret_cast<double2 *>(smem + c.ltab);
    uint64_t *mbar = reinterpret_cast<uint64_t *>(smem + c.bar);
    const int tid = threadIdx.x, lane = tid & 31;
    if constexpr (sizeof(T) == 8 && NS == 3) {  // dense fp64: the 8-fold table of log_tab8, or log_tab's
        if (a.lt8)
            for (int i = tid; i < 8 * kLogTab8; i += NT) s_lt[i] = a.log_tab[kLogTab + kLogTab32 + (i >> 3)];
        else
            for (int i = tid; i < kLogTab; i += NT) s_lt[i] = a.log_tab[i];
    }
    float lc = 0.f;  // fp64: this lane's entry of the 32-entry shuffle table (log_shfl)
    double lL = 0.0;
    if constexpr (sizeof(T) == 8) {
        const double2 e = a.log_tab[kLogTab + lane];
        lc = (float)e.x;
        lL = e.y;
    }

    auto issue = [&](int ti, int b) {  // one elected thread: arm buffer b and bulk-copy tile ti's record
        const int slot = a.tile_slot[ti];
        unsigned char *buf = smem + c.buf0 + b * c.bufsz;
        const uint32_t rb = a.reg_off[slot], nent = a.reg_off[slot + 1] - rb;
        const uint32_t tb = a.tgt_pack_off[slot], ntp = a.tgt_pack_off[slot + 1] - tb;
        const uint32_t ib = NS == 3 ? a.item_off[slot] : 0u, nit = NS == 3 ? a.item_off[slot + 1] - ib : 0u;
        const uint32_t b_tab = (uint32_t)c.tstride * 2u, b_uv = nent * 2 * (uint32_t)sizeof(T), b_ix = nent * 4u;
        const uint32_t b_tuv = ntp * 2 * (uint32_t)sizeof(T), b_t16 = ntp * 2u, b_it = nit * 2u;
        const uint32_t bar = smem_addr(mbar + b);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                     "r"(b_tab + b_uv + b_ix + b_tuv + 2 * b_t16 + b_it)
                     : "memory");
#define P2P_BULK(dst, src, bytes)                                                                        \
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" \
                 ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(bar)                                   \
                 : "memory")
        P2P_BULK(buf + c.table, a.reg_table + (size_t)slot * c.tstride, b_tab);
        if (nent) {
            P2P_BULK(buf + c.uv, a.reg_uv + 2 * (size_t)rb, b_uv);
            P2P_BULK(buf + c.idx, a.reg_idx + rb, b_ix);
        }
        if (ntp) {
            P2P_BULK(buf + c.tuv, a.tgt_ruv + 2 * (size_t)tb, b_tuv);
            P2P_BULK(buf + c.tbl, a.tgt_bl + tb, b_t16);
            P2P_BULK(buf + c.oix, a.tgt_oix + tb, b_t16);
        }
        if (nit) P2P_BULK(buf + c.items, a.items + ib, b_it);
#undef P2P_BULK
    };

    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(mbar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(mbar + 1)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const int t0 = atomicAdd(a.queue, 1);
        s_next[0] = t0;
        if (t0 < a.ntiles) {
            s_base_next[0] = a.tile_tgt_base[a.tile_slot[t0]];
            s_part_next[0] = a.tile_part[t0];
            issue(t0, 0);
        }
    }
    __syncthreads();
    int cur = s_next[0], buf = 0, tb = s_base_next[0], pinfo = s_part_next[0], it = 0;
    uint32_t parity = 0u;  // bit b = phase parity of buffer b's mbarrier

    while (cur < a.ntiles) {
        unsigned long long *trc = (a.trace && tid == 0) ? a.trace + 8 * (size_t)cur : nullptr;
        if (trc) {
            trc[0] = (unsigned long long)smid() << 32 | blockIdx.x;
            trc[1] = gtimer();
        }
        const unsigned char *B = smem + c.buf0 + buf * c.bufsz;
        const uint16_t *table = reinterpret_cast<const uint16_t *>(B + c.table);
        const T *s_uv = reinterpret_cast<const T *>(B + c.uv);
        const int32_t *s_idx = reinterpret_cast<const int32_t *>(B + c.idx);
        const T *tuv = reinterpret_cast<const T *>(B + c.tuv);
        const uint16_t *tbl = reinterpret_cast<const uint16_t *>(B + c.tbl);
        const uint16_t *oix = reinterpret_cast<const uint16_t *>(B + c.oix);
        const uint16_t *items = reinterpret_cast<const uint16_t *>(B + c.items);
        if (tid == 0) {  // next tile; with two buffers its record streams in while this tile computes
            const int nx = atomicAdd(a.queue, 1);
            s_next[(it + 1) & 1] = nx;
            if (nx < a.ntiles) {
                s_base_next[(it + 1) & 1] = a.tile_tgt_base[a.tile_slot[nx]];
                s_part_next[(it + 1) & 1] = a.tile_part[nx];
                if (db) issue(nx, buf ^ 1);
            }
        }
        {
            const uint32_t bar = smem_addr(mbar + buf);
            asm volatile(
                "{\n\t.reg .pred P;\n"
                "WAIT_%=:\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
                "@!P bra WAIT_%=;\n}" ::"r"(bar),
                "r"((parity >> buf) & 1u)
                : "memory");
            parity ^= 1u << buf;
        }
        if (trc) trc[2] = gtimer();
        const int nent = (int)table[RR], nslot = (int)table[RR + 1], nu = nslot / TPI;
        gather_weights(s_idx, a.q, s_q, nent, tid, NT);  // weights through the per-entry index
        __syncthreads();
        const int npart = pinfo >> 16, ipart = pinfo & 0xffff;
        // lean, plan order, whole tile: the slots are n9-sorted, so their outputs are scattered; stage
        // them in shared memory and store the tile's contiguous output range coalesced instead
        const bool stage = LEAN && a.out_idx == nullptr && npart == 1;
        int ub = 0, ue = nu;
        if (npart > 1) {  // tail tile split into npart unit ranges (nu * npart < 2^31)
            ub = (nu * ipart) / npart;
            ue = (nu * (ipart + 1)) / npart;
        }
        if (trc) {
            trc[3] = gtimer();
            trc[6] = nu;
            trc[7] = (unsigned long long)nent;
        }

        // TPI partial sums of unit u over its row-run `row`
        auto unit_row = [&](int u, int row, T *res) {
            const int t0 = TPI * u, j0 = tbl[t0] + row * R;
            const int i0 = table[j0], i1 = table[j0 + 3];
            if constexpr (PAD) {
                const float4 *A = reinterpret_cast<const float4 *>(s_uv);
                const float2 *Q = reinterpret_cast<const float2 *>(s_q);
                if constexpr (TPI == 2)
                    span2_f32(A, Q, i0 >> 1, i1 >> 1, tuv[2 * t0], tuv[2 * t0 + 1], tuv[2 * t0 + 2], tuv[2 * t0 + 3],
                              res[0], res[1]);
                else
                    res[0] = span_f32(A, Q, i0 >> 1, i1 >> 1, tuv[2 * t0], tuv[2 * t0 + 1]);
            } else if constexpr (sizeof(T) == 4) {
                res[0] = span1_f32(reinterpret_cast<const float2 *>(s_uv), reinterpret_cast<const float *>(s_q), i0,
                                   i1, tuv[2 * t0], tuv[2 * t0 + 1]);
            } else if constexpr (TPI == 2) {  // dense fp64: two targets per source load
                span1x2_f64(reinterpret_cast<const double2 *>(s_uv), reinterpret_cast<const double *>(s_q), i0, i1,
                            tuv[2 * t0], tuv[2 * t0 + 1], tuv[2 * t0 + 2], tuv[2 * t0 + 3], a.eps2, s_lt, lane & 7,
                            a.lt8, res[0], res[1]);
            } else {
                if (a.lt8)
                    res[0] = span1_f64r(reinterpret_cast<const double2 *>(s_uv), reinterpret_cast<const double *>(s_q),
                                        i0, i1, tuv[2 * t0], tuv[2 * t0 + 1], a.eps2, s_lt, lane & 7);
                else
                    res[0] = span1_f64(reinterpret_cast<const double2 *>(s_uv), reinterpret_cast<const double *>(s_q),
                                       i0, i1, tuv[2 * t0], tuv[2 * t0 + 1], a.eps2, s_lt);
            }
        };
        // final value of slot t from its row-ordered sum (fp32: guarded redo if non-finite),
        // written to the slot's tile-local output index (duplicate slots write nothing)
        auto finish = [&](int t, T acc) {
            const int o = oix[t];
            if (TPI > 1 && o == 0xFFFF) return;
            if constexpr (sizeof(T) == 4) {
                if (!isfinite(acc)) {
                    const int jb = tbl[t];
                    acc = 0.f;
                    for (int row = 0; row < 3; ++row) {
                        const int j0 = jb + row * R;
                        if constexpr (PAD)
                            acc += span_f32_guarded(reinterpret_cast<const float4 *>(s_uv),
                                                    reinterpret_cast<const float2 *>(s_q), table[j0] >> 1,
                                                    table[j0 + 3] >> 1, tuv[2 * t], tuv[2 * t + 1], a.eps2);
                        else
                            acc += span1_f32_guarded(reinterpret_cast<const float2 *>(s_uv),
                                                     reinterpret_cast<const float *>(s_q), table[j0], table[j0 + 3],
                                                     tuv[2 * t], tuv[2 * t + 1], a.eps2);
                    }
                }
                acc = (-0.5f * kLn2) * acc;
            } else {
                if (TPI == 2 && !isfinite(acc)) {  // dense fp64: a pair flagged closer than eps (span1x2_f64)
                    const int jb = tbl[t];
                    acc = 0.0;
                    for (int row = 0; row < 3; ++row) {
                        const int j0 = jb + row * R;
                        const double2 *UV = reinterpret_cast<const double2 *>(s_uv);
                        const double *Qd = reinterpret_cast<const double *>(s_q);
                        acc += a.lt8 ? span1_f64r(UV, Qd, table[j0], table[j0 + 3], tuv[2 * t], tuv[2 * t + 1], a.eps2,
                                                  s_lt, lane & 7)
                                     : span1_f64(UV, Qd, table[j0], table[j0 + 3], tuv[2 * t], tuv[2 * t + 1], a.eps2,
                                                 s_lt);
                    }
                }
                acc = -0.5 * acc;
            }
            if (LEAN && stage) {  // staged in output order, stored coalesced after the tile's barrier
                part[o] = acc;
                return;
            }
            const int oi = a.out_idx ? a.out_idx[tb + o] : tb + o;
            a.out[oi] = a.accumulate ? a.out[oi] + acc : acc;
        };

        if constexpr (LEAN && sizeof(T) == 8) {  // fp64: flattened runs, whole-warp rounds (log_shfl)
            for (int base = ub + (tid & ~31); base < ue; base += NT) {
                const int t = base + lane;
                const bool has = t < ue;
                const int jb = has ? tbl[t] : 0;
                const Runs3 runs(table[jb], table[jb + 3], table[jb + R], table[jb + R + 3], table[jb + 2 * R],
                                 table[jb + 2 * R + 3]);
                const double acc = sweep_f64w(
                    reinterpret_cast<const double2 *>(s_uv), reinterpret_cast<const double *>(s_q), has ? runs.n : 0,
                    [&](int v) { return runs.at(runs.v0 + v); }, has ? (double)tuv[2 * t] : 0.0,
                    has ? (double)tuv[2 * t + 1] : 0.0, (double)a.eps2, lc, lL);
                if (has) finish(t, (T)acc);
            }
        } else if constexpr (LEAN) {  // one thread per target (boxes by n9): three row-runs, flattened or in turn
            for (int t = ub + tid; t < ue; t += NT) {
                const int jb = tbl[t];
                const T ux = tuv[2 * t], uy = tuv[2 * t + 1];
                T acc = (T)0;
                if (a.flat) {
                    const Runs3 runs(table[jb], table[jb + 3], table[jb + R], table[jb + R + 3], table[jb + 2 * R],
                                     table[jb + 2 * R + 3]);
                    if constexpr (sizeof(T) == 4)
                        acc = span3_f32(reinterpret_cast<const float2 *>(s_uv), reinterpret_cast<const float *>(s_q),
                                        runs, ux, uy);
                    else
                        acc = span3_f64(reinterpret_cast<const double2 *>(s_uv),
                                        reinterpret_cast<const double *>(s_q), runs, ux, uy, a.eps2, s_lt);
                } else {
#pragma unroll
                    for (int row = 0; row < 3; ++row) {
                        const int j0 = jb + row * R;
                        if constexpr (sizeof(T) == 4)
                            acc += span1_f32(reinterpret_cast<const float2 *>(s_uv),
                                             reinterpret_cast<const float *>(s_q), table[j0], table[j0 + 3], ux, uy);
                        else
                            acc += span1_f64(reinterpret_cast<const double2 *>(s_uv),
                                             reinterpret_cast<const double *>(s_q), table[j0], table[j0 + 3], ux, uy,
                                             a.eps2, s_lt);
                    }
                }
                finish(t, acc);
            }
        } else if constexpr (NS == 1) {  // one item per unit, rows in order
            for (int u = ub + tid; u < ue; u += NT) {
                T acc[TPI], r[TPI];
#pragma unroll
                for (int x = 0; x < TPI; ++x) acc[x] = (T)0;
                for (int row = 0; row < 3; ++row) {
                    unit_row(u, row, r);
#pragma unroll
                    for (int x = 0; x < TPI; ++x) acc[x] += r[x];
                }
#pragma unroll
                for (int x = 0; x < TPI; ++x) finish(TPI * u + x, acc[x]);
            }
        } else {  // (unit, row) items in the plan's order, then the fixed-order reduction of the partials
            for (int it = 3 * ub + tid; it < 3 * ue; it += NT) {  // the plan's LPT-dealt batches, static
                const int w = items[it], u = w >> 2, row = w & 3;
                T res[TPI];
                unit_row(u, row, res);
#pragma unroll
                for (int x = 0; x < TPI; ++x) part[row * nslot + TPI * u + x] = res[x];
            }
            __syncthreads();
            for (int u = ub + tid; u < ue; u += NT) {
#pragma unroll
                for (int x = 0; x < TPI; ++x) {
                    const int sl = TPI * u + x;
                    finish(sl, part[sl] + part[nslot + sl] + part[2 * nslot + sl]);
                }
            }
        }
        __syncthreads();  // buffer `buf` and the work arrays are free; s_next / s_base_next visible
        if (trc) trc[5] = gtimer();
        const int tb_done = tb;
        ++it;
        cur = s_next[it & 1];
        tb = s_base_next[it & 1];
        pinfo = s_part_next[it & 1];
        if (db) buf ^= 1;
        else if (tid == 0 && cur < a.ntiles) issue(cur, 0);
        if (LEAN && stage)  // the staged results (the next writes to `part` follow the next barrier)
            for (int i = tid; i < nslot; i += NT) {
                T *o = a.out + tb_done + i;
                *o = a.accumulate ? *o + part[i] : part[i];
            }
    }
    if (tid == 0) queue_exit(a.queue);
}

// ---------------------------------------------------------------- TILED Helmholtz kernel (NEXT-3)
// G(r) = (i/4) H0^(1)(kappa r) = (-Y0(kappa r) + i J0(kappa r)) / 4 (include/p2p.h; R23),
// complex weights and results as (re, im) pairs.  Same TILED record, queue and TMA staging as the
// lean Laplace path; one thread per target slot (boxes ordered by n9), its three row-runs swept
// as one flattened sequence.  Per pair: r^2, guard, sqrt, J0 and Y0 (CUDA's j0f/y0f, j0/y0:
// rational / asymptotic approximations on the FMA pipe + one sincos and one log beyond the
// small-argument branch), 4 FMA for the complex multiply-add.
template <typename T>
__device__ void bessel_j0y0(T x, T &J, T &Y);
template <>
__device__ __forceinline__ void bessel_j0y0<float>(float x, float &J, float &Y) {
    J = j0f(x);
    Y = y0f(x);
}
// fp64, x > 6 (the series covers x <= 6): the modulus / phase form of H0^(1) = J0 + i Y0
// (A&S 9.2.17, 9.2.28-30): J0 = M cos(theta), Y0 = M sin(theta), M = sqrt(2 / (pi x)) m(w),
// theta = x - pi/4 + g(w) / x, w = (6 / x)^2; m and g are degree-15 / 17 polynomials in w fitted
// to 60-digit mpmath values (tools/gen_hankel_coeffs.py; |error| < 2e-17 on x >= 6), so J0 and
// Y0 carry the ~1e-16 relative error of the fp64 x itself (CUDA's j0 / y0: 5e-12 absolute).
__constant__ double kHankM[16] = {-1.009491152938711e-08, 8.57361572380178e-08, -3.3621255599445164e-07,
    8.119914966752918e-07, -1.3646187307687262e-06, 1.7230350554592675e-06, -1.7496035271524972e-06,
    1.5517824092842689e-06, -1.3504203538737336e-06, 1.3405018556771033e-06, -1.764884373894713e-06,
    3.481928813934044e-06, -1.1635076105372948e-05, 7.987316710141125e-05, -0.0017361111111073842, 1.0};
__constant__ double kHankG[18] = {1.0760822573387157e-07, -1.0085244871057431e-06, 4.380518381796627e-06,
    -1.1732236951590672e-05, 2.1778454372757905e-05, -2.993602677569589e-05, 3.194496675304352e-05,
    -2.764766382910038e-05, 2.0464690083447213e-05, -1.3981396693431658e-05, 9.833845375076344e-06,
    -8.117210709175648e-06, 8.851138042211988e-06, -1.3976003481602903e-05, 3.510941725411511e-05,
    -0.00016170548761511877, 0.001808449074070366, -0.125};
template <>
__device__ __noinline__ void bessel_j0y0<double>(double x, double &J, double &Y) {  // cold: kappa r > 6 only
    const double rx = 1.0 / x, w = 36.0 * rx * rx;
    double m = kHankM[0], g = kHankG[0];
#pragma unroll
    for (int i = 1; i < 16; ++i) m = fma(m, w, kHankM[i]);
#pragma unroll
    for (int i = 1; i < 18; ++i) g = fma(g, w, kHankG[i]);
    const double th = (x - 0.78539816339744830962) + g * rx;
    double s, c;
    sincos(th, &s, &c);
    const double M = m * sqrt(0.63661977236758134308 * rx);  // sqrt(2 / (pi x))
    J = M * c;
    Y = M * s;
}

// Small arguments (z = (kappa r / 2)^2 <= kHelmZmax): J0 and Y0 from their ascending series
// (Abramowitz & Stegun 9.1.12, 9.1.13) sharing one log and one z:
//   J0 = sum_k (-z)^k / (k!)^2,
//   Y0 = (2/pi) [ (ln(x/2) + gamma) J0 + sum_{k>=1} (-1)^{k+1} H_k z^k / (k!)^2 ],  ln(x/2) = ln(z)/2,
// Horner in z: 2 x 11 FFMA + one MUFU.LG2 (fp32, x <= 4.5: |error| <= 8e-7), 2 x 19 DFMA + the
// table log (fp64, x <= 6: <= 1.1e-14); larger arguments take CUDA's j0/y0.
template <typename T>
struct HelmSeries;
template <>
struct HelmSeries<float> {
    static constexpr float kZmax = 4.5f * 4.5f / 4.f;
    static __device__ __forceinline__ void eval(float z, float &J, float &Y, const double2 *) {
        constexpr float A[11] = {1.0f, -1.0f, 0.25f, -0.027777777777777776f, 0.001736111111111111f,
                                 -6.944444444444444e-05f, 1.9290123456790124e-06f, -3.936759889140842e-08f,
                                 6.151187326782565e-10f, -7.594058428126624e-12f, 7.594058428126623e-14f};
        constexpr float B[11] = {0.0f, 1.0f, -0.375f, 0.05092592592592592f, -0.003616898148148148f,
                                 0.0001585648148148148f, -4.72608024691358e-06f, 1.0207455998272325e-07f,
                                 -1.6718048413148328e-09f, 2.1483350211950277e-11f, -2.224275605476294e-13f};
        float j = A[10], s = B[10];
#pragma unroll
        for (int k = 9; k >= 0; --k) {
            j = fmaf(j, z, A[k]);
            s = fmaf(s, z, B[k]);
        }
        const float hl = fmaf(lg2_approx(z), 0.5f * kLn2, 0.5772156649015329f);  // ln(x/2) + gamma
        J = j;
        Y = 0.6366197723675814f * fmaf(hl, j, s);
    }    // two arguments at once: each Horner chain packed over the two sources (f32x2), the two
    // chains (J, S) independent
    static __device__ __forceinline__ void eval2(float za, float zc, float &Ja, float &Ya, float &Jc, float &Yc) {
        constexpr float A[11] = {1.0f, -1.0f, 0.25f, -0.027777777777777776f, 0.001736111111111111f,
                                 -6.944444444444444e-05f, 1.9290123456790124e-06f, -3.936759889140842e-08f,
                                 6.151187326782565e-10f, -7.594058428126624e-12f, 7.594058428126623e-14f};
        constexpr float B[11] = {0.0f, 1.0f, -0.375f, 0.05092592592592592f, -0.003616898148148148f,
                                 0.0001585648148148148f, -4.72608024691358e-06f, 1.0207455998272325e-07f,
                                 -1.6718048413148328e-09f, 2.1483350211950277e-11f, -2.224275605476294e-13f};
        const f2_t Z = f2_pack(za, zc);
        f2_t j = f2_pack(A[10], A[10]), s = f2_pack(B[10], B[10]);
#pragma unroll
        for (int k = 9; k >= 0; --k) {
            j = f2_fma(j, Z, f2_pack(A[k], A[k]));
            s = f2_fma(s, Z, f2_pack(B[k], B[k]));
        }
        const f2_t hl = f2_fma(f2_pack(lg2_approx(za), lg2_approx(zc)), f2_pack(0.5f * kLn2, 0.5f * kLn2),
                               f2_pack(0.5772156649015329f, 0.5772156649015329f));
        const f2_t Y = f2_mul(f2_pack(0.6366197723675814f, 0.6366197723675814f), f2_fma(hl, j, s));
        f2_unpack(j, Ja, Jc);
        f2_unpack(Y, Ya, Yc);
    }
};
// fp64 series coefficients (a_k, b_k of HelmSeries<float>, 19 terms) in the constant bank
__constant__ double kHelmA64[19] = {1.0, -1.0, 0.25, -0.027777777777777776, 0.001736111111111111,
                          -6.944444444444444e-05, 1.9290123456790124e-06, -3.936759889140842e-08,
                          6.151187326782565e-10, -7.594058428126624e-12, 7.594058428126623e-14,
                          -6.276081345559193e-16, 4.358389823304995e-18, -2.5789288895295828e-20,
                          1.3157800456783586e-22, -5.8479113141260385e-25, 2.2843403570804838e-27,
                          -7.904291893012054e-30, 2.4395962632753253e-32};
__constant__ double kHelmB64[19] = {0.0, 1.0, -0.375, 0.05092592592592592, -0.003616898148148148,
                          0.0001585648148148148, -4.72608024691358e-06, 1.0207455998272325e-07,
                          -1.6718048413148328e-09, 2.1483350211950277e-11, -2.224275605476294e-13,
                          1.895299587006153e-15, -1.3525001839484812e-17, 8.201338813682637e-20,
                          -4.278340826570208e-22, 1.9404708872364884e-24, -7.722735675585063e-27,
                          2.71872271202985e-29, -8.52665260731113e-32};
template <>
struct HelmSeries<double> {
    static constexpr double kZmax = 6.0 * 6.0 / 4.0;
    static __device__ __forceinline__ void eval(double z, double &J, double &Y, const double2 *LT) {
        const double *A = kHelmA64, *B = kHelmB64;  // constant-bank operands of DFMA (no UMOV pairs)
        double j = A[18], s = B[18];
#pragma unroll
        for (int k = 17; k >= 0; --k) {
            j = fma(j, z, A[k]);
            s = fma(s, z, B[k]);
        }
        const double hl = fma(log_tab(z, LT), 0.5, 0.5772156649015329);  // ln(x/2) + gamma
        J = j;
        Y = 0.6366197723675814 * fma(hl, j, s);
    }
};

template <typename T, int NT>
__global__ void __launch_bounds__(NT) p2p_tiled_helm_kernel(const P2PArgs<T> a) {
    using C2 = typename V2<T>::type;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ int s_next[2], s_base_next[2];
    const int k = a.k, W = 1 << k, R = W + 2, RR = R * R;
    const HCarve hc = helm_carve(k, a.src_cap, a.tgt_cap, (int)sizeof(T));
    const TCarve &c = hc.t;
    C2 *s_q = reinterpret_cast<C2 *>(smem + hc.q);
    double2 *s_lt = reinterpret_cast<double2 *>(smem + hc.ltab);
    uint64_t *mbar = reinterpret_cast<uint64_t *>(smem + hc.bar);
    if constexpr (sizeof(T) == 8)
        for (int i = threadIdx.x; i < kLogTab; i += NT) s_lt[i] = a.log_tab[i];
    const C2 *q2 = reinterpret_cast<const C2 *>(a.q);
    C2 *out2 = reinterpret_cast<C2 *>(a.out);
    const int tid = threadIdx.x;

    auto issue = [&](int ti) {  // one elected thread: bulk-copy tile ti's record (no item list)
        const int slot = a.tile_slot[ti];
        unsigned char *buf = smem + c.buf0;
        const uint32_t rb = a.reg_off[slot], nent = a.reg_off[slot + 1] - rb;
        const uint32_t tb = a.tgt_pack_off[slot], ntp = a.tgt_pack_off[slot + 1] - tb;
        const uint32_t b_tab = (uint32_t)c.tstride * 2u, b_uv = nent * 2 * (uint32_t)sizeof(T), b_ix = nent * 4u;
        const uint32_t b_tuv = ntp * 2 * (uint32_t)sizeof(T), b_t16 = ntp * 2u;
        const uint32_t bar = smem_addr(mbar);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                     "r"(b_tab + b_uv + b_ix + b_tuv + 2 * b_t16)
                     : "memory");
#define P2P_BULK(dst, src, bytes)                                                                        \
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" \
                 ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(bar)                                   \
                 : "memory")
        P2P_BULK(buf + c.table, a.reg_table + (size_t)slot * c.tstride, b_tab);
        if (nent) {
            P2P_BULK(buf + c.uv, a.reg_uv + 2 * (size_t)rb, b_uv);
            P2P_BULK(buf + c.idx, a.reg_idx + rb, b_ix);
        }
        if (ntp) {
            P2P_BULK(buf + c.tuv, a.tgt_ruv + 2 * (size_t)tb, b_tuv);
            P2P_BULK(buf + c.tbl, a.tgt_bl + tb, b_t16);
            P2P_BULK(buf + c.oix, a.tgt_oix + tb, b_t16);
        }
#undef P2P_BULK
    };

    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const int t0 = atomicAdd(a.queue, 1);
        s_next[0] = t0;
        if (t0 < a.ntiles) {
            s_base_next[0] = a.tile_tgt_base[a.tile_slot[t0]];
            issue(t0);
        }
    }
    __syncthreads();
    int cur = s_next[0], tb = s_base_next[0], it = 0;
    uint32_t parity = 0u;
    const T kap = a.kappa, kq = (T)0.25 * a.kappa * a.kappa, quarter = (T)0.25;
    while (cur < a.ntiles) {
        const unsigned char *B = smem + c.buf0;
        const uint16_t *table = reinterpret_cast<const uint16_t *>(B + c.table);
        const C2 *s_uv = reinterpret_cast<const C2 *>(B + c.uv);
        const int32_t *s_idx = reinterpret_cast<const int32_t *>(B + c.idx);
        const T *tuv = reinterpret_cast<const T *>(B + c.tuv);
        const uint16_t *tbl = reinterpret_cast<const uint16_t *>(B + c.tbl);
        const uint16_t *oix = reinterpret_cast<const uint16_t *>(B + c.oix);
        if (tid == 0) {
            const int nx = atomicAdd(a.queue, 1);
            s_next[(it + 1) & 1] = nx;
            if (nx < a.ntiles) s_base_next[(it + 1) & 1] = a.tile_tgt_base[a.tile_slot[nx]];
        }
        {
            const uint32_t bar = smem_addr(mbar);
            asm volatile(
                "{\n\t.reg .pred P;\n"
                "WAIT_%=:\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
                "@!P bra WAIT_%=;\n}" ::"r"(bar),
                "r"(parity)
                : "memory");
            parity ^= 1u;
        }
        const int nent = (int)table[RR], nu = (int)table[RR + 1];
        // complex weights through the per-entry index, 4 loads in flight per thread
        for (int base = tid; base < nent; base += 4 * NT) {
            C2 v[4];
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                const int i = base + x * NT;
                const int32_t j = i < nent ? s_idx[i] : -1;
                if (j >= 0) v[x] = q2[j];
                else v[x].x = v[x].y = (T)0;
            }
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                const int i = base + x * NT;
                if (i < nent) s_q[i] = v[x];
            }
        }
        __syncthreads();
        const int pinfo = a.tile_part[cur], npart = pinfo >> 16, ipart = pinfo & 0xffff;
        int ub = 0, ue = nu;
        if (npart > 1) {
            ub = (nu * ipart) / npart;
            ue = (nu * (ipart + 1)) / npart;
        }
        for (int t = ub + tid; t < ue; t += NT) {
            const int jb = tbl[t];
            const T ux = tuv[2 * t], uy = tuv[2 * t + 1];
            const Runs3 runs(table[jb], table[jb + 3], table[jb + R], table[jb + R + 3], table[jb + 2 * R],
                             table[jb + 2 * R + 3]);
            T re = (T)0, im = (T)0;
            const int v1 = runs.v0 + runs.n;
            auto one = [&](int j) {
                const C2 sp = s_uv[j];
                const T du = ux - sp.x, dv = uy - sp.y;
                const T r2 = du * du + dv * dv;
                if (r2 < a.eps2) return;  // coincident points contribute 0 (R3)
                T J, Y;
                const T z = kq * r2;  // (kappa r / 2)^2
                if (z <= HelmSeries<T>::kZmax) HelmSeries<T>::eval(z, J, Y, s_lt);
                else bessel_j0y0<T>(kap * sqrt(r2), J, Y);
                const C2 qv = s_q[j];
                re = fma(-qv.x, Y, fma(-qv.y, J, re));
                im = fma(qv.x, J, fma(-qv.y, Y, im));
            };
            int v = runs.v0;
            if constexpr (sizeof(T) == 4 && P2P_HELM_PAIR) {
                // two sources per step: both series in packed f32x2 FMAs (two independent chains)
                for (; v + 1 < v1; v += 2) {
                    const int ja = runs.at(v), jc = runs.at(v + 1);
                    const float2 pa = reinterpret_cast<const float2 *>(s_uv)[ja];
                    const float2 pc = reinterpret_cast<const float2 *>(s_uv)[jc];
                    const float dua = ux - pa.x, dva = uy - pa.y, duc = ux - pc.x, dvc = uy - pc.y;
                    const float r2a = fmaf(dva, dva, dua * dua), r2c = fmaf(dvc, dvc, duc * duc);
                    const float za = kq * r2a, zc = kq * r2c;
                    if (r2a >= a.eps2 && r2c >= a.eps2 && za <= HelmSeries<float>::kZmax &&
                        zc <= HelmSeries<float>::kZmax) {
                        float Ja, Ya, Jc, Yc;
                        HelmSeries<float>::eval2(za, zc, Ja, Ya, Jc, Yc);
                        const float2 qa = reinterpret_cast<const float2 *>(s_q)[ja];
                        const float2 qc = reinterpret_cast<const float2 *>(s_q)[jc];
                        re = fmaf(-qa.x, Ya, fmaf(-qa.y, Ja, re));
                        im = fmaf(qa.x, Ja, fmaf(-qa.y, Ya, im));
                        re = fmaf(-qc.x, Yc, fmaf(-qc.y, Jc, re));
                        im = fmaf(qc.x, Jc, fmaf(-qc.y, Yc, im));
                    } else {
                        one(ja);
                        one(jc);
                    }
                }
            }
            for (; v < v1; ++v) one(runs.at(v));
            const int o = oix[t];
            const int oi = a.out_idx ? a.out_idx[tb + o] : tb + o;
            C2 r;
            r.x = quarter * re;
            r.y = quarter * im;
            if (a.accumulate) {
                const C2 p = out2[oi];
                r.x += p.x;
                r.y += p.y;
            }
            out2[oi] = r;
        }
        __syncthreads();
        ++it;
        cur = s_next[it & 1];
        tb = s_base_next[it & 1];
        if (tid == 0 && cur < a.ntiles) issue(cur);
    }
    if (tid == 0) queue_exit(a.queue);
}

// ---------------------------------------------------------------- 3D box kernel (NEXT-3)
// Octree leaf grid of the unit cube (include/p2p.h LAPLACE_3D / HELMHOLTZ_3D; R24).
// Persistent CTAs pull target boxes from the queue (longest first); per box the 27 neighbour
// boxes' CSR segments are staged into shared memory, each source shifted by its box offset so
// all coordinates are relative to the target box origin in units of h (x, y, z, q); the box's
// targets are then swept against the staged sources -- every lane of a warp reads the same
// source (a broadcast, no bank conflicts).  Boxes with fewer targets than threads split the
// sources into C = NT / n_t chunks per target (fixed chunking, fixed-order reduction: results
// are bit-reproducible).  Per pair: Laplace 1 MUFU.RSQ + 7 FP32; Helmholtz adds r, the phase
// kappa h r reduced to [-pi, pi] and __sincosf (2 MUFU).  fp64: rsqrt, sincos.
__device__ __forceinline__ uint32_t compact3(uint32_t v) {
    uint32_t r = 0;
#pragma unroll
    for (int b = 0; b < 10; ++b) r |= ((v >> (3 * b)) & 1u) << b;
    return r;
}
__device__ __forceinline__ uint32_t spread3d(uint32_t v) {
    uint32_t r = 0;
#pragma unroll
    for (int b = 0; b < 10; ++b) r |= ((v >> b) & 1u) << (3 * b);
    return r;
}

template <typename T, bool HELM>
__device__ __forceinline__ void box3d_pairs(const T *__restrict__ P, const T *__restrict__ QI, int s0, int s1, T tx,
                                            T ty, T tz, T eps2, T kh, T &re, T &im) {
    for (int s = s0; s < s1; ++s) {
        T px, py, pz, q;
        if constexpr (sizeof(T) == 4) {
            const float4 v = reinterpret_cast<const float4 *>(P)[s];
            px = v.x; py = v.y; pz = v.z; q = v.w;
        } else {
            const double2 a = reinterpret_cast<const double2 *>(P)[2 * s], b = reinterpret_cast<const double2 *>(P)[2 * s + 1];
            px = a.x; py = a.y; pz = b.x; q = b.y;
        }
        const T dx = tx - px, dy = ty - py, dz = tz - pz;
        const T r2 = fma(dz, dz, fma(dy, dy, dx * dx));
        if (!(r2 >= eps2)) continue;  // coincident points contribute 0 (R3)
        const T rs = rsqrt(r2);
        if constexpr (!HELM) {
            re = fma(q, rs, re);
        } else {
            const T qi = QI[s];
            T sn, cs;
            const T ph = kh * (r2 * rs);
            if constexpr (sizeof(T) == 4) {
                __sincosf(ph, &sn, &cs);  // |ph| <= 2 sqrt(3) kappa h: MUFU accuracy holds
            } else {
                sincos(ph, &sn, &cs);
            }
            const T gc = cs * rs, gs = sn * rs;
            re = fma(q, gc, fma(-qi, gs, re));
            im = fma(q, gs, fma(qi, gc, im));
        }
    }
}

// fp32 Laplace, two targets per thread sharing each broadcast source load, f32x2 math:
// 3 FADD2 + FMUL2 + 2 FFMA2 + 2 MUFU.RSQ + FFMA2 per two pairs.  No guard in the loop: a
// coincident pair gives rsqrt(0) = inf and a non-finite sum, and that unit is recomputed with
// the guard (R17).
__device__ __forceinline__ float rsq_approx(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
// fp32 Helmholtz 3D, two targets per thread sharing each source load: distances in f32x2, then
// per target rsqrt + sincos (3 MUFU) and the complex multiply-add.  Guarded in the loop.
__device__ __forceinline__ void box3d_pairs2_helm_f32(const float4 *__restrict__ P, const float *__restrict__ QI,
                                                      int s0, int s1, float x0, float y0, float z0, float x1,
                                                      float y1, float z1, float eps2, float kh, float &re0,
                                                      float &im0, float &re1, float &im1) {
    const f2_t X = f2_pack(x0, x1), Y = f2_pack(y0, y1), Z = f2_pack(z0, z1);
    re0 = im0 = re1 = im1 = 0.f;
    for (int s = s0; s < s1; ++s) {
        const float4 p = P[s];
        const float qi = QI[s];
        const f2_t dx = f2_sub(X, f2_pack(p.x, p.x)), dy = f2_sub(Y, f2_pack(p.y, p.y)), dz = f2_sub(Z, f2_pack(p.z, p.z));
        float r20, r21;
        f2_unpack(f2_fma(dz, dz, f2_fma(dy, dy, f2_mul(dx, dx))), r20, r21);
        if (r20 >= eps2) {
            const float rs = rsq_approx(r20);
            float sn, cs;
            __sincosf(kh * (r20 * rs), &sn, &cs);
            const float gc = cs * rs, gs = sn * rs;
            re0 = fmaf(p.w, gc, fmaf(-qi, gs, re0));
            im0 = fmaf(p.w, gs, fmaf(qi, gc, im0));
        }
        if (r21 >= eps2) {
            const float rs = rsq_approx(r21);
            float sn, cs;
            __sincosf(kh * (r21 * rs), &sn, &cs);
            const float gc = cs * rs, gs = sn * rs;
            re1 = fmaf(p.w, gc, fmaf(-qi, gs, re1));
            im1 = fmaf(p.w, gs, fmaf(qi, gc, im1));
        }
    }
}
__device__ __forceinline__ void box3d_pairs2_f32(const float4 *__restrict__ P, int s0, int s1, float x0, float y0,
                                                 float z0, float x1, float y1, float z1, float &a0, float &a1) {
    const f2_t X = f2_pack(x0, x1), Y = f2_pack(y0, y1), Z = f2_pack(z0, z1);
    f2_t acc = 0ull;
#pragma unroll 4
    for (int s = s0; s < s1; ++s) {
        const float4 p = P[s];
        const f2_t dx = f2_sub(X, f2_pack(p.x, p.x)), dy = f2_sub(Y, f2_pack(p.y, p.y)), dz = f2_sub(Z, f2_pack(p.z, p.z));
        const f2_t r2 = f2_fma(dz, dz, f2_fma(dy, dy, f2_mul(dx, dx)));
        float u0, u1;
        f2_unpack(r2, u0, u1);
        acc = f2_fma(f2_pack(p.w, p.w), f2_pack(rsq_approx(u0), rsq_approx(u1)), acc);
    }
    f2_unpack(acc, a0, a1);
}

template <typename T, bool HELM, int NT>
__global__ void __launch_bounds__(NT) p2p_box3d_kernel(const P2PArgs<T> a) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_box;
    constexpr int comps = HELM ? 2 : 1;
    // partial sums: 2 per thread for complex values and for the fp32 two-target units
    const B3Carve c = box3d_carve(a.src_cap, (int)sizeof(T), comps, NT, box3d_parts(HELM, sizeof(T)));
    T *s_p = reinterpret_cast<T *>(smem + c.p);
    T *s_qi = reinterpret_cast<T *>(smem + c.qi);
    T *s_part = reinterpret_cast<T *>(smem + c.part);
    int *s_nbs = reinterpret_cast<int *>(smem + c.nbs), *s_pre = reinterpret_cast<int *>(smem + c.pre);
    int *s_nbd = reinterpret_cast<int *>(smem + c.nbd);
    const int tid = threadIdx.x;
    const int64_t S = a.S;
    for (;;) {
        if (tid == 0) {
            const int e = atomicAdd(a.queue, 1);
            s_box = e < a.ntiles ? a.tiles[e] : -1;
        }
        __syncthreads();
        const int b = s_box;
        if (b < 0) break;
        if (tid < 32) {  // neighbour boxes: start, count (0 outside the cube), shift; prefix of counts
            int cnt = 0, st = 0, code = 0;
            if (tid < 27) {
                const int dx = tid % 3 - 1, dy = (tid / 3) % 3 - 1, dz = tid / 9 - 1;
                const int64_t x = (int64_t)compact3((uint32_t)b) + dx, y = (int64_t)compact3((uint32_t)b >> 1) + dy,
                              z = (int64_t)compact3((uint32_t)b >> 2) + dz;
                if (x >= 0 && y >= 0 && z >= 0 && x < S && y < S && z < S) {
                    const uint32_t m = spread3d((uint32_t)x) | spread3d((uint32_t)y) << 1 | spread3d((uint32_t)z) << 2;
                    st = a.src_off[m];
                    cnt = a.src_off[m + 1] - st;
                }
                code = (dx + 1) | (dy + 1) << 2 | (dz + 1) << 4;
            }
            int incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (tid >= o) incl += v;
            }
            if (tid < 27) {
                s_nbs[tid] = st;
                s_pre[tid] = incl - cnt;
                s_nbd[tid] = code;
            }
            if (tid == 26) s_pre[27] = incl;
        }
        __syncthreads();
        const int total = s_pre[27];
        for (int i = tid; i < total; i += NT) {  // stage: source i of neighbour nb, shifted into the target box frame
            int nb = 0;
#pragma unroll
            for (int step = 16; step; step >>= 1)
                if (nb + step < 27 && s_pre[nb + step] <= i) nb += step;
            const int j = s_nbs[nb] + (i - s_pre[nb]);
            const int code = s_nbd[nb];
            // fp32: the frame is shifted by one box (x + 1, y + 1, z + 1): every target then sits
            // >= 1 from the origin, so two staged coordinates either coincide or differ by
            // >= 2^-24 > eps S, and the unguarded loop's r^2 = 0 check is the whole guard (R17)
            constexpr int SH = sizeof(T) == 4 ? 0 : 1;
            const T sx = (T)((code & 3) - SH), sy = (T)(((code >> 2) & 3) - SH), sz = (T)(((code >> 4) & 3) - SH);
            const int jq = a.src_idx ? a.src_idx[j] : j;
            T q, qi = (T)0;
            if constexpr (HELM) {
                q = a.q[2 * (int64_t)jq];
                qi = a.q[2 * (int64_t)jq + 1];
                s_qi[i] = qi;
            } else {
                q = a.q[jq];
            }
            const T *sp = a.src_p4 + 4 * (int64_t)j;
            if constexpr (sizeof(T) == 4) {
                const float4 v = *reinterpret_cast<const float4 *>(sp);
                reinterpret_cast<float4 *>(s_p)[i] = make_float4(v.x + sx, v.y + sy, v.z + sz, q);
            } else {
                const double2 u = reinterpret_cast<const double2 *>(sp)[0], w = reinterpret_cast<const double2 *>(sp)[1];
                reinterpret_cast<double2 *>(s_p)[2 * i] = make_double2(u.x + sx, u.y + sy);
                reinterpret_cast<double2 *>(s_p)[2 * i + 1] = make_double2(w.x + sz, q);
            }
        }
        __syncthreads();
        const int t0 = a.tgt_off[b], nt = a.tgt_off[b + 1] - t0;
        constexpr bool PAIR = sizeof(T) == 4 && !HELM;  // two targets per thread (f32x2)
        constexpr bool HPAIR = sizeof(T) == 4 && HELM && P2P_BOX3_HELM_PAIR;  // Helmholtz, two targets per thread
        const int nu = (PAIR || HPAIR) ? (nt + 1) / 2 : nt;  // work units (odd box: the last unit's second slot idle)
        const int C = nu >= NT ? 1 : NT / nu;           // source chunks per unit
        auto finish = [&](int t, T re, T im) {
            const int64_t o = a.out_idx ? a.out_idx[t0 + t] : t0 + t;
            re *= a.scale;
            if constexpr (HELM) {
                im *= a.scale;
                if (a.accumulate) {
                    re += a.out[2 * o];
                    im += a.out[2 * o + 1];
                }
                a.out[2 * o] = re;
                a.out[2 * o + 1] = im;
            } else {
                a.out[o] = a.accumulate ? a.out[o] + re : re;
            }
        };
        for (int it = tid; it < nu * C; it += NT) {
            const int u = it % nu, ch = it / nu;
            const int c0 = (int)((int64_t)total * ch / C), c1 = (int)((int64_t)total * (ch + 1) / C);
            if constexpr (HPAIR) {
                const int ta = 2 * u, tb = min(2 * u + 1, nt - 1);
                const float4 pa4 = reinterpret_cast<const float4 *>(a.tgt_p4)[t0 + ta];
                const float4 pb4 = reinterpret_cast<const float4 *>(a.tgt_p4)[t0 + tb];
                const float pa[3] = {pa4.x + 1.f, pa4.y + 1.f, pa4.z + 1.f};  // fp32 frame shift (R17)
                const float pb[3] = {pb4.x + 1.f, pb4.y + 1.f, pb4.z + 1.f};
                float r0, i0, r1, i1;
                box3d_pairs2_helm_f32(reinterpret_cast<const float4 *>(s_p), reinterpret_cast<const float *>(s_qi), c0,
                                      c1, pa[0], pa[1], pa[2], pb[0], pb[1], pb[2], (float)a.eps2, (float)a.kh, r0, i0,
                                      r1, i1);
                if (C == 1) {
                    finish(ta, (T)r0, (T)i0);
                    if (tb != ta) finish(tb, (T)r1, (T)i1);
                } else {
                    s_part[4 * it] = (T)r0;
                    s_part[4 * it + 1] = (T)i0;
                    s_part[4 * it + 2] = (T)r1;
                    s_part[4 * it + 3] = (T)i1;
                }
            } else if constexpr (PAIR) {
                const int ta = 2 * u, tb = min(2 * u + 1, nt - 1);
                const float4 pa4 = reinterpret_cast<const float4 *>(a.tgt_p4)[t0 + ta];
                const float4 pb4 = reinterpret_cast<const float4 *>(a.tgt_p4)[t0 + tb];
                const float pa[3] = {pa4.x + 1.f, pa4.y + 1.f, pa4.z + 1.f};  // fp32 frame shift (R17)
                const float pb[3] = {pb4.x + 1.f, pb4.y + 1.f, pb4.z + 1.f};
                float r0, r1, dummy;
                box3d_pairs2_f32(reinterpret_cast<const float4 *>(s_p), c0, c1, pa[0], pa[1], pa[2], pb[0], pb[1],
                                 pb[2], r0, r1);
                if (!isfinite(r0)) {
                    r0 = 0.f;
                    box3d_pairs<float, false>(reinterpret_cast<const float *>(s_p), nullptr, c0, c1, pa[0], pa[1],
                                              pa[2], (float)a.eps2, 0.f, r0, dummy);
                }
                if (!isfinite(r1)) {
                    r1 = 0.f;
                    box3d_pairs<float, false>(reinterpret_cast<const float *>(s_p), nullptr, c0, c1, pb[0], pb[1],
                                              pb[2], (float)a.eps2, 0.f, r1, dummy);
                }
                if (C == 1) {
                    finish(ta, (T)r0, (T)0);
                    if (tb != ta) finish(tb, (T)r1, (T)0);
                } else {
                    s_part[2 * it] = (T)r0;
                    s_part[2 * it + 1] = (T)r1;
                }
            } else {
                const T *tq = a.tgt_p4 + 4 * (int64_t)(t0 + u);
                constexpr T SH = sizeof(T) == 4 ? (T)1 : (T)0;  // fp32 frame shift (R17)
                const T tp[3] = {tq[0] + SH, tq[1] + SH, tq[2] + SH};
                T re = (T)0, im = (T)0;
                box3d_pairs<T, HELM>(s_p, s_qi, c0, c1, tp[0], tp[1], tp[2], a.eps2, a.kh, re, im);
                if (C == 1) {
                    finish(u, re, im);
                } else {
                    s_part[comps * it] = re;
                    if constexpr (HELM) s_part[comps * it + 1] = im;
                }
            }
        }
        if (C > 1) {
            __syncthreads();
            for (int t = tid; t < nt; t += NT) {  // chunks summed in order
                T re = (T)0, im = (T)0;
                for (int ch = 0; ch < C; ++ch) {
                    if constexpr (HPAIR) {
                        re += s_part[4 * (ch * nu + t / 2) + 2 * (t & 1)];
                        im += s_part[4 * (ch * nu + t / 2) + 2 * (t & 1) + 1];
                    } else if constexpr (PAIR) {
                        re += s_part[2 * (ch * nu + t / 2) + (t & 1)];
                    } else {
                        re += s_part[comps * (ch * nu + t)];
                        if constexpr (HELM) im += s_part[comps * (ch * nu + t) + 1];
                    }
                }
                finish(t, re, im);
            }
        }
        __syncthreads();
    }
    if (tid == 0) queue_exit(a.queue);
}

// ---------------------------------------------------------------- ADAPTIVE kernel (NEXT-4)
// CT-driven quadtree (include/p2p.h P2P_LAYOUT_ADAPTIVE; R25).  Persistent CTAs pull
// target leaves (most pairs first); per leaf the sources of its U-list leaves are staged into
// shared memory as (x, y, q) relative to the target leaf's origin -- exact integer cell offsets
// times the finest cell size plus the in-cell offset, rounded once -- and the leaf's targets
// (<= CT) sweep them, C = NT / n_t source chunks per target with a fixed-order reduction.
template <typename T, int NT>
__global__ void __launch_bounds__(NT) p2p_adaptive_kernel(const P2PArgs<T> a) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_leaf;
    const int sbytes = ((a.src_cap * 4 * (int)sizeof(T)) + 15) & ~15;
    T *s_p = reinterpret_cast<T *>(smem);
    int *s_st = reinterpret_cast<int *>(smem + sbytes);
    int *s_pre = s_st + kMaxUlist;
    T *s_part = reinterpret_cast<T *>(smem + sbytes + 8 * kMaxUlist + 16);  // 16-B aligned
    const int tid = threadIdx.x;
    using C2 = typename V2<T>::type;
    const C2 *suv = reinterpret_cast<const C2 *>(a.src_uv), *tuv = reinterpret_cast<const C2 *>(a.tgt_uv);
    const T hf = a.h;
    for (;;) {
        if (tid == 0) {
            const int e = atomicAdd(a.queue, 1);
            s_leaf = e < a.ntiles ? a.tiles[e] : -1;
        }
        __syncthreads();
        const int b = s_leaf;
        if (b < 0) break;
        const int u0 = a.ul_off[b], nu = a.ul_off[b + 1] - u0;
        const int2 org = a.leaf_org[b];
        if (tid < 32) {  // U-list source starts and prefix: lanes load 32 entries at a time, warp scan
            int run = 0;
            for (int k0 = 0; k0 < nu; k0 += 32) {
                const int k = k0 + tid;
                int st = 0, cnt = 0;
                if (k < nu) {
                    const int4 r = a.leaf_rng[a.ul_leaf[u0 + k]];
                    st = r.x;
                    cnt = r.y - r.x;
                }
                int incl = cnt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, incl, o);
                    if (tid >= o) incl += v;
                }
                if (k < nu) {
                    s_st[k] = st;
                    s_pre[k] = run + incl - cnt;
                }
                run += __shfl_sync(0xffffffffu, incl, 31);
            }
            if (tid == 0) s_pre[nu] = run;
        }
        __syncthreads();
        const int total = s_pre[nu];
        for (int i = tid; i < total; i += NT) {  // stage (x, y, q) relative to the leaf origin
            int k = 0;
#pragma unroll
            for (int step = 128; step; step >>= 1)
                if (k + step < nu && s_pre[k + step] <= i) k += step;
            const int j = s_st[k] + (i - s_pre[k]);
            const int2 cl = a.src_cell[j];
            const C2 o = suv[j];
            const T x = fma((T)(cl.x - org.x), hf, o.x), y = fma((T)(cl.y - org.y), hf, o.y);
            const T q = a.q[a.src_idx ? a.src_idx[j] : j];
            s_p[4 * i] = x;
            s_p[4 * i + 1] = y;
            s_p[4 * i + 2] = q;
        }
        __syncthreads();
        const int4 tr = a.leaf_rng[b];
        const int t0 = tr.z, nt = tr.w - tr.z;
        const int C = nt >= NT ? 1 : NT / nt;
        auto finish = [&](int t, T acc) {
            const int64_t o = a.out_idx ? a.out_idx[t0 + t] : t0 + t;
            const T v = sizeof(T) == 4 ? (T)(-0.5f * kLn2) * acc : (T)-0.5 * acc;
            a.out[o] = a.accumulate ? a.out[o] + v : v;
        };
        for (int it = tid; it < nt * C; it += NT) {
            const int t = it % nt, ch = it / nt;
            const int2 cl = a.tgt_cell[t0 + t];
            const C2 o = tuv[t0 + t];
            const T tx = fma((T)(cl.x - org.x), hf, o.x), ty = fma((T)(cl.y - org.y), hf, o.y);
            const int s0 = (int)((int64_t)total * ch / C), s1 = (int)((int64_t)total * (ch + 1) / C);
            T acc = (T)0;
            for (int s = s0; s < s1; ++s) {
                const T dx = tx - s_p[4 * s], dy = ty - s_p[4 * s + 1];
                const T r2 = fma(dy, dy, dx * dx);
                if (r2 < a.eps2) continue;  // coincident points contribute 0 (R3)
                if constexpr (sizeof(T) == 4) acc = fmaf(s_p[4 * s + 2], lg2_approx(r2), acc);
                else acc = fma(s_p[4 * s + 2], log(r2), acc);
            }
            if (C == 1) finish(t, acc);
            else s_part[it] = acc;
        }
        if (C > 1) {
            __syncthreads();
            for (int t = tid; t < nt; t += NT) {
                T acc = (T)0;
                for (int ch = 0; ch < C; ++ch) acc += s_part[ch * nt + t];
                finish(t, acc);
            }
        }
        __syncthreads();
    }
    if (tid == 0) queue_exit(a.queue);
}

// ADAPTIVE, one WARP per target leaf (small leaves, CT <= 64): each warp claims leaves from the
// queue on its own and stages into its own shared-memory slice, with __syncwarp between phases --
// NT / 32 leaves in flight per CTA instead of one, no CTA-wide barriers.
template <typename T, int NT>
__global__ void __launch_bounds__(NT) p2p_adaptive_warp_kernel(const P2PArgs<T> a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sbytes = align16(a.src_cap * 4 * (int)sizeof(T));
    unsigned char *base = smem + (size_t)warp * adaptive_warp_slice(a.src_cap, (int)sizeof(T));
    T *s_p = reinterpret_cast<T *>(base);
    int *s_st = reinterpret_cast<int *>(base + sbytes);
    int *s_pre = s_st + kMaxUlist;
    T *s_part = reinterpret_cast<T *>(base + sbytes + 8 * kMaxUlist + 16);
    using C2 = typename V2<T>::type;
    const C2 *suv = reinterpret_cast<const C2 *>(a.src_uv), *tuv = reinterpret_cast<const C2 *>(a.tgt_uv);
    const T hf = a.h;
    for (;;) {
        int b = -1;
        if (lane == 0) {
            const int e = atomicAdd(a.queue, 1);
            b = e < a.ntiles ? a.tiles[e] : -1;
        }
        b = __shfl_sync(0xffffffffu, b, 0);
        if (b < 0) break;
        const int u0 = a.ul_off[b], nu = a.ul_off[b + 1] - u0;
        const int2 org = a.leaf_org[b];
        int run = 0;
        for (int k0 = 0; k0 < nu; k0 += 32) {  // U-list starts and prefix (warp scan)
            const int k = k0 + lane;
            int st = 0, cnt = 0;
            if (k < nu) {
                const int4 r = a.leaf_rng[a.ul_leaf[u0 + k]];
                st = r.x;
                cnt = r.y - r.x;
            }
            int incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            if (k < nu) {
                s_st[k] = st;
                s_pre[k] = run + incl - cnt;
            }
            run += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) s_pre[nu] = run;
        __syncwarp();
        const int total = run;
        for (int i = lane; i < total; i += 32) {
            int k = 0;
#pragma unroll
            for (int step = 128; step; step >>= 1)
                if (k + step < nu && s_pre[k + step] <= i) k += step;
            const int j = s_st[k] + (i - s_pre[k]);
            const int2 cl = a.src_cell[j];
            const C2 o = suv[j];
            s_p[4 * i] = fma((T)(cl.x - org.x), hf, o.x);
            s_p[4 * i + 1] = fma((T)(cl.y - org.y), hf, o.y);
            s_p[4 * i + 2] = a.q[a.src_idx ? a.src_idx[j] : j];
        }
        __syncwarp();
        const int4 tr = a.leaf_rng[b];
        const int t0 = tr.z, nt = tr.w - tr.z;
        const int C = nt >= 32 ? 1 : 32 / nt;
        auto finish = [&](int t, T acc) {
            const int64_t o = a.out_idx ? a.out_idx[t0 + t] : t0 + t;
            const T v = sizeof(T) == 4 ? (T)(-0.5f * kLn2) * acc : (T)-0.5 * acc;
            a.out[o] = a.accumulate ? a.out[o] + v : v;
        };
        for (int it = lane; it < nt * C; it += 32) {
            const int t = it % nt, ch = it / nt;
            const int2 cl = a.tgt_cell[t0 + t];
            const C2 o = tuv[t0 + t];
            const T tx = fma((T)(cl.x - org.x), hf, o.x), ty = fma((T)(cl.y - org.y), hf, o.y);
            const int s0 = (int)((int64_t)total * ch / C), s1 = (int)((int64_t)total * (ch + 1) / C);
            T acc = (T)0;
            for (int s = s0; s < s1; ++s) {
                const T dx = tx - s_p[4 * s], dy = ty - s_p[4 * s + 1];
                const T r2 = fma(dy, dy, dx * dx);
                if (r2 < a.eps2) continue;  // coincident points contribute 0 (R3)
                if constexpr (sizeof(T) == 4) acc = fmaf(s_p[4 * s + 2], lg2_approx(r2), acc);
                else acc = fma(s_p[4 * s + 2], log(r2), acc);
            }
            if (C == 1) finish(t, acc);
            else s_part[it] = acc;
        }
        if (C > 1) {
            __syncwarp();
            for (int t = lane; t < nt; t += 32) {
                T acc = (T)0;
                for (int ch = 0; ch < C; ++ch) acc += s_part[ch * nt + t];
                finish(t, acc);
            }
        }
        __syncwarp();
    }
    __syncthreads();
    if (threadIdx.x == 0) queue_exit(a.queue);
}

// ---------------------------------------------------------------- the paper's kernels (NEXT-1)
// Reproduced as the paper describes them, global memory only ("none of ... pre-fetching,
// exploiting Shared Memory ... were employed"), fp64, the library log.
//   Indexing (§3.2): "A GPU thread is assigned to a single box" -- it walks the
//   box's target index list and, per target, the box's E1 source index list.
//   Repetition (§3.3): one thread per target reads its own fixed-stride record
//   [x_t, y_t, count, (x_s, y_s, q_s) ...].
__global__ void paper_indexing_kernel(int64_t nbox, const int32_t *__restrict__ tgt_off,
                                      const int32_t *__restrict__ tgt_idx, const int32_t *__restrict__ nei_off,
                                      const int32_t *__restrict__ nei_idx, const double2 *__restrict__ src_xy,
                                      const double2 *__restrict__ tgt_xy, const double *__restrict__ q,
                                      double *__restrict__ out, double eps2, int accumulate) {
    const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= nbox) return;
    for (int32_t i = tgt_off[b]; i < tgt_off[b + 1]; ++i) {
        const int32_t t = tgt_idx[i];
        const double2 pt = tgt_xy[t];
        double acc = 0.0;
        for (int32_t e = nei_off[b]; e < nei_off[b + 1]; ++e) {
            const int32_t sidx = nei_idx[e];
            const double2 ps = src_xy[sidx];
            const double du = pt.x - ps.x, dv = pt.y - ps.y;
            const double r2 = fma(dv, dv, du * du);
            if (r2 >= eps2) acc = fma(q[sidx], log(r2), acc);
        }
        out[t] = accumulate ? out[t] - 0.5 * acc : -0.5 * acc;
    }
}

// The per-execution part of the Repetition collection: the weights into the records' q slots.
__global__ void paper_rep_pack_kernel(int64_t n_tgt, int64_t maxn, int64_t stride, const int32_t *__restrict__ slot,
                                      const double *__restrict__ q, double *__restrict__ records) {
    const int64_t n = n_tgt * maxn;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t sidx = slot[i];
        if (sidx >= 0) records[(i / maxn) * stride + 3 + 3 * (i % maxn) + 2] = q[sidx];
    }
}

__global__ void paper_repetition_kernel(int64_t n_tgt, int64_t stride, const double *__restrict__ records,
                                        double *__restrict__ out, double eps2, int accumulate) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n_tgt) return;
    const double *rec = records + r * stride;
    const double xt = rec[0], yt = rec[1];
    const int count = (int)(uint32_t)__double_as_longlong(rec[2]);  // integer in the slot's low 4 bytes
    double acc = 0.0;
    for (int k = 0; k < count; ++k) {
        const double du = xt - rec[3 + 3 * k], dv = yt - rec[4 + 3 * k];
        const double r2 = fma(dv, dv, du * du);
        if (r2 >= eps2) acc = fma(rec[5 + 3 * k], log(r2), acc);
    }
    out[r] = accumulate ? out[r] - 0.5 * acc : -0.5 * acc;
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
// Peer-memory halo (p2p_apply_dist_peer): q_local[lidx[h]] = peer[owner[h]][oidx[h]], the
// owners' buffers read directly (NVLink P2P loads on a multi-GPU node, CUDA IPC mappings).
template <typename T>
struct PeerPtrs {
    const T *p[16];
};
template <typename T>
__global__ void halo_peer_kernel(PeerPtrs<T> peers, const int32_t *__restrict__ owner, const int32_t *__restrict__ oidx,
                                 const int32_t *__restrict__ lidx, T *__restrict__ q_local, int64_t n) {
    for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < n; h += (int64_t)gridDim.x * blockDim.x)
        q_local[lidx[h]] = peers.p[owner[h]][oidx[h]];
}

// ---- device-synchronised peer exchange (p2p_apply_peer_sync / p2p_gather; include/p2p.h).
// Every rank owns a signal block in its own HBM, mapped by its peers (CUDA IPC; NVLink on a
// node): [kSigReady + x] the epoch up to which it has published buffer x (0 = halo weights,
// 1 = results), [kSigDone + x*16 + s] the epoch up to which reader s has finished reading it,
// [kSigCount + x] its own epoch counter.  An owner publishes epoch e only after every reader has
// finished e - 1; a reader reads only after the owner has published e.  Flags are written with
// st.release.sys after a system-scope fence and polled with ld.acquire.sys; the peers' data is
// read with ld.global.cv (never a stale L1 line).  No host synchronisation anywhere: the whole
// exchange is stream-ordered kernels (graph-capturable).  A wait longer than kPeerTimeoutNs
// sets the error word and gives up (a dead peer cannot hang the device).
constexpr int kSigReady = 0, kSigCount = 2, kSigDone = 4, kSigWords = 4 + 2 * 16;
constexpr unsigned long long kPeerTimeoutNs = 20ull * 1000 * 1000 * 1000;
struct SigPtrs {
    unsigned long long *p[16];
};
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void wait_epoch(const unsigned long long *flag, unsigned long long e, int *err) {
    const unsigned long long t0 = gtimer();
    while (ld_acquire_sys(flag) < e) {
        if (gtimer() - t0 > kPeerTimeoutNs) {
            atomicExch(err, 1);
            return;
        }
        __nanosleep(128);
    }
}
// Publish buffer x for epoch e = counter + 1: wait for the readers in `readers` (bit mask) to be
// done with e - 1, pub[i] = src[idx ? idx[i] : i], then (last CTA) counter = e and ready = e.
template <typename V>
__global__ void peer_publish_kernel(const int32_t *__restrict__ idx, const V *__restrict__ src, V *__restrict__ pub,
                                    int64_t n, unsigned long long *sig, int x, unsigned readers, unsigned *ctr,
                                    int *err) {
    const unsigned long long e = sig[kSigCount + x] + 1;  // stable: only this kernel's last CTA writes it
    if (threadIdx.x == 0)
        for (int s = 0; s < 16; ++s)
            if (readers >> s & 1u) wait_epoch(sig + kSigDone + 16 * x + s, e - 1, err);
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        pub[i] = src[idx ? idx[i] : i];
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        if (atomicAdd(ctr, 1u) == gridDim.x - 1) {
            *ctr = 0u;
            sig[kSigCount + x] = e;
            __threadfence_system();
            st_release_sys(sig + kSigReady + x, e);
        }
    }
}

// Read epoch e (= this rank's counter, already advanced by its publish kernel) of the owners in
// `owners`: dst[didx ? didx[h] : h] = pub[owner(h)][oidx(h)], where owner / oidx come from the
// arrays or, without them, from `nseg` contiguous segments (seg_begin[r] .. seg_begin[r + 1]
// read from rank r's buffer at offset h - seg_begin[r]); then (last CTA) done = e at every owner.
template <typename V>
__global__ void peer_pull_kernel(PeerPtrs<V> pub, SigPtrs sig, const unsigned long long *own_sig, int x, int me,
                                 unsigned owners, const int32_t *__restrict__ owner, const int32_t *__restrict__ oidx,
                                 const int64_t *__restrict__ seg_begin, int nseg, const int32_t *__restrict__ didx,
                                 V *__restrict__ dst, int64_t n, unsigned *ctr, int *err) {
    const unsigned long long e = own_sig[kSigCount + x];
    if (threadIdx.x == 0)
        for (int o = 0; o < 16; ++o)
            if (owners >> o & 1u) wait_epoch(sig.p[o] + kSigReady + x, e, err);
    __syncthreads();
    for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < n; h += (int64_t)gridDim.x * blockDim.x) {
        int o;
        int64_t j;
        if (owner) {
            o = owner[h];
            j = oidx[h];
        } else {
            o = 0;
            while (o + 1 < nseg && seg_begin[o + 1] <= h) ++o;
            j = h - seg_begin[o];
        }
        dst[didx ? didx[h] : h] = __ldcv(pub.p[o] + j);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        if (atomicAdd(ctr, 1u) == gridDim.x - 1) {
            *ctr = 0u;
            for (int o = 0; o < 16; ++o)
                if (owners >> o & 1u) st_release_sys(sig.p[o] + kSigDone + 16 * x + me, e);
        }
    }
}

template <typename T>
__global__ void gather_kernel(const int32_t *__restrict__ idx, const T *__restrict__ src, T *__restrict__ dst,
                              int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[idx[i]];
}

// out[idx[i]] = v[i] for any element type (complex weights of the distributed Helmholtz apply)
template <typename V>
__global__ void copy_scatter_kernel(const int32_t *__restrict__ idx, const V *__restrict__ v, V *__restrict__ out,
                                    int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[idx[i]] = v[i];
}

// dst[i] = i2 < n_owned ? owned[i2] : halo[i2 - n_owned], i2 = qidx[i]  (distributed import)
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
