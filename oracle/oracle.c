/*
 * oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for the MLFMA
 * near-field P2P operator of arXiv 2403.01596.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2403_01596_b200/) never links, imports or calls it,
 * and shares no code, header, table or helper with it.
 *
 * What it computes (§4.1, the CPU
 * baseline: "for each target point in a box ... for each source point in the
 * E_1 neighborhood, the potential function is executed once and its value is
 * added"):
 *
 *   phi_t = sum_{s : |ix_s-ix_t|<=1 and |iy_s-iy_t|<=1 and r_ts >= eps}  q_s * ln(1/r_ts)
 *
 * with the leaf grid S = 2^(L-1) per side ("4^{L-1}" boxes,
 * root = level 1), box(p) = (min(floor(x*S), S-1), min(floor(y*S), S-1))
 * (half-open cells closed at the upper edge), the kernel
 * G = q ln(1/r), 0 when r < eps ("electrical
 * potential function on a two-dimensional PEC"), E1 = the 3x3 block of boxes
 * clipped at the domain edge ("The number 9 above refers to the
 * number of adjacent neighboring boxes").  ln(1/r) is evaluated as
 * -0.5*log(r^2) with the C library log (<= 1 ulp).
 *
 * Pins: see tests/test_oracle_pins.py (closed-form lattice, SPEC worked
 * values, brute force, reciprocity, linearity, permutation, pair-count closed
 * form, SPEC geometry examples).
 */
#define _DEFAULT_SOURCE /* j0 / y0 (XSI Bessel functions of glibc's libm) under -std=c11 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---- geometry: PAPER.md §3.1 L67 ("division factor of 4"), SPEC.md L120 ---- */

static int64_t grid_side(int L) { return (int64_t)1 << (L - 1); }

static int64_t cell_of(double x, int64_t S)
{
    /* floor(x*S) is exact in fp64 because S is a power of two. */
    int64_t c = (int64_t)floor(x * (double)S);
    if (c > S - 1) c = S - 1; /* closed at x = 1 */
    if (c < 0) c = 0;
    return c;
}

/* Sources bucketed into an S x S array of lists, each list in original index
 * order ("per-box insertion order").  Plain counting: count,
 * prefix, fill.  Caller frees *start and *items. */
static int bucket_sources(int64_t ns, const double *src_xy, int64_t S,
                          int64_t **start_out, int64_t **items_out)
{
    int64_t cells = S * S;
    int64_t *start = (int64_t *)calloc((size_t)(cells + 1), sizeof(int64_t));
    int64_t *items = (int64_t *)malloc((size_t)(ns > 0 ? ns : 1) * sizeof(int64_t));
    int64_t *fill = (int64_t *)malloc((size_t)(cells > 0 ? cells : 1) * sizeof(int64_t));
    if (!start || !items || !fill) { free(start); free(items); free(fill); return -1; }
    for (int64_t s = 0; s < ns; ++s) {
        int64_t c = cell_of(src_xy[2 * s + 1], S) * S + cell_of(src_xy[2 * s], S);
        start[c + 1] += 1;
    }
    for (int64_t c = 0; c < cells; ++c) start[c + 1] += start[c];
    memcpy(fill, start, (size_t)cells * sizeof(int64_t));
    for (int64_t s = 0; s < ns; ++s) {
        int64_t c = cell_of(src_xy[2 * s + 1], S) * S + cell_of(src_xy[2 * s], S);
        items[fill[c]++] = s;
    }
    free(fill);
    *start_out = start;
    *items_out = items;
    return 0;
}

/* ---- C-2 step 3: the direct sum over the 3x3 neighbourhood ----------------
 * For each selected target (all if sel == NULL): loop over the 3x3 block of
 * cells around its cell (rows dy = -1..1, then columns dx = -1..1), over the
 * sources of each cell in original index order; skip r^2 < eps^2; otherwise
 * acc += q*log(r^2).  phi = -0.5*acc.  pairs_out (optional) receives the
 * number of (t, s) pairs visited, guarded pairs included.
 * Returns 0, or -1 on allocation failure. */
int oracle_direct(int64_t ns, const double *src_xy, const double *q,
                  int64_t nt, const double *tgt_xy, int L, double eps,
                  int64_t nsel, const int64_t *sel, double *phi_out,
                  int nthreads, int64_t *pairs_out)
{
    int64_t S = grid_side(L);
    int64_t *start = NULL, *items = NULL;
    if (bucket_sources(ns, src_xy, S, &start, &items)) return -1;
    int64_t count = sel ? nsel : nt;
    double eps2 = eps * eps;
    int64_t pairs = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : pairs)
    for (int64_t k = 0; k < count; ++k) {
        int64_t t = sel ? sel[k] : k;
        double xt = tgt_xy[2 * t], yt = tgt_xy[2 * t + 1];
        int64_t ix = cell_of(xt, S), iy = cell_of(yt, S);
        double acc = 0.0;
        for (int64_t dy = -1; dy <= 1; ++dy) {
            int64_t cy = iy + dy;
            if (cy < 0 || cy >= S) continue;
            for (int64_t dx = -1; dx <= 1; ++dx) {
                int64_t cx = ix + dx;
                if (cx < 0 || cx >= S) continue;
                int64_t c = cy * S + cx;
                for (int64_t j = start[c]; j < start[c + 1]; ++j) {
                    int64_t s = items[j];
                    double ddx = xt - src_xy[2 * s], ddy = yt - src_xy[2 * s + 1];
                    double r2 = ddx * ddx + ddy * ddy;
                    pairs += 1;
                    if (r2 < eps2) continue; /* 0 when r < epsilon */
                    acc += q[s] * log(r2);
                }
            }
        }
        phi_out[k] = -0.5 * acc;
    }
    free(start);
    free(items);
    if (pairs_out) *pairs_out = pairs;
    return 0;
}

/* ---- C-2 step 4: brute force, no buckets -----------------------------------
 * Every (t, s) pair, filtered by the 3x3 box-adjacency predicate. */
int oracle_bruteforce(int64_t ns, const double *src_xy, const double *q,
                      int64_t nt, const double *tgt_xy, int L, double eps,
                      double *phi_out, int64_t *pairs_out)
{
    int64_t S = grid_side(L);
    double eps2 = eps * eps;
    int64_t pairs = 0;
    for (int64_t t = 0; t < nt; ++t) {
        int64_t ixt = cell_of(tgt_xy[2 * t], S), iyt = cell_of(tgt_xy[2 * t + 1], S);
        double acc = 0.0;
        for (int64_t s = 0; s < ns; ++s) {
            int64_t ixs = cell_of(src_xy[2 * s], S), iys = cell_of(src_xy[2 * s + 1], S);
            if (llabs(ixs - ixt) > 1 || llabs(iys - iyt) > 1) continue;
            pairs += 1;
            double ddx = tgt_xy[2 * t] - src_xy[2 * s];
            double ddy = tgt_xy[2 * t + 1] - src_xy[2 * s + 1];
            double r2 = ddx * ddx + ddy * ddy;
            if (r2 < eps2) continue;
            acc += q[s] * log(r2);
        }
        phi_out[t] = -0.5 * acc;
    }
    if (pairs_out) *pairs_out = pairs;
    return 0;
}

/* ---- single pair: SPEC.md L150 pair_potential ------------------------------ */
double oracle_pair_potential(double xt, double yt, double xs, double ys, double q, double eps)
{
    double ddx = xt - xs, ddy = yt - ys;
    double r2 = ddx * ddx + ddy * ddy;
    if (r2 < eps * eps) return 0.0;
    return -0.5 * q * log(r2);
}

/* ---- C-2 step 5: plan-indexing oracle (bit-exact plan checks) --------------
 * Morton code by a bit loop: bit b of ix goes to bit 2b, bit b of iy to bit
 * 2b+1 ("x occupies even bit positions").  */
uint64_t oracle_morton(uint64_t ix, uint64_t iy, int L)
{
    uint64_t code = 0;
    for (int b = 0; b < L - 1; ++b) {
        code |= ((ix >> b) & 1u) << (2 * b);
        code |= ((iy >> b) & 1u) << (2 * b + 1);
    }
    return code;
}

void oracle_morton_decode(uint64_t code, int L, uint64_t *ix, uint64_t *iy)
{
    uint64_t x = 0, y = 0;
    for (int b = 0; b < L - 1; ++b) {
        x |= ((code >> (2 * b)) & 1u) << b;
        y |= ((code >> (2 * b + 1)) & 1u) << b;
    }
    *ix = x;
    *iy = y;
}

typedef struct { uint64_t code; int64_t idx; } keyed;

static int cmp_keyed(const void *a, const void *b)
{
    const keyed *x = (const keyed *)a, *y = (const keyed *)b;
    if (x->code != y->code) return x->code < y->code ? -1 : 1;
    if (x->idx != y->idx) return x->idx < y->idx ? -1 : 1;
    return 0;
}

/* Sort points by (Morton code, original index) -> perm[plan] = original index;
 * off[B+1] = CSR box offsets over all B = 4^(L-1) boxes in Morton order. */
int oracle_sort_points(int64_t n, const double *xy, int L, int64_t *perm, int64_t *off)
{
    int64_t S = grid_side(L), B = S * S;
    keyed *k = (keyed *)malloc((size_t)(n > 0 ? n : 1) * sizeof(keyed));
    if (!k) return -1;
    for (int64_t i = 0; i < n; ++i) {
        k[i].code = oracle_morton((uint64_t)cell_of(xy[2 * i], S), (uint64_t)cell_of(xy[2 * i + 1], S), L);
        k[i].idx = i;
    }
    qsort(k, (size_t)n, sizeof(keyed), cmp_keyed);
    for (int64_t b = 0; b <= B; ++b) off[b] = 0;
    for (int64_t i = 0; i < n; ++i) {
        perm[i] = k[i].idx;
        off[k[i].code + 1] += 1;
    }
    for (int64_t b = 0; b < B; ++b) off[b + 1] += off[b];
    free(k);
    return 0;
}

/* E1 neighbour list of every box, ascending Morton, -1 padded to 9
 * (SPEC.md L91-99 neighbors_e1). nb must hold 9*4^(L-1) entries. */
void oracle_neighbors(int L, int64_t *nb)
{
    int64_t S = grid_side(L), B = S * S;
    for (int64_t m = 0; m < B; ++m) {
        uint64_t ix, iy;
        oracle_morton_decode((uint64_t)m, L, &ix, &iy);
        int64_t list[9];
        int cnt = 0;
        for (int64_t dy = -1; dy <= 1; ++dy)
            for (int64_t dx = -1; dx <= 1; ++dx) {
                int64_t cx = (int64_t)ix + dx, cy = (int64_t)iy + dy;
                if (cx < 0 || cy < 0 || cx >= S || cy >= S) continue;
                list[cnt++] = (int64_t)oracle_morton((uint64_t)cx, (uint64_t)cy, L);
            }
        for (int i = 1; i < cnt; ++i) /* insertion sort, ascending Morton */
            for (int j = i; j > 0 && list[j - 1] > list[j]; --j) {
                int64_t tmp = list[j]; list[j] = list[j - 1]; list[j - 1] = tmp;
            }
        for (int i = 0; i < 9; ++i) nb[9 * m + i] = i < cnt ? list[i] : -1;
    }
}

/* ---- PAPER.md §3.1 L67-69 tree-construction loop ----------
 * Start at l_start; while some leaf box holds more than ct sources or ct
 * targets, L += 1.  Returns L, or -1 if l_max is exceeded. */
int oracle_ct_level(int64_t ns, const double *src_xy, int64_t nt, const double *tgt_xy,
                    int ct, int l_start, int l_max)
{
    for (int L = l_start; L <= l_max; ++L) {
        int64_t S = grid_side(L), B = S * S;
        int32_t *cs = (int32_t *)calloc((size_t)B, sizeof(int32_t));
        int32_t *ctg = (int32_t *)calloc((size_t)B, sizeof(int32_t));
        if (!cs || !ctg) { free(cs); free(ctg); return -2; }
        int ok = 1;
        for (int64_t i = 0; i < ns && ok; ++i)
            if (++cs[cell_of(src_xy[2 * i + 1], S) * S + cell_of(src_xy[2 * i], S)] > ct) ok = 0;
        for (int64_t i = 0; i < nt && ok; ++i)
            if (++ctg[cell_of(tgt_xy[2 * i + 1], S) * S + cell_of(tgt_xy[2 * i], S)] > ct) ok = 0;
        free(cs);
        free(ctg);
        if (ok) return L;
    }
    return -1;
}

/* Number of (t, s) pairs with box(s) in E1(box(t)) -- the pair-interaction
 * count the metric divides by. */
int64_t oracle_pair_count(int64_t ns, const double *src_xy, int64_t nt, const double *tgt_xy, int L)
{
    int64_t S = grid_side(L);
    int64_t *start = NULL, *items = NULL;
    if (bucket_sources(ns, src_xy, S, &start, &items)) return -1;
    int64_t pairs = 0;
    for (int64_t t = 0; t < nt; ++t) {
        int64_t ix = cell_of(tgt_xy[2 * t], S), iy = cell_of(tgt_xy[2 * t + 1], S);
        for (int64_t cy = iy - 1; cy <= iy + 1; ++cy)
            for (int64_t cx = ix - 1; cx <= ix + 1; ++cx)
                if (cx >= 0 && cy >= 0 && cx < S && cy < S)
                    pairs += start[cy * S + cx + 1] - start[cy * S + cx];
    }
    free(start);
    free(items);
    return pairs;
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---- the paper's layout byte accounting ----------
 * Eq. 3 (§3.2): Memory_indexing = 5N Double + 4^(L-1)(2 + t + 9t)
 * Integer = 40N + 4^L (2 + 10t) bytes (Double = 8 B, Integer = 4 B, L97).
 * Eq. 8 (§3.3): Memory_Repetition = N(3 + 27 CT) Double
 * = 8N(3 + 27 CT) bytes.  t = the maximum number of points in a leaf box
 * ("maximum points in the boxes after applying CT"). */
int64_t oracle_indexing_bytes(int64_t n, int L, int64_t t)
{
    int64_t four_L = 1;
    for (int i = 0; i < L; ++i) four_L *= 4;
    return 40 * n + four_L * (2 + 10 * t);
}

int64_t oracle_repetition_bytes(int64_t n, int64_t ct)
{
    return 8 * n * (3 + 27 * ct);
}

/* t of Eq. 3-5: max over leaf boxes of max(#sources, #targets) in the box. */
int64_t oracle_box_tmax(int64_t ns, const double *src_xy, int64_t nt, const double *tgt_xy, int L)
{
    const int64_t S = grid_side(L);
    int64_t *cs = calloc((size_t)(S * S), sizeof(int64_t));
    int64_t *ctg = calloc((size_t)(S * S), sizeof(int64_t));
    int64_t t = 0;
    if (!cs || !ctg) {
        free(cs);
        free(ctg);
        return -1;
    }
    for (int64_t i = 0; i < ns; ++i)
        cs[cell_of(src_xy[2 * i + 1], S) * S + cell_of(src_xy[2 * i], S)] += 1;
    for (int64_t i = 0; i < nt; ++i)
        ctg[cell_of(tgt_xy[2 * i + 1], S) * S + cell_of(tgt_xy[2 * i], S)] += 1;
    for (int64_t b = 0; b < S * S; ++b) {
        if (cs[b] > t) t = cs[b];
        if (ctg[b] > t) t = ctg[b];
    }
    free(cs);
    free(ctg);
    return t;
}

/* ---- NEXT-3: the 2D Helmholtz kernel -------------------------------
 * Outside the paper's own (electrostatic) kernel -- SPEC.md L176 lists oscillatory kernels as a
 * non-goal of its CPU program -- but the workloads the paper motivates its redundancy with are
 * the "high-frequency" MLFMA problems (refs [2], [3] at L390-391).  The 2D
 * Helmholtz free-space Green's function (the textbook fundamental solution of
 * (Delta + kappa^2) G = -delta):
 *
 *     G(r) = (i/4) H0^(1)(kappa r) = (i/4) (J0(kappa r) + i Y0(kappa r)) = (-Y0(kappa r) + i J0(kappa r)) / 4
 *
 *     phi_t = sum_{s : box(s) in E1(box(t)), r_ts >= eps} q_s G(r_ts),   q_s, phi_t complex
 *
 * with the same leaf grid, E1 and guard as the Laplace oracle above (R23).  J0 and Y0
 * are the C library's j0 / y0 (glibc, double).  q and phi are interleaved (re, im) pairs.
 * (a + ib)(-Y + iJ)/4 = (-aY - bJ)/4 + i (aJ - bY)/4. */
static void helmholtz_pair(double r2, double kappa, double qr, double qi, double *re, double *im)
{
    double x = kappa * sqrt(r2);
    double J = j0(x), Y = y0(x);
    *re += 0.25 * (-qr * Y - qi * J);
    *im += 0.25 * (qr * J - qi * Y);
}

int oracle_direct_helmholtz(int64_t ns, const double *src_xy, const double *q,
                            int64_t nt, const double *tgt_xy, int L, double eps, double kappa,
                            int64_t nsel, const int64_t *sel, double *phi_out,
                            int nthreads, int64_t *pairs_out)
{
    int64_t S = grid_side(L);
    int64_t *start = NULL, *items = NULL;
    if (bucket_sources(ns, src_xy, S, &start, &items)) return -1;
    int64_t count = sel ? nsel : nt;
    double eps2 = eps * eps;
    int64_t pairs = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : pairs)
    for (int64_t k = 0; k < count; ++k) {
        int64_t t = sel ? sel[k] : k;
        double xt = tgt_xy[2 * t], yt = tgt_xy[2 * t + 1];
        int64_t ix = cell_of(xt, S), iy = cell_of(yt, S);
        double re = 0.0, im = 0.0;
        for (int64_t dy = -1; dy <= 1; ++dy) {
            int64_t cy = iy + dy;
            if (cy < 0 || cy >= S) continue;
            for (int64_t dx = -1; dx <= 1; ++dx) {
                int64_t cx = ix + dx;
                if (cx < 0 || cx >= S) continue;
                int64_t c = cy * S + cx;
                for (int64_t j = start[c]; j < start[c + 1]; ++j) {
                    int64_t s = items[j];
                    double ddx = xt - src_xy[2 * s], ddy = yt - src_xy[2 * s + 1];
                    double r2 = ddx * ddx + ddy * ddy;
                    pairs += 1;
                    if (r2 < eps2) continue; /* coincident points contribute 0 (R3) */
                    helmholtz_pair(r2, kappa, q[2 * s], q[2 * s + 1], &re, &im);
                }
            }
        }
        phi_out[2 * k] = re;
        phi_out[2 * k + 1] = im;
    }
    free(start);
    free(items);
    if (pairs_out) *pairs_out = pairs;
    return 0;
}

/* Brute force (no buckets): every (t, s) pair filtered by the 3x3 adjacency predicate. */
int oracle_bruteforce_helmholtz(int64_t ns, const double *src_xy, const double *q,
                                int64_t nt, const double *tgt_xy, int L, double eps, double kappa,
                                double *phi_out, int64_t *pairs_out)
{
    int64_t S = grid_side(L);
    double eps2 = eps * eps;
    int64_t pairs = 0;
    for (int64_t t = 0; t < nt; ++t) {
        int64_t ixt = cell_of(tgt_xy[2 * t], S), iyt = cell_of(tgt_xy[2 * t + 1], S);
        double re = 0.0, im = 0.0;
        for (int64_t s = 0; s < ns; ++s) {
            int64_t ixs = cell_of(src_xy[2 * s], S), iys = cell_of(src_xy[2 * s + 1], S);
            if (llabs(ixs - ixt) > 1 || llabs(iys - iyt) > 1) continue;
            pairs += 1;
            double ddx = tgt_xy[2 * t] - src_xy[2 * s];
            double ddy = tgt_xy[2 * t + 1] - src_xy[2 * s + 1];
            double r2 = ddx * ddx + ddy * ddy;
            if (r2 < eps2) continue;
            helmholtz_pair(r2, kappa, q[2 * s], q[2 * s + 1], &re, &im);
        }
        phi_out[2 * t] = re;
        phi_out[2 * t + 1] = im;
    }
    if (pairs_out) *pairs_out = pairs;
    return 0;
}

/* One pair: out[0] + i out[1] = q G(r), q = qr + i qi; 0 when r < eps. */
void oracle_pair_helmholtz(double xt, double yt, double xs, double ys, double qr, double qi,
                           double eps, double kappa, double *out)
{
    double ddx = xt - xs, ddy = yt - ys;
    double r2 = ddx * ddx + ddy * ddy;
    out[0] = 0.0;
    out[1] = 0.0;
    if (r2 < eps * eps) return;
    helmholtz_pair(r2, kappa, qr, qi, &out[0], &out[1]);
}

/* ---- NEXT-3: the 3D kernels on an octree leaf grid (R24) ---
 * The 3D analogue of the paper's operator (the "4x4x4 leaf boxes" reading of BASELINE.json's
 * tiny config, and the 3D EM workloads of the prior art): leaf grid S = 2^(L-1)
 * per side on the unit cube, box(p) = (cell(x), cell(y), cell(z)) as in 2D, E1 =
 * the 3x3x3 block of boxes clipped at the domain edge (27 in the interior), and
 *   LAPLACE_3D:   G(r) = 1 / (4 pi r)                 (real q, phi)
 *   HELMHOLTZ_3D: G(r) = exp(i kappa r) / (4 pi r)     (complex q, phi; the outgoing free-space
 *                                                       Green's function of Delta + kappa^2)
 * with the same guard (r < eps contributes 0).  Points are [n][3]; complex values (re, im). */
static void kernel3(double r2, int helm, double kappa, const double *q, double *acc)
{
    double r = sqrt(r2);
    double g = 1.0 / (4.0 * M_PI * r);
    if (!helm) {
        acc[0] += q[0] * g;
        return;
    }
    double c = cos(kappa * r) * g, s = sin(kappa * r) * g; /* G = (c + i s) */
    acc[0] += q[0] * c - q[1] * s;
    acc[1] += q[0] * s + q[1] * c;
}

int oracle_direct_3d(int64_t ns, const double *src, const double *q, int64_t nt, const double *tgt,
                     int L, double eps, int helm, double kappa, int64_t nsel, const int64_t *sel,
                     double *phi_out, int nthreads, int64_t *pairs_out)
{
    int64_t S = grid_side(L), cells = S * S * S;
    int64_t *start = (int64_t *)calloc((size_t)(cells + 1), sizeof(int64_t));
    int64_t *items = (int64_t *)malloc((size_t)(ns > 0 ? ns : 1) * sizeof(int64_t));
    int64_t *fill = (int64_t *)malloc((size_t)cells * sizeof(int64_t));
    if (!start || !items || !fill) { free(start); free(items); free(fill); return -1; }
    for (int64_t s = 0; s < ns; ++s) {  /* bucket the sources, original index order per cell */
        int64_t c = (cell_of(src[3 * s + 2], S) * S + cell_of(src[3 * s + 1], S)) * S + cell_of(src[3 * s], S);
        start[c + 1] += 1;
    }
    for (int64_t c = 0; c < cells; ++c) start[c + 1] += start[c];
    memcpy(fill, start, (size_t)cells * sizeof(int64_t));
    for (int64_t s = 0; s < ns; ++s) {
        int64_t c = (cell_of(src[3 * s + 2], S) * S + cell_of(src[3 * s + 1], S)) * S + cell_of(src[3 * s], S);
        items[fill[c]++] = s;
    }
    free(fill);
    int64_t count = sel ? nsel : nt, pairs = 0;
    int w = helm ? 2 : 1;
    double eps2 = eps * eps;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : pairs)
    for (int64_t k = 0; k < count; ++k) {
        int64_t t = sel ? sel[k] : k;
        double xt = tgt[3 * t], yt = tgt[3 * t + 1], zt = tgt[3 * t + 2];
        int64_t ix = cell_of(xt, S), iy = cell_of(yt, S), iz = cell_of(zt, S);
        double acc[2] = {0.0, 0.0};
        for (int64_t dz = -1; dz <= 1; ++dz)
            for (int64_t dy = -1; dy <= 1; ++dy)
                for (int64_t dx = -1; dx <= 1; ++dx) {
                    int64_t cx = ix + dx, cy = iy + dy, cz = iz + dz;
                    if (cx < 0 || cy < 0 || cz < 0 || cx >= S || cy >= S || cz >= S) continue;
                    int64_t c = (cz * S + cy) * S + cx;
                    for (int64_t j = start[c]; j < start[c + 1]; ++j) {
                        int64_t s = items[j];
                        double ddx = xt - src[3 * s], ddy = yt - src[3 * s + 1], ddz = zt - src[3 * s + 2];
                        double r2 = ddx * ddx + ddy * ddy + ddz * ddz;
                        pairs += 1;
                        if (r2 < eps2) continue;
                        kernel3(r2, helm, kappa, &q[w * s], acc);
                    }
                }
        for (int i = 0; i < w; ++i) phi_out[w * k + i] = acc[i];
    }
    free(start);
    free(items);
    if (pairs_out) *pairs_out = pairs;
    return 0;
}

/* Brute force: every (t, s) pair filtered by the 3x3x3 adjacency predicate. */
int oracle_bruteforce_3d(int64_t ns, const double *src, const double *q, int64_t nt, const double *tgt,
                         int L, double eps, int helm, double kappa, double *phi_out, int64_t *pairs_out)
{
    int64_t S = grid_side(L), pairs = 0;
    int w = helm ? 2 : 1;
    double eps2 = eps * eps;
    for (int64_t t = 0; t < nt; ++t) {
        double acc[2] = {0.0, 0.0};
        for (int64_t s = 0; s < ns; ++s) {
            int near = 1;
            for (int d = 0; d < 3; ++d)
                if (llabs(cell_of(src[3 * s + d], S) - cell_of(tgt[3 * t + d], S)) > 1) near = 0;
            if (!near) continue;
            pairs += 1;
            double ddx = tgt[3 * t] - src[3 * s], ddy = tgt[3 * t + 1] - src[3 * s + 1];
            double ddz = tgt[3 * t + 2] - src[3 * s + 2];
            double r2 = ddx * ddx + ddy * ddy + ddz * ddz;
            if (r2 < eps2) continue;
            kernel3(r2, helm, kappa, &q[w * s], acc);
        }
        for (int i = 0; i < w; ++i) phi_out[w * t + i] = acc[i];
    }
    if (pairs_out) *pairs_out = pairs;
    return 0;
}

/* ---- NEXT-4: CT-driven adaptive quadtree (R25) -------------
 * The tree construction of PAPER.md §3.1 L67-69 applied per box instead of globally: a box is
 * split into its 4 children while it holds more than CT sources or more than CT targets and its
 * level is below l_max; the leaves partition the unit square.  E1 generalises to the U-list: a
 * target in leaf A interacts with every source in a leaf B whose closed square touches A's
 * closed square (A itself included) -- on a uniform tree this is exactly the 3x3 block.
 * Everything below is brute force: counts by scanning all points, touching by comparing
 * closed intervals, the sum over all (t, s) pairs. */
typedef struct { int64_t level, ix, iy; } leaf_t;

static int in_box(double x, double y, int64_t L, int64_t ix, int64_t iy)
{
    int64_t S = grid_side((int)L);
    return cell_of(x, S) == ix && cell_of(y, S) == iy;
}

static void split_box(int64_t L, int64_t ix, int64_t iy, int64_t ns, const double *src, int64_t nt,
                      const double *tgt, int64_t ct, int64_t lmax, leaf_t *out, int64_t *n_out)
{
    int64_t a = 0, b = 0;
    for (int64_t s = 0; s < ns; ++s) a += in_box(src[2 * s], src[2 * s + 1], L, ix, iy);
    for (int64_t t = 0; t < nt; ++t) b += in_box(tgt[2 * t], tgt[2 * t + 1], L, ix, iy);
    if ((a > ct || b > ct) && L < lmax) {
        for (int c = 0; c < 4; ++c) /* children in Morton order: x bit first */
            split_box(L + 1, 2 * ix + (c & 1), 2 * iy + (c >> 1), ns, src, nt, tgt, ct, lmax, out, n_out);
        return;
    }
    out[*n_out].level = L;
    out[*n_out].ix = ix;
    out[*n_out].iy = iy;
    *n_out += 1;
}

/* Leaves of the tree in Morton (depth-first) order: leaves_out[3*i..] = (level, ix, iy); returns
 * the number of leaves (capacity cap; -1 if exceeded). */
int64_t oracle_adaptive_tree(int64_t ns, const double *src, int64_t nt, const double *tgt, int64_t ct,
                             int64_t lmax, int64_t *leaves_out, int64_t cap)
{
    int64_t bound = 1 + 3 * (ns + nt) * lmax + 4; /* leaves <= 1 + 3 * (internal nodes) */
    leaf_t *lv = (leaf_t *)malloc((size_t)bound * sizeof(leaf_t));
    if (!lv) return -1;
    int64_t n = 0;
    split_box(1, 0, 0, ns, src, nt, tgt, ct, lmax, lv, &n);
    if (n > cap) { free(lv); return -1; }
    for (int64_t i = 0; i < n; ++i) {
        leaves_out[3 * i] = lv[i].level;
        leaves_out[3 * i + 1] = lv[i].ix;
        leaves_out[3 * i + 2] = lv[i].iy;
    }
    free(lv);
    return n;
}

/* closed squares of two leaves touch (in units of the level-lmax grid) */
static int leaves_touch(const int64_t *A, const int64_t *B, int64_t lmax)
{
    int64_t sa = (int64_t)1 << (lmax - A[0]), sb = (int64_t)1 << (lmax - B[0]);
    int64_t ax0 = A[1] * sa, ax1 = ax0 + sa, ay0 = A[2] * sa, ay1 = ay0 + sa;
    int64_t bx0 = B[1] * sb, bx1 = bx0 + sb, by0 = B[2] * sb, by1 = by0 + sb;
    return ax0 <= bx1 && bx0 <= ax1 && ay0 <= by1 && by0 <= ay1;
}

static int64_t leaf_of(double x, double y, const int64_t *leaves, int64_t nl)
{
    for (int64_t i = 0; i < nl; ++i)
        if (in_box(x, y, leaves[3 * i], leaves[3 * i + 1], leaves[3 * i + 2])) return i;
    return -1;
}

/* phi_t = sum over sources in leaves touching t's leaf (r >= eps) of -1/2 q ln r^2. */
int oracle_adaptive_direct(int64_t ns, const double *src, const double *q, int64_t nt, const double *tgt,
                           int64_t ct, int64_t lmax, double eps, double *phi_out, int64_t *pairs_out)
{
    int64_t cap = 1 + 3 * (ns + nt) * lmax + 4;
    int64_t *leaves = (int64_t *)malloc((size_t)(3 * cap) * sizeof(int64_t));
    int64_t *ls = (int64_t *)malloc((size_t)(ns > 0 ? ns : 1) * sizeof(int64_t));
    if (!leaves || !ls) { free(leaves); free(ls); return -1; }
    int64_t nl = oracle_adaptive_tree(ns, src, nt, tgt, ct, lmax, leaves, cap);
    if (nl < 0) { free(leaves); free(ls); return -1; }
    for (int64_t s = 0; s < ns; ++s) ls[s] = leaf_of(src[2 * s], src[2 * s + 1], leaves, nl);
    double eps2 = eps * eps;
    int64_t pairs = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : pairs)
    for (int64_t t = 0; t < nt; ++t) {
        int64_t lt = leaf_of(tgt[2 * t], tgt[2 * t + 1], leaves, nl);
        double acc = 0.0;
        for (int64_t s = 0; s < ns; ++s) {
            if (!leaves_touch(&leaves[3 * lt], &leaves[3 * ls[s]], lmax)) continue;
            pairs += 1;
            double ddx = tgt[2 * t] - src[2 * s], ddy = tgt[2 * t + 1] - src[2 * s + 1];
            double r2 = ddx * ddx + ddy * ddy;
            if (r2 < eps2) continue;
            acc += q[s] * log(r2);
        }
        phi_out[t] = -0.5 * acc;
    }
    free(leaves);
    free(ls);
    if (pairs_out) *pairs_out = pairs;
    return 0;
}
