/*
 * p2p_peaks.h -- roofline-denominator microbenchmarks for the P2P operator
 * (SURVEY.md §7 step 0).  Separate library (libp2p_peaks.so); not part of the
 * P2P operator's ABI.  Each call runs on `device` (host-synchronous), times
 * its kernel with CUDA events after one warm-up, and returns 0 on success
 * (non-zero: a CUDA call failed).  Outputs are whole-device rates.
 */
#ifndef P2P_PEAKS_H
#define P2P_PEAKS_H
#ifdef __cplusplus
extern "C" {
#endif

typedef int p2p_peak_status;

/* MUFU lg2.approx.ftz.f32 results per second (8 independent chains per thread). */
p2p_peak_status p2p_peak_mufu_lg2(int device, double *ops_per_s);
/* Packed fp32 fma.rn.f32x2 FLOP/s (2 lanes x 2 flops per instruction). */
p2p_peak_status p2p_peak_ffma2(int device, double *flops);
/* fp64 FMA FLOP/s. */
p2p_peak_status p2p_peak_dfma(int device, double *flops);
/* The P2P fp32 inner loop alone (tpi = 1 or 2 targets per thread, nsrc
 * sources resident in shared memory): pair-interactions per second.  The
 * lanes of a warp form `groups` groups reading source pairs `gstride` apart
 * (groups = 1: every lane reads the same source, a broadcast). */
p2p_peak_status p2p_peak_span(int device, int tpi, int nsrc, int groups, int gstride, double *pairs_per_s);
/* Streaming read of a 2 GiB buffer (bytes/s). */
p2p_peak_status p2p_peak_hbm_read(int device, double *bytes_per_s);

#ifdef __cplusplus
}
#endif
#endif
