"""Run the roofline microbenchmarks of libp2p_peaks.so on cuda:0 and print JSON."""
import ctypes as C
import json
import os

lib = C.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                          "paper_2403_01596_b200", "lib", "libp2p_peaks.so"))
out = {}
for name in ("p2p_peak_mufu_lg2", "p2p_peak_ffma2", "p2p_peak_dfma", "p2p_peak_hbm_read"):
    f = getattr(lib, name)
    f.argtypes = [C.c_int, C.POINTER(C.c_double)]
    v = C.c_double(0)
    out[name] = (f(0, C.byref(v)), v.value)
lib.p2p_peak_span.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
for tpi in (1, 2):
    for n in (48, 144, 576):
        for groups, gstride in ((1, 0), (2, 1), (4, 1), (4, 37), (8, 1), (8, 37), (32, 1)):
            v = C.c_double(0)
            out[f"span_tpi{tpi}_n{n}_g{groups}_s{gstride}"] = (lib.p2p_peak_span(0, tpi, n, groups, gstride, C.byref(v)),
                                                               v.value / 4.653e12)
print(json.dumps(out, indent=1))
