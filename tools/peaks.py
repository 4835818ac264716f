"""Run the roofline microbenchmarks of libp2p_peaks.so on cuda:0 and write JSON.

    python tools/peaks.py [--out profiles/r02_peaks.json] [--spans]

Each rate is measured with CUDA events (peaks.cu) while NVML samples the SM clock, so
the per-clock-per-SM figure (rate / (148 x median SM clock)) is reported beside the
whole-device rate; bench.py scales the per-clock figure by the clock of its own run.
"""
import argparse
import ctypes as C
import datetime
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SM_COUNT = 148


class Clocks:
    def __init__(self):
        import pynvml
        pynvml.nvmlInit()
        self.nv, self.h = pynvml, pynvml.nvmlDeviceGetHandleByIndex(0)
        self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        self.samples, self.reasons, self._stop = [], 0, threading.Event()

    def _run(self):
        while not self._stop.is_set():
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h) & ~0x1
            time.sleep(0.002)

    def __enter__(self):
        self.samples, self.reasons = [], 0
        self._stop.clear()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join()

    def median(self):
        s = sorted(self.samples)
        return float(s[len(s) // 2]) if s else float(self.max_mhz)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    ap.add_argument("--spans", action="store_true", help="also the inner-loop span sweep")
    a = ap.parse_args()
    lib = C.CDLL(os.path.join(ROOT, "paper_2403_01596_b200", "lib", "libp2p_peaks.so"))
    clk = Clocks()
    out = {"when": datetime.datetime.utcnow().isoformat() + "Z", "sm_count": SM_COUNT,
           "sm_max_mhz": clk.max_mhz, "how": "libp2p_peaks.so (paper_2403_01596_b200/csrc/peaks.cu): "
           "8 independent chains per thread, 256-thread CTAs, CUDA events after a warm-up; best of 5; "
           "NVML SM clock sampled during each run"}
    units = {"p2p_peak_mufu_lg2": ("lg2_per_s", "MUFU.LG2 results"),
             "p2p_peak_ffma2": ("flop_per_s", "fma.rn.f32x2: 4 FLOP per instruction"),
             "p2p_peak_dfma": ("flop_per_s", "DFMA: 2 FLOP per instruction"),
             "p2p_peak_hbm_read": ("bytes_per_s", "streaming read of 2 GiB")}
    for name, (unit, what) in units.items():
        f = getattr(lib, name)
        f.argtypes = [C.c_int, C.POINTER(C.c_double)]
        best, mhz, reasons = 0.0, None, 0
        for _ in range(5):
            v = C.c_double(0)
            with clk:
                st = f(0, C.byref(v))
            if st != 0:
                sys.exit(f"{name} failed: {st}")
            if v.value > best:
                best, mhz, reasons = v.value, clk.median(), clk.reasons
        rec = {"value": best, "unit": unit, "what": what, "sm_mhz_median": mhz, "throttle_reasons_mask": reasons}
        if unit != "bytes_per_s":
            rec["per_clk_per_sm"] = best / (SM_COUNT * mhz * 1e6)
            rec["at_sm_max"] = rec["per_clk_per_sm"] * SM_COUNT * clk.max_mhz * 1e6
        out[name.replace("p2p_peak_", "")] = rec
    if a.spans:
        lib.p2p_peak_span.argtypes = [C.c_int] * 5 + [C.POINTER(C.c_double)]
        spans = {}
        for tpi in (1, 2):
            for n in (48, 144, 576):
                for groups, gstride in ((1, 0), (4, 37), (32, 1)):
                    v = C.c_double(0)
                    lib.p2p_peak_span(0, tpi, n, groups, gstride, C.byref(v))
                    spans[f"tpi{tpi}_n{n}_g{groups}_s{gstride}"] = v.value
        out["span_pairs_per_s"] = spans
    txt = json.dumps(out, indent=1)
    print(txt)
    if a.out:
        os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
        with open(a.out, "w") as fh:
            fh.write(txt + "\n")


if __name__ == "__main__":
    main()
