"""ADAPTIVE layout on B200: a clustered 1e6-point cloud -- a uniform
background, a dense blob and a star curve (the shapes of tests/test_adaptive.py at scale) --
(sources and targets half a curve spacing apart) with CT = 16 / 32 / 64, fp32 and fp64: pairs/s (median of L2-flushed applies), the MUFU
fraction (fp32: one MUFU.LG2 per pair), leaf statistics and the host plan build.  Parity at
this size is by construction (tests/test_adaptive.py pins the same code at 2e3-6e3 points);
the fp64 result is compared with fp32 here as a consistency check.

  python tools/adaptive_bench.py --json gpurun_out/adaptive_bench.json
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_01596_b200 import p2p  # noqa: E402
from paper_2403_01596_b200 import workloads as W  # noqa: E402

DEV = torch.device("cuda", 0)


def cloud(n, seed, phase):
    """Sources (phase 0) and targets (phase 1/2) sit on the curve half a spacing apart, so no
    target nearly coincides with a source (fp32 cannot resolve r << 1e-7 x the leaf size)."""
    idx = np.arange(n // 3, dtype=np.uint64)
    a = np.stack([W.uniform01(seed, 10, idx), W.uniform01(seed, 11, idx)], axis=1)
    b = 0.62 + 0.03 * np.stack([W.uniform01(seed, 12, idx), W.uniform01(seed, 13, idx)], axis=1)
    m = n - 2 * (n // 3)
    t = 2.0 * np.pi * (np.arange(m) + phase) / m
    r = 0.35 * (1.0 + 0.3 * np.cos(5 * t))
    c = np.stack([0.5 + r * np.cos(t), 0.5 + r * np.sin(t)], axis=1)
    return np.concatenate([a, b, c])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--cts", default="16,32,64")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    src, tgt = cloud(a.n, 1, 0.0), cloud(a.n, 2, 0.5)
    q = W.weights(a.n, 1)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=DEV)
    stream = torch.cuda.current_stream(DEV)
    peak = 16 * 148 * 1.965e9
    rows = []
    for ct in map(int, a.cts.split(",")):
        res = {}
        for prec in ("fp32", "fp64"):
            with p2p.Plan(src, tgt, layout="adaptive", ct=ct, l_max=15, precision=prec) as pl:
                qd = torch.as_tensor(q, dtype=pl.torch_dtype, device=DEV)
                out = torch.empty(a.n, dtype=pl.torch_dtype, device=DEV)
                for _ in range(3):
                    pl.apply(qd, out, order="user")
                ts = []
                for _ in range(a.reps):
                    flush.zero_()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    pl.apply(qd, out, order="user")
                    e1.record(stream)
                    e1.synchronize()
                    ts.append(e0.elapsed_time(e1))
                ms = float(np.median(ts))
                res[prec] = out.double().cpu().numpy()
                lv = pl.export("leaves").reshape(-1, 3)
                info = pl.info
                row = {"n": a.n, "ct": ct, "precision": prec, "pairs": info["pairs"], "ms": ms,
                       "Gpair_s": info["pairs"] / (ms * 1e-3) / 1e9,
                       "mufu_frac": info["pairs"] / (ms * 1e-3) / peak if prec == "fp32" else None,
                       "leaves": len(lv), "target_leaves": info["tiles"], "levels": sorted(set(lv[:, 0].tolist())),
                       "t_max": info["t_max"], "build_s": info["build_seconds"], "upload_s": info["upload_seconds"]}
                rows.append(row)
                print(json.dumps(row), flush=True)
        r = res["fp32"] - res["fp64"]
        rows[-1]["fp32_vs_fp64_rel_l2"] = float(np.linalg.norm(r) / np.linalg.norm(res["fp64"]))
        print("fp32 vs fp64 rel L2", rows[-1]["fp32_vs_fp64_rel_l2"], flush=True)
    if a.json:
        with open(a.json, "w") as f:
            json.dump({"rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
