"""The paper's own comparison on B200 (§4.3 Figs. 3-4, §4.6 Fig. 6).

For each problem: the Indexing kernel (one thread per box, the seven arrays) and the Repetition
kernel (one thread per target, 3 + 27 CT records) -- kernel alone, the Repetition apply with its
weight pack, and the paper's "total" = collection (host plan build) + transfer (upload) + one
apply -- next to this build's optimised NR / R / TILED fp64 applies.  N sweep: N = 1e3..1e6 at
CT = 15; grid: N = 4^L, CT = 15, leaf level = CT-loop level + i,
i in -3..3.  Uniform points on the unit square.

  python tools/paper_sweep.py --mode n --json profiles/r01_paper_nsweep.json
  python tools/paper_sweep.py --mode grid --json profiles/r01_paper_grid.json
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_01596_b200 import p2p  # noqa: E402
from paper_2403_01596_b200 import workloads as W  # noqa: E402

LIB = p2p.load_library()
LIB.p2p_internal_paper_kernel_only.argtypes = [C.c_void_p, C.c_int]
DEV = torch.device("cuda", 0)
FLUSH = torch.empty(256 << 20, dtype=torch.uint8, device=DEV)


def time_apply(pl, qd, out, reps):
    for _ in range(2):
        pl.apply(qd, out, order="user")
    ts = []
    for _ in range(reps):
        FLUSH.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        pl.apply(qd, out, order="user")
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def run(src, tgt, q, level, ct, reps):
    row = {"n": len(src), "level": level}
    qd = torch.as_tensor(q, dtype=torch.float64, device=DEV)
    out = torch.empty(len(tgt), dtype=torch.float64, device=DEV)
    for lay in ("paper_i", "paper_r", "nr", "r", "tiled"):
        try:
            t0 = time.perf_counter()
            pl = p2p.Plan(src, tgt, level=level, layout=lay, precision="fp64", ct=ct, device=0)
            create_s = time.perf_counter() - t0
        except p2p.P2PError as e:
            row[lay] = {"unavailable": str(e).split(":")[-1].strip()[:120]}
            continue
        i = pl.info
        ms = time_apply(pl, qd, out, reps)
        ent = {"apply_ms": ms, "collect_s": i["build_seconds"], "transfer_s": i["upload_seconds"],
               "create_s": create_s, "pairs": i["pairs"], "Gpair_s": i["pairs"] / (ms * 1e-3) / 1e9,
               "device_MB": i["device_bytes"] / 1e6}
        if lay.startswith("paper"):
            ent["model_bytes"] = i["paper_model_bytes"]
            ent["total_ms"] = (i["build_seconds"] + i["upload_seconds"]) * 1e3 + ms
        if lay == "paper_r":
            LIB.p2p_internal_paper_kernel_only(pl.handle, 1)
            ent["kernel_ms"] = time_apply(pl, qd, out, reps)
            LIB.p2p_internal_paper_kernel_only(pl.handle, 0)
            ent["stride"] = i["record_stride"]
        elif lay == "paper_i":
            ent["kernel_ms"] = ms
        row["t_max"] = i["t_max"]
        row[lay] = ent
        pl.close()
    pi, pr = row.get("paper_i", {}), row.get("paper_r", {})
    if "kernel_ms" in pi and "kernel_ms" in pr:
        row["R_over_I_kernel_speedup"] = pi["kernel_ms"] / pr["kernel_ms"]
        row["R_over_I_total_speedup"] = pi["total_ms"] / pr["total_ms"]
    return row


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", choices=["n", "grid"], default="n")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--json", default="")
    args = ap.parse_args()
    rows = []
    if args.mode == "n":
        for n in (1000, 10000, 100000, 1000000):
            src, tgt, q = W.uniform_unit(n, 20240303)
            with p2p.Plan(src, tgt, level=0, ct=15, device=-1) as h:
                L = h.info["level"]
            rows.append(run(src, tgt, q, L, 15, args.reps))
            print(json.dumps(rows[-1])[:400], flush=True)
    else:
        for L in range(4, 10):
            n = 4 ** L
            src, tgt, q = W.uniform_unit(n, 20240303)
            with p2p.Plan(src, tgt, level=0, ct=15, device=-1) as h:
                L0 = h.info["level"]
            for i in range(-3, 4):
                if L0 + i < 1 or L0 + i > 15:
                    continue
                r = run(src, tgt, q, L0 + i, 15, args.reps)
                r.update(L=L, i=i)
                rows.append(r)
                print(json.dumps({k: r[k] for k in ("L", "i", "n", "level", "t_max") if k in r}),
                      {k: round(v, 3) for k, v in r.items() if k.startswith("R_over")}, flush=True)
    if args.json:
        json.dump(rows, open(args.json, "w"), indent=1)


if __name__ == "__main__":
    main()
