"""Plan build on the host (p2p_plan_create) vs on the GPU (p2p_plan_create_device), SURVEY.md
§8(f) NEXT-2: the paper's "collection" step (§3.2, §3.3; alpha ~ 0.82 of its
total, L337-343) at the BASELINE.json sizes.

Per config and layout: host build (C++ builder on all host cores) + upload; the H2D copy of
the coordinates from pinned host memory; the device build from coordinates in HBM; and the
paper-style "total" = plan + one apply.  Device numbers are the median of `--reps` builds after one warm-up build (the first build in a process pays CUDA/CUB set-up).

  python tools/plan_build_bench.py --json gpurun_out/plan_build.json
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_01596_b200 import p2p  # noqa: E402
from paper_2403_01596_b200 import workloads as W  # noqa: E402

DEV = torch.device("cuda", 0)


def apply_ms(pl, q):
    qd = torch.as_tensor(q, dtype=pl.torch_dtype, device=DEV)
    out = torch.empty(pl.info["n_tgt"], dtype=pl.torch_dtype, device=DEV)
    torch.cuda.synchronize()
    t = time.perf_counter()
    pl.apply(qd, out, order="user")
    torch.cuda.synchronize()
    return (time.perf_counter() - t) * 1e3, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="d16_1e6,d64_1e6,lowd1_1e7,lowd025_1e7,surf_2e7,d32_7e7")
    ap.add_argument("--layouts", default="tiled,nr")
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    cores = len(os.sched_getaffinity(0))
    src, tgt, q = W.make_problem("tiny")
    p2p.Plan(src, tgt, level=4, layout="tiled", build="device").close()  # warm-up: CUDA context, CUB
    rows = []
    for name in a.configs.split(","):
        cfg = W.CONFIGS[name]
        src, tgt, q = W.make_problem(cfg)
        hs = torch.from_numpy(src).pin_memory()
        ht = torch.from_numpy(tgt).pin_memory()
        for layout in a.layouts.split(","):
            kw = dict(level=cfg.level, layout=layout, precision=a.precision)
            t = time.perf_counter()
            hp = p2p.Plan(src, tgt, **kw)
            host_wall = time.perf_counter() - t
            hinfo = dict(hp.info)
            h_apply, h_out = apply_ms(hp, q)
            h_out = h_out.cpu()
            hp.close()
            dev_build, dev_e2e, d_apply, h2d = [], [], [], []
            for _ in range(a.reps):
                torch.cuda.synchronize()
                t = time.perf_counter()
                ds = hs.to(DEV, non_blocking=True)
                dt = ht.to(DEV, non_blocking=True)
                torch.cuda.synchronize()
                h2d.append(time.perf_counter() - t)
                pl = p2p.Plan(ds, dt, build="device", **kw)
                e2e = time.perf_counter() - t
                dev_build.append(pl.info["build_seconds"])
                dev_e2e.append(e2e)
                ms, d_out = apply_ms(pl, q)
                d_apply.append(ms)
                same = bool(torch.equal(d_out.cpu(), h_out))
                pairs = pl.info["pairs"]
                pl.close()
                del ds, dt
            row = {
                "config": name, "layout": layout, "precision": a.precision, "n": cfg.n,
                "pairs": pairs, "tiles": hinfo["tiles"], "tile_log2": hinfo["tile_log2"],
                "host_build_s": hinfo["build_seconds"], "host_upload_s": hinfo["upload_seconds"],
                "host_plan_wall_s": host_wall, "host_cores": cores,
                "device_build_s": float(np.median(dev_build)), "device_build_min_s": float(np.min(dev_build)),
                "device_build_with_h2d_s": float(np.median(dev_e2e)), "h2d_coords_s": float(np.median(h2d)),
                "first_apply_ms_host_plan": h_apply, "first_apply_ms_device_plan": float(np.median(d_apply)),
                "speedup_build": (hinfo["build_seconds"] + hinfo["upload_seconds"]) / float(np.median(dev_e2e)),
                "results_bit_identical": same,
            }
            row["total_host_s"] = host_wall + h_apply / 1e3
            row["total_device_s"] = row["device_build_with_h2d_s"] + row["first_apply_ms_device_plan"] / 1e3
            rows.append(row)
            print(json.dumps(row), flush=True)
    if a.json:
        with open(a.json, "w") as f:
            json.dump({"cores": cores, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
