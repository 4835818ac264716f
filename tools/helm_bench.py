"""2D Helmholtz near field on B200: G = (i/4) H0^(1)(kappa r), complex
weights, TILED layout.  Workload: the d16_1e6 and d4_1e6 plates with the leaf box a quarter
wavelength (kappa h = pi/2, R23), iid points, fp32 and fp64; per config the median of
`--reps` L2-flushed applies (CUDA events), pairs/s, the oracle on a sample of targets (all host
cores) and the fp32 relative L2 error on that sample.

  python tools/helm_bench.py --json gpurun_out/helm_bench.json
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure: the CPU baseline and the error check)
from paper_2403_01596_b200 import p2p  # noqa: E402
from paper_2403_01596_b200 import workloads as W  # noqa: E402

DEV = torch.device("cuda", 0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="d16_1e6,d4_1e6")
    ap.add_argument("--kh", type=float, default=math.pi / 2)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--sample", type=int, default=20000)
    ap.add_argument("--precisions", default="fp32,fp64")
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=DEV)
    stream = torch.cuda.current_stream(DEV)
    rows = []
    for name in a.configs.split(","):
        cfg = W.CONFIGS[name]
        src, tgt, _ = W.make_problem(cfg)
        q = W.weights(cfg.n, cfg.seed) + 1j * W.weights(cfg.n, cfg.seed, stream=5)
        kappa = a.kh * (1 << (cfg.level - 1))
        sel = np.random.default_rng(0).choice(cfg.n, min(a.sample, cfg.n), replace=False)
        t = time.perf_counter()
        ref, sp = oracle.direct_helmholtz(src, q, tgt, cfg.level, kappa, targets=sel)
        cpu_s = time.perf_counter() - t
        for prec in a.precisions.split(","):
            with p2p.Plan(torch.as_tensor(src, device=DEV), torch.as_tensor(tgt, device=DEV), level=cfg.level,
                          layout="tiled", precision=prec, kernel="helmholtz", wavenumber=kappa,
                          build="device") as pl:
                qd = torch.as_tensor(q[pl.export("src_perm")], dtype=pl.torch_dtype, device=DEV)
                out = torch.empty(pl.info["n_tgt_local"], dtype=pl.torch_dtype, device=DEV)
                for _ in range(3):
                    pl.apply(qd, out)
                ts = []
                for _ in range(a.reps):
                    flush.zero_()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    pl.apply(qd, out)
                    e1.record(stream)
                    e1.synchronize()
                    ts.append(e0.elapsed_time(e1))
                ms = float(np.median(ts))
                phi = torch.empty_like(out)
                pl.apply(torch.as_tensor(q, dtype=pl.torch_dtype, device=DEV), phi, order="user")
                got = phi.cpu().numpy().astype(np.complex128)[sel]
                err = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
                pairs = pl.info["pairs"]
                row = {"config": name, "precision": prec, "kappa": kappa, "kappa_h": a.kh, "pairs": pairs,
                       "ms": ms, "Gpair_s": pairs / (ms * 1e-3) / 1e9, "rel_l2_sample": err,
                       "cpu_oracle_pair_s": sp / cpu_s, "cpu_cores": oracle.num_threads(),
                       "cta_threads": pl.info["cta_threads"], "tile_log2": pl.info["tile_log2"]}
                rows.append(row)
                print(json.dumps(row), flush=True)
    if a.json:
        with open(a.json, "w") as f:
            json.dump({"rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
