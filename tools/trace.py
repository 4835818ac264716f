"""Per-tile timeline of the TILED kernel (diagnostics): phase durations, concurrency, tail."""
import argparse
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_01596_b200 import p2p  # noqa: E402
from paper_2403_01596_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="d16_1e6")
ap.add_argument("--layout", default="tiled")
ap.add_argument("--flush", action="store_true", help="flush L2 (256 MiB write) right before the traced apply")
args = ap.parse_args()
lib = p2p.load_library()
lib.p2p_internal_set_trace.argtypes = [C.c_void_p, C.c_void_p]
for name in args.configs.split(","):
    cfg = W.CONFIGS[name]
    src, tgt, q = W.make_problem(cfg)
    pl = p2p.Plan(src, tgt, level=cfg.level, layout=args.layout, device=0)
    nt = pl.info["tiles"]
    tr = torch.zeros(nt * 8, dtype=torch.int64, device="cuda")
    qd = torch.as_tensor(q[pl.export("src_perm")], dtype=pl.torch_dtype, device="cuda")
    out = torch.empty(pl.info["n_tgt_local"], dtype=pl.torch_dtype, device="cuda")
    for _ in range(3):
        pl.apply(qd, out)
    lib.p2p_internal_set_trace(pl.handle, C.c_void_p(tr.data_ptr()))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if args.flush:
        torch.empty(256 << 20, dtype=torch.uint8, device="cuda").zero_()
    e0.record()
    pl.apply(qd, out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    t = tr.view(nt, 8).cpu().numpy().astype(np.int64)
    sm = (t[:, 0] >> 32)
    t0 = t[:, 1].min()
    claim, data, units, end = (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3, (t[:, 3] - t0) / 1e3, (t[:, 5] - t0) / 1e3
    dur = end - claim
    print(f"== {name}: kernel {ms * 1e3:.1f} us (events), trace span {end.max():.1f} us, tiles {nt}, "
          f"grid {len(np.unique(t[:, 0] & 0xffffffff))} CTAs on {len(np.unique(sm))} SMs")
    print(f"  tile duration us: mean {dur.mean():.2f} p10 {np.percentile(dur, 10):.2f} p90 {np.percentile(dur, 90):.2f}")
    print(f"  phases mean us: wait-data {np.mean(data - claim):.2f}  gather+units {np.mean(units - data):.2f}  "
          f"compute+reduce {np.mean(end - units):.2f}")
    print(f"  first-wave start spread {np.percentile(claim, 1):.2f}..{np.sort(claim)[min(len(claim) - 1, 1000)]:.2f} us; "
          f"last tile ends {end.max():.2f}; 90% of tiles done by {np.percentile(end, 90):.2f} us")
    # per-SM busy time: union of tile intervals per SM
    busy = []
    for s_ in np.unique(sm):
        m = sm == s_
        busy.append(end[m].max() - claim[m].min())
    busy = np.array(busy)
    print(f"  per-SM active span us: min {busy.min():.1f} mean {busy.mean():.1f} max {busy.max():.1f}")
    first = np.argsort(claim)[:min(len(claim), 1332)]
    print(f"  first wave: wait-data mean {np.mean((data - claim)[first]):.2f} us, max {np.max((data - claim)[first]):.2f}; "
          f"later tiles {np.mean(np.delete(data - claim, first)):.2f} us")
    # concurrency: average number of tiles in flight per SM
    conc = dur.sum() / (len(np.unique(sm)) * end.max())
    print(f"  mean tiles in flight per SM {conc:.2f}; pairs {pl.info['pairs']}, "
          f"{pl.info['pairs'] / (ms * 1e-3) / 1e12:.3f} Tpair/s")
    lib.p2p_internal_set_trace(pl.handle, None)
    pl.close()
