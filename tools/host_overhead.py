"""Host-side cost of one apply call through the ctypes binding (no synchronisation in the loop)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2403_01596_b200 import p2p, workloads as W
cfg = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "d16_1e6"]
src, tgt, q = W.make_problem(cfg)
pl = p2p.Plan(torch.as_tensor(src, device="cuda"), torch.as_tensor(tgt, device="cuda"), level=cfg.level,
              layout="tiled", precision="fp32", build="device")
qd = torch.as_tensor(q[pl.export("src_perm")], dtype=torch.float32, device="cuda")
out = torch.empty(pl.info["n_tgt_local"], dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    p2p.p2p_apply(pl.handle, qd.data_ptr(), out.data_ptr(), 0, 0, s)
torch.cuda.synchronize()
for label, body in [("apply only", lambda: p2p.p2p_apply(pl.handle, qd.data_ptr(), out.data_ptr(), 0, 0, s)),
                    ("flush only", lambda: flush.zero_()),
                    ("event record", lambda: torch.cuda.Event(enable_timing=True).record())]:
    n = 50
    t = time.perf_counter()
    for _ in range(n):
        body()
    dt = (time.perf_counter() - t) / n * 1e3
    torch.cuda.synchronize()
    print(f"{label:14s} {dt:.4f} ms per call (host)")
