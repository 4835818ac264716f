"""Timeline of the bench's e2e step (three configs, one stream each): per stream, when its H2D,
P2P apply (user order: permutation kernels + P2P kernel) and D2H start/end, relative to the step
start.  Replays p2p_apply_host_async's sequence with torch copies + p2p_apply on device buffers."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_01596_b200 import p2p  # noqa: E402
from paper_2403_01596_b200 import workloads as W  # noqa: E402

names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["d16_1e6", "d32_1e6", "d64_1e6"]
dev = torch.device("cuda", 0)
jobs = []
for n in names:
    c = W.CONFIGS[n]
    s, t, q = W.make_problem(c)
    pl = p2p.Plan(s, t, level=c.level, layout="tiled", device=0)
    jobs.append(dict(pl=pl, hq=torch.as_tensor(q, dtype=torch.float32).pin_memory(),
                     ho=torch.empty(len(t), dtype=torch.float32).pin_memory(),
                     dq=torch.empty(len(s), dtype=torch.float32, device=dev),
                     do=torch.empty(len(t), dtype=torch.float32, device=dev), st=torch.cuda.Stream(dev)))
main = torch.cuda.current_stream(dev)


def step(record):
    start = torch.cuda.Event(enable_timing=True)
    start.record(main)
    evs = []
    for j in jobs:
        st = j["st"]
        st.wait_event(start)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        with torch.cuda.stream(st):
            e[0].record(st)
            j["dq"].copy_(j["hq"], non_blocking=True)
            e[1].record(st)
            p2p.p2p_apply(j["pl"].handle, j["dq"].data_ptr(), j["do"].data_ptr(), p2p.P2P_ORDER_USER, 0,
                          st.cuda_stream)
            e[2].record(st)
            j["ho"].copy_(j["do"], non_blocking=True)
            e[3].record(st)
        main.wait_event(e[3])
        evs.append(e)
    end = torch.cuda.Event(enable_timing=True)
    end.record(main)
    return start, evs, end


for _ in range(5):
    step(False)
torch.cuda.synchronize()
rows = []
for _ in range(10):
    start, evs, end = step(True)
    torch.cuda.synchronize()
    rows.append([[start.elapsed_time(x) * 1e3 for x in e] for e in evs] + [[start.elapsed_time(end) * 1e3] * 4])
r = np.median(np.array(rows), axis=0)
for n, x in zip(names + ["step"], r):
    print(f"{n:10s} h2d {x[0]:7.1f}..{x[1]:7.1f}  apply ..{x[2]:7.1f}  d2h ..{x[3]:7.1f} us")
