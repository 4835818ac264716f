"""Multi-process (gloo, CPU) test of the Morton-range partition and the halo
weight exchange bookkeeping.

Each rank builds a host-only plan for its partition, sends the owned weights
AND coordinates its peers need (per the plan's send lists) through a real
torch.distributed process group, assembles its local source set from what it
owns plus what it received, and evaluates its owned targets with the oracle
on that local set only.  The result must equal the global oracle: this proves
the exchanged halo is exactly the E1 neighbourhood the kernel needs.  (The
apply itself needs a GPU; tests/test_gpu_parity.py checks the device path of
the same exchange.)"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg_name, n, level, results):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    from paper_2403_01596_b200 import p2p
    from paper_2403_01596_b200 import workloads as W

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        src, tgt, q = W.make_problem(cfg_name, n=n)
        pl = p2p.Plan(src, tgt, level=level, device=-1, part_world=world, part_rank=rank)
        full = p2p.Plan(src, tgt, level=level, device=-1)
        gperm = full.export("src_perm")  # global plan index -> user index
        part = pl.export("partition").reshape(2, world + 1)
        lo, hi = part[0, rank], part[0, rank + 1]
        own_user = gperm[lo:hi]
        # this rank only "has" its owned points and weights from here on
        own_xy, own_q = src[own_user], q[own_user]
        counts = pl.export("halo_counts").reshape(2, world)
        send_idx = pl.export("send_index")
        splits = np.cumsum(counts[1])[:-1]
        outbox = [(own_xy[i], own_q[i]) for i in np.split(send_idx, splits)]
        gathered = [None] * world
        dist.all_gather_object(gathered, outbox)
        inbox = [gathered[o][rank] for o in range(world)]  # from each owner, ascending
        for o in range(world):
            assert len(inbox[o][1]) == counts[0, o]
        halo_xy = np.concatenate([b[0] for b in inbox]) if world > 1 else np.zeros((0, 2))
        halo_q = np.concatenate([b[1] for b in inbox]) if world > 1 else np.zeros(0)
        # assemble the local source set in local plan order (what the gather2 kernel does)
        gl = pl.export("src_global")
        loc_xy = np.empty((len(gl), 2))
        loc_q = np.empty(len(gl))
        h = 0
        for i, g in enumerate(gl):
            if lo <= g < hi:
                loc_xy[i], loc_q[i] = own_xy[g - lo], own_q[g - lo]
            else:
                loc_xy[i], loc_q[i] = halo_xy[h], halo_q[h]
                h += 1
        assert h == len(halo_q) == pl.info["n_halo"]
        my_t = pl.export("tgt_perm")
        got, _ = oracle.direct(loc_xy, loc_q, tgt, level, targets=my_t)
        ref, _ = oracle.direct(src, q, tgt, level, targets=my_t)
        err = np.max(np.abs(got - ref)) if len(ref) else 0.0
        results[rank] = (float(err), int(len(my_t)), int(pl.info["n_halo"]), int(pl.info["pairs"]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_halo_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, "d16_1e6", 30000, 7, results)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    res = [results[r] for r in range(world)]
    assert sum(r[1] for r in res) == 30000
    assert all(r[2] > 0 for r in res)
    for err, *_ in res:
        assert err <= 1e-12
