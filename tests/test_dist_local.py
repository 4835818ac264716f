"""Partitioned plans from each rank's OWN points (gloo, world 2 and 3, CPU; SURVEY.md §8(e),
north_star "a one-time exchange distributes halo source points").

Every rank holds only an interleaved share of the sources and targets (global id % world ==
rank) -- not its partition's points, and never the global set.  DistributedP2P.from_local
counts boxes, sums the counts over the ranks, routes each point to the ranks that need it
(one all-to-all of coordinates + ids) and builds its plan from what arrived.  Checked:
  * the plan equals the global-input builder's plan for the same rank (tiles, partition, local
    order, halo and send lists, TILED records): the GPU applies are then bit-identical;
  * the rank's targets evaluated by the oracle on the received points only (weights looked up
    by id) equal the global oracle -- the routed halo is exactly the E1 neighbourhood."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


SAME = ["src_global", "tiles", "partition", "halo_counts", "send_index", "halo_index", "halo_offsets",
        "region_offsets", "region_index", "region_table", "slot_offsets", "slot_base", "slot_output",
        "item_offsets", "items", "launch"]
INFO = ["n_src_local", "n_tgt_local", "n_src_owned", "src_owned_begin", "tgt_begin", "n_halo", "n_send", "pairs",
        "pairs_global", "tiles", "tile_log2", "smem_bytes", "halo_entries", "interior_launches", "launches",
        "n_src", "n_tgt", "occupied_src_boxes", "occupied_tgt_boxes", "t_max"]


def _worker(rank, world, port, layout, kind, results):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    import oracle
    from paper_2403_01596_b200 import p2p
    from paper_2403_01596_b200 import workloads as W
    from paper_2403_01596_b200.dist import DistributedP2P

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        if kind == "disjoint":  # sources uniform, targets in one quarter (owned boxes outside every region)
            rng = np.random.default_rng(5)
            src, tgt = rng.uniform(0, 1, (12000, 2)), rng.uniform(0.5, 1, (9000, 2))
            q = rng.uniform(-1, 1, len(src))
            level = 7
        else:
            src, tgt, q = W.make_problem("d16_1e6", n=30000)
            level = 7
        # this rank holds an interleaved share only (the global arrays below are used for checks);
        # "empty": the last rank holds no points at all (it still owns a Morton range)
        if kind == "empty":
            holders = world - 1
            sid = np.arange(rank, len(src), holders) if rank < holders else np.zeros(0, dtype=np.int64)
            tid = np.arange(rank, len(tgt), holders) if rank < holders else np.zeros(0, dtype=np.int64)
        else:
            sid = np.arange(rank, len(src), world)
            tid = np.arange(rank, len(tgt), world)
        dp = DistributedP2P.from_local(src[sid], tgt[tid], sid, tid, level=level, device=-1, host_staged=True,
                                       layout=layout, precision="fp32")
        ref = p2p.Plan(src, tgt, level=level, layout=layout, precision="fp32", device=-1, part_world=world,
                       part_rank=rank)
        li, gi = dp.plan.info, ref.info
        bad = [k for k in INFO if li[k] != gi[k]]
        for kind_ in SAME:
            if not np.array_equal(dp.plan.export(kind_), ref.export(kind_)):
                bad.append(kind_)
        # local order: ids of the local sources / targets = the global plan's user indices
        if not np.array_equal(dp.src_ids[dp.plan.export("src_perm")], ref.export("src_perm")):
            bad.append("src_perm")
        if not np.array_equal(dp.target_ids(), ref.export("tgt_perm")):
            bad.append("tgt_perm")
        # oracle on the received points only
        rs_xy = dp.src_xy_local  # the coordinates that arrived, with their ids
        if not np.array_equal(rs_xy, src[dp.src_ids]) or not np.array_equal(dp.tgt_xy_local, tgt[dp.tgt_ids]):
            bad.append("routed coordinates")
        got, _ = oracle.direct(rs_xy, q[dp.src_ids], tgt, level, targets=dp.target_ids())
        exp, _ = oracle.direct(src, q, tgt, level, targets=dp.target_ids())
        err = float(np.max(np.abs(got - exp))) if len(exp) else 0.0
        results[rank] = (bad, err, li["n_src_local"], len(sid))
        ref.close()
        dp.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("layout", ["tiled", "nr", "r"])
@pytest.mark.parametrize("world,kind", [(2, "iid"), (3, "iid"), (3, "disjoint"), (3, "empty")])
def test_plan_from_local_points(layout, world, kind):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, layout, kind, results)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    for r in range(world):
        bad, err, n_local, n_held = results[r]
        assert not bad, (r, bad)
        assert err <= 1e-12, (r, err)
