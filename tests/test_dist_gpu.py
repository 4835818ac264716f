"""DistributedP2P end to end on the GPU (NCCL when every rank has its own GPU; else the ranks share
the box's GPU with a gloo, host-staged exchange):
each rank exchanges halo weights (synchronously, and pipelined through exchange_async on a
communication stream as bench.py does; and with the peer-memory halo, the owners' buffers read
through CUDA IPC mappings), applies its partition, and gathers all targets; the gathered result
must be bit-identical to the single-plan apply (same tiles, same sum order) and match the fp64
oracle within the north_star gates."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, level, prec, results, kernel="laplace"):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    from paper_2403_01596_b200 import p2p
    from paper_2403_01596_b200 import workloads as W
    from paper_2403_01596_b200.dist import DistributedP2P

    # NCCL (device tensors, the bench path) whenever every rank has a GPU of its own; otherwise
    # the ranks share the box's GPU and the exchange is host-staged over gloo (test mode)
    nccl = torch.cuda.device_count() >= world
    dev = rank if nccl else 0
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl" if nccl else "gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world, **({"device_id": torch.device("cuda", dev)} if nccl else {}))
    try:
        src, tgt, q = W.make_problem(W.widened(W.CONFIGS["tiny"], 4))
        kw = {}
        if kernel == "helmholtz":  # complex weights through the same exchange (re, im pairs)
            q = W.weights_complex(len(src), 1)
            kw = dict(kernel="helmholtz", wavenumber=1.2 * (1 << (level - 1)))
        dp = DistributedP2P(src, tgt, device=dev, host_staged=not nccl, level=level, layout="tiled", precision=prec,
                            **kw)
        dt = dp.plan.torch_dtype
        lo, hi = dp.owned_source_range()
        full = p2p.Plan(src, tgt, level=level, device=-1)
        q_owned = torch.as_tensor(q[full.export("src_perm")[lo:hi]], dtype=dt, device=f"cuda:{dev}")
        full.close()
        out_sync = dp.apply(q_owned)
        side = torch.cuda.Stream()  # an explicit stream that is not the current one
        side.wait_stream(torch.cuda.current_stream())
        out_side = dp.apply(q_owned, stream=side.cuda_stream)
        torch.cuda.synchronize()
        assert torch.equal(out_side, out_sync)
        comm = torch.cuda.Stream()
        ev = dp.exchange_async(q_owned, comm)
        out_async = dp.apply(q_owned, halo_ready=ev)
        torch.cuda.synchronize()
        out_peer = dp.apply_peer(q_owned)  # halo read from the peers' memory (CUDA IPC)
        torch.cuda.synchronize()
        conv = (lambda t: t.cpu().numpy().astype(np.complex128)) if kernel == "helmholtz" else \
            (lambda t: t.double().cpu().numpy())
        g_sync, g_async, g_peer = conv(dp.gather(out_sync)), conv(dp.gather(out_async)), conv(dp.gather(out_peer))
        g_gp = conv(dp.gather_peer(out_peer))  # allgatherv over peer memory
        assert np.array_equal(g_gp, g_peer)
        # device-synchronised peer exchange + p2p_gather: five epochs enqueued back to back with
        # no host synchronisation; weights scaled by powers of two (results scale exactly)
        scales = (1.0, -2.0, 0.5, 4.0, 1.0)
        outs, gs = [], []
        for f in scales:
            o = dp.apply_sync(q_owned * f)
            outs.append(o)
            gs.append(dp.gather_sync(o))
        torch.cuda.synchronize()
        dp.check()
        for f, o, g in zip(scales, outs, gs):
            assert np.array_equal(conv(o), conv(out_sync) * f)
            assert np.array_equal(conv(g)[: len(g_sync)], g_sync * f)
        # the same step captured in a CUDA graph (no host work per apply at all) and replayed
        qs, og = q_owned.clone(), torch.empty_like(out_sync)
        gg = torch.empty_like(gs[0])
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # warm-up epoch outside the capture
            dp.apply_sync(qs, og)
            dp.gather_sync(og, gg)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            dp.apply_sync(qs, og)
            dp.gather_sync(og, gg)
        for f in (2.0, -1.0, 0.25):
            qs.copy_(q_owned * f)
            graph.replay()
            torch.cuda.synchronize()
            assert np.array_equal(conv(og), conv(out_sync) * f)
            assert np.array_equal(conv(gg)[: len(g_sync)], g_sync * f)
        dp.check()
        if rank == 0:
            results.put((g_sync, g_async, g_peer))
        dp.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(240)
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("level,prec,kernel", [(5, "fp32", "laplace"), (7, "fp32", "laplace"), (5, "fp64", "laplace"),
                                               (5, "fp32", "helmholtz"), (6, "fp64", "helmholtz")])
def test_distributed_apply_bit_identical(world, level, prec, kernel):
    from paper_2403_01596_b200 import p2p
    from paper_2403_01596_b200 import workloads as W
    src, tgt, q = W.make_problem(W.widened(W.CONFIGS["tiny"], 4))
    kw = {}
    if kernel == "helmholtz":
        q = W.weights_complex(len(src), 1)
        kw = dict(kernel="helmholtz", wavenumber=1.2 * (1 << (level - 1)))
    with p2p.Plan(src, tgt, level=level, layout="tiled", precision=prec, **kw) as pl:
        qd = torch.as_tensor(q[pl.export("src_perm")], dtype=pl.torch_dtype, device="cuda")
        out = pl.apply(qd)
        ref = out.cpu().numpy().astype(np.complex128) if kernel == "helmholtz" else out.double().cpu().numpy()
    ctx = mp.get_context("spawn")
    results = ctx.Queue()
    procs = mp.start_processes(_worker, args=(world, _free_port(), level, prec, results, kernel), nprocs=world,
                               start_method="spawn", join=False)
    g_sync, g_async, g_peer = results.get(timeout=180)  # drain before joining (a blocked queue pipe deadlocks)
    while not procs.join():
        pass
    assert np.array_equal(g_sync, ref)
    assert np.array_equal(g_async, ref)
    assert np.array_equal(g_peer, ref)
    # and against the fp64 oracle itself (SURVEY §8(c) gates), global plan order
    import oracle
    with p2p.Plan(src, tgt, level=level, device=-1) as host:
        tperm = host.export("tgt_perm")
    if kernel == "helmholtz":
        oref = oracle.direct_helmholtz(src, q, tgt, level, kw["wavenumber"])[0][tperm]
    else:
        oref = oracle.direct(src, q, tgt, level)[0][tperm]
    tol = 1e-5 if prec == "fp32" else 1e-12
    for g in (g_sync, g_async, g_peer):
        assert np.linalg.norm(g - oref) / np.linalg.norm(oref) <= tol


def _local_worker(rank, world, port, prec, results):
    """from_local plans on the GPU: each rank passes only an interleaved share of the points."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    from paper_2403_01596_b200 import workloads as W
    from paper_2403_01596_b200.dist import DistributedP2P

    nccl = torch.cuda.device_count() >= world
    dev = rank if nccl else 0
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl" if nccl else "gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world, **({"device_id": torch.device("cuda", dev)} if nccl else {}))
    try:
        src, tgt, q = W.make_problem(W.widened(W.CONFIGS["tiny"], 4))
        sid, tid = np.arange(rank, len(src), world), np.arange(rank, len(tgt), world)
        dp = DistributedP2P.from_local(src[sid], tgt[tid], sid, tid, level=6, device=dev, host_staged=not nccl,
                                       layout="tiled", precision=prec)
        q_owned = torch.as_tensor(q[dp.owned_source_ids()], dtype=dp.plan.torch_dtype, device=f"cuda:{dev}")
        out = dp.apply_sync(q_owned)
        g = dp.gather_sync(out)
        torch.cuda.synchronize()
        dp.check()
        if rank == 0:
            results.put((g.double().cpu().numpy(), dp.target_ids()))
        dp.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(240)
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_local_points_plan_apply(world, prec):
    """DistributedP2P.from_local (no rank holds the global point set) + the device-synchronised
    exchange and gather: bit-identical to the single plan, and within the gate of the oracle."""
    import oracle
    from paper_2403_01596_b200 import p2p
    from paper_2403_01596_b200 import workloads as W
    src, tgt, q = W.make_problem(W.widened(W.CONFIGS["tiny"], 4))
    with p2p.Plan(src, tgt, level=6, layout="tiled", precision=prec) as pl:
        qd = torch.as_tensor(q[pl.export("src_perm")], dtype=pl.torch_dtype, device="cuda")
        ref = pl.apply(qd).double().cpu().numpy()
        tperm = pl.export("tgt_perm")
    ctx = mp.get_context("spawn")
    results = ctx.Queue()
    procs = mp.start_processes(_local_worker, args=(world, _free_port(), prec, results), nprocs=world,
                               start_method="spawn", join=False)
    g, _ = results.get(timeout=180)
    while not procs.join():
        pass
    assert np.array_equal(g[: len(ref)], ref)
    oref = oracle.direct(src, q, tgt, 6)[0][tperm]
    assert np.linalg.norm(g[: len(ref)] - oref) / np.linalg.norm(oref) <= (1e-5 if prec == "fp32" else 1e-12)
