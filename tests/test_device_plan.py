"""The plan built on the GPU (p2p_plan_create_device) against the
host builder (p2p_plan_create) and the fp64 oracle.

Bar: the device-built plan is bit-identical to the host-built one -- every info field but the
timings, every exported array (permutations, CSR offsets, partition, launch queue, TILED tables,
regions, slots, items) -- and so are its apply results; at the tiny sizes both also meet the
oracle's tolerance (relative L2 1e-5 fp32, 1e-12 fp64)."""
import numpy as np
import pytest

from paper_2403_01596_b200 import p2p
from paper_2403_01596_b200 import workloads as W

COMMON = ["src_perm", "tgt_perm", "src_box_offsets", "tgt_box_offsets", "partition", "src_global",
          "halo_counts", "tiles", "launch"]
TILED = ["region_offsets", "region_index", "region_table", "slot_offsets", "slot_base", "slot_output",
         "item_offsets", "items"]
SKIP_INFO = {"build_seconds", "upload_seconds", "device_bytes"}


def _desc(n_src, n_tgt, **kw):
    d = p2p.p2p_plan_desc_init()
    d.n_src, d.n_tgt = n_src, n_tgt
    for k, v in kw.items():
        setattr(d, k, v)
    return d


# ------------------------------------------------------------------ host-only (no GPU needed)
@pytest.mark.parametrize("kw,status", [
    (dict(layout=p2p.P2P_LAYOUT_REDUNDANT), p2p.P2P_ERROR_NOT_SUPPORTED),
    (dict(layout=p2p.P2P_LAYOUT_PAPER_INDEXING, precision=p2p.P2P_FP64), p2p.P2P_ERROR_NOT_SUPPORTED),
    (dict(part_world=2), p2p.P2P_ERROR_NOT_SUPPORTED),
    (dict(layout=p2p.P2P_LAYOUT_ADAPTIVE), p2p.P2P_ERROR_NOT_SUPPORTED),
    (dict(kernel=p2p.P2P_KERNEL_LAPLACE_3D), p2p.P2P_ERROR_NOT_SUPPORTED),
    (dict(epsilon=0.0), p2p.P2P_ERROR_INVALID_ARGUMENT),
    (dict(device=-1), p2p.P2P_ERROR_NO_DEVICE),
])
def test_device_build_rejects_before_touching_the_gpu(kw, status):
    d = _desc(4, 4, **kw)
    with pytest.raises(p2p.P2PError) as ei:
        p2p.p2p_plan_create_device(d, 1 << 20, 1 << 20)  # never dereferenced: rejected first
    assert ei.value.status == status


def test_device_build_rejects_null_and_empty():
    with pytest.raises(p2p.P2PError) as ei:
        p2p.p2p_plan_create_device(_desc(4, 4), 0, 0)
    assert ei.value.status == p2p.P2P_ERROR_INVALID_ARGUMENT
    with pytest.raises(p2p.P2PError) as ei:
        p2p.p2p_plan_create_device(_desc(0, 4), 1 << 20, 1 << 20)
    assert ei.value.status == p2p.P2P_ERROR_INVALID_ARGUMENT


# ------------------------------------------------------------------ GPU: bit-identity with the host builder
def _compare(src, tgt, q, **kw):
    import torch
    host = p2p.Plan(src, tgt, **kw)
    dev = p2p.Plan(src, tgt, build="device", **kw)
    try:
        for k, v in host.info.items():
            if k not in SKIP_INFO:
                assert dev.info[k] == v, (k, dev.info[k], v)
        kinds = COMMON + (TILED if kw.get("layout") == "tiled" else [])
        if host.info["boxes"] <= 1 << 16:
            kinds = kinds + ["neighbors"]
        for kind in kinds:
            a, b = host.export(kind), dev.export(kind)
            assert a.shape == b.shape and np.array_equal(a, b), kind
        dt = host.torch_dtype
        qp = torch.as_tensor(q[host.export("src_perm")], dtype=dt, device="cuda")
        qu = torch.as_tensor(q, dtype=dt, device="cuda")
        for order, qq in (("plan", qp), ("user", qu)):
            a = host.apply(qq, order=order)
            b = dev.apply(qq, order=order)
            torch.cuda.synchronize()
            assert torch.equal(a, b), order
        return host.info
    finally:
        host.close()
        dev.close()


SMALL = {
    "d16": W.PlateConfig("d16_s", 64, 48, 8, 64 * 48 * 16, seed=7),
    "d64": W.PlateConfig("d64_s", 32, 32, 7, 32 * 32 * 64, seed=8),
    "d1": W.PlateConfig("d1_s", 300, 200, 10, 60_000, seed=9),
    "d025": W.PlateConfig("d025_s", 400, 400, 10, 40_000, seed=10),
    "d4": W.PlateConfig("d4_s", 200, 125, 9, 100_000, seed=11),
}


@pytest.mark.gpu
@pytest.mark.parametrize("layout", ["nr", "tiled"])
@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("level", [4, 6])
def test_tiny_matches_host_and_oracle(layout, prec, level):
    import torch
    import oracle
    src, tgt, q = W.make_problem("tiny")
    _compare(src, tgt, q, level=level, layout=layout, precision=prec)
    with p2p.Plan(src, tgt, level=level, layout=layout, precision=prec, build="device") as pl:
        out = pl.apply(torch.as_tensor(q, dtype=pl.torch_dtype, device="cuda"), order="user")
        torch.cuda.synchronize()
        ref, pairs = oracle.direct(src, q, tgt, level)
        got = out.double().cpu().numpy()
        assert pl.info["pairs"] == pairs
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= (1e-5 if prec == "fp32" else 1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(SMALL))
@pytest.mark.parametrize("layout", ["nr", "tiled"])
@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("kind", ["iid", "stratified"])
def test_workload_shapes_match_host(name, layout, prec, kind):
    cfg = SMALL[name]
    if kind == "stratified" and cfg.n % (cfg.sx * cfg.sy):
        pytest.skip("stratified needs an integer density")
    src, tgt, q = W.make_problem(cfg, kind=kind)
    _compare(src, tgt, q, level=cfg.level, layout=layout, precision=prec)


@pytest.mark.gpu
@pytest.mark.parametrize("delta", [-1, 0, 1])
@pytest.mark.parametrize("layout", ["nr", "tiled"])
def test_ct_loop_matches_host(delta, layout):
    src, tgt, q = W.uniform_unit(20_000, seed=3)
    info = _compare(src, tgt, q, level=0, ct=15, level_delta=delta, layout=layout, precision="fp32")
    assert info["level"] >= 3


@pytest.mark.gpu
@pytest.mark.parametrize("tile_log2", [0, 1, 3])
def test_explicit_tile_size_matches_host(tile_log2):
    cfg = SMALL["d16"]
    src, tgt, q = W.make_problem(cfg)
    _compare(src, tgt, q, level=cfg.level, layout="tiled", precision="fp32", tile_log2=tile_log2)


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("name", ["d16", "d1"])
def test_morton_queue_with_split_tail_matches_host(monkeypatch, prec, name):
    monkeypatch.setenv("P2P_LPT", "0")  # Morton-order queue; its last tiles split in 4 parts
    cfg = SMALL[name]
    src, tgt, q = W.make_problem(cfg)
    info = _compare(src, tgt, q, level=cfg.level, layout="tiled", precision=prec)
    with p2p.Plan(src, tgt, level=cfg.level, layout="tiled", precision=prec, build="device") as pl:
        launch = pl.export("launch")
    nparts = launch[info["launches"]:] >> 16
    assert (nparts >= 4).any()  # the split tail (small problems also split heavy tiles)


@pytest.mark.gpu
def test_collocated_single_point_and_one_box():
    src, _, q = W.make_problem("tiny")
    _compare(src, None, q, level=4, layout="tiled", precision="fp32")  # targets = sources
    one = np.array([[0.25, 0.75]])
    _compare(one, one, np.array([0.5]), level=3, layout="tiled", precision="fp64")
    _compare(src, src, q, level=1, layout="nr", precision="fp32")  # one box


@pytest.mark.gpu
def test_device_build_errors():
    import torch
    src, tgt, _ = W.make_problem("tiny")
    bad = src.copy()
    bad[17, 1] = np.nan
    with pytest.raises(p2p.P2PError) as ei:
        p2p.Plan(bad, tgt, level=4, build="device")
    assert ei.value.status == p2p.P2P_ERROR_INVALID_ARGUMENT and "coordinate 17" in str(ei.value)
    same = np.full((64, 2), 0.3)  # 64 coincident points: no level separates them
    with pytest.raises(p2p.P2PError) as ei:
        p2p.Plan(same, same, level=0, ct=15, l_max=8, build="device")
    assert ei.value.status == p2p.P2P_ERROR_CONSTRUCTION_FAILURE
    # device tensors are accepted as they are
    with p2p.Plan(torch.as_tensor(src, device="cuda"), torch.as_tensor(tgt, device="cuda"), level=4,
                  layout="tiled", build="device") as pl:
        assert pl.info["pairs"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("name,layout", [("d16_1e6", "tiled"), ("d32_1e6", "nr"), ("lowd1_1e7", "tiled")])
def test_full_size_matches_host(name, layout):
    """BASELINE.json sizes, the launch configuration bench.py times."""
    cfg = W.CONFIGS[name]
    src, tgt, q = W.make_problem(cfg)
    _compare(src, tgt, q, level=cfg.level, layout=layout, precision="fp32")
