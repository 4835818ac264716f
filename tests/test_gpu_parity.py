"""Parity of the sm_100a P2P kernels (through the C ABI) with the fp64 oracle.

Gate (BASELINE.json north_star): relative L2 <= 1e-12 (fp64), <= 1e-5 (fp32).
Diagnostic, element-wise: |phi_gpu - phi_oracle| <= tol_el * sum_s |q_s ln(1/r)|
(the absolute-sum bound; for L >= 3 every E1 pair has r < 1, so the oracle
applied to |q| is exactly that sum)."""
import numpy as np
import pytest

import oracle
from paper_2403_01596_b200 import p2p
from paper_2403_01596_b200 import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

TOL = {"fp32": 1e-5, "fp64": 1e-12}
TOL_EL = {"fp32": 2e-5, "fp64": 1e-12}
COMBOS = [(lay, prec) for lay in ("nr", "r", "tiled") for prec in ("fp32", "fp64")]


def rel_l2(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def gpu_apply(plan, q_user, order="plan"):
    dt = plan.torch_dtype
    if order == "plan":
        q_plan = q_user[plan.export("src_perm")]
        qd = torch.as_tensor(q_plan, dtype=dt, device="cuda")
    else:
        qd = torch.as_tensor(q_user, dtype=dt, device="cuda")
    out = plan.apply(qd, order=order)
    torch.cuda.synchronize()
    return out.double().cpu().numpy()


def check(plan, src, tgt, q, level, targets_plan=None, abs_bound=True):
    """Compare the plan-order GPU result with the oracle (optionally on a sample of plan indices)."""
    phi = gpu_apply(plan, q)
    tperm = plan.export("tgt_perm")
    sel = tperm if targets_plan is None else tperm[targets_plan]
    ref, _ = oracle.direct(src, q, tgt, level, targets=sel)
    got = phi if targets_plan is None else phi[targets_plan]
    err = rel_l2(got, ref)
    assert err <= TOL[plan.precision], (plan.layout, plan.precision, err)
    if abs_bound and level >= 3:
        bound, _ = oracle.direct(src, np.abs(q), tgt, level, targets=sel)
        assert np.all(np.abs(got - ref) <= TOL_EL[plan.precision] * np.maximum(bound, 1e-300) + 1e-300)
    return err


@pytest.mark.parametrize("layout,prec", COMBOS)
@pytest.mark.parametrize("kind", ["iid", "stratified"])
def test_tiny(layout, prec, kind):
    src, tgt, q = W.make_problem("tiny", kind=kind)
    with p2p.Plan(src, tgt, level=4, layout=layout, precision=prec) as pl:
        check(pl, src, tgt, q, 4)


@pytest.mark.parametrize("layout,prec", COMBOS)
@pytest.mark.parametrize("level,tile", [(5, -1), (6, 0), (6, 1), (7, 2), (7, 3), (8, -1)])
def test_ragged_multi_tile(layout, prec, level, tile):
    src, tgt, q = W.uniform_unit(6007, 100 + level)
    with p2p.Plan(src, tgt, level=level, layout=layout, precision=prec, tile_log2=tile) as pl:
        assert pl.info["tiles"] > 1
        check(pl, src, tgt, q, level)


@pytest.mark.parametrize("layout,prec", COMBOS)
def test_collocated_guard(layout, prec):
    """targets = sources: every target has a guarded self pair (fp32 slow path)."""
    src, _, q = W.make_problem("tiny", seed=7)
    with p2p.Plan(src, src, level=4, layout=layout, precision=prec) as pl:
        check(pl, src, src, q, 4)


@pytest.mark.parametrize("layout,prec", COMBOS)
def test_lattice_closed_form(layout, prec):
    level = 5
    S = 1 << (level - 1)
    h = 1.0 / S
    ix, iy = np.meshgrid(np.arange(S), np.arange(S), indexing="xy")
    pts = np.stack([(ix.ravel() + 0.5) * h, (iy.ravel() + 0.5) * h], axis=1)
    with p2p.Plan(pts, pts, level=level, layout=layout, precision=prec) as pl:
        phi_plan = gpu_apply(pl, np.ones(len(pts)))
        phi = np.empty_like(phi_plan)
        phi[pl.export("tgt_perm")] = phi_plan
    lnh, ln2 = np.log(h), np.log(2.0)
    onx = (ix.ravel() == 0) | (ix.ravel() == S - 1)
    ony = (iy.ravel() == 0) | (iy.ravel() == S - 1)
    exp = np.where(onx & ony, -3 * lnh - 0.5 * ln2, np.where(onx | ony, -5 * lnh - ln2, -8 * lnh - 2 * ln2))
    assert rel_l2(phi, exp) <= TOL[prec]


@pytest.mark.parametrize("layout,prec", COMBOS)
def test_degenerate_cases(layout, prec):
    one = np.array([[0.3, 0.7]])
    with p2p.Plan(one, one, level=3, layout=layout, precision=prec) as pl:  # n = 1, coincident -> 0
        assert gpu_apply(pl, np.array([0.9]))[0] == 0.0
    src, tgt, q = W.uniform_unit(777, 5)
    with p2p.Plan(src, tgt, level=1, layout=layout, precision=prec) as pl:  # L = 1: one box, all pairs
        check(pl, src, tgt, q, 1)
    rng = np.random.default_rng(3)
    clus = 0.6 + rng.uniform(0, 0.05, (600, 2))  # everything in one L=3 cell
    qq = rng.uniform(-1, 1, 600)
    with p2p.Plan(clus, clus[::-1].copy(), level=3, layout=layout, precision=prec) as pl:
        check(pl, clus, clus[::-1].copy(), qq, 3)
    # plate smaller than the grid: most tiles empty, sources without targets and vice versa
    s2 = rng.uniform(0, 0.2, (500, 2))
    t2 = rng.uniform(0.1, 0.3, (400, 2))
    q2 = rng.uniform(-1, 1, 500)
    with p2p.Plan(s2, t2, level=7, layout=layout, precision=prec) as pl:
        check(pl, s2, t2, q2, 7)


@pytest.mark.parametrize("layout,prec", COMBOS)
def test_user_order_accumulate_host(layout, prec):
    src, tgt, q = W.make_problem("tiny", seed=2)
    ref, _ = oracle.direct(src, q, tgt, 4)
    with p2p.Plan(src, tgt, level=4, layout=layout, precision=prec) as pl:
        dt = pl.torch_dtype
        qd = torch.as_tensor(q, dtype=dt, device="cuda")
        out = pl.apply(qd, order="user")
        assert rel_l2(out.double().cpu().numpy(), ref) <= TOL[prec]
        # accumulate (near + far): a far-field-sized base, compared in fp64 at the plain gate
        base_h = np.linspace(-3.0, 5.0, len(tgt)).astype(pl.np_dtype)
        out2 = torch.as_tensor(base_h, device="cuda")
        pl.apply(qd, out2, order="user", accumulate=True)
        exp = base_h.astype(np.float64) + ref
        assert rel_l2(out2.double().cpu().numpy(), exp) <= TOL[prec]
        hq = q.astype(pl.np_dtype)
        hout = pl.apply_host(hq, order="user")
        assert rel_l2(hout.astype(np.float64), ref) <= TOL[prec]
        hp = pl.apply_host(np.ascontiguousarray(hq[pl.export("src_perm")]), order="plan")
        assert rel_l2(hp.astype(np.float64), ref[pl.export("tgt_perm")]) <= TOL[prec]


@pytest.mark.parametrize("layout,prec", COMBOS)
def test_deterministic(layout, prec):
    src, tgt, q = W.make_problem("d16_1e6", n=50000)
    with p2p.Plan(src, tgt, level=8, layout=layout, precision=prec) as pl:
        a = gpu_apply(pl, q)
        b = gpu_apply(pl, q)
    np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("layout,prec", [("nr", "fp32"), ("r", "fp32"), ("tiled", "fp32"), ("nr", "fp64")])
@pytest.mark.parametrize("world", [2, 3])
def test_partitions_bit_identical(layout, prec, world):
    """Results are bit-identical for any number of partitions:
    replicated-weight applies and the distributed (owned + halo) apply."""
    src, tgt, q = W.make_problem("d32_1e6", n=60000)
    level = 8
    with p2p.Plan(src, tgt, level=level, layout=layout, precision=prec) as full:
        ref = gpu_apply(full, q)
        q_plan = torch.as_tensor(q[full.export("src_perm")], dtype=full.torch_dtype, device="cuda")
    plans = [p2p.Plan(src, tgt, level=level, layout=layout, precision=prec, part_world=world, part_rank=r)
             for r in range(world)]
    parts = [pl.apply(q_plan).double().cpu().numpy() for pl in plans]
    np.testing.assert_array_equal(np.concatenate(parts), ref)
    # distributed: each rank packs the weights its peers need; exchange by hand (one GPU)
    part = plans[0].export("partition").reshape(2, world + 1)
    owned = [q_plan[part[0, r]:part[0, r + 1]].contiguous() for r in range(world)]
    sends = []
    for r, pl in enumerate(plans):
        buf = torch.empty(pl.info["n_send"], dtype=pl.torch_dtype, device="cuda")
        pl.halo_pack(owned[r], buf)
        cnt = pl.export("halo_counts").reshape(2, world)[1]
        sends.append(torch.split(buf, cnt.tolist()))
    for r, pl in enumerate(plans):
        halo = torch.cat([sends[o][r] for o in range(world)]) if world > 1 else torch.empty(0)
        assert halo.numel() == pl.info["n_halo"]
        out = torch.empty(pl.info["n_tgt_local"], dtype=pl.torch_dtype, device="cuda")
        pl.apply_dist(owned[r], halo.contiguous(), out)
        np.testing.assert_array_equal(out.double().cpu().numpy(), parts[r])
    for pl in plans:
        pl.close()


FULL = ["d16_1e6", "d32_1e6", "d64_1e6", "lowd025_1e7", "lowd1_1e7", "lowd2_1e7", "lowd4_1e7"]


@pytest.mark.parametrize("cfg", FULL)
@pytest.mark.parametrize("layout,prec", [("nr", "fp32"), ("r", "fp32"), ("tiled", "fp32"), ("nr", "fp64"), ("tiled", "fp64")])
def test_full_size_sampled(cfg, layout, prec):
    """BASELINE.json sizes, bench launch configuration; oracle on 3000 sampled targets."""
    c = W.CONFIGS[cfg]
    src, tgt, q = W.make_problem(c)
    with p2p.Plan(src, tgt, level=c.level, layout=layout, precision=prec) as pl:
        rng = np.random.default_rng(0)
        sample = np.sort(rng.choice(len(tgt), 3000, replace=False))
        check(pl, src, tgt, q, c.level, targets_plan=sample)


@pytest.mark.parametrize("cfg", ["surf_2e7", "d32_7e7"])
@pytest.mark.parametrize("layout,prec", [("tiled", "fp32"), ("tiled", "fp64"), ("nr", "fp32"), ("r", "fp32")])
def test_full_size_sampled_large(cfg, layout, prec):
    """BASELINE.json configs[3] / configs[4] (the headline bench workloads) at full size, plans
    built as bench.py builds them (on the device for NR / TILED); oracle on 3000 sampled targets."""
    c = W.CONFIGS[cfg]
    src, tgt, q = W.make_problem(c)
    kw = dict(level=c.level, layout=layout, precision=prec)
    if layout == "r":
        pl = p2p.Plan(src, tgt, **kw)
    else:
        pl = p2p.Plan(torch.as_tensor(src, device="cuda"), torch.as_tensor(tgt, device="cuda"), build="device", **kw)
    with pl:
        rng = np.random.default_rng(1)
        sample = np.sort(rng.choice(len(tgt), 3000, replace=False))
        check(pl, src, tgt, q, c.level, targets_plan=sample)


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("level", [5, 7])
def test_tail_split_bit_identical(prec, level, monkeypatch):
    """Tail tiles split into unit ranges (forced: the plan's default splits only Morton-ordered
    queues) give bit-identical results to the unsplit plan, and match the oracle."""
    src, tgt, q = W.make_problem(W.widened(W.CONFIGS["tiny"], 4))
    with p2p.Plan(src, tgt, level=level, layout="tiled", precision=prec) as pl:
        base = gpu_apply(pl, q)
    for tiles, parts in ((4, 3), (1000, 5)):
        monkeypatch.setenv("P2P_TAIL_TILES", str(tiles))
        monkeypatch.setenv("P2P_TAIL_PARTS", str(parts))
        with p2p.Plan(src, tgt, level=level, layout="tiled", precision=prec) as pl:
            launch = pl.export("launch").reshape(2, -1)
            assert np.any((launch[1] >> 16) >= parts)  # heavy tiles may split further
            assert np.array_equal(gpu_apply(pl, q), base)
            check(pl, src, tgt, q, level)


@pytest.mark.parametrize("layout", ["paper_i", "paper_r"])
@pytest.mark.parametrize("level", [1, 3, 4, 6])
def test_paper_layouts_parity(layout, level):
    """The paper's own Indexing / Repetition kernels vs the oracle, fp64,
    plan and user order, accumulate."""
    src, tgt, q = W.make_problem("tiny")
    with p2p.Plan(src, tgt, level=level, layout=layout, precision="fp64") as pl:
        check(pl, src, tgt, q, level)
        ref, _ = oracle.direct(src, q, tgt, level)
        got = gpu_apply(pl, q, order="user")
        assert rel_l2(got, ref) <= TOL["fp64"]
        out = torch.full((len(tgt),), 2.0, dtype=torch.float64, device="cuda")
        pl.apply(torch.as_tensor(q, dtype=torch.float64, device="cuda"), out, order="user", accumulate=True)
        torch.cuda.synchronize()
        assert rel_l2(out.cpu().numpy() - 2.0, ref) <= TOL["fp64"]
        # host buffers in plan order: the weights land in the plan's staging buffer
        for _ in range(2):
            hp = pl.apply_host(np.ascontiguousarray(q[pl.export("src_perm")]), order="plan")
            assert rel_l2(hp, ref[pl.export("tgt_perm")]) <= TOL["fp64"]
        hu = pl.apply_host(np.ascontiguousarray(q), order="user")
        assert rel_l2(hu, ref) <= TOL["fp64"]


@pytest.mark.parametrize("layout", ["paper_i", "paper_r"])
def test_paper_layouts_parity_sparse_and_ct(layout):
    """20k points at ~1 per box, and the CT loop's own level (CT = 15)."""
    c = W.CONFIGS["lowd1_1e7"]
    src, tgt, q = W.make_problem(c, n=20000)
    with p2p.Plan(src, tgt, level=c.level - 5, layout=layout, precision="fp64") as pl:
        check(pl, src, tgt, q, c.level - 5)
    with p2p.Plan(src, tgt, level=0, layout=layout, precision="fp64", ct=15) as pl:
        check(pl, src, tgt, q, pl.info["level"])


@pytest.mark.parametrize("layout,prec", [("tiled", "fp32"), ("nr", "fp64"), ("r", "fp32")])
def test_workspace_slots_pipelined(layout, prec):
    """p2p_plan_set_workspaces: applies of one plan in flight on different streams (host buffers
    and device buffers), no host synchronisation between them; every result equals the
    one-slot result for its weights (scaled by powers of two: exact)."""
    src, tgt, q = W.make_problem("d16_1e6", n=40000)
    with p2p.Plan(src, tgt, level=8, layout=layout, precision=prec) as pl:
        qd = torch.as_tensor(q, dtype=pl.torch_dtype, device="cuda")
        ref = pl.apply(qd, order="user").double().cpu().numpy()
        pl.set_workspaces(3)
        streams = [torch.cuda.Stream() for _ in range(3)]
        scales = [1.0, 2.0, -0.5, 4.0, 0.25, -1.0]
        hq = [(q * f).astype(pl.np_dtype) for f in scales]
        hq = [torch.from_numpy(a).pin_memory() for a in hq]
        ho = [torch.empty(len(tgt), dtype=pl.torch_dtype).pin_memory() for _ in scales]
        outs = []
        for k, f in enumerate(scales):
            st = streams[k % 3]
            p2p.p2p_apply_host_async(pl.handle, hq[k].data_ptr(), ho[k].data_ptr(), p2p.P2P_ORDER_USER, 0,
                                     st.cuda_stream)
            with torch.cuda.stream(st):
                outs.append(pl.apply(qd * f, order="user", stream=st.cuda_stream))
        torch.cuda.synchronize()
        for k, f in enumerate(scales):
            assert np.array_equal(ho[k].double().numpy(), ref * f)
            assert np.array_equal(outs[k].double().cpu().numpy(), ref * f)
