"""3D kernels on the octree leaf grid (include/p2p.h LAPLACE_3D /
HELMHOLTZ_3D; R24): plan indexing bit-exact against an independent recomputation,
GPU results against the pinned 3D oracle (relative L2 1e-5 fp32, 1e-12 fp64)."""
import math

import numpy as np
import pytest

import oracle
from paper_2403_01596_b200 import p2p
from paper_2403_01596_b200 import workloads as W

TINY = W.CONFIGS["tiny3d"]          # 4 x 4 x 4 leaf boxes, 16 points per box
MID = W.CubeConfig("cube_s", 12, 5, 12 ** 3 * 16, seed=3)


def _morton3(ix, iy, iz):
    code = np.zeros_like(ix)
    for b in range(10):
        code |= ((ix >> b) & 1) << (3 * b) | ((iy >> b) & 1) << (3 * b + 1) | ((iz >> b) & 1) << (3 * b + 2)
    return code


def test_plan_indexing_bit_exact():
    src, tgt, _ = W.make_problem(MID)
    with p2p.Plan(src, tgt, level=MID.level, layout="nr", kernel="laplace3d", device=-1) as pl:
        S = pl.info["side"]
        assert pl.info["boxes"] == S ** 3
        for pts, pk, ok in ((src, "src_perm", "src_box_offsets"), (tgt, "tgt_perm", "tgt_box_offsets")):
            c = np.minimum(np.floor(pts * S), S - 1).astype(np.int64)
            code = _morton3(c[:, 0], c[:, 1], c[:, 2])
            assert np.array_equal(pl.export(pk), np.argsort(code, kind="stable"))
            assert np.array_equal(pl.export(ok), np.searchsorted(np.sort(code), np.arange(S ** 3 + 1)))
        _, pairs = oracle.direct_3d(src, np.ones(len(src)), tgt, MID.level)
        assert pl.info["pairs"] == pairs
        with pytest.raises(p2p.P2PError):
            pl.export("neighbors")


def test_3d_envelope_errors():
    src, tgt, _ = W.make_problem(TINY)
    for kw, st in ((dict(layout="tiled"), p2p.P2P_ERROR_NOT_SUPPORTED),
                   (dict(layout="nr", level=0), p2p.P2P_ERROR_NOT_SUPPORTED),
                   (dict(layout="nr", level=10), p2p.P2P_ERROR_NOT_SUPPORTED)):
        kw = {"level": 3, **kw}
        with pytest.raises(p2p.P2PError) as ei:
            p2p.Plan(src, tgt, kernel="laplace3d", device=-1, **kw)
        assert ei.value.status == st, kw
    with pytest.raises(p2p.P2PError) as ei:
        p2p.Plan(src, tgt, level=3, layout="nr", kernel="helmholtz3d", device=-1)  # no wavenumber
    assert ei.value.status == p2p.P2P_ERROR_INVALID_ARGUMENT
    bad = src.copy()
    bad[5, 2] = 1.5
    with pytest.raises(p2p.P2PError) as ei:
        p2p.Plan(bad, tgt, level=3, layout="nr", kernel="laplace3d", device=-1)
    assert ei.value.status == p2p.P2P_ERROR_INVALID_ARGUMENT


def _run(pl, q, order):
    import torch
    qq = q if order == "user" else q[pl.export("src_perm")]
    out = pl.apply(torch.as_tensor(qq, dtype=pl.torch_dtype, device="cuda"), order=order)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    return got if order == "user" else got[np.argsort(pl.export("tgt_perm"))]


@pytest.mark.gpu
@pytest.mark.parametrize("kernel", ["laplace3d", "helmholtz3d"])
@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("cfg", [TINY, MID], ids=lambda c: c.name)
def test_against_oracle(kernel, prec, cfg):
    src, tgt, q = W.make_problem(cfg)
    helm = kernel == "helmholtz3d"
    kappa = (math.pi / 2) * cfg.side if helm else 0.0
    if helm:
        q = W.weights_complex(cfg.n, cfg.seed)
    ref, pairs = oracle.direct_3d(src, q, tgt, cfg.level, "helmholtz" if helm else "laplace", kappa)
    with p2p.Plan(src, tgt, level=cfg.level, layout="nr", precision=prec, kernel=kernel, wavenumber=kappa) as pl:
        assert pl.info["pairs"] == pairs
        tol = 1e-5 if prec == "fp32" else 1e-12
        for order in ("user", "plan"):
            got = _run(pl, q, order)
            assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= tol, (order, np.linalg.norm(got - ref) / np.linalg.norm(ref))


@pytest.mark.gpu
def test_collocated_accumulate_and_determinism():
    import torch
    src, _, q = W.make_problem(TINY)
    ref, _ = oracle.direct_3d(src, q, src, TINY.level)  # self pairs guarded
    with p2p.Plan(src, src, level=TINY.level, layout="nr", precision="fp64", kernel="laplace3d") as pl:
        a = _run(pl, q, "user")
        assert np.linalg.norm(a - ref) / np.linalg.norm(ref) <= 1e-12
        assert np.array_equal(a, _run(pl, q, "user"))
        base = torch.full((len(src),), 2.5, dtype=torch.float64, device="cuda")
        out = pl.apply(torch.as_tensor(q, device="cuda"), base, order="user", accumulate=True)
        torch.cuda.synchronize()
        assert np.allclose(out.cpu().numpy(), a + 2.5, rtol=0, atol=1e-12)
        assert np.array_equal(pl.apply_host(q, order="user"), a)


@pytest.mark.gpu
@pytest.mark.parametrize("kernel", ["laplace3d", "helmholtz3d"])
def test_full_size_sampled(kernel):
    cfg = W.CONFIGS["cube3d_1e6"]
    src, tgt, q = W.make_problem(cfg)
    helm = kernel == "helmholtz3d"
    kappa = (math.pi / 2) * cfg.side if helm else 0.0
    if helm:
        q = W.weights_complex(cfg.n, cfg.seed)
    with p2p.Plan(src, tgt, level=cfg.level, layout="nr", precision="fp32", kernel=kernel, wavenumber=kappa) as pl:
        got = _run(pl, q, "user")
    sel = np.random.default_rng(2).choice(cfg.n, 3000, replace=False)
    ref, _ = oracle.direct_3d(src, q, tgt, cfg.level, "helmholtz" if helm else "laplace", kappa, targets=sel)
    assert np.linalg.norm(got[sel] - ref) / np.linalg.norm(ref) <= 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("level", [1, 2])
@pytest.mark.parametrize("kernel", ["laplace3d", "helmholtz3d"])
def test_coarse_levels(level, kernel):
    """One box (L = 1) and 2x2x2 boxes (L = 2): every box neighbours every other."""
    import torch
    rng = np.random.default_rng(level)
    src, tgt = rng.random((300, 3)), rng.random((200, 3))
    helm = kernel == "helmholtz3d"
    q = rng.uniform(-1, 1, 300) + (1j * rng.uniform(-1, 1, 300) if helm else 0)
    ref, pairs = oracle.direct_3d(src, q, tgt, level, "helmholtz" if helm else "laplace", 3.0)
    assert pairs == 300 * 200
    with p2p.Plan(src, tgt, level=level, layout="nr", precision="fp64", kernel=kernel, wavenumber=3.0) as pl:
        out = pl.apply(torch.as_tensor(q, dtype=pl.torch_dtype, device="cuda"), order="user")
        torch.cuda.synchronize()
        got = out.cpu().numpy()
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-12
