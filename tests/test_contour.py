"""Curve-concentrated clouds (workloads.ContourConfig): boundary nodes of
a 2D scatterer, collocated sources and targets, most leaf boxes empty.  Same bars as the plate
workloads: parity with the fp64 oracle (relative L2 1e-5 fp32 / 1e-12 fp64), the device-built
plan bit-identical to the host-built one."""
import math

import numpy as np
import pytest

import oracle
from paper_2403_01596_b200 import p2p
from paper_2403_01596_b200 import workloads as W

SMALL = W.ContourConfig("contour_s", 20_000, 11, seed=5)


def test_contour_points_lie_on_the_curve():
    c = W.CONFIGS["contour_2e5"]
    p = W.contour_points(c)
    assert p.shape == (c.n, 2) and p.min() > 0.04 and p.max() < 0.96
    d = p - 0.5
    t = np.arctan2(d[:, 1], d[:, 0])
    r = np.hypot(d[:, 0], d[:, 1])
    assert np.allclose(r, c.r0 * (1 + c.a * np.cos(c.m * t)), rtol=0, atol=1e-12)
    s, tg, q = W.make_problem(c)
    assert np.array_equal(s, tg) and len(q) == c.n  # collocated


@pytest.mark.gpu
@pytest.mark.parametrize("layout", ["nr", "tiled"])
@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_small_contour_against_oracle(layout, prec):
    import torch
    src, tgt, q = W.make_problem(SMALL)
    ref, pairs = oracle.direct(src, q, tgt, SMALL.level)
    with p2p.Plan(src, tgt, level=SMALL.level, layout=layout, precision=prec) as h, \
            p2p.Plan(src, tgt, level=SMALL.level, layout=layout, precision=prec, build="device") as d:
        assert h.info["pairs"] == pairs == d.info["pairs"]
        qd = torch.as_tensor(q, dtype=h.torch_dtype, device="cuda")
        a, b = h.apply(qd, order="user"), d.apply(qd, order="user")
        torch.cuda.synchronize()
        assert torch.equal(a, b)
        got = a.double().cpu().numpy()
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= (1e-5 if prec == "fp32" else 1e-12)
        for kind in ("tgt_perm", "tiles", "launch"):
            assert np.array_equal(h.export(kind), d.export(kind))


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_small_contour_helmholtz(prec):
    import torch
    src, tgt, _ = W.make_problem(SMALL)
    q = W.weights_complex(SMALL.n, SMALL.seed)
    kappa = (math.pi / 2) * SMALL.side
    ref, _ = oracle.direct_helmholtz(src, q, tgt, SMALL.level, kappa)
    with p2p.Plan(src, tgt, level=SMALL.level, layout="tiled", precision=prec, kernel="helmholtz",
                  wavenumber=kappa, build="device") as pl:
        out = pl.apply(torch.as_tensor(q, dtype=pl.torch_dtype, device="cuda"), order="user")
        torch.cuda.synchronize()
        got = out.cpu().numpy().astype(np.complex128)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= (1e-5 if prec == "fp32" else 1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("name,kernel", [("contour_2e5", "laplace"), ("contour_1e5", "helmholtz")])
def test_full_contour_sampled(name, kernel):
    """The bench configs (device-built plans, fp32) on 5000 sampled targets."""
    import torch
    cfg = W.CONFIGS[name]
    src, tgt, q = W.make_problem(cfg)
    kw = {}
    if kernel == "helmholtz":
        q = W.weights_complex(cfg.n, cfg.seed)
        kw = dict(kernel="helmholtz", wavenumber=(math.pi / 2) * cfg.side)
    with p2p.Plan(src, tgt, level=cfg.level, layout="tiled", precision="fp32", build="device", **kw) as pl:
        out = pl.apply(torch.as_tensor(q, dtype=pl.torch_dtype, device="cuda"), order="user")
        torch.cuda.synchronize()
        got = out.cpu().numpy()
    sel = np.random.default_rng(1).choice(cfg.n, 5000, replace=False)
    if kernel == "helmholtz":
        ref, _ = oracle.direct_helmholtz(src, q, tgt, cfg.level, kw["wavenumber"], targets=sel)
    else:
        ref, _ = oracle.direct(src, q, tgt, cfg.level, targets=sel)
    assert np.linalg.norm(got[sel] - ref) / np.linalg.norm(ref) <= 1e-5
