"""The 2D Helmholtz near field (include/p2p.h P2P_KERNEL_HELMHOLTZ_2D)
through the C ABI against the fp64 oracle (oracle.direct_helmholtz, pinned in
tests/test_oracle_helmholtz.py).

Gate (R23; north_star): relative L2 <= 1e-5 (fp32), <= 1e-12 (fp64) at every kappa:
the fp64 kernel takes the ascending series up to kappa r = 6 and the modulus / phase form of
H0^(1) beyond (|error| < 2e-17 + the rounding of kappa r itself)."""
import math

import numpy as np
import pytest

import oracle
from paper_2403_01596_b200 import p2p
from paper_2403_01596_b200 import workloads as W


def _kappa(level, kh):
    return kh * (1 << (level - 1))  # kappa h = kh


# ------------------------------------------------------------------ host-only checks
def test_helmholtz_envelope_errors():
    src, tgt, _ = W.make_problem("tiny")
    for kw, st in ((dict(layout="nr", wavenumber=5.0), p2p.P2P_ERROR_NOT_SUPPORTED),
                   (dict(layout="tiled", wavenumber=0.0), p2p.P2P_ERROR_INVALID_ARGUMENT),
                   (dict(layout="tiled", wavenumber=float("nan")), p2p.P2P_ERROR_INVALID_ARGUMENT)):
        with pytest.raises(p2p.P2PError) as ei:
            p2p.Plan(src, tgt, level=4, device=-1, kernel="helmholtz", **kw)
        assert ei.value.status == st, kw


def test_helmholtz_host_plan_info():
    src, tgt, _ = W.make_problem("tiny")
    with p2p.Plan(src, tgt, level=4, device=-1, layout="tiled", kernel="helmholtz", wavenumber=7.5) as pl:
        i = pl.info
        assert (i["kernel"], i["components"], i["wavenumber"]) == (p2p.P2P_KERNEL_HELMHOLTZ_2D, 2, 7.5)
        assert i["slots_per_unit"] == 1 and i["items_per_unit"] == 1 and i["flags"] == 3
        assert i["pairs"] == oracle.pair_count(src, tgt, 4)
    with p2p.Plan(src, tgt, level=4, device=-1, layout="tiled") as pl:
        assert pl.info["components"] == 1 and pl.info["kernel"] == p2p.P2P_KERNEL_LAPLACE_2D


# ------------------------------------------------------------------ GPU parity
def _q(n, seed):
    return W.weights(n, seed) + 1j * W.weights(n, seed, stream=5)


def _tol(prec, kappa, level):
    return 1e-5 if prec == "fp32" else 1e-12


def _run(pl, q, order="user", out=None, accumulate=False):
    import torch
    qq = q if order == "user" else q[pl.export("src_perm")]
    qd = torch.as_tensor(qq, dtype=pl.torch_dtype, device="cuda")
    r = pl.apply(qd, out, order=order, accumulate=accumulate)
    torch.cuda.synchronize()
    return r.cpu().numpy().astype(np.complex128)


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("level", [4, 6])
@pytest.mark.parametrize("kh", [0.05, 1.0, 2.0, 6.0])
@pytest.mark.parametrize("build", ["host", "device"])
def test_tiny_against_oracle(prec, level, kh, build):
    src, tgt, _ = W.make_problem("tiny")
    q = _q(len(src), 1)
    kappa = _kappa(level, kh)
    ref, pairs = oracle.direct_helmholtz(src, q, tgt, level, kappa)
    with p2p.Plan(src, tgt, level=level, layout="tiled", precision=prec, kernel="helmholtz",
                  wavenumber=kappa, build=build) as pl:
        assert pl.info["pairs"] == pairs
        got = _run(pl, q, "user")
        assert _rel(got, ref) <= _tol(prec, kappa, level), _rel(got, ref)
        got_p = _run(pl, q, "plan")
        assert np.array_equal(got_p, got[pl.export("tgt_perm")])  # same sums, plan order


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("kind", ["iid", "stratified"])
def test_plate_against_oracle(prec, kind):
    cfg = W.PlateConfig("helm_s", 96, 64, 8, 96 * 64 * 16, seed=12)
    src, tgt, _ = W.make_problem(cfg, kind=kind)
    q = _q(len(src), 12)
    kappa = _kappa(cfg.level, math.pi / 2)  # leaf box = a quarter wavelength
    ref, _ = oracle.direct_helmholtz(src, q, tgt, cfg.level, kappa)
    with p2p.Plan(src, tgt, level=cfg.level, layout="tiled", precision=prec, kernel="helmholtz",
                  wavenumber=kappa) as pl:
        got = _run(pl, q)
        assert _rel(got, ref) <= _tol(prec, kappa, cfg.level)


@pytest.mark.gpu
def test_accumulate_determinism_and_device_build_identity():
    import torch
    cfg = W.PlateConfig("helm_a", 64, 48, 8, 64 * 48 * 4, seed=13)
    src, tgt, _ = W.make_problem(cfg)
    q = _q(len(src), 13)
    kappa = _kappa(cfg.level, 1.2)
    kw = dict(level=cfg.level, layout="tiled", precision="fp32", kernel="helmholtz", wavenumber=kappa)
    with p2p.Plan(src, tgt, **kw) as h, p2p.Plan(src, tgt, build="device", **kw) as d:
        a = _run(h, q)
        assert np.array_equal(a, _run(h, q))                     # bit-reproducible
        assert np.array_equal(a, _run(d, q))                     # device-built plan: same bits
        for kind in ("region_index", "slot_base", "launch", "tgt_perm"):
            assert np.array_equal(h.export(kind), d.export(kind))
        base = torch.full((len(tgt),), 1.0 - 2.0j, dtype=h.torch_dtype, device="cuda")
        acc = _run(h, q, "user", out=base.clone(), accumulate=True)
        assert np.allclose(acc, a + (1.0 - 2.0j), rtol=0, atol=1e-5)
        # host buffers through the C ABI
        out = h.apply_host(q.astype(np.complex64), order="user")
        assert np.array_equal(out.astype(np.complex128), a)


@pytest.mark.gpu
def test_full_size_sample():
    """BASELINE.json d16_1e6 plate at a quarter-wavelength leaf box, fp32, on sampled targets."""
    cfg = W.CONFIGS["d16_1e6"]
    src, tgt, _ = W.make_problem(cfg)
    q = _q(len(src), 14)
    kappa = _kappa(cfg.level, math.pi / 2)
    with p2p.Plan(src, tgt, level=cfg.level, layout="tiled", precision="fp32", kernel="helmholtz",
                  wavenumber=kappa, build="device") as pl:
        got = _run(pl, q)
    sel = np.random.default_rng(0).choice(len(tgt), 4000, replace=False)
    ref, _ = oracle.direct_helmholtz(src, q, tgt, cfg.level, kappa, targets=sel)
    assert _rel(got[sel], ref) <= 1e-5
