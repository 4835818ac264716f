"""Pins of the 3D oracle (oracle.c oracle_direct_3d, R24):
phi_t = sum over the 3x3x3 neighbour boxes of q_s G(r), G = 1/(4 pi r) (Laplace) or
e^{i kappa r}/(4 pi r) (Helmholtz), on the octree leaf grid of the unit cube.

Against something other than the oracle: the box-centre lattice closed forms (the 26 neighbour
offsets at distances h, sqrt(2) h, sqrt(3) h, clipped at the faces), brute force over all pairs,
(Delta + kappa^2) G = 0 off the source, the unit point-source flux, the small-kappa limit, and
reciprocity."""
import itertools
import math

import numpy as np
import pytest

import oracle


def _centres(level):
    S = 1 << (level - 1)
    g = (np.arange(S) + 0.5) / S
    z, y, x = np.meshgrid(g, g, g, indexing="ij")
    return np.stack([x.ravel(), y.ravel(), z.ravel()], axis=1), S


@pytest.mark.parametrize("kernel,kappa", [("laplace", 0.0), ("helmholtz", 9.0)])
def test_box_centre_lattice_closed_form(kernel, kappa):
    level = 4
    p, S = _centres(level)
    h = 1.0 / S
    q = np.ones(len(p), dtype=complex if kernel == "helmholtz" else float)
    phi, pairs = oracle.direct_3d(p, q, p, level, kernel, kappa)
    idx = np.floor(p * S).astype(int)
    for t in range(len(p)):
        want = 0.0
        for o in itertools.product((-1, 0, 1), repeat=3):
            if o == (0, 0, 0) or any(not (0 <= idx[t, d] + o[d] < S) for d in range(3)):
                continue
            r = h * math.sqrt(sum(v * v for v in o))
            want += (np.exp(1j * kappa * r) if kernel == "helmholtz" else 1.0) / (4 * math.pi * r)
        assert abs(phi[t] - want) <= 1e-12 * abs(want)
    interior = (4 * math.pi * h) ** -1 * (6 + 12 / math.sqrt(2) + 8 / math.sqrt(3))
    if kernel == "laplace":
        assert phi.max() == pytest.approx(interior, rel=1e-14)
    assert pairs == sum(np.prod([3 - (i == 0) - (i == S - 1) for i in row]) for row in idx)


@pytest.mark.parametrize("seed,level,kernel", [(1, 3, "laplace"), (2, 4, "laplace"), (3, 3, "helmholtz"),
                                              (4, 4, "helmholtz")])
def test_direct_matches_bruteforce(seed, level, kernel):
    rng = np.random.default_rng(seed)
    s, t = rng.random((700, 3)), rng.random((650, 3))
    q = rng.uniform(-1, 1, 700) + (1j * rng.uniform(-1, 1, 700) if kernel == "helmholtz" else 0)
    a, pa = oracle.direct_3d(s, q, t, level, kernel, 17.0)
    b, pb = oracle.bruteforce_3d(s, q, t, level, kernel, 17.0)
    assert pa == pb and np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(b))


def _G(x, kappa):
    src = np.array([[0.5, 0.5, 0.5]])
    phi, _ = oracle.direct_3d(src, np.array([1.0 + 0j]), np.asarray(x, float).reshape(1, 3), 1, "helmholtz", kappa)
    return phi[0]


@pytest.mark.parametrize("kappa", [1.0, 30.0])
def test_helmholtz_equation_and_unit_source(kappa):
    d = np.array([0.3, -0.2, 0.6]) / np.linalg.norm([0.3, -0.2, 0.6])
    for r in (0.5 / kappa, 2.0 / kappa):
        r = min(r, 0.2)
        x = np.array([0.5, 0.5, 0.5]) + r * d
        e = 1e-3 * r
        lap = sum(_G(x + e * u, kappa) + _G(x - e * u, kappa) - 2 * _G(x, kappa) for u in np.eye(3)) / e ** 2
        assert abs(lap + kappa ** 2 * _G(x, kappa)) <= 1e-5 * kappa ** 2 * abs(_G(x, kappa))
    rho, dr = 1e-5, 1e-8
    c = np.array([0.5, 0.5, 0.5])
    flux = 4 * math.pi * rho ** 2 * (_G(c + (rho + dr) * d, kappa) - _G(c + (rho - dr) * d, kappa)) / (2 * dr)
    assert flux.real == pytest.approx(-1.0, abs=1e-5)


def test_small_kappa_limit_and_reciprocity():
    rng = np.random.default_rng(5)
    s, t = rng.random((500, 3)), rng.random((500, 3))
    q = rng.uniform(-1, 1, 500)
    lap, _ = oracle.direct_3d(s, q, t, 3, "laplace")
    kappa = 1e-5
    hel, _ = oracle.direct_3d(s, q.astype(complex), t, 3, "helmholtz", kappa)
    assert np.allclose(hel.real, lap, rtol=0, atol=1e-9 * np.abs(lap).max())
    # Im G = sin(kappa r) / (4 pi r) -> kappa / (4 pi): sum of q over the neighbour set
    qsum = hel.imag * 4 * math.pi / kappa
    brute = np.array([sum(q[j] for j in range(500)
                          if np.all(np.abs(np.floor(s[j] * 4) - np.floor(t[i] * 4)) <= 1)) for i in range(40)])
    assert np.allclose(qsum[:40], brute, atol=1e-6)
    w = rng.uniform(-1, 1, 500) + 1j * rng.uniform(-1, 1, 500)
    qc = q + 1j * rng.uniform(-1, 1, 500)
    A, _ = oracle.direct_3d(s, qc, t, 3, "helmholtz", 12.0)
    AT, _ = oracle.direct_3d(t, w, s, 3, "helmholtz", 12.0)
    assert np.sum(w * A) == pytest.approx(np.sum(qc * AT), rel=1e-12)
