"""Pins of the 2D Helmholtz oracle (oracle.c; R23):
G(r) = (i/4) H0^(1)(kappa r) = (-Y0(kappa r) + i J0(kappa r)) / 4, phi_t = sum_{E1} q_s G(r_ts).

Each pin checks the oracle against something other than itself:
  * tabulated Bessel values and zeros (Abramowitz & Stegun, tests/golden/helmholtz_bessel.json);
  * the defining properties of the fundamental solution: (Delta + kappa^2) G = 0 off the source
    (finite differences), unit flux 2 pi rho dG/drho -> -1 (the delta source), Im G(0+) = 1/4,
    and the outgoing (Sommerfeld) far-field phase of H0^(1) (not H0^(2));
  * the small-kappa limit against the (separately pinned) Laplace oracle:
    Re phi = phi_laplace / (2 pi) - (ln(kappa/2) + gamma) / (2 pi) * sum_{E1} q_s + O((kappa r)^2 ln);
  * brute force over all pairs, reciprocity (G symmetric, bilinear form), complex linearity."""
import json
import math
import os

import numpy as np
import pytest

import oracle
from paper_2403_01596_b200 import workloads as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "helmholtz_bessel.json")))


@pytest.mark.parametrize("row", GOLD["values"], ids=lambda r: f"x={r['x']}")
def test_tabulated_bessel_values(row):
    kappa = 3.0
    g = oracle.pair_helmholtz((0.1, 0.2), (0.1 + row["x"] / kappa, 0.2), 1.0, kappa)
    assert g.real == pytest.approx(-row["Y0"] / 4, rel=1e-12, abs=1e-14)
    assert g.imag == pytest.approx(row["J0"] / 4, rel=1e-12, abs=1e-14)
    # q = i rotates: i G = (-J0 - i Y0)/4
    gi = oracle.pair_helmholtz((0.1, 0.2), (0.1, 0.2 + row["x"] / kappa), 1j, kappa)
    assert gi.real == pytest.approx(-row["J0"] / 4, rel=1e-12, abs=1e-14)
    assert gi.imag == pytest.approx(-row["Y0"] / 4, rel=1e-12, abs=1e-14)


def test_zeros():
    z = GOLD["zeros"]
    kappa = 2.0
    assert abs(oracle.pair_helmholtz((0, 0), (z["j01"] / kappa, 0), 1.0, kappa).imag) < 1e-15
    assert abs(oracle.pair_helmholtz((0, 0), (0, z["y01"] / kappa), 1.0, kappa).real) < 1e-15


@pytest.mark.parametrize("kappa", [0.7, 5.0, 40.0])
def test_helmholtz_equation_off_the_source(kappa):
    """(Delta + kappa^2) G = 0 at r > 0 (5-point stencil, O(delta^2))."""
    for r in (0.3 / kappa, 1.0 / kappa, 4.0 / kappa):
        t = np.array([0.5 + r * 0.6, 0.5 + r * 0.8])
        d = 1e-3 * r
        G = lambda p: oracle.pair_helmholtz(p, (0.5, 0.5), 1.0, kappa)  # noqa: E731
        g0 = G(t)
        lap = (G(t + [d, 0]) + G(t - [d, 0]) + G(t + [0, d]) + G(t - [0, d]) - 4 * g0) / d ** 2
        assert abs(lap + kappa ** 2 * g0) <= 1e-5 * kappa ** 2 * max(abs(g0), 0.05)


def test_unit_source_and_regular_part():
    """Delta G + kappa^2 G = -delta: the flux through a small circle is -1; Im G(0+) = J0(0)/4."""
    kappa = 2.5
    rho = 1e-5
    d = 1e-8
    G = lambda r: oracle.pair_helmholtz((0.0, 0.0), (r, 0.0), 1.0, kappa)  # noqa: E731
    flux = 2 * math.pi * rho * (G(rho + d) - G(rho - d)) / (2 * d)
    assert flux.real == pytest.approx(-1.0, abs=1e-6)
    assert G(1e-9).imag == pytest.approx(0.25, abs=1e-12)


def test_outgoing_far_field():
    """H0^(1)(x) ~ sqrt(2/(pi x)) e^{i(x - pi/4)}: G e^{-i kappa r} sqrt(r) -> (i/4) sqrt(2/(pi kappa)) e^{-i pi/4}."""
    kappa = 1.0
    lim = 0.25j * math.sqrt(2 / (math.pi * kappa)) * np.exp(-0.25j * math.pi)
    for x in (500.0, 2000.0):
        g = oracle.pair_helmholtz((0.0, 0.0), (x / kappa, 0.0), 1.0, kappa)
        v = g * np.exp(-1j * x) * math.sqrt(x / kappa)
        assert abs(v - lim) <= 0.2 / x  # next term: O(1/x)
        assert abs(v - np.conj(lim)) > 0.1  # not the incoming H0^(2)


def test_small_kappa_limit_matches_laplace_oracle():
    src, tgt, q = W.make_problem("tiny")
    kappa, level = 1e-4, 4
    phi_h, pairs_h = oracle.direct_helmholtz(src, q.astype(complex), tgt, level, kappa)
    phi_l, pairs_l = oracle.direct(src, q, tgt, level)
    assert pairs_h == pairs_l
    gamma = 0.5772156649015329
    qsum = 4 * phi_h.imag  # sum_{E1} q_s J0(kappa r) = sum q_s (1 + O((kappa r)^2))
    pred = phi_l / (2 * math.pi) - (math.log(kappa / 2) + gamma) / (2 * math.pi) * qsum
    assert np.max(np.abs(phi_h.real - pred)) <= 1e-7 * np.max(np.abs(phi_h.real))


@pytest.mark.parametrize("seed,level,kappa", [(1, 3, 5.0), (2, 4, 20.0), (3, 5, 60.0)])
def test_direct_matches_bruteforce(seed, level, kappa):
    src, tgt, qr = W.uniform_unit(600, seed)
    q = qr + 1j * W.weights(600, seed, stream=5)
    a, pa = oracle.direct_helmholtz(src, q, tgt, level, kappa)
    b, pb = oracle.bruteforce_helmholtz(src, q, tgt, level, kappa)
    assert pa == pb
    assert np.max(np.abs(a - b)) <= 1e-13 * max(1.0, np.max(np.abs(b)))


def test_reciprocity_and_linearity():
    src, tgt, _ = W.uniform_unit(500, 7)
    rng = np.random.default_rng(0)
    q = rng.standard_normal(500) + 1j * rng.standard_normal(500)
    w = rng.standard_normal(500) + 1j * rng.standard_normal(500)
    level, kappa = 4, 12.0
    Aq, _ = oracle.direct_helmholtz(src, q, tgt, level, kappa)
    ATw, _ = oracle.direct_helmholtz(tgt, w, src, level, kappa)
    assert np.sum(w * Aq) == pytest.approx(np.sum(q * ATw), rel=1e-12)
    q2 = rng.standard_normal(500) + 1j * rng.standard_normal(500)
    al, be = 0.3 - 1.2j, -2.0 + 0.5j
    lhs, _ = oracle.direct_helmholtz(src, al * q + be * q2, tgt, level, kappa)
    Aq2, _ = oracle.direct_helmholtz(src, q2, tgt, level, kappa)
    assert np.allclose(lhs, al * Aq + be * Aq2, rtol=1e-12, atol=1e-12)


def test_coincident_points_contribute_zero():
    assert oracle.pair_helmholtz((0.3, 0.3), (0.3, 0.3), 1.0, 4.0) == 0
