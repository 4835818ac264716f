"""The fp64 kernels' table-driven log (csrc/p2p_kernels.cuh log_tab) replayed on the
host step by step: x = m 2^e, k = top 8 mantissa bits, t = fma(m, c_inv_k, -1), degree-5 log1p,
fma(e, ln2, L_k + log1p(t)).  Checked against math.log over many exponents and every table cell."""
import math

import numpy as np


def _table():
    k = np.arange(256)
    cinv = 1.0 / (1.0 + (k + 0.5) / 256.0)
    L = -np.log(cinv.astype(np.longdouble))  # 64-bit mantissa, as the plan builder's logl
    return cinv, L.astype(np.float64)


def _fma(a, b, c):  # exact a*b + c rounded once (long double holds the 106-bit product closely enough here)
    return (np.longdouble(a) * np.longdouble(b) + np.longdouble(c)).astype(np.float64)


def log_tab(x):
    cinv, L = _table()
    b = np.asarray(x, dtype=np.float64).view(np.int64)
    e = (b >> 52) - 1023
    k = (b >> 44) & 255
    m = ((b & 0x000FFFFFFFFFFFFF) | 0x3FF0000000000000).view(np.float64)
    t = _fma(m, cinv[k], -1.0)
    q = _fma(t, 0.2, -0.25)
    q = _fma(t, q, 1.0 / 3.0)
    q = _fma(t, q, -0.5)
    p = _fma(t * t, q, t)
    de = e.astype(np.float64)
    return _fma(de, 6.93147180559945309417e-01, L[k] + p)


def test_t_range():
    cinv, _ = _table()
    k = np.arange(256)
    lo, hi = 1.0 + k / 256.0, 1.0 + (k + 1) / 256.0
    assert np.all(np.abs(lo * cinv - 1) < 2 ** -9) and np.all(np.abs(hi * cinv - 1) < 2 ** -9)


def test_log_table_accuracy():
    rng = np.random.default_rng(7)
    # r^2 of near-field pairs: 1e-24 (the guard) .. 1 (the root box), plus every table cell at 1
    x = np.concatenate([10.0 ** rng.uniform(-24, 0.5, 200000), 1.0 + (np.arange(256) + rng.random(256)) / 256,
                        np.nextafter(1.0, 0.0) - np.arange(64) * 2.0 ** -52, [1.0, 2.0, 0.5, 1e-24]])
    got = log_tab(x)
    ref = np.array([math.log(v) for v in x])
    err = np.abs(got - ref)
    # absolute error ~ the ulp of the larger of |log x| and |e ln2|: never more than a few ulp of 1
    assert np.max(err / np.maximum(1.0, np.abs(ref))) < 4 * 2.0 ** -52
