"""Synthetic workload generator (host only): the weak-scaling plates keep the density."""
import numpy as np
import pytest

from paper_2403_01596_b200 import workloads as W


@pytest.mark.parametrize("name", ["d16_1e6", "d32_1e6", "d64_1e6", "surf_2e7"])
@pytest.mark.parametrize("factor", [1, 2, 4, 8])
def test_widened_keeps_density(name, factor):
    base = W.CONFIGS[name]
    c = W.widened(base, factor)
    assert c.n == base.n * factor
    assert c.sx * c.sy == base.sx * base.sy * factor
    assert c.density == base.density
    assert max(c.sx, c.sy) <= c.side <= 2 * max(c.sx, c.sy) or c.level == base.level
    assert c.level <= W.MAX_LEVEL


def test_widened_points_on_plate():
    c = W.widened(W.CONFIGS["tiny"], 4)
    src, tgt, q = W.make_problem(c)
    h = 1.0 / c.side
    for p in (src, tgt):
        assert p[:, 0].max() < c.sx * h and p[:, 1].max() < c.sy * h and p.min() >= 0
    # iid occupancy: the mean count per plate box is the base density
    ix = np.floor(tgt[:, 0] / h).astype(int)
    iy = np.floor(tgt[:, 1] / h).astype(int)
    assert np.bincount(iy * c.sx + ix, minlength=c.sx * c.sy).mean() == pytest.approx(W.CONFIGS["tiny"].density)


def test_widened_level_cap():
    with pytest.raises(ValueError):
        W.widened(W.CONFIGS["lowd025_1e7"], 8)


@pytest.mark.parametrize("kind", ["iid", "stratified"])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_problem_share_is_a_subset(kind, world):
    """A rank's share (DistributedP2P.from_local input) is exactly the global points at its ids."""
    c = W.CONFIGS["tiny"]
    s, t, q = W.make_problem(c, kind=kind)
    seen = []
    for r in range(world):
        a, b, i, j = W.problem_share(c, r, world, kind)
        assert np.array_equal(a, s[i]) and np.array_equal(b, t[j])
        assert np.array_equal(W.weights(c.n, c.seed, index=i), q[i])
        seen.append(i)
    assert np.array_equal(np.sort(np.concatenate(seen)), np.arange(c.n))
