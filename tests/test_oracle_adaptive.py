"""Pins of the adaptive-tree oracle (oracle.c oracle_adaptive_*; SURVEY.md §8(f) NEXT-4,
DESIGN.md R25): CT-driven leaves, U-lists = leaves touching the target's leaf.

Against something other than itself: a stratified cloud filling the whole grid at exactly CT
points per box builds the uniform tree at that level, where the U-list is the 3x3 block -- the
result must equal the (separately pinned) uniform-grid oracle; a hand-built two-level tree with
its leaves and adjacencies counted by hand; reciprocity (the touching relation is symmetric)."""
import numpy as np
import pytest

import oracle
from paper_2403_01596_b200 import workloads as W


@pytest.mark.parametrize("level,d", [(3, 4), (4, 6)])
def test_uniform_tree_reduces_to_the_grid_oracle(level, d):
    S = 1 << (level - 1)
    cfg = W.PlateConfig("full", S, S, level, S * S * d, seed=level)
    src, tgt, q = W.make_problem(cfg, kind="stratified")
    leaves = oracle.adaptive_tree(src, tgt, ct=d, l_max=12)
    assert len(leaves) == S * S and np.all(leaves[:, 0] == level)
    a, pa = oracle.adaptive_direct(src, q, tgt, ct=d, l_max=12)
    b, pb = oracle.direct(src, q, tgt, level)
    assert pa == pb and np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(b))


def test_hand_built_two_level_tree():
    """Five points in the lower-left quarter, none elsewhere, CT = 1, l_max = 3: the root splits;
    the lower-left child (level 2) holds 5 > 1 and splits again into four level-3 boxes; the other
    three level-2 children are leaves.  7 leaves in Morton order."""
    pts = np.array([[0.05, 0.05], [0.2, 0.05], [0.05, 0.2], [0.2, 0.2], [0.21, 0.21]])
    leaves = oracle.adaptive_tree(pts, pts, ct=1, l_max=3)
    assert leaves.tolist() == [[3, 0, 0], [3, 1, 0], [3, 0, 1], [3, 1, 1], [2, 1, 0], [2, 0, 1], [2, 1, 1]]
    # q = 1 at every point; all four level-3 boxes touch each other, so every target sees all 5
    # sources (its own removed by the guard)
    phi, pairs = oracle.adaptive_direct(pts, np.ones(5), pts, ct=1, l_max=3)
    assert pairs == 25  # every leaf holding points touches every other (all within [0, 0.5]^2)
    want0 = -0.5 * sum(np.log(np.sum((pts[0] - p) ** 2)) for p in pts[1:])
    assert phi[0] == pytest.approx(want0, rel=1e-14)


def test_reciprocity_and_linearity():
    rng = np.random.default_rng(3)
    # clustered: a dense blob and a sparse background -> leaves at several levels
    s = np.concatenate([rng.random((300, 2)), 0.3 + 0.05 * rng.random((500, 2))])
    t = np.concatenate([rng.random((250, 2)), 0.3 + 0.05 * rng.random((450, 2))])
    q, w = rng.uniform(-1, 1, len(s)), rng.uniform(-1, 1, len(t))
    leaves = oracle.adaptive_tree(s, t, ct=12, l_max=10)
    assert len(set(leaves[:, 0])) >= 3
    A, _ = oracle.adaptive_direct(s, q, t, ct=12, l_max=10)
    AT, _ = oracle.adaptive_direct(t, w, s, ct=12, l_max=10)  # same tree: max(#src, #tgt) is symmetric
    assert np.dot(w, A) == pytest.approx(np.dot(q, AT), rel=1e-12)
    B, _ = oracle.adaptive_direct(s, 2 * q - 1, t, ct=12, l_max=10)
    ones, _ = oracle.adaptive_direct(s, np.ones(len(s)), t, ct=12, l_max=10)
    assert np.allclose(B, 2 * A - ones, rtol=0, atol=1e-10)
