"""ADAPTIVE layout (include/p2p.h P2P_LAYOUT_ADAPTIVE; R25):
the CT-driven quadtree and its U-lists bit-exact against the pinned oracle's tree and a brute-force
touching test; GPU results against the oracle (relative L2 1e-5 fp32, 1e-12 fp64)."""
import numpy as np
import pytest

import oracle
from paper_2403_01596_b200 import p2p
from paper_2403_01596_b200 import workloads as W


def _clustered(n, seed):
    """A uniform background, a dense blob and a curve: leaves at many levels."""
    rng = np.random.default_rng(seed)
    a = rng.random((n // 3, 2))
    b = 0.62 + 0.03 * rng.random((n // 3, 2))
    c = W.contour_points(W.ContourConfig("c", n - 2 * (n // 3), 12, seed=seed))
    return np.concatenate([a, b, c])


CASES = [(2000, 3, 10, 9), (6000, 4, 16, 11), (6000, 5, 6, 12)]


def _touch(A, B, lmax):
    sa, sb = 1 << (lmax - A[0]), 1 << (lmax - B[0])
    return (A[1] * sa <= (B[1] + 1) * sb and B[1] * sb <= (A[1] + 1) * sa and
            A[2] * sa <= (B[2] + 1) * sb and B[2] * sb <= (A[2] + 1) * sa)


@pytest.mark.parametrize("n,seed,ct,lmax", CASES)
def test_tree_and_ulists_bit_exact(n, seed, ct, lmax):
    src, tgt = _clustered(n, seed), _clustered(n, seed + 100)
    with p2p.Plan(src, tgt, layout="adaptive", ct=ct, l_max=lmax, device=-1) as pl:
        leaves = pl.export("leaves").reshape(-1, 3)
        assert np.array_equal(leaves, oracle.adaptive_tree(src, tgt, ct, lmax))
        assert len(set(leaves[:, 0])) >= 3
        off, ul = pl.export("ulist_offsets"), pl.export("ulist")
        # target leaves: those holding a target (oracle cell test)
        has_t = np.zeros(len(leaves), bool)
        for x, y in tgt:
            for i, (L, ix, iy) in enumerate(leaves):
                S = 1 << (L - 1)
                if min(int(x * S), S - 1) == ix and min(int(y * S), S - 1) == iy:
                    has_t[i] = True
                    break
        for i in range(len(leaves)):
            want = [j for j in range(len(leaves)) if _touch(leaves[i], leaves[j], lmax)] if has_t[i] else []
            assert ul[off[i]:off[i + 1]].tolist() == want, i
        _, pairs = oracle.adaptive_direct(src, np.ones(len(src)), tgt, ct, lmax)
        assert pl.info["pairs"] == pairs


def test_adaptive_envelope():
    src, tgt = _clustered(300, 1), _clustered(300, 2)
    for kw, st in ((dict(kernel="helmholtz", wavenumber=3.0), p2p.P2P_ERROR_NOT_SUPPORTED),
                   (dict(part_world=2), p2p.P2P_ERROR_NOT_SUPPORTED),
                   (dict(ct=0), p2p.P2P_ERROR_INVALID_ARGUMENT)):
        with pytest.raises(p2p.P2PError) as ei:
            p2p.Plan(src, tgt, layout="adaptive", device=-1, **kw)
        assert ei.value.status == st, kw


@pytest.mark.gpu
@pytest.mark.parametrize("n,seed,ct,lmax", CASES)
@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_against_oracle(n, seed, ct, lmax, prec):
    import torch
    src, tgt = _clustered(n, seed), _clustered(n, seed + 100)
    q = W.weights(n, seed)
    ref, pairs = oracle.adaptive_direct(src, q, tgt, ct, lmax)
    with p2p.Plan(src, tgt, layout="adaptive", ct=ct, l_max=lmax, precision=prec) as pl:
        assert pl.info["pairs"] == pairs
        out = pl.apply(torch.as_tensor(q, dtype=pl.torch_dtype, device="cuda"), order="user")
        torch.cuda.synchronize()
        got = out.double().cpu().numpy()
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= (1e-5 if prec == "fp32" else 1e-12)
        qp = torch.as_tensor(q[pl.export("src_perm")], dtype=pl.torch_dtype, device="cuda")
        outp = pl.apply(qp)
        torch.cuda.synchronize()
        assert np.array_equal(outp.double().cpu().numpy(), got[pl.export("tgt_perm")])
        assert np.array_equal(pl.apply_host(q.astype(pl.np_dtype), order="user").astype(np.float64), got)


@pytest.mark.gpu
def test_uniform_tree_matches_the_grid_path():
    """A full stratified grid at CT points per box builds the uniform tree: same sums as the
    uniform TILED plan at that level (both fp64, tolerance-level agreement)."""
    import torch
    level, d = 6, 8
    S = 1 << (level - 1)
    cfg = W.PlateConfig("full", S, S, level, S * S * d, seed=4)
    src, tgt, q = W.make_problem(cfg, kind="stratified")
    with p2p.Plan(src, tgt, layout="adaptive", ct=d, l_max=12, precision="fp64") as pa, \
            p2p.Plan(src, tgt, level=level, layout="tiled", precision="fp64") as pt:
        assert pa.info["pairs"] == pt.info["pairs"]
        qd = torch.as_tensor(q, device="cuda")
        a, b = pa.apply(qd, order="user"), pt.apply(qd, order="user")
        torch.cuda.synchronize()
        assert torch.allclose(a, b, rtol=0, atol=1e-12 * float(b.abs().max()))


@pytest.mark.gpu
def test_single_leaf_and_deep_cap():
    """CT >= n: the root is the only leaf (every pair interacts); l_max = 1 caps the split."""
    import torch
    rng = np.random.default_rng(5)
    src, tgt = rng.random((400, 2)), rng.random((300, 2))
    q = rng.uniform(-1, 1, 400)
    for ct, lmax in ((1000, 12), (5, 1)):
        ref, pairs = oracle.adaptive_direct(src, q, tgt, ct, lmax)
        assert pairs == 400 * 300
        with p2p.Plan(src, tgt, layout="adaptive", ct=ct, l_max=lmax, precision="fp64") as pl:
            assert pl.export("leaves").tolist() == [1, 0, 0]
            out = pl.apply(torch.as_tensor(q, device="cuda"), order="user")
            torch.cuda.synchronize()
            assert np.linalg.norm(out.cpu().numpy() - ref) / np.linalg.norm(ref) <= 1e-12
