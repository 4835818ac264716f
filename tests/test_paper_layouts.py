"""The paper's own layouts (PAPER_INDEXING = §3.2, PAPER_REPETITION = §3.3; SURVEY.md §8(f)
NEXT-1) on host-only plans: byte accounting against the oracle's Eq. 3 / Eq. 8, and the
interaction sets against the oracle's independent box assignment and neighbour lists."""
import numpy as np
import pytest

import oracle
from paper_2403_01596_b200 import p2p
from paper_2403_01596_b200 import workloads as W


def _e1_sources_by_box(src, level):
    """Per Morton box: original source indices of its E1 neighbourhood, neighbour boxes ascending
    Morton, sources in original index order (oracle sort + oracle neighbour lists)."""
    perm, off = oracle.sort_points(src, level)
    nb = oracle.neighbors(level)
    return [[int(perm[i]) for m in nb[b] if m >= 0 for i in range(off[m], off[m + 1])] for b in range(len(off) - 1)]


def _box_of(points, level):
    S = 1 << (level - 1)
    ix = np.minimum(np.floor(points[:, 0] * S), S - 1).astype(np.int64)
    iy = np.minimum(np.floor(points[:, 1] * S), S - 1).astype(np.int64)
    return np.array([oracle.morton(int(x), int(y), level) for x, y in zip(ix, iy)])


@pytest.mark.parametrize("level", [1, 3, 4, 5])
def test_paper_indexing_layout(level):
    src, tgt, _ = W.make_problem("tiny")
    with p2p.Plan(src, tgt, level=level, layout="paper_i", precision="fp64", device=-1) as pl:
        t = oracle.box_tmax(src, tgt, level)
        assert pl.info["paper_model_bytes"] == oracle.indexing_bytes(len(src), level, t)   # Eq. 3
        off, idx = pl.export("paper_nei_offsets"), pl.export("paper_nei_index")
        ref = _e1_sources_by_box(src, level)
        assert len(off) == len(ref) + 1 and off[-1] == len(idx)
        for b, lst in enumerate(ref):
            assert idx[off[b]:off[b + 1]].tolist() == lst
        # target lists: the plan's Morton target order, per box (tgt_box_offsets)
        tperm, toff = oracle.sort_points(tgt, level)
        assert np.array_equal(pl.export("tgt_perm"), tperm) and np.array_equal(pl.export("tgt_box_offsets"), toff)


@pytest.mark.parametrize("level,ct", [(3, 15), (4, 15), (5, 4), (4, 64)])
def test_paper_repetition_layout(level, ct):
    src, tgt, _ = W.make_problem("tiny")
    with p2p.Plan(src, tgt, level=level, layout="paper_r", precision="fp64", device=-1, ct=ct) as pl:
        t = oracle.box_tmax(src, tgt, level)
        C = max(ct, t)
        stride = pl.info["record_stride"]
        assert stride == 3 + 27 * C
        assert pl.info["paper_model_bytes"] == oracle.repetition_bytes(len(tgt), ct)      # Eq. 8
        words = pl.export("paper_records").reshape(len(tgt), stride)
        rec = words.view(np.float64)
        count = (words[:, 2] & 0xFFFFFFFF).astype(np.int64)
        assert np.all((words[:, 2] >> 32) == 0) and np.all(count <= 9 * C)          # count slot convention
        ref = _e1_sources_by_box(src, level)
        box = _box_of(tgt, level)
        for r in range(len(tgt)):
            assert rec[r, 0] == tgt[r, 0] and rec[r, 1] == tgt[r, 1]
            lst = ref[box[r]]
            assert count[r] == len(lst)
            trip = rec[r, 3:3 + 3 * count[r]].reshape(-1, 3)
            assert np.array_equal(trip[:, :2], src[lst])                            # same sources, same order
            assert np.all(rec[r, 3 + 3 * count[r]:] == 0)                            # zero-filled tail


def test_paper_layout_bytes_vs_ours():
    """The redundancy premise (SPEC.md layouts invariant): Repetition bytes >= Indexing bytes for D >= 1."""
    src, tgt, _ = W.make_problem("tiny")
    for level in (3, 4):
        with p2p.Plan(src, tgt, level=level, layout="paper_i", precision="fp64", device=-1) as a, \
                p2p.Plan(src, tgt, level=level, layout="paper_r", precision="fp64", device=-1) as b:
            assert b.info["paper_model_bytes"] >= a.info["paper_model_bytes"]


def test_paper_layouts_reject_fp32_and_partitions():
    src, tgt, _ = W.make_problem("tiny")
    for lay in ("paper_i", "paper_r"):
        with pytest.raises(p2p.P2PError):
            p2p.Plan(src, tgt, level=4, layout=lay, precision="fp32", device=-1)
        with pytest.raises(p2p.P2PError):
            p2p.Plan(src, tgt, level=4, layout=lay, precision="fp64", device=-1, part_world=2, part_rank=0)
