"""Host plan builder vs the oracle's independent indexing (bit-exact), on
host-only plans (device = -1): no GPU needed.

SURVEY.md §8(c) C-2 step 5: the oracle computes Morton codes by a bit loop and
sorts by (code, index) with qsort; the plan builder uses magic-number bit
spreading and a counting sort.  Permutations, box offsets and neighbour lists
must agree bit for bit."""
import numpy as np
import pytest

import oracle
from paper_2403_01596_b200 import p2p
from paper_2403_01596_b200 import workloads as W


def _plan(src, tgt, **kw):
    kw.setdefault("device", -1)
    return p2p.Plan(src, tgt, **kw)


@pytest.mark.parametrize("cfg,kind,level", [
    ("tiny", "iid", 4), ("tiny", "stratified", 4), ("tiny", "iid", 6), ("tiny", "iid", 1),
])
def test_indexing_bit_exact(cfg, kind, level):
    src, tgt, _ = W.make_problem(cfg, kind=kind)
    pl = _plan(src, tgt, level=level)
    for xy, perm_kind, off_kind in ((src, "src_perm", "src_box_offsets"), (tgt, "tgt_perm", "tgt_box_offsets")):
        perm, off = oracle.sort_points(xy, level)
        np.testing.assert_array_equal(pl.export(perm_kind), perm)
        np.testing.assert_array_equal(pl.export(off_kind), off)
    np.testing.assert_array_equal(pl.export("neighbors").reshape(-1, 9), oracle.neighbors(level))


def test_indexing_bit_exact_random_unit():
    src, tgt, _ = W.uniform_unit(3000, 17)
    for level in (2, 5, 7):
        pl = _plan(src, tgt, level=level)
        perm, off = oracle.sort_points(src, level)
        np.testing.assert_array_equal(pl.export("src_perm"), perm)
        np.testing.assert_array_equal(pl.export("src_box_offsets"), off)


def test_duplicates_and_edges_bit_exact():
    # points on cell edges, at x = 1, and exact duplicates exercise the boundary rule and stability
    pts = np.array([[0.0, 0.0], [1.0, 1.0], [0.5, 0.5], [0.5, 0.5], [0.25, 1.0], [1.0, 0.0],
                    [0.125, 0.375], [0.5, 0.5], [np.nextafter(0.5, 0), 0.5]])
    for level in (1, 2, 3, 4):
        pl = _plan(pts, pts, level=level)
        perm, off = oracle.sort_points(pts, level)
        np.testing.assert_array_equal(pl.export("src_perm"), perm)
        np.testing.assert_array_equal(pl.export("tgt_box_offsets"), off)


@pytest.mark.parametrize("seed,n", [(1, 1000), (2, 5000), (3, 20000)])
def test_ct_loop_matches_oracle(seed, n):
    src, tgt, _ = W.uniform_unit(n, seed)
    for ct in (4, 15):
        L = oracle.ct_level(src, tgt, ct, 3, 15)
        assert _plan(src, tgt, ct=ct).info["level"] == L
        assert _plan(src, tgt, ct=ct, level_delta=1).info["level"] == L + 1


def test_spec_stats():
    one = np.array([[0.3, 0.3]])
    info = _plan(one, one, ct=15).info
    assert info["level"] == 3 and info["boxes"] == 16
    src, tgt, _ = W.uniform_unit(4096, 3)
    info = _plan(src, tgt, level=6).info
    assert info["density"] == 4.0
    assert info["density"] * info["boxes"] == 4096


@pytest.mark.parametrize("cfg,kind", [("tiny", "iid"), ("tiny", "stratified"), ("d64_1e6", None)])
def test_pair_count(cfg, kind):
    c = W.CONFIGS[cfg]
    if kind is None:  # a smaller stratified plate at the d64 level
        c = W.PlateConfig("s", 40, 23, c.level, 40 * 23 * 64, seed=5)
        kind = "stratified"
    src, tgt, _ = W.make_problem(c, kind=kind)
    info = _plan(src, tgt, level=c.level).info
    assert info["pairs"] == info["pairs_global"] == oracle.pair_count(src, tgt, c.level)
    if kind == "stratified":
        assert info["pairs"] == c.stratified_pairs()


def _e1_sources(src, tgt_point, level):
    S = 1 << (level - 1)
    bs = np.minimum(np.floor(src * S), S - 1)
    bt = np.minimum(np.floor(tgt_point * S), S - 1)
    return set(np.nonzero((np.abs(bs[:, 0] - bt[0]) <= 1) & (np.abs(bs[:, 1] - bt[1]) <= 1))[0].tolist())


def test_redundant_halo_interaction_set():
    """the pairs implied by the R layout equal the brute-force E1 enumeration."""
    src, tgt, _ = W.uniform_unit(1500, 23)
    level = 5
    pl = _plan(src, tgt, level=level, layout="r")
    hidx = pl.export("halo_index")
    hoff = pl.export("halo_offsets")
    sperm = pl.export("src_perm")
    tperm = pl.export("tgt_perm")
    toff = pl.export("tgt_box_offsets")
    for b in range(len(toff) - 1):
        if toff[b + 1] == toff[b]:
            continue
        ent = hidx[hoff[b]:hoff[b + 1]]
        got = set(sperm[ent[ent >= 0]].tolist())
        assert len(got) == (ent >= 0).sum()  # no duplicates
        assert len(ent) % 2 == 0
        for t in tperm[toff[b]:toff[b + 1]]:
            assert got == _e1_sources(src, tgt[t], level)
    info = pl.info
    assert info["halo_entries"] >= info["pairs"] / 1e9  # trivial sanity
    assert info["halo_entries"] % 4 == 0


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_partition_covers_everything(world):
    src, tgt, _ = W.make_problem("d16_1e6", n=40000)
    level = 7
    plans = [_plan(src, tgt, level=level, part_world=world, part_rank=r) for r in range(world)]
    infos = [p.info for p in plans]
    part = plans[0].export("partition").reshape(2, world + 1)
    for p in plans[1:]:
        np.testing.assert_array_equal(p.export("partition").reshape(2, world + 1), part)
    assert part[0, 0] == 0 and part[0, -1] == len(src) and part[1, -1] == len(tgt)
    assert sum(i["pairs"] for i in infos) == infos[0]["pairs_global"]
    assert sum(i["n_tgt_local"] for i in infos) == len(tgt)
    # balance: no rank above 1/world + one tile's worth of pairs
    assert max(i["pairs"] for i in infos) <= infos[0]["pairs_global"] / world * 1.2
    # owned targets concatenate to the global plan order
    full = _plan(src, tgt, level=level)
    np.testing.assert_array_equal(np.concatenate([p.export("tgt_perm") for p in plans]), full.export("tgt_perm"))
    # halo bookkeeping: what r receives from q is what q sends to r
    counts = [p.export("halo_counts").reshape(2, world) for p in plans]
    for r in range(world):
        for q in range(world):
            assert counts[r][0, q] == counts[q][1, r]
    # each rank's local sources cover the E1 sources of every owned target
    for p in plans:
        loc = set(p.export("src_perm").tolist())
        tp = p.export("tgt_perm")
        for t in tp[:: max(1, len(tp) // 50)]:
            assert _e1_sources(src, tgt[t], level) <= loc


def test_tiled_region_interaction_set():
    """TILED layout: the packed region of each tile holds exactly the sources of
    the tile's boxes and their one-box ring (each once), so every target's E1
    set is covered."""
    src, tgt, _ = W.uniform_unit(2500, 29)
    level = 6
    for tile in (0, 1, 2):
        pl = _plan(src, tgt, level=level, layout="tiled", tile_log2=tile)
        roff = pl.export("region_offsets")
        ridx = pl.export("region_index")
        sperm = pl.export("src_perm")
        tiles_launch = pl.export("tiles")
        assert roff[-1] == len(ridx) and np.all(np.diff(roff) % 4 == 0)
        S = 1 << (level - 1)
        W_ = 1 << tile
        for slot, t in enumerate(np.unique(tiles_launch)):  # slots are Morton tile order (tail tiles repeat)
            ent = ridx[roff[slot]:roff[slot + 1]]
            got = sperm[ent[ent >= 0]]
            assert len(set(got.tolist())) == len(got)
            tx, ty = oracle.morton_decode(int(t), level - tile)
            x0, y0 = tx * W_ - 1, ty * W_ - 1
            bs = np.minimum(np.floor(src * S), S - 1)
            inside = (bs[:, 0] >= x0) & (bs[:, 0] <= x0 + W_ + 1) & (bs[:, 1] >= y0) & (bs[:, 1] <= y0 + W_ + 1)
            assert set(got.tolist()) == set(np.nonzero(inside)[0].tolist())


def _tiled_layout_checks(pl, level, nt):
    """Invariants of the TILED target slots and item lists (plan builder, host only)."""
    k = pl.info["tile_log2"]
    W_, WW = 1 << k, 1 << (2 * k)
    R, RR = W_ + 2, (W_ + 2) ** 2
    stride = (RR + 2 + 7) & ~7
    tiles = np.unique(pl.export("tiles"))  # Morton slot order
    soff, sbase, sout = pl.export("slot_offsets"), pl.export("slot_base"), pl.export("slot_output")
    table = pl.export("region_table").reshape(len(tiles), stride)
    toff = pl.export("tgt_box_offsets")
    ioff, items = pl.export("item_offsets"), pl.export("items")
    launch = pl.export("launch").reshape(2, -1)
    nparts = {int(s): int(p) >> 16 for s, p in zip(launch[0], launch[1])}
    assert np.all(soff % 8 == 0)
    tpi = pl.info["slots_per_unit"]
    assert (len(items) > 0) == (pl.info["items_per_unit"] == 3)
    for i, t in enumerate(tiles):
        nslot = int(table[i, RR + 1])
        assert soff[i] + nslot <= soff[i + 1]
        o, b = sout[soff[i]:soff[i] + nslot], sbase[soff[i]:soff[i] + nslot]
        g0, n = toff[t * WW], toff[(t + 1) * WW] - toff[t * WW]
        real = o[o >= 0]
        assert np.array_equal(np.sort(real), np.arange(n))           # every target exactly once
        for x, j0 in zip(o, b):                                          # row-run base = the target's box
            if x < 0:
                continue
            box = np.searchsorted(toff, g0 + x, side="right") - 1
            bx, by = oracle.morton_decode(int(box - t * WW), k + 1)  # level k + 1: k bits per axis
            assert j0 == by * R + bx
        if tpi == 2:                                                     # units: 2 slots of one box
            assert nslot % 2 == 0 and np.all(b[0::2] == b[1::2]) and np.all(o[0::2] >= 0)
        else:
            assert np.all(o >= 0)
        if len(items) == 0:
            continue
        nu = nslot // tpi
        it = items[ioff[i]:ioff[i] + 3 * nu]
        np_ = nparts[i]
        for ip in range(np_):
            ub, ue = nu * ip // np_, nu * (ip + 1) // np_
            part = it[3 * ub:3 * ue]
            assert sorted(part.tolist()) == sorted(u << 2 | r for u in range(ub, ue) for r in range(3))
            # balanced batches: every warp's summed batch maxima within one batch of the others
            j0 = b[tpi * (part >> 2)] + (part & 3) * R
            ln = table[i, j0 + 3].astype(np.int64) - table[i, j0]
            loads = np.zeros(nt // 32, dtype=np.int64)
            for s in range(0, len(part), 32):
                loads[(s % nt) // 32] += ln[s:s + 32].max()
            if len(part) > nt:
                assert loads.max() - loads.min() <= ln.max()


@pytest.mark.parametrize("split", [False, True])
@pytest.mark.parametrize("level,precision", [(4, "fp32"), (5, "fp32"), (6, "fp32"), (4, "fp64"), (6, "fp64")])
def test_tiled_slots_and_items(level, precision, split, monkeypatch):
    if split:  # force tail splitting (the default splits only Morton-ordered queues)
        monkeypatch.setenv("P2P_TAIL_TILES", "1000")
        monkeypatch.setenv("P2P_TAIL_PARTS", "3")
    src, tgt, _ = W.make_problem(W.widened(W.CONFIGS["tiny"], 4))
    level += 1  # the widened tiny plate needs one more level
    for tile in (-1, 0, 1, 2):
        pl = _plan(src, tgt, level=level, layout="tiled", precision=precision, tile_log2=tile)
        _tiled_layout_checks(pl, level, pl.info["cta_threads"])
        pl.close()


@pytest.mark.parametrize("layout", ["nr", "r", "tiled"])
@pytest.mark.parametrize("world", [2, 3])
def test_owned_sources_contiguous_disjoint_clouds(layout, world):
    """Sources and targets from different distributions (uniform sources, targets in the upper
    right quarter): owned boxes without targets lie outside every owned tile region.  The owned
    sources must still be one contiguous block of the local set, [owned_local_begin,
    + n_src_owned), holding exactly the global plan range [part_src[r], part_src[r+1]) in order --
    the distributed applies copy the owned weights there as one block."""
    rng = np.random.default_rng(11)
    src = rng.uniform(0, 1, (20000, 2))
    tgt = rng.uniform(0.5, 1, (20000, 2))
    for r in range(world):
        pl = _plan(src, tgt, level=8, layout=layout, part_world=world, part_rank=r)
        info = pl.info
        part = pl.export("partition").reshape(2, world + 1)
        sg = pl.export("src_global")
        assert len(sg) == info["n_src_local"] == info["n_src_owned"] + info["n_halo"]
        lo = np.searchsorted(sg, part[0, r])
        np.testing.assert_array_equal(sg[lo:lo + info["n_src_owned"]], np.arange(part[0, r], part[0, r + 1]))
        assert np.all(np.diff(sg) > 0)
        pl.close()


@pytest.mark.parametrize("world", [2, 3, 5])
@pytest.mark.parametrize("level", [5, 7])
def test_interior_launches_read_owned_sources_only(world, level):
    """Distributed TILED plans put interior tiles first: their regions hold owned sources only
    (they run before the halo arrives); every boundary tile reads at least one halo source."""
    src, tgt, _ = W.make_problem(W.widened(W.CONFIGS["tiny"], 4))
    for r in range(world):
        pl = _plan(src, tgt, level=level, layout="tiled", part_world=world, part_rank=r)
        info = pl.info
        launch = pl.export("launch").reshape(2, -1)
        roff, ridx = pl.export("region_offsets"), pl.export("region_index")
        sg = pl.export("src_global")
        lo, hi = info["src_owned_begin"], info["src_owned_begin"] + info["n_src_owned"]
        n_int = info["interior_launches"]
        assert 0 <= n_int <= info["launches"] == launch.shape[1]
        for e, slot in enumerate(launch[0]):
            ent = ridx[roff[slot]:roff[slot + 1]]
            g = sg[ent[ent >= 0]]
            owned = np.all((g >= lo) & (g < hi))
            assert owned == (e < n_int), (r, e, n_int)
        pl.close()


def _compact_bits(v):
    v = v & 0x55555555
    v = (v | (v >> 1)) & 0x33333333
    v = (v | (v >> 2)) & 0x0F0F0F0F
    v = (v | (v >> 4)) & 0x00FF00FF
    return (v | (v >> 8)) & 0x0000FFFF


def test_heavy_tiles_are_split():
    """A curve cloud concentrates its pairs in few tiles: every tile above 1/1184 of the pairs runs
    as ceil(pairs / share) consecutive launch entries (<= 32), each a unit range, so no single CTA
    serialises a large share of the work (tile pair counts recomputed here from the offsets)."""
    cfg = W.CONFIGS["contour_2e5"]
    src, tgt, _ = W.make_problem(cfg)
    pl = _plan(src, tgt, level=cfg.level, layout="tiled", precision="fp32")
    info = pl.info
    k, S = info["tile_log2"], info["side"]
    so, to = pl.export("src_box_offsets"), pl.export("tgt_box_offsets")
    ns, nt_ = np.diff(so), np.diff(to)
    b = np.arange(S * S, dtype=np.int64)
    ix, iy = _compact_bits(b), _compact_bits(b >> 1)
    grid = np.zeros((S + 2, S + 2), dtype=np.int64)
    grid[iy + 1, ix + 1] = ns
    n9 = sum(grid[iy + 1 + dy, ix + 1 + dx] for dy in (-1, 0, 1) for dx in (-1, 0, 1))
    tile_pairs = np.bincount(b >> (2 * k), weights=nt_ * n9, minlength=(S * S) >> (2 * k)).astype(np.int64)
    assert tile_pairs.sum() == info["pairs"]
    share = -(-info["pairs"] // 1184)
    tiles, launch = pl.export("tiles"), pl.export("launch").reshape(2, -1)
    parts, q = launch[1] >> 16, launch[1] & 0xFFFF
    e = 0
    n_split = 0
    while e < len(tiles):
        np_ = parts[e]
        want = min(32, max(1, -(-tile_pairs[tiles[e]] // share)))
        assert np_ == want, (e, np_, want)
        assert list(q[e:e + np_]) == list(range(np_)) and len(set(tiles[e:e + np_])) == 1
        n_split += np_ > 1
        e += np_
    assert n_split > 0
    pl.close()


@pytest.mark.parametrize("density,tpi,items,nt", [(2, 1, 1, None), (4, 2, 3, 64), (6, 2, 3, 128), (16, 2, 3, 128)])
def test_tiled_fp32_kernel_choice(density, tpi, items, nt):
    """TILED fp32 kernel choice by occupied-box density (measured on 1e7-point
    plates): the lean one-target path below 3 points per occupied box, the 2-target dense path
    from 3 (64-thread CTAs below 5 points per box, 128 above)."""
    cfg = W.PlateConfig("kc", 64, 64, 8, 64 * 64 * density, seed=11)
    src, tgt, _ = W.make_problem(cfg)
    pl = _plan(src, tgt, level=cfg.level, layout="tiled", precision="fp32")
    i = pl.info
    assert (i["slots_per_unit"], i["items_per_unit"]) == (tpi, items), (density, i["density_occupied"])
    if nt is not None:
        assert i["cta_threads"] == nt
    else:
        assert i["flags"] & 1 and i["cta_threads"] in (32, 64)  # n9-ordered lean slots
    pl.close()


@pytest.mark.parametrize("density,tpi,items,nt", [(2, 1, 1, 128), (4, 2, 3, 256), (16, 2, 3, 256)])
def test_tiled_fp64_kernel_choice(density, tpi, items, nt):
    """TILED fp64: the lean path (flattened runs, register-table log) below 4 points per occupied
    box, 2-target units with (unit, row) items and 256-thread CTAs from 4."""
    cfg = W.PlateConfig("kc", 64, 64, 8, 64 * 64 * density, seed=11)
    src, tgt, _ = W.make_problem(cfg)
    pl = _plan(src, tgt, level=cfg.level, layout="tiled", precision="fp64")
    i = pl.info
    assert (i["slots_per_unit"], i["items_per_unit"], i["cta_threads"]) == (tpi, items, nt), i["density_occupied"]
    pl.close()
