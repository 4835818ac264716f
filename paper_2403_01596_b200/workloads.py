"""Seeded synthetic workloads for the near-field P2P operator.

This module is the ONLY code shared by the CUDA path's callers (bench, tests)
and the oracle's callers: it produces point sets and weights and holds none of
the method's arithmetic (no box assignment, no Morton codes, no kernel).

Workload shape (§4 "a PEC square plate which
the source and target points are distributed randomly on it"):

* The root box is the unit square [0,1]^2.  The leaf level L
  gives a grid of S = 2^(L-1) boxes per side, box side h = 1/S.
* A *plate* of sx x sy leaf boxes sits at the origin.  Points lie on the
  plate, so the density per occupied box D = N / (sx*sy) is exact.
* ``iid``: coordinates uniform on the plate (paper-faithful, Poisson occupancy).
* ``stratified``: exactly D points per plate box, uniform inside the box
  (exact pair counts, no load imbalance).
* Weights q ~ U[-1, 1).
* Targets and sources are independent sets of equal size (PAPER.md L65,
  "assumed equal for both"); ``collocated=True`` makes targets = sources.

Random numbers come from a counter-based SplitMix64 keyed by
(seed, stream, index), so any rank can regenerate any point:
stream 0/1 = target x/y, 2/3 = source x/y, 4 = q.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_STREAM_MUL = np.uint64(0xD1B54A32D192ED03)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix64(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def uniform01(seed: int, stream: int, index: np.ndarray) -> np.ndarray:
    """Counter-based U[0,1) doubles: SplitMix64(key(seed, stream) + (i+1)*golden)."""
    with np.errstate(over="ignore"):
        key = _mix64(np.array([np.uint64(seed) * _GOLDEN ^ (np.uint64(stream) * _STREAM_MUL)],
                              dtype=np.uint64))[0]
        idx = np.asarray(index, dtype=np.uint64)
        z = _mix64(key + (idx + np.uint64(1)) * _GOLDEN)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


@dataclass(frozen=True)
class PlateConfig:
    """One BASELINE.json workload: an sx x sy plate of leaf boxes at level L."""
    name: str
    sx: int
    sy: int
    level: int
    n: int
    seed: int = 20240303

    @property
    def side(self) -> int:
        return 1 << (self.level - 1)

    @property
    def density(self) -> float:
        return self.n / (self.sx * self.sy)

    def stratified_pairs(self) -> int:
        """Exact pair count of the stratified generator: D^2 (3sx-2)(3sy-2)."""
        d = self.n // (self.sx * self.sy)
        return d * d * (3 * self.sx - 2) * (3 * self.sy - 2)


@dataclass(frozen=True)
class ContourConfig:
    """a curve-concentrated ("surface-like") 2D cloud -- the nodes of a
    boundary discretisation of a 2D scatterer (the 2D MLFMA / EFIE setting of PAPER.md refs
    [2], [4]-[6]): n points on the closed star curve r(t) = r0 (1 + a cos(m t)) around
    (1/2, 1/2), equispaced in t with a seeded jitter of +-1/8 spacing; sources = targets
    (collocation; the self pair is removed by the eps guard).  Most leaf boxes are empty; the
    occupied ones hold about n h / (curve length) points (curve length ~ 3.16)."""
    name: str
    n: int
    level: int
    r0: float = 0.35
    a: float = 0.3
    m: int = 5
    seed: int = 20240303

    @property
    def side(self) -> int:
        return 1 << (self.level - 1)


@dataclass(frozen=True)
class CubeConfig:
    """SURVEY.md §8(f) NEXT-3 (3D kernels): n points uniform in an s x s x s block of leaf boxes of
    the octree leaf grid at level L (grid 2^(L-1) per side on the unit cube), embedded at the
    origin -- the "4x4x4 uniform leaf boxes" reading of BASELINE.json's tiny config in 3D, and a
    1e6-point volume at 16 points per box."""
    name: str
    s: int
    level: int
    n: int
    seed: int = 20240303

    @property
    def side(self) -> int:
        return 1 << (self.level - 1)

    @property
    def density(self) -> float:
        return self.n / self.s ** 3


def cube_points(cfg: CubeConfig, streams=(0, 1, 7), seed: int | None = None) -> np.ndarray:
    """[n, 3] float64 points uniform in the box block of ``cfg``."""
    seed = cfg.seed if seed is None else seed
    idx = np.arange(cfg.n, dtype=np.uint64)
    w = cfg.s / cfg.side
    return np.stack([_below(w, uniform01(seed, st, idx) * w) for st in streams], axis=1)


def contour_points(cfg: ContourConfig, seed: int | None = None, n: int | None = None) -> np.ndarray:
    """[n, 2] float64 points on the star curve of ``cfg`` (inside [0.045, 0.955]^2)."""
    seed = cfg.seed if seed is None else seed
    n = cfg.n if n is None else n
    u = uniform01(seed, 6, np.arange(n, dtype=np.uint64))
    t = 2.0 * np.pi * (np.arange(n, dtype=np.float64) + 0.5 + 0.25 * (u - 0.5)) / n
    r = cfg.r0 * (1.0 + cfg.a * np.cos(cfg.m * t))
    return np.stack([0.5 + r * np.cos(t), 0.5 + r * np.sin(t)], axis=1)


# SURVEY.md §8(d) table; BASELINE.json "configs".
CONFIGS: dict[str, PlateConfig | ContourConfig] = {
    c.name: c for c in [
        PlateConfig("tiny", 8, 8, 4, 1024, seed=1),
        PlateConfig("d16_1e6", 250, 250, 9, 1_000_000),
        PlateConfig("d32_1e6", 250, 125, 9, 1_000_000),
        PlateConfig("d64_1e6", 125, 125, 8, 1_000_000),
        PlateConfig("lowd025_1e7", 8000, 5000, 14, 10_000_000),
        PlateConfig("lowd1_1e7", 4000, 2500, 13, 10_000_000),
        PlateConfig("lowd2_1e7", 2500, 2000, 13, 10_000_000),
        PlateConfig("lowd4_1e7", 2000, 1250, 12, 10_000_000),
        PlateConfig("surf_2e7", 1250, 1000, 12, 20_000_000),
        PlateConfig("d32_7e7", 1750, 1250, 12, 70_000_000),
        # NEXT-3 (Helmholtz): a 1e6-point plate at 4 points per leaf box (leaf = a quarter
        # wavelength at the helmholtz workload's kappa: ~8 samples per wavelength along x and y)
        PlateConfig("d4_1e6", 500, 500, 10, 1_000_000),
        # kernel-choice sweeps between the low-density and the density configs (not BASELINE
        # workloads): 1e7 points at 3 and 6 points per leaf box
        PlateConfig("lowd3_1e7", 2000, 1667, 12, 10_000_000),
        PlateConfig("lowd6_1e7", 1291, 1291, 12, 10_000_000),
    ]
}
# NEXT-4 curve clouds: Laplace at ~12 points per occupied leaf box (t = 43); Helmholtz with the
# leaf box a quarter wavelength at ~7.7 samples per wavelength along the curve (~1.8 points per
# occupied box).
CONFIGS.update({c.name: c for c in [
    CubeConfig("tiny3d", 4, 3, 1024, seed=1),
    CubeConfig("cube3d_1e6", 40, 7, 1_024_000),
    ContourConfig("contour_2e5", 200_000, 13),
    ContourConfig("contour_1e5", 100_000, 15, seed=20240304),
]})


MAX_LEVEL = 15  # the plan builder's level cap (R16)


def widened(cfg: PlateConfig, factor: int) -> PlateConfig:
    """The plate ``factor`` times longer (same points per box, ``factor`` x the points):
    the weak-scaling problem for ``factor`` GPUs.  The leaf level rises only if the
    wider plate no longer fits the grid (boxes stay boxes: D is unchanged)."""
    if factor == 1:
        return cfg
    if not isinstance(cfg, PlateConfig):
        raise ValueError(f"{cfg.name}: weak scaling widens plates only")
    sx, sy = cfg.sx, cfg.sy
    if sx <= sy:
        sx *= factor
    else:
        sy *= factor
    level = max(cfg.level, int(np.ceil(np.log2(max(sx, sy)))) + 1)
    if level > MAX_LEVEL:
        raise ValueError(f"{cfg.name} x{factor}: a {sx}x{sy} plate needs level {level} > {MAX_LEVEL}")
    return PlateConfig(f"{cfg.name}_x{factor}", sx, sy, level, cfg.n * factor, cfg.seed)


def _below(limit: float, x: np.ndarray) -> np.ndarray:
    """Clamp x strictly below ``limit`` (guards against round-up at the plate edge)."""
    return np.minimum(x, np.nextafter(limit, 0.0))


def plate_points(cfg: PlateConfig, stream_x: int, stream_y: int, kind: str = "iid",
                 seed: int | None = None, n: int | None = None, index=None) -> np.ndarray:
    """[n, 2] float64 points on the plate of ``cfg`` (``index``: only those points of the set,
    e.g. one rank's share -- the counter-based generator makes any subset directly)."""
    seed = cfg.seed if seed is None else seed
    n = cfg.n if n is None else n
    h = 1.0 / cfg.side
    idx = np.arange(n, dtype=np.uint64) if index is None else np.asarray(index, dtype=np.uint64)
    n = len(idx)
    ux = uniform01(seed, stream_x, idx)
    uy = uniform01(seed, stream_y, idx)
    xy = np.empty((n, 2), dtype=np.float64)
    if kind == "iid":
        wx, wy = cfg.sx * h, cfg.sy * h
        xy[:, 0] = _below(wx, ux * wx)
        xy[:, 1] = _below(wy, uy * wy)
    elif kind == "stratified":
        boxes = cfg.sx * cfg.sy
        if (cfg.n if index is not None else n) % boxes:
            raise ValueError("stratified generator needs an integer density")
        d = (cfg.n if index is not None else n) // boxes
        j = idx.astype(np.int64) // d
        bx = (j % cfg.sx).astype(np.float64)
        by = (j // cfg.sx).astype(np.float64)
        # (b + u) < b + 1 keeps the point inside its cell; scaling by h = 2^-(L-1) is exact.
        xy[:, 0] = np.minimum(bx + ux, np.nextafter(bx + 1.0, 0.0)) * h
        xy[:, 1] = np.minimum(by + uy, np.nextafter(by + 1.0, 0.0)) * h
    else:
        raise ValueError(f"unknown generator kind {kind!r}")
    return xy


def weights(n: int, seed: int, stream: int = 4, index=None) -> np.ndarray:
    """q ~ U[-1, 1) as float64; ``index``: only those weights."""
    idx = np.arange(n, dtype=np.uint64) if index is None else np.asarray(index, dtype=np.uint64)
    return 2.0 * uniform01(seed, stream, idx) - 1.0


def weights_complex(n: int, seed: int, index=None) -> np.ndarray:
    """Complex weights for the Helmholtz kernel (NEXT-3): re, im ~ U[-1, 1) (streams 4 and 5)."""
    return weights(n, seed, index=index) + 1j * weights(n, seed, stream=5, index=index)


def problem_share(cfg: PlateConfig | str, rank: int, world: int, kind: str = "iid"):
    """One rank's interleaved share of a workload (global ids rank, rank + world, ...): (src_xy,
    tgt_xy, src_ids, tgt_ids) -- what DistributedP2P.from_local takes; the rank never
    generates the other points."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    ids = np.arange(rank, cfg.n, world, dtype=np.int64)
    return plate_points(cfg, 2, 3, kind, index=ids), plate_points(cfg, 0, 1, kind, index=ids), ids, ids.copy()


def make_problem(cfg: PlateConfig | str, kind: str = "iid", seed: int | None = None,
                 collocated: bool = False, n: int | None = None):
    """(src_xy, tgt_xy, q) float64 arrays for one workload."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    seed = cfg.seed if seed is None else seed
    n = cfg.n if n is None else n
    if isinstance(cfg, CubeConfig):  # 3D: targets streams (0, 1, 7), sources (2, 3, 8)
        return cube_points(cfg, (2, 3, 8), seed), cube_points(cfg, (0, 1, 7), seed), weights(cfg.n, seed)
    if isinstance(cfg, ContourConfig):  # collocated boundary nodes (kind does not apply)
        src = contour_points(cfg, seed, n)
        return src, src.copy(), weights(n, seed)
    src = plate_points(cfg, 2, 3, kind, seed, n)
    tgt = src.copy() if collocated else plate_points(cfg, 0, 1, kind, seed, n)
    q = weights(n, seed)
    return src, tgt, q


def uniform_unit(n: int, seed: int):
    """SPEC.md L51 generate_points: n sources and n targets uniform in [0,1]^2, q in [-1,1)."""
    idx = np.arange(n, dtype=np.uint64)
    tgt = np.stack([uniform01(seed, 0, idx), uniform01(seed, 1, idx)], axis=1)
    src = np.stack([uniform01(seed, 2, idx), uniform01(seed, 3, idx)], axis=1)
    return src, tgt, weights(n, seed)
