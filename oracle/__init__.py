"""Python access to the fp64 CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs.  The product package
(paper_2403_01596_b200) never imports this module.

Every function here marshals numpy arrays into the C oracle; the arithmetic
lives in oracle.c, which cites the paper passage each step follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")


def _cpu_tag() -> str:
    """-march=native binaries are CPU-specific: key the library by the host CPU."""
    import hashlib
    try:
        info = open("/proc/cpuinfo").read()
        model = [l for l in info.splitlines() if l.startswith(("model name", "flags"))][:2]
    except OSError:
        model = []
    return hashlib.sha1("\n".join(model).encode()).hexdigest()[:10]


_LIB = os.path.join(_HERE, f"liboracle_{_cpu_tag()}.so")

CFLAGS = ["-O3", "-march=native", "-fopenmp", "-fPIC", "-shared", "-std=c11"]  # no -ffast-math


def build(force: bool = False) -> str:
    """Compile oracle.c into oracle/liboracle.so (gcc, OpenMP, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.run(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"], check=True)
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        i64, i32, f64 = C.c_int64, C.c_int, C.c_double
        P = C.c_void_p
        _lib.oracle_direct.argtypes = [i64, P, P, i64, P, i32, f64, i64, P, P, i32, P]
        _lib.oracle_direct.restype = i32
        _lib.oracle_bruteforce.argtypes = [i64, P, P, i64, P, i32, f64, P, P]
        _lib.oracle_bruteforce.restype = i32
        _lib.oracle_pair_potential.argtypes = [f64] * 6
        _lib.oracle_pair_potential.restype = f64
        _lib.oracle_morton.argtypes = [C.c_uint64, C.c_uint64, i32]
        _lib.oracle_morton.restype = C.c_uint64
        _lib.oracle_morton_decode.argtypes = [C.c_uint64, i32, P, P]
        _lib.oracle_sort_points.argtypes = [i64, P, i32, P, P]
        _lib.oracle_sort_points.restype = i32
        _lib.oracle_neighbors.argtypes = [i32, P]
        _lib.oracle_ct_level.argtypes = [i64, P, i64, P, i32, i32, i32]
        _lib.oracle_ct_level.restype = i32
        _lib.oracle_pair_count.argtypes = [i64, P, i64, P, i32]
        _lib.oracle_indexing_bytes.argtypes = [i64, i32, i64]
        _lib.oracle_indexing_bytes.restype = i64
        _lib.oracle_repetition_bytes.argtypes = [i64, i64]
        _lib.oracle_repetition_bytes.restype = i64
        _lib.oracle_box_tmax.argtypes = [i64, P, i64, P, i32]
        _lib.oracle_box_tmax.restype = i64
        _lib.oracle_pair_count.restype = i64
        _lib.oracle_num_threads.restype = i32
        _lib.oracle_direct_helmholtz.argtypes = [i64, P, P, i64, P, i32, f64, f64, i64, P, P, i32, P]
        _lib.oracle_direct_helmholtz.restype = i32
        _lib.oracle_bruteforce_helmholtz.argtypes = [i64, P, P, i64, P, i32, f64, f64, P, P]
        _lib.oracle_bruteforce_helmholtz.restype = i32
        _lib.oracle_pair_helmholtz.argtypes = [f64] * 8 + [P]
        _lib.oracle_pair_helmholtz.restype = None
        _lib.oracle_direct_3d.argtypes = [i64, P, P, i64, P, i32, f64, i32, f64, i64, P, P, i32, P]
        _lib.oracle_direct_3d.restype = i32
        _lib.oracle_bruteforce_3d.argtypes = [i64, P, P, i64, P, i32, f64, i32, f64, P, P]
        _lib.oracle_bruteforce_3d.restype = i32
        _lib.oracle_adaptive_tree.argtypes = [i64, P, i64, P, i64, i64, P, i64]
        _lib.oracle_adaptive_tree.restype = i64
        _lib.oracle_adaptive_direct.argtypes = [i64, P, P, i64, P, i64, i64, f64, P, P]
        _lib.oracle_adaptive_direct.restype = i32
    return _lib


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def direct(src_xy, q, tgt_xy, level: int, eps: float = 1e-12, targets=None,
           nthreads: int = 0) -> tuple[np.ndarray, int]:
    """phi for all targets (or the index subset ``targets``) and the pair count."""
    src_xy, q, tgt_xy = _f64(src_xy), _f64(q), _f64(tgt_xy)
    sel = None if targets is None else np.ascontiguousarray(targets, dtype=np.int64)
    n_out = len(tgt_xy) if sel is None else len(sel)
    phi = np.empty(n_out, dtype=np.float64)
    pairs = C.c_int64(0)
    rc = lib().oracle_direct(len(src_xy), _ptr(src_xy), _ptr(q), len(tgt_xy), _ptr(tgt_xy),
                             level, eps, 0 if sel is None else len(sel),
                             None if sel is None else _ptr(sel), _ptr(phi), nthreads,
                             C.byref(pairs))
    if rc:
        raise MemoryError("oracle_direct allocation failed")
    return phi, pairs.value


def bruteforce(src_xy, q, tgt_xy, level: int, eps: float = 1e-12) -> tuple[np.ndarray, int]:
    src_xy, q, tgt_xy = _f64(src_xy), _f64(q), _f64(tgt_xy)
    phi = np.empty(len(tgt_xy), dtype=np.float64)
    pairs = C.c_int64(0)
    lib().oracle_bruteforce(len(src_xy), _ptr(src_xy), _ptr(q), len(tgt_xy), _ptr(tgt_xy),
                            level, eps, _ptr(phi), C.byref(pairs))
    return phi, pairs.value


def pair_potential(t, s, q: float, eps: float = 1e-12) -> float:
    return lib().oracle_pair_potential(float(t[0]), float(t[1]), float(s[0]), float(s[1]),
                                       float(q), eps)


def morton(ix: int, iy: int, level: int) -> int:
    return int(lib().oracle_morton(ix, iy, level))


def morton_decode(code: int, level: int) -> tuple[int, int]:
    x, y = C.c_uint64(0), C.c_uint64(0)
    lib().oracle_morton_decode(code, level, C.byref(x), C.byref(y))
    return x.value, y.value


def sort_points(xy, level: int) -> tuple[np.ndarray, np.ndarray]:
    """(perm[plan] = original index, box offsets[4^(L-1)+1]) in Morton order."""
    xy = _f64(xy)
    perm = np.empty(len(xy), dtype=np.int64)
    off = np.empty((1 << (2 * (level - 1))) + 1, dtype=np.int64)
    if lib().oracle_sort_points(len(xy), _ptr(xy), level, _ptr(perm), _ptr(off)):
        raise MemoryError
    return perm, off


def neighbors(level: int) -> np.ndarray:
    nb = np.empty((1 << (2 * (level - 1))) * 9, dtype=np.int64)
    lib().oracle_neighbors(level, _ptr(nb))
    return nb.reshape(-1, 9)


def ct_level(src_xy, tgt_xy, ct: int = 15, l_start: int = 3, l_max: int = 16) -> int:
    src_xy, tgt_xy = _f64(src_xy), _f64(tgt_xy)
    return int(lib().oracle_ct_level(len(src_xy), _ptr(src_xy), len(tgt_xy), _ptr(tgt_xy),
                                     ct, l_start, l_max))


def pair_count(src_xy, tgt_xy, level: int) -> int:
    src_xy, tgt_xy = _f64(src_xy), _f64(tgt_xy)
    return int(lib().oracle_pair_count(len(src_xy), _ptr(src_xy), len(tgt_xy), _ptr(tgt_xy), level))


def indexing_bytes(n: int, level: int, t: int) -> int:
    """PAPER.md Eq. 3 (L96): 40N + 4^L (2 + 10t) bytes."""
    return int(lib().oracle_indexing_bytes(n, level, t))


def repetition_bytes(n: int, ct: int) -> int:
    """PAPER.md Eq. 8 (L126): 8N(3 + 27 CT) bytes."""
    return int(lib().oracle_repetition_bytes(n, ct))


def box_tmax(src_xy, tgt_xy, level: int) -> int:
    """t of Eqs. 3-5: max over leaf boxes of max(#sources, #targets)."""
    s, t = _f64(src_xy), _f64(tgt_xy)
    return int(lib().oracle_box_tmax(len(s), _ptr(s), len(t), _ptr(t), level))


def num_threads() -> int:
    return int(lib().oracle_num_threads())


# ---- NEXT-3: the 2D Helmholtz kernel G = (i/4) H0^(1)(kappa r) (oracle.c) ----
def _c128(a) -> np.ndarray:
    """complex input -> interleaved (re, im) float64"""
    a = np.ascontiguousarray(a, dtype=np.complex128)
    return a.view(np.float64)


def direct_helmholtz(src_xy, q, tgt_xy, level: int, kappa: float, eps: float = 1e-12, targets=None,
                     nthreads: int = 0) -> tuple[np.ndarray, int]:
    """complex phi for all targets (or the index subset ``targets``) and the pair count."""
    src_xy, tgt_xy = _f64(src_xy), _f64(tgt_xy)
    qi = _c128(q)
    sel = None if targets is None else np.ascontiguousarray(targets, dtype=np.int64)
    n_out = len(tgt_xy) if sel is None else len(sel)
    phi = np.empty(n_out, dtype=np.complex128)
    pairs = C.c_int64(0)
    rc = lib().oracle_direct_helmholtz(len(src_xy), _ptr(src_xy), _ptr(qi), len(tgt_xy), _ptr(tgt_xy),
                                       level, eps, kappa, 0 if sel is None else len(sel),
                                       None if sel is None else _ptr(sel), _ptr(phi), nthreads,
                                       C.byref(pairs))
    if rc:
        raise MemoryError("oracle_direct_helmholtz allocation failed")
    return phi, pairs.value


def bruteforce_helmholtz(src_xy, q, tgt_xy, level: int, kappa: float, eps: float = 1e-12):
    src_xy, tgt_xy = _f64(src_xy), _f64(tgt_xy)
    qi = _c128(q)
    phi = np.empty(len(tgt_xy), dtype=np.complex128)
    pairs = C.c_int64(0)
    lib().oracle_bruteforce_helmholtz(len(src_xy), _ptr(src_xy), _ptr(qi), len(tgt_xy), _ptr(tgt_xy),
                                      level, eps, kappa, _ptr(phi), C.byref(pairs))
    return phi, pairs.value


def pair_helmholtz(t, s, q: complex, kappa: float, eps: float = 1e-12) -> complex:
    out = np.zeros(2, dtype=np.float64)
    q = complex(q)
    lib().oracle_pair_helmholtz(float(t[0]), float(t[1]), float(s[0]), float(s[1]), q.real, q.imag,
                                eps, kappa, _ptr(out))
    return complex(out[0], out[1])


# ---- NEXT-3: 3D kernels on the octree leaf grid (oracle.c oracle_direct_3d) ----
def direct_3d(src_xyz, q, tgt_xyz, level: int, kernel: str = "laplace", kappa: float = 0.0,
              eps: float = 1e-12, targets=None, nthreads: int = 0):
    """phi (real for "laplace": 1/(4 pi r); complex for "helmholtz": e^{i kappa r}/(4 pi r)) and
    the pair count, over the 3x3x3 neighbour boxes."""
    src, tgt = _f64(src_xyz), _f64(tgt_xyz)
    helm = kernel == "helmholtz"
    qa = _c128(q) if helm else _f64(q)
    sel = None if targets is None else np.ascontiguousarray(targets, dtype=np.int64)
    n_out = len(tgt) if sel is None else len(sel)
    phi = np.empty(n_out, dtype=np.complex128 if helm else np.float64)
    pairs = C.c_int64(0)
    rc = lib().oracle_direct_3d(len(src), _ptr(src), _ptr(qa), len(tgt), _ptr(tgt), level, eps, int(helm),
                                kappa, 0 if sel is None else len(sel), None if sel is None else _ptr(sel),
                                _ptr(phi), nthreads, C.byref(pairs))
    if rc:
        raise MemoryError("oracle_direct_3d allocation failed")
    return phi, pairs.value


def bruteforce_3d(src_xyz, q, tgt_xyz, level: int, kernel: str = "laplace", kappa: float = 0.0,
                  eps: float = 1e-12):
    src, tgt = _f64(src_xyz), _f64(tgt_xyz)
    helm = kernel == "helmholtz"
    qa = _c128(q) if helm else _f64(q)
    phi = np.empty(len(tgt), dtype=np.complex128 if helm else np.float64)
    pairs = C.c_int64(0)
    lib().oracle_bruteforce_3d(len(src), _ptr(src), _ptr(qa), len(tgt), _ptr(tgt), level, eps, int(helm),
                               kappa, _ptr(phi), C.byref(pairs))
    return phi, pairs.value


# ---- NEXT-4: CT-driven adaptive quadtree (oracle.c oracle_adaptive_*) ----
def adaptive_tree(src_xy, tgt_xy, ct: int, l_max: int) -> np.ndarray:
    """Leaves [(level, ix, iy)] in Morton (depth-first) order."""
    s, t = _f64(src_xy), _f64(tgt_xy)
    cap = 1 + 3 * (len(s) + len(t)) * l_max + 4
    out = np.empty(3 * cap, dtype=np.int64)
    n = lib().oracle_adaptive_tree(len(s), _ptr(s), len(t), _ptr(t), ct, l_max, _ptr(out), cap)
    if n < 0:
        raise MemoryError
    return out[:3 * n].reshape(-1, 3)


def adaptive_direct(src_xy, q, tgt_xy, ct: int, l_max: int, eps: float = 1e-12):
    """phi over the U-lists (leaves touching the target's leaf) and the pair count (brute force)."""
    s, t, qq = _f64(src_xy), _f64(tgt_xy), _f64(q)
    phi = np.empty(len(t), dtype=np.float64)
    pairs = C.c_int64(0)
    if lib().oracle_adaptive_direct(len(s), _ptr(s), _ptr(qq), len(t), _ptr(t), ct, l_max, eps, _ptr(phi),
                                    C.byref(pairs)):
        raise MemoryError
    return phi, pairs.value
