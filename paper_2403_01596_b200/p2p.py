"""Thin ctypes binding of the C ABI in include/p2p.h.

Argument marshalling only: every step of plan building runs in the C++ host
builder and every step of apply runs in the sm_100a kernels of
libp2p_b200.so.  There is no CPU fallback: if the library is missing the
import fails loudly, and applying a host-only plan raises P2PError.

The function names mirror the C ABI (p2p_plan_create, p2p_apply, ...); the
`Plan` class is a convenience wrapper that takes numpy points and torch
device tensors.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("P2P_LIB") or os.path.join(_PKG, "lib", "libp2p_b200.so")  # P2P_LIB: experiments

P2P_SUCCESS = 0
P2P_ERROR_INVALID_ARGUMENT = 1
P2P_ERROR_CONSTRUCTION_FAILURE = 2
P2P_ERROR_LAYOUT_CORRUPT = 3
P2P_ERROR_OUT_OF_MEMORY = 4
P2P_ERROR_CUDA = 5
P2P_ERROR_NOT_SUPPORTED = 6
P2P_ERROR_NO_DEVICE = 7

P2P_KERNEL_LAPLACE_2D = 0
P2P_KERNEL_HELMHOLTZ_2D = 1
P2P_KERNEL_LAPLACE_3D = 2
P2P_KERNEL_HELMHOLTZ_3D = 3
KERNELS = {"laplace": P2P_KERNEL_LAPLACE_2D, "helmholtz": P2P_KERNEL_HELMHOLTZ_2D,
           "laplace3d": P2P_KERNEL_LAPLACE_3D, "helmholtz3d": P2P_KERNEL_HELMHOLTZ_3D}
P2P_LAYOUT_NONREDUNDANT = 0
P2P_LAYOUT_REDUNDANT = 1
P2P_LAYOUT_TILED = 2
P2P_LAYOUT_PAPER_INDEXING = 3
P2P_LAYOUT_PAPER_REPETITION = 4
P2P_LAYOUT_ADAPTIVE = 5
P2P_FP64 = 0
P2P_FP32 = 1
P2P_ORDER_PLAN = 0
P2P_ORDER_USER = 1

EXPORT = {
    "src_perm": 0, "tgt_perm": 1, "src_box_offsets": 2, "tgt_box_offsets": 3,
    "neighbors": 4, "partition": 5, "src_global": 6, "halo_counts": 7, "tiles": 8,
    "halo_index": 9, "send_index": 10, "halo_offsets": 11, "region_offsets": 12, "region_index": 13,
    "region_table": 14, "slot_offsets": 15, "slot_base": 16, "slot_output": 17, "item_offsets": 18,
    "items": 19, "launch": 20, "paper_nei_offsets": 21, "paper_nei_index": 22, "paper_records": 23,
    "leaves": 24, "ulist_offsets": 25, "ulist": 26,
}

# Symbols declared in include/p2p.h (checked by tests/test_abi.py).
ABI_SYMBOLS = (
    "p2p_plan_desc_init", "p2p_plan_create", "p2p_plan_create_device", "p2p_apply", "p2p_apply_host", "p2p_apply_host_async",
    "p2p_apply_dist", "p2p_apply_dist_interior", "p2p_apply_dist_boundary",
    "p2p_halo_pack", "p2p_apply_dist_peer", "p2p_gather_peer", "p2p_ipc_export", "p2p_ipc_open", "p2p_ipc_close", "p2p_destroy", "p2p_plan_get_info", "p2p_plan_export",
    "p2p_status_string", "p2p_last_error", "p2p_abi_version",
    "p2p_peer_buffers", "p2p_peer_connect", "p2p_apply_peer_sync", "p2p_gather", "p2p_peer_check",
    "p2p_box_counts", "p2p_partition_route", "p2p_plan_create_local", "p2p_plan_set_workspaces",
)


class PlanDesc(C.Structure):
    _fields_ = [
        ("struct_size", C.c_uint32), ("abi_version", C.c_int32),
        ("n_src", C.c_int64), ("n_tgt", C.c_int64),
        ("src_xy", C.c_void_p), ("tgt_xy", C.c_void_p),
        ("level", C.c_int32), ("ct", C.c_int32), ("l_start", C.c_int32), ("l_max", C.c_int32),
        ("level_delta", C.c_int32), ("kernel", C.c_int32), ("epsilon", C.c_double),
        ("layout", C.c_int32), ("precision", C.c_int32), ("device", C.c_int32),
        ("tile_log2", C.c_int32), ("stream", C.c_void_p),
        ("part_world", C.c_int32), ("part_rank", C.c_int32), ("wavenumber", C.c_double),
    ]


class PlanInfo(C.Structure):
    _fields_ = [
        ("struct_size", C.c_uint32),
        ("level", C.c_int32), ("tile_log2", C.c_int32), ("layout", C.c_int32), ("precision", C.c_int32),
        ("device", C.c_int32), ("part_world", C.c_int32), ("part_rank", C.c_int32),
        ("side", C.c_int64), ("boxes", C.c_int64), ("n_src", C.c_int64), ("n_tgt", C.c_int64),
        ("n_src_local", C.c_int64), ("n_tgt_local", C.c_int64), ("n_src_owned", C.c_int64),
        ("src_owned_begin", C.c_int64), ("tgt_begin", C.c_int64), ("n_halo", C.c_int64),
        ("n_send", C.c_int64), ("occupied_src_boxes", C.c_int64), ("occupied_tgt_boxes", C.c_int64),
        ("t_max", C.c_int64), ("density", C.c_double), ("density_occupied", C.c_double),
        ("pairs", C.c_int64), ("pairs_global", C.c_int64), ("tiles", C.c_int64),
        ("smem_bytes", C.c_int64), ("halo_entries", C.c_int64), ("alg_bytes_kernel", C.c_int64),
        ("layout_bytes_apply", C.c_int64), ("device_bytes", C.c_int64), ("build_seconds", C.c_double),
        ("upload_seconds", C.c_double), ("cta_threads", C.c_int32), ("slots_per_unit", C.c_int32),
        ("items_per_unit", C.c_int32), ("flags", C.c_int32), ("interior_launches", C.c_int64),
        ("paper_model_bytes", C.c_int64), ("record_stride", C.c_int64), ("launches", C.c_int64),
        ("kernel", C.c_int32), ("components", C.c_int32), ("wavenumber", C.c_double),
    ]


class P2PError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        self.status = status
        super().__init__(f"{where}: {_status_name(status)}: {detail}")


_lib = None


def load_library() -> C.CDLL:
    """Load libp2p_b200.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    if os.environ.get("P2P_LIB"):  # A/B experiments with older builds: skip symbols they lack
        class _Tolerant:
            def __init__(self, l):
                object.__setattr__(self, "_l", l)

            def __getattr__(self, name):
                try:
                    return getattr(self._l, name)
                except AttributeError:
                    return C.CFUNCTYPE(None)()  # placeholder; calling it is an error

            def __setattr__(self, name, v):
                setattr(self._l, name, v)
        lib = _Tolerant(lib)
    P, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    lib.p2p_plan_desc_init.argtypes = [C.POINTER(PlanDesc)]
    lib.p2p_plan_desc_init.restype = None
    lib.p2p_plan_create.argtypes = [C.POINTER(PlanDesc), C.POINTER(P)]
    lib.p2p_plan_create_device.argtypes = [C.POINTER(PlanDesc), P, P, C.POINTER(P)]
    lib.p2p_apply.argtypes = [P, P, P, i32, i32, P]
    lib.p2p_apply_host.argtypes = [P, P, P, i32, i32, P]
    lib.p2p_apply_host_async.argtypes = [P, P, P, i32, i32, P]
    lib.p2p_apply_dist.argtypes = [P, P, P, P, i32, P]
    lib.p2p_apply_dist_interior.argtypes = [P, P, P, i32, P]
    lib.p2p_apply_dist_boundary.argtypes = [P, P, P, i32, P]
    lib.p2p_halo_pack.argtypes = [P, P, P, P]
    lib.p2p_apply_dist_peer.argtypes = [P, P, C.POINTER(P), P, i32, P]
    lib.p2p_gather_peer.argtypes = [P, C.POINTER(P), P, P]
    lib.p2p_ipc_export.argtypes = [P, P, C.POINTER(i64)]
    lib.p2p_ipc_open.argtypes = [P, i64, i32, C.POINTER(P)]
    lib.p2p_ipc_close.argtypes = [P, i64]
    lib.p2p_peer_buffers.argtypes = [P, C.POINTER(P), C.POINTER(P), C.POINTER(P)]
    lib.p2p_peer_connect.argtypes = [P, C.POINTER(P), C.POINTER(P), C.POINTER(P), C.POINTER(i64)]
    lib.p2p_apply_peer_sync.argtypes = [P, P, P, i32, P]
    lib.p2p_gather.argtypes = [P, P, P, P]
    lib.p2p_peer_check.argtypes = [P]
    lib.p2p_box_counts.argtypes = [i32, i64, P, P]
    lib.p2p_plan_set_workspaces.argtypes = [P, i32]
    lib.p2p_partition_route.argtypes = [C.POINTER(PlanDesc), P, P, P, P, i64, i64, P, P]
    lib.p2p_plan_create_local.argtypes = [C.POINTER(PlanDesc), P, P, P, P, i64, i64, C.POINTER(P)]
    lib.p2p_destroy.argtypes = [P]
    lib.p2p_plan_get_info.argtypes = [P, C.POINTER(PlanInfo)]
    lib.p2p_plan_export.argtypes = [P, i32, P, C.POINTER(C.c_size_t)]
    lib.p2p_status_string.argtypes = [i32]
    lib.p2p_status_string.restype = C.c_char_p
    lib.p2p_last_error.restype = C.c_char_p
    lib.p2p_abi_version.restype = i32
    for name in ("p2p_plan_create", "p2p_plan_create_device", "p2p_apply", "p2p_apply_host", "p2p_apply_host_async", "p2p_apply_dist", "p2p_apply_dist_interior",
                 "p2p_apply_dist_boundary", "p2p_halo_pack", "p2p_apply_dist_peer", "p2p_gather_peer", "p2p_ipc_export",
                 "p2p_ipc_open", "p2p_ipc_close", "p2p_peer_buffers", "p2p_peer_connect", "p2p_apply_peer_sync",
                 "p2p_gather", "p2p_peer_check", "p2p_box_counts", "p2p_partition_route", "p2p_plan_create_local",
                 "p2p_plan_set_workspaces", "p2p_destroy", "p2p_plan_get_info", "p2p_plan_export"):
        getattr(lib, name).restype = i32
    _lib = lib
    return lib


def _status_name(s: int) -> str:
    try:
        return load_library().p2p_status_string(s).decode()
    except Exception:
        return str(s)


def _check(status: int, where: str):
    if status != P2P_SUCCESS:
        raise P2PError(status, where, load_library().p2p_last_error().decode())


# ------------------------------------------------------------- C-ABI mirror
def p2p_plan_desc_init() -> PlanDesc:
    d = PlanDesc()
    load_library().p2p_plan_desc_init(C.byref(d))
    return d


def p2p_plan_create(desc: PlanDesc) -> C.c_void_p:
    h = C.c_void_p()
    _check(load_library().p2p_plan_create(C.byref(desc), C.byref(h)), "p2p_plan_create")
    return h


def p2p_plan_create_device(desc: PlanDesc, d_src_xy: int, d_tgt_xy: int) -> C.c_void_p:
    """Plan built on the GPU from device coordinates (fp64 [n][2] on desc.device)."""
    h = C.c_void_p()
    _check(load_library().p2p_plan_create_device(C.byref(desc), d_src_xy, d_tgt_xy, C.byref(h)),
           "p2p_plan_create_device")
    return h


def p2p_apply(plan, d_q: int, d_out: int, order: int = P2P_ORDER_PLAN, accumulate: int = 0, stream: int = 0):
    _check(load_library().p2p_apply(plan, d_q, d_out, order, accumulate, stream or None), "p2p_apply")


def p2p_apply_host(plan, h_q: int, h_out: int, order: int = P2P_ORDER_PLAN, accumulate: int = 0, stream: int = 0):
    _check(load_library().p2p_apply_host(plan, h_q, h_out, order, accumulate, stream or None), "p2p_apply_host")


def p2p_apply_host_async(plan, h_q: int, h_out: int, order: int = P2P_ORDER_PLAN, accumulate: int = 0,
                         stream: int = 0):
    _check(load_library().p2p_apply_host_async(plan, h_q, h_out, order, accumulate, stream or None),
           "p2p_apply_host_async")


def p2p_apply_dist_interior(plan, d_q_owned: int, d_out: int, accumulate: int = 0, stream: int = 0):
    _check(load_library().p2p_apply_dist_interior(plan, d_q_owned or None, d_out, accumulate, stream or None),
           "p2p_apply_dist_interior")


def p2p_apply_dist_boundary(plan, d_q_halo: int, d_out: int, accumulate: int = 0, stream: int = 0):
    _check(load_library().p2p_apply_dist_boundary(plan, d_q_halo or None, d_out, accumulate, stream or None),
           "p2p_apply_dist_boundary")


def p2p_apply_dist(plan, d_q_owned: int, d_q_halo: int, d_out: int, accumulate: int = 0, stream: int = 0):
    _check(load_library().p2p_apply_dist(plan, d_q_owned or None, d_q_halo or None, d_out, accumulate,
                                         stream or None), "p2p_apply_dist")


def p2p_halo_pack(plan, d_q_owned: int, d_send: int, stream: int = 0):
    _check(load_library().p2p_halo_pack(plan, d_q_owned or None, d_send or None, stream or None), "p2p_halo_pack")


def p2p_apply_dist_peer(plan, d_q_owned: int, peer_ptrs, d_out: int, accumulate: int = 0, stream: int = 0):
    arr = (C.c_void_p * len(peer_ptrs))(*[p or None for p in peer_ptrs])
    _check(load_library().p2p_apply_dist_peer(plan, d_q_owned or None, arr, d_out, accumulate, stream or None),
           "p2p_apply_dist_peer")


def p2p_gather_peer(plan, peer_out_ptrs, d_global: int, stream: int = 0):
    arr = (C.c_void_p * len(peer_out_ptrs))(*[p or None for p in peer_out_ptrs])
    _check(load_library().p2p_gather_peer(plan, arr, d_global, stream or None), "p2p_gather_peer")


def p2p_peer_buffers(plan) -> tuple[int, int, int]:
    """(published send buffer, published result buffer, signal block) device pointers."""
    a, b, c = C.c_void_p(), C.c_void_p(), C.c_void_p()
    _check(load_library().p2p_peer_buffers(plan, C.byref(a), C.byref(b), C.byref(c)), "p2p_peer_buffers")
    return a.value, b.value, c.value


def p2p_peer_connect(plan, pub_w, pub_o, sig, displ):
    n = len(pub_w)
    arr = lambda v: (C.c_void_p * n)(*[p or None for p in v])  # noqa: E731
    d = (C.c_int64 * n)(*[int(x) for x in displ])
    _check(load_library().p2p_peer_connect(plan, arr(pub_w), arr(pub_o), arr(sig), d), "p2p_peer_connect")


def p2p_apply_peer_sync(plan, d_q_owned: int, d_out: int, accumulate: int = 0, stream: int = 0):
    _check(load_library().p2p_apply_peer_sync(plan, d_q_owned or None, d_out, accumulate, stream or None),
           "p2p_apply_peer_sync")


def p2p_gather(plan, d_local: int, d_global: int, stream: int = 0):
    _check(load_library().p2p_gather(plan, d_local or None, d_global, stream or None), "p2p_gather")


def p2p_peer_check(plan):
    _check(load_library().p2p_peer_check(plan), "p2p_peer_check")


def p2p_plan_set_workspaces(plan, n: int):
    _check(load_library().p2p_plan_set_workspaces(plan, n), "p2p_plan_set_workspaces")


def p2p_box_counts(level: int, xy) -> np.ndarray:
    """int32 per-box counts [4^(level-1)] (Morton order) of the points xy [n, 2]."""
    xy = np.ascontiguousarray(xy, dtype=np.float64).reshape(-1, 2)
    out = np.empty(1 << (2 * (level - 1)), dtype=np.int32)
    _check(load_library().p2p_box_counts(level, len(xy), xy.ctypes.data if len(xy) else None, out.ctypes.data),
           "p2p_box_counts")
    return out


def _local_args(src_ids, tgt_ids, src_counts, tgt_counts):
    a = [np.ascontiguousarray(src_ids, dtype=np.int64), np.ascontiguousarray(tgt_ids, dtype=np.int64),
         np.ascontiguousarray(src_counts, dtype=np.int32), np.ascontiguousarray(tgt_counts, dtype=np.int32)]
    ptr = [x.ctypes.data if x.size else None for x in a]
    return a, ptr, int(a[2].sum(dtype=np.int64)), int(a[3].sum(dtype=np.int64))


def p2p_partition_route(desc, src_ids, tgt_ids, src_counts, tgt_counts):
    """(source masks, target masks): per passed point, the bit mask of the ranks that need it."""
    keep, ptr, ns, nt = _local_args(src_ids, tgt_ids, src_counts, tgt_counts)
    sm = np.zeros(max(1, desc.n_src), dtype=np.uint32)
    tm = np.zeros(max(1, desc.n_tgt), dtype=np.uint32)
    _check(load_library().p2p_partition_route(C.byref(desc), *ptr, ns, nt, sm.ctypes.data, tm.ctypes.data),
           "p2p_partition_route")
    return sm[:desc.n_src], tm[:desc.n_tgt]


def p2p_plan_create_local(desc, src_ids, tgt_ids, src_counts, tgt_counts):
    keep, ptr, ns, nt = _local_args(src_ids, tgt_ids, src_counts, tgt_counts)
    h = C.c_void_p()
    _check(load_library().p2p_plan_create_local(C.byref(desc), *ptr, ns, nt, C.byref(h)), "p2p_plan_create_local")
    return h


def p2p_ipc_export(d_ptr: int) -> tuple[bytes, int]:
    """(64-byte IPC handle of the allocation holding d_ptr, d_ptr's offset in it)."""
    buf = C.create_string_buffer(64)
    off = C.c_int64(0)
    _check(load_library().p2p_ipc_export(d_ptr, buf, C.byref(off)), "p2p_ipc_export")
    return buf.raw, off.value


def p2p_ipc_open(handle: bytes, offset: int, device: int) -> int:
    out = C.c_void_p()
    _check(load_library().p2p_ipc_open(C.c_char_p(handle), offset, device, C.byref(out)), "p2p_ipc_open")
    return out.value


def p2p_ipc_close(d_ptr: int, offset: int):
    _check(load_library().p2p_ipc_close(d_ptr or None, offset), "p2p_ipc_close")


def p2p_destroy(plan):
    _check(load_library().p2p_destroy(plan), "p2p_destroy")


def p2p_plan_get_info(plan) -> dict:
    info = PlanInfo()
    _check(load_library().p2p_plan_get_info(plan, C.byref(info)), "p2p_plan_get_info")
    return {name: getattr(info, name) for name, _ in PlanInfo._fields_ if name != "struct_size"}


def p2p_plan_export(plan, kind) -> np.ndarray:
    k = EXPORT[kind] if isinstance(kind, str) else int(kind)
    nbytes = C.c_size_t(0)
    lib = load_library()
    _check(lib.p2p_plan_export(plan, k, None, C.byref(nbytes)), "p2p_plan_export")
    out = np.empty(nbytes.value // 8, dtype=np.int64)
    if out.size:
        _check(lib.p2p_plan_export(plan, k, out.ctypes.data_as(C.c_void_p), C.byref(nbytes)), "p2p_plan_export")
    return out


# ------------------------------------------------------------- convenience
_LAYOUTS = {"nr": P2P_LAYOUT_NONREDUNDANT, "r": P2P_LAYOUT_REDUNDANT, "tiled": P2P_LAYOUT_TILED,
            "paper_i": P2P_LAYOUT_PAPER_INDEXING, "paper_r": P2P_LAYOUT_PAPER_REPETITION,
            "adaptive": P2P_LAYOUT_ADAPTIVE}


def make_desc(src_xy, tgt_xy, *, level: int = 0, ct: int = 15, l_start: int = 3, l_max: int = 15,
              level_delta: int = 0, epsilon: float = 1e-12, layout: str = "nr", precision: str = "fp32",
              device: int = 0, tile_log2: int = -1, stream: int = 0, part_world: int = 1, part_rank: int = 0,
              kernel: str = "laplace", wavenumber: float = 0.0) -> PlanDesc:
    """A p2p_plan_desc over host point arrays (kept alive by the caller while it is used)."""
    d = p2p_plan_desc_init()
    d.n_src, d.n_tgt = len(src_xy), len(tgt_xy)
    d.src_xy = src_xy.ctypes.data if len(src_xy) else None
    d.tgt_xy = tgt_xy.ctypes.data if len(tgt_xy) else None
    d.level, d.ct, d.l_start, d.l_max, d.level_delta = level, ct, l_start, l_max, level_delta
    d.epsilon = epsilon
    d.layout = _LAYOUTS[layout]
    d.precision = {"fp32": P2P_FP32, "fp64": P2P_FP64}[precision]
    d.device, d.tile_log2, d.stream = device, tile_log2, stream or None
    d.part_world, d.part_rank = part_world, part_rank
    d.kernel = KERNELS[kernel]
    d.wavenumber = wavenumber
    return d


class Plan:
    """A P2P plan: ``Plan(src_xy, tgt_xy, level=...)`` then ``plan.apply(q, out)``.

    src_xy / tgt_xy: numpy float64 [n, 2] in [0,1]^2 (copied by the library).
    layout: "nr" (non-redundant), "r" (redundant per box) or "tiled" (redundant on
    the tile ring only); "paper_i" / "paper_r": the paper's own Indexing / Repetition
    layouts and kernels (fp64); precision: "fp32" or "fp64".
    kernel: "laplace" (the paper's ln(1/r)) or "helmholtz" ((i/4) H0^(1)(kappa r) with
    ``wavenumber`` = kappa; complex q / phi; TILED layout); "laplace3d" (1/(4 pi r)) or
    "helmholtz3d" (e^{i kappa r}/(4 pi r)) on the octree leaf grid: points [n, 3], layout "nr".
    device: CUDA ordinal, or -1 for a host-only plan (build + export only).
    build: "host" (p2p_plan_create: the C++ builder on the CPU) or "device"
    (p2p_plan_create_device: the same plan built by GPU kernels; src_xy / tgt_xy may then
    be CUDA float64 [n, 2] tensors, numpy input is copied to the device first), or "local"
    (p2p_plan_create_local: a partition's plan from the points this rank received; pass
    ``local=(src_ids, tgt_ids, src_counts, tgt_counts)`` -- their global ids and the global
    per-box counts; see dist.DistributedP2P.from_local).
    """

    def __init__(self, src_xy, tgt_xy=None, *, level: int = 0, ct: int = 15, l_start: int = 3,
                 l_max: int = 15, level_delta: int = 0, epsilon: float = 1e-12, layout: str = "nr",
                 precision: str = "fp32", device: int = 0, tile_log2: int = -1, stream: int = 0,
                 part_world: int = 1, part_rank: int = 0, build: str = "host", kernel: str = "laplace",
                 wavenumber: float = 0.0, local=None):
        if build not in ("host", "device", "local"):
            raise ValueError("build must be 'host', 'device' or 'local'")
        dim = 3 if kernel.endswith("3d") else 2
        d = p2p_plan_desc_init()
        if build == "device":
            import torch
            dev = torch.device("cuda", device)
            self._src = torch.as_tensor(src_xy, dtype=torch.float64, device=dev).contiguous()
            self._tgt = self._src if tgt_xy is None else \
                torch.as_tensor(tgt_xy, dtype=torch.float64, device=dev).contiguous()
            if self._src.dim() != 2 or self._src.shape[1] != dim or self._tgt.dim() != 2 or self._tgt.shape[1] != dim:
                raise ValueError(f"points must be [n, {dim}] arrays")
            d.n_src, d.n_tgt = self._src.shape[0], self._tgt.shape[0]
        else:
            self._src = np.ascontiguousarray(src_xy, dtype=np.float64)
            self._tgt = self._src if tgt_xy is None else np.ascontiguousarray(tgt_xy, dtype=np.float64)
            if self._src.ndim != 2 or self._src.shape[1] != dim or self._tgt.ndim != 2 or self._tgt.shape[1] != dim:
                raise ValueError(f"points must be [n, {dim}] arrays")
            d.n_src, d.n_tgt = len(self._src), len(self._tgt)
            d.src_xy = self._src.ctypes.data
            d.tgt_xy = self._tgt.ctypes.data
        d.level, d.ct, d.l_start, d.l_max, d.level_delta = level, ct, l_start, l_max, level_delta
        d.epsilon = epsilon
        d.layout = {"nr": P2P_LAYOUT_NONREDUNDANT, "r": P2P_LAYOUT_REDUNDANT, "tiled": P2P_LAYOUT_TILED,
                    "paper_i": P2P_LAYOUT_PAPER_INDEXING, "paper_r": P2P_LAYOUT_PAPER_REPETITION,
                    "adaptive": P2P_LAYOUT_ADAPTIVE}[layout]
        d.precision = {"fp32": P2P_FP32, "fp64": P2P_FP64}[precision]
        d.device, d.tile_log2, d.stream = device, tile_log2, stream or None
        d.part_world, d.part_rank = part_world, part_rank
        d.kernel = KERNELS[kernel]
        d.wavenumber = wavenumber
        self.kernel = kernel
        self.layout, self.precision, self.device, self.build = layout, precision, device, build
        if build == "device":
            if not stream:
                import torch
                d.stream = torch.cuda.current_stream(device).cuda_stream or None
            self._h = p2p_plan_create_device(d, self._src.data_ptr(), self._tgt.data_ptr())
            self._src = self._tgt = None  # read during the call only
        elif build == "local":
            self._h = p2p_plan_create_local(d, *local)
        else:
            self._h = p2p_plan_create(d)
        self.info = p2p_plan_get_info(self._h)

    @property
    def handle(self):
        return self._h

    @property
    def torch_dtype(self):
        """Element type of q and phi: real, or complex for the Helmholtz kernel."""
        import torch
        if self.kernel.startswith("helmholtz"):
            return torch.complex64 if self.precision == "fp32" else torch.complex128
        return torch.float32 if self.precision == "fp32" else torch.float64

    @property
    def np_dtype(self):
        if self.kernel.startswith("helmholtz"):
            return np.complex64 if self.precision == "fp32" else np.complex128
        return np.float32 if self.precision == "fp32" else np.float64

    def export(self, kind) -> np.ndarray:
        return p2p_plan_export(self._h, kind)

    def set_workspaces(self, n: int):
        """Up to n applies of this plan in flight on different streams (p2p_plan_set_workspaces)."""
        p2p_plan_set_workspaces(self._h, n)

    def _stream(self, stream):
        if stream is not None:
            return int(stream)
        import torch
        return torch.cuda.current_stream(self.device).cuda_stream

    def _check_tensor(self, t, n, name):
        import torch
        if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != self.torch_dtype or not t.is_contiguous():
            raise TypeError(f"{name} must be a contiguous CUDA {self.torch_dtype} tensor")
        if t.numel() != n:
            raise ValueError(f"{name} has {t.numel()} elements, expected {n}")

    def apply(self, q, out=None, *, order: str = "plan", accumulate: bool = False, stream=None):
        """phi = A q on the device (asynchronous on the current torch stream)."""
        import torch
        o = P2P_ORDER_USER if order == "user" else P2P_ORDER_PLAN
        n_out = self.info["n_tgt"] if o == P2P_ORDER_USER else self.info["n_tgt_local"]
        self._check_tensor(q, self.info["n_src"], "q")
        if out is None:
            out = torch.zeros(n_out, dtype=self.torch_dtype, device=q.device)
        self._check_tensor(out, n_out, "out")
        p2p_apply(self._h, q.data_ptr(), out.data_ptr(), o, int(accumulate), self._stream(stream))
        return out

    def apply_host(self, q: np.ndarray, out: np.ndarray | None = None, *, order: str = "plan",
                   accumulate: bool = False, stream=None) -> np.ndarray:
        """phi = A q from/to host buffers (H2D, apply, D2H, synchronise)."""
        o = P2P_ORDER_USER if order == "user" else P2P_ORDER_PLAN
        n_out = self.info["n_tgt"] if o == P2P_ORDER_USER else self.info["n_tgt_local"]
        if q.dtype != self.np_dtype or q.size != self.info["n_src"] or not q.flags.c_contiguous:
            raise TypeError("q: wrong dtype/size/layout")
        if out is None:
            out = np.zeros(n_out, dtype=self.np_dtype)
        p2p_apply_host(self._h, q.ctypes.data, out.ctypes.data, o, int(accumulate), self._stream(stream))
        return out

    def apply_dist(self, q_owned, q_halo, out, *, accumulate: bool = False, stream=None):
        self._check_tensor(out, self.info["n_tgt_local"], "out")
        p2p_apply_dist(self._h, q_owned.data_ptr() if q_owned.numel() else 0,
                       q_halo.data_ptr() if q_halo.numel() else 0, out.data_ptr(), int(accumulate),
                       self._stream(stream))
        return out

    def apply_dist_interior(self, q_owned, out, *, accumulate: bool = False, stream=None):
        self._check_tensor(out, self.info["n_tgt_local"], "out")
        p2p_apply_dist_interior(self._h, q_owned.data_ptr() if q_owned.numel() else 0, out.data_ptr(),
                                int(accumulate), self._stream(stream))
        return out

    def apply_dist_boundary(self, q_halo, out, *, accumulate: bool = False, stream=None):
        self._check_tensor(out, self.info["n_tgt_local"], "out")
        p2p_apply_dist_boundary(self._h, q_halo.data_ptr() if q_halo.numel() else 0, out.data_ptr(),
                                int(accumulate), self._stream(stream))
        return out

    def halo_pack(self, q_owned, send, stream=None):
        p2p_halo_pack(self._h, q_owned.data_ptr() if q_owned.numel() else 0,
                      send.data_ptr() if send.numel() else 0, self._stream(stream))
        return send

    def close(self):
        if getattr(self, "_h", None):
            p2p_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
