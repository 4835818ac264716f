"""The C-ABI library loads, exports every symbol include/p2p.h declares, and
behaves per its documented error contract -- all without a GPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2403_01596_b200 import p2p
from paper_2403_01596_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "p2p.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(p2p_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = p2p.load_library()
    declared = _declared_functions()
    assert len(declared) >= 12
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in include/p2p.h but not exported"
    assert set(declared) == set(p2p.ABI_SYMBOLS)
    assert lib.p2p_abi_version() == 1


def test_struct_layouts_match():
    d = p2p.p2p_plan_desc_init()
    assert d.struct_size == C.sizeof(p2p.PlanDesc)
    assert d.ct == 15 and d.l_start == 3 and d.epsilon == 1e-12 and d.part_world == 1
    h = p2p.Plan(np.array([[0.5, 0.5]]), level=2, device=-1)
    info = p2p.PlanInfo()
    p2p.load_library().p2p_plan_get_info(h.handle, C.byref(info))
    assert info.struct_size == C.sizeof(p2p.PlanInfo)


def test_status_strings():
    lib = p2p.load_library()
    assert lib.p2p_status_string(0) == b"P2P_SUCCESS"
    assert lib.p2p_status_string(7) == b"P2P_ERROR_NO_DEVICE"


@pytest.mark.parametrize("bad,status", [
    (dict(src=np.zeros((0, 2))), p2p.P2P_ERROR_INVALID_ARGUMENT),
    (dict(src=np.array([[0.5, 1.5]])), p2p.P2P_ERROR_INVALID_ARGUMENT),
    (dict(src=np.array([[np.nan, 0.5]])), p2p.P2P_ERROR_INVALID_ARGUMENT),
    (dict(level=3, level_delta=-3), p2p.P2P_ERROR_INVALID_ARGUMENT),
    (dict(level=16), p2p.P2P_ERROR_NOT_SUPPORTED),
])
def test_invalid_arguments(bad, status):
    src = bad.get("src", np.array([[0.25, 0.75], [0.5, 0.5]]))
    with pytest.raises(p2p.P2PError) as ei:
        p2p.Plan(src, level=bad.get("level", 3), level_delta=bad.get("level_delta", 0), device=-1)
    assert ei.value.status == status
    assert p2p.load_library().p2p_last_error() != b""


def test_ct_loop_construction_failure():
    pts = np.full((40, 2), 0.3)  # 40 coincident points can never satisfy CT = 15
    with pytest.raises(p2p.P2PError) as ei:
        p2p.Plan(pts, ct=15, device=-1)
    assert ei.value.status == p2p.P2P_ERROR_CONSTRUCTION_FAILURE


def test_host_only_plan_refuses_apply():
    plan = p2p.Plan(np.array([[0.5, 0.5]]), level=2, device=-1)
    with pytest.raises(p2p.P2PError) as ei:
        p2p.p2p_apply(plan.handle, 8, 8)  # pointers are never touched
    assert ei.value.status == p2p.P2P_ERROR_NO_DEVICE
    with pytest.raises(p2p.P2PError):
        p2p.p2p_apply(None, 8, 8)


def test_destroy_null_is_noop():
    p2p.p2p_destroy(None)


def test_plan_info_struct_size_prefix():
    """A caller with an older, smaller p2p_plan_info gets only its prefix (include/p2p.h)."""
    src, tgt, _ = W.make_problem("tiny")
    with p2p.Plan(src, tgt, level=4, device=-1) as h:
        lib = p2p.load_library()
        cut = p2p.PlanInfo.cta_threads.offset
        buf = (C.c_uint8 * C.sizeof(p2p.PlanInfo))(*([0xAB] * C.sizeof(p2p.PlanInfo)))
        info = p2p.PlanInfo.from_buffer(buf)
        info.struct_size = cut
        assert lib.p2p_plan_get_info(h.handle, C.byref(info)) == 0
        assert info.struct_size == cut and info.level == 4
        assert bytes(buf[cut:]) == bytes([0xAB] * (C.sizeof(p2p.PlanInfo) - cut))
        info.struct_size = 2  # smaller than the struct_size field itself: rejected
        assert lib.p2p_plan_get_info(h.handle, C.byref(info)) == p2p.P2P_ERROR_INVALID_ARGUMENT


def test_plan_info_field_order_matches_header():
    """The ctypes PlanInfo follows include/p2p.h field by field (names and order)."""
    hdr = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "p2p.h")).read()
    body = hdr[hdr.index("typedef struct {", hdr.index("p2p_status p2p_destroy")):hdr.index("} p2p_plan_info;")]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    names = []
    for decl in body.split(";"):
        decl = decl.replace("typedef struct {", "").strip()
        if not decl:
            continue
        parts = decl.split(None, 1)
        names += [n.strip() for n in parts[1].split(",")]
    assert names == [n for n, _ in p2p.PlanInfo._fields_]
