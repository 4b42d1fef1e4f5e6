"""The C-ABI library loads and exports every symbol include/gmp.h declares.

Runs on CPU: only argument-validation paths are exercised (they return before
any CUDA call), never a compute launch.
"""

import ctypes
import re
from pathlib import Path

import pytest

from paper_1909_01315_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "gmp.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(gmp_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 12
    for name in names:
        assert hasattr(lib, name), name
    assert set(_lib.EXPORTED) == set(names)


def test_version_and_strerror():
    lib = _lib.load()
    assert lib.gmp_version() == 1
    assert lib.gmp_strerror(0) == b"ok"
    assert lib.gmp_strerror(1) == b"invalid argument"


def test_invalid_arguments_rejected_without_gpu():
    lib = _lib.load()
    adj = _lib.GmpAdj(3, 3, None, None, None)
    x = _lib.GmpOperand(ctypes.c_void_p(16), 1, 1, _lib.TARGETS["src"])
    # unknown reducer
    st = lib.gmp_gspmm(ctypes.byref(adj), None, 0, 9, 0, ctypes.byref(x), None, None, 1, 1,
                       None, None, None, None, None)
    assert st == _lib.GMP_EINVAL and b"reducer" in lib.gmp_last_error()
    # dot with unequal dims
    y = _lib.GmpOperand(ctypes.c_void_p(16), 2, 2, _lib.TARGETS["dst"])
    coo = _lib.GmpCoo(3, 3, None, None)
    st = lib.gmp_gsddmm(ctypes.byref(coo), _lib.OPS["dot"], 0, ctypes.byref(x), ctypes.byref(y),
                        None, 1, 1, None, None)
    assert st == _lib.GMP_EINVAL and b"dot needs equal operand dims" in lib.gmp_last_error()
    # non-broadcastable dims
    z = _lib.GmpOperand(ctypes.c_void_p(16), 3, 3, _lib.TARGETS["edge"])
    st = lib.gmp_gsddmm(ctypes.byref(coo), _lib.OPS["add"], 0, ctypes.byref(y), ctypes.byref(z),
                        None, 3, 3, None, None)
    assert st == _lib.GMP_EINVAL and b"not broadcastable" in lib.gmp_last_error()
    # same targets
    st = lib.gmp_gsddmm(ctypes.byref(coo), _lib.OPS["mul"], 0, ctypes.byref(x), ctypes.byref(x),
                        None, 1, 1, None, None)
    assert st == _lib.GMP_EINVAL and b"differ" in lib.gmp_last_error()
    # div without an error slot
    st = lib.gmp_gspmm(ctypes.byref(adj), None, _lib.OPS["div"], 0, 0, ctypes.byref(x),
                       ctypes.byref(_lib.GmpOperand(ctypes.c_void_p(16), 1, 1, 2)),
                       ctypes.c_void_p(16), 1, 1, None, None, None, None, None)
    assert st == _lib.GMP_EINVAL and b"err_pos" in lib.gmp_last_error()
    with pytest.raises(_lib.GmpError, match="invalid argument"):
        _lib.check(st, "gmp_gspmm")


def test_error_string_is_thread_local():
    import threading
    lib = _lib.load()
    coo = _lib.GmpCoo(3, 3, None, None)
    lib.gmp_gsddmm(ctypes.byref(coo), 42, 0, None, None, None, 1, 1, None, None)
    seen = []

    def other():
        seen.append(lib.gmp_last_error())

    t = threading.Thread(target=other)
    t.start()
    t.join()
    assert seen == [b""]
    assert b"unknown op" in lib.gmp_last_error()


def test_round1_entry_points_validate_without_gpu():
    """The entry points added this round reject bad arguments before any
    CUDA call, with a detail string."""
    lib = _lib.load()
    p = ctypes.c_void_p(256)
    adj = _lib.GmpAdj(3, 3, p, p, p)
    # gat aggregate: leading dimension smaller than the width
    st = lib.gmp_gat_aggregate(ctypes.byref(adj), None, 0, 0, p, 2, 4, p, 1, p, p, 4, None, 0,
                               None, None, None)
    assert st == _lib.GMP_EINVAL and b"leading" in lib.gmp_last_error()
    # uv stats: null el / er
    st = lib.gmp_edge_softmax_uv_stats(ctypes.byref(adj), None, 0, None, 1, None, 1, 1, p, 64,
                                       None)
    assert st == _lib.GMP_EINVAL and b"el / er" in lib.gmp_last_error()
    # pack: tile must be a power of two is checked by the launcher; bad ld here
    st = lib.gmp_pack_tiles(10, 8, 0, 64, p, 4, p, None)
    assert st == _lib.GMP_EINVAL and b"bad sizes" in lib.gmp_last_error()
    # binary extrema backward: copy is not a binary op
    coo = _lib.GmpCoo(3, 3, p, p)
    x = _lib.GmpOperand(p, 4, 4, _lib.TARGETS["src"])
    w = _lib.GmpOperand(p, 1, 1, _lib.TARGETS["edge"])
    st = lib.gmp_extrema_bwd_binary(ctypes.byref(coo), 3, 4, 0, p, p, 4, _lib.OPS["copy_lhs"], 0,
                                    ctypes.byref(x), ctypes.byref(w), p, 4, 4, 3, None, 0, None)
    assert st == _lib.GMP_EINVAL and b"binary extrema backward" in lib.gmp_last_error()
    # dot: d_out must be 1
    st = lib.gmp_extrema_bwd_binary(ctypes.byref(coo), 3, 4, 0, p, p, 4, _lib.OPS["dot"], 0,
                                    ctypes.byref(x), ctypes.byref(x), p, 4, 4, 3, None, 0, None)
    assert st == _lib.GMP_EINVAL and b"d_out must be 1" in lib.gmp_last_error()
    # neighbour sample: negative sizes
    st = lib.gmp_neighbor_sample(p, -1, p, 1, p, 0, p, p, None)
    assert st == _lib.GMP_EINVAL and b"bad sizes" in lib.gmp_last_error()
    # extrema backward of source rows needs the sort workspace
    st = lib.gmp_extrema_bwd_copy(3, 4, 0, p, p, 4, p, 3, p, 4, None, 0, None)
    assert st == _lib.GMP_EINVAL and b"workspace too small" in lib.gmp_last_error()
    assert lib.gmp_extrema_bwd_workspace_size(0, 4) == 0
    assert lib.gmp_extrema_bwd_workspace_size(1000, 4) >= 4 * 8 * 4000
    # staged g-SpMM: reducer, stage mode and accumulator are validated
    st = lib.gmp_gspmm_staged(ctypes.byref(adj), None, 0, _lib.RHOS["max"], 0, ctypes.byref(x),
                              None, p, 4, 0, None, p, 4, 4, None, None, None)
    assert st == _lib.GMP_EINVAL and b"sum / mean" in lib.gmp_last_error()
    st = lib.gmp_gspmm_staged(ctypes.byref(adj), None, 0, 0, 0, ctypes.byref(x), None, p, 4, 2,
                              None, p, 4, 4, None, None, None)
    assert st == _lib.GMP_EINVAL and b"stage mode" in lib.gmp_last_error()
    st = lib.gmp_gspmm_staged(ctypes.byref(adj), None, 0, 0, 0, ctypes.byref(x), None, None, 4,
                              0, None, p, 4, 4, None, None, None)
    assert st == _lib.GMP_EINVAL and b"accumulator" in lib.gmp_last_error()
    # rowdot: B must be the dtype or f64
    st = lib.gmp_rowdot(3, 4, 1, p, 4, 0, p, 4, None, p, 1, 0, None)
    assert st == _lib.GMP_EINVAL and b"B must be" in lib.gmp_last_error()
    # windowed softmax workspace: no schedule -> the plain size
    assert lib.gmp_edge_softmax_workspace_size_ex(ctypes.byref(adj), None, 8, 0, 0) == \
        lib.gmp_edge_softmax_workspace_size(3, 8)


def test_segplan_workspace_size():
    """gmp_edge_softmax_workspace_size_ex with a gmp_segplan in the schedule
    reserves the per-piece partials ((max, sum) per head) after the per-row
    statistics; a plan without arrays is ignored (pure size arithmetic, no
    device access)."""
    lib = _lib.load()
    adj = _lib.GmpAdj(3, 5, None, None, None)
    plan = _lib.GmpSegplan(256, 1000, 4096, 16, 1, 1, 1, 1, 1)
    sched = _lib.GmpSched()
    sched.n_heavy = 1
    sched.segplan = ctypes.addressof(plan)
    base = lib.gmp_edge_softmax_workspace_size(3, 8)
    for dtype, F in ((0, 4), (1, 8)):
        got = lib.gmp_edge_softmax_workspace_size_ex(ctypes.byref(adj), ctypes.byref(sched), 8,
                                                     dtype, 0)
        assert got >= base + 256 + 1000 * 8 * (F + 8)
    plan.perm = None
    assert lib.gmp_edge_softmax_workspace_size_ex(ctypes.byref(adj), ctypes.byref(sched), 8, 0,
                                                  0) == base
