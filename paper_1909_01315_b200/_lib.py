"""ctypes binding of libgmp.so (include/gmp.h).

This module is the "reference-side binding" INTEGRATION.md describes: plain
ctypes over the C-ABI, device pointers and sizes only. It fails loudly when
the shared library is missing - there is no CPU fallback behind it.
"""

import ctypes
import os
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libgmp.so"

# enums (include/gmp.h)
GMP_OK, GMP_EINVAL, GMP_ECUDA, GMP_EUNSUPPORTED = 0, 1, 2, 3
OPS = {"copy_lhs": 0, "copy_rhs": 1, "add": 2, "sub": 3, "mul": 4, "div": 5, "dot": 6}
TARGETS = {None: -1, "src": 0, "dst": 1, "edge": 2, "edge_pos": 3}
RHOS = {"sum": 0, "max": 1, "min": 2, "mean": 3}
GMP_F32, GMP_F64 = 0, 1
STAGE_FIRST, STAGE_MID, STAGE_LAST = 0, 1, 3

EXPORTED = ("gmp_schedule_workspace_size", "gmp_build_schedule", "gmp_gspmm", "gmp_gspmm_staged",
            "gmp_gsddmm",
            "gmp_edge_softmax_workspace_size", "gmp_edge_softmax_workspace_size_ex", "gmp_edge_softmax_fwd", "gmp_edge_softmax_uv_fwd", "gmp_edge_softmax_bwd", "gmp_route_extrema",
            "gmp_extrema_bwd_workspace_size", "gmp_extrema_bwd_copy", "gmp_gather_rows", "gmp_neighbor_sample",
            "gmp_edge_softmax_uv_stats", "gmp_gat_aggregate", "gmp_pack_tiles", "gmp_unpack_tiles",
            "gmp_extrema_bwd_binary", "gmp_rowdot", "gmp_last_error", "gmp_strerror", "gmp_launch_count",
            "gmp_version", "gmp_probe_l2_gather", "gmp_gspmm_ring_workspace_size",
            "gmp_gspmm_ring_prepare", "gmp_gspmm_ring", "gmp_gather_adj_workspace_size",
            "gmp_gather_adj")


class GmpAdj(ctypes.Structure):
    _fields_ = [("n_rows", ctypes.c_int64), ("m", ctypes.c_int64),
                ("indptr", ctypes.c_void_p), ("indices", ctypes.c_void_p),
                ("eids", ctypes.c_void_p)]


class GmpSched(ctypes.Structure):
    _fields_ = [("order", ctypes.c_void_p), ("n_heavy", ctypes.c_int64),
                ("n_medium", ctypes.c_int64), ("n_nonempty", ctypes.c_int64),
                ("heavy_threshold", ctypes.c_int32), ("light_threshold", ctypes.c_int32),
                ("sorted_eids", ctypes.c_void_p), ("max_degree", ctypes.c_int64),
                ("segplan", ctypes.c_void_p)]


class GmpSegplan(ctypes.Structure):
    _fields_ = [("n_pos", ctypes.c_int64), ("n_pieces", ctypes.c_int64), ("win", ctypes.c_int64),
                ("group", ctypes.c_int64),
                ("perm", ctypes.c_void_p), ("starts", ctypes.c_void_p),
                ("chunk_piece", ctypes.c_void_p), ("row_ptr", ctypes.c_void_p),
                ("row_pieces", ctypes.c_void_p)]


class GmpCoo(ctypes.Structure):
    _fields_ = [("n_nodes", ctypes.c_int64), ("m", ctypes.c_int64),
                ("src", ctypes.c_void_p), ("dst", ctypes.c_void_p)]


class GmpOperand(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("ld", ctypes.c_int64),
                ("dim", ctypes.c_int32), ("target", ctypes.c_int32)]


class GmpTuning(ctypes.Structure):
    _fields_ = [("tile_cols", ctypes.c_int32), ("warps_per_cta", ctypes.c_int32),
                ("l2_budget_mb", ctypes.c_int32)]


class GmpError(RuntimeError):
    """A libgmp call returned a non-zero status."""


_lib = None
_lock = threading.Lock()
_P = ctypes.POINTER


def _declare(lib):
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    c_int = ctypes.c_int
    lib.gmp_schedule_workspace_size.argtypes = [i64]
    lib.gmp_schedule_workspace_size.restype = ctypes.c_size_t
    lib.gmp_build_schedule.argtypes = [_P(GmpAdj), i32, i32, vp, vp, ctypes.c_size_t,
                                       _P(GmpSched), vp]
    lib.gmp_gspmm.argtypes = [_P(GmpAdj), _P(GmpSched), c_int, c_int, c_int,
                              _P(GmpOperand), _P(GmpOperand), vp, i64, i32, vp, vp, vp,
                              _P(GmpTuning), vp]
    lib.gmp_gspmm_staged.argtypes = [_P(GmpAdj), _P(GmpSched), c_int, c_int, c_int,
                                     _P(GmpOperand), _P(GmpOperand), vp, i64, c_int, vp, vp, i64,
                                     i32, vp, _P(GmpTuning), vp]
    lib.gmp_gsddmm.argtypes = [_P(GmpCoo), c_int, c_int, _P(GmpOperand), _P(GmpOperand),
                               vp, i64, i32, vp, vp]
    lib.gmp_edge_softmax_workspace_size.argtypes = [i64, i32]
    lib.gmp_edge_softmax_workspace_size.restype = ctypes.c_size_t
    lib.gmp_edge_softmax_workspace_size_ex.argtypes = [_P(GmpAdj), _P(GmpSched), i32, c_int, c_int]
    lib.gmp_edge_softmax_workspace_size_ex.restype = ctypes.c_size_t
    lib.gmp_edge_softmax_fwd.argtypes = [_P(GmpAdj), _P(GmpCoo), _P(GmpSched), c_int, vp, i64, i32,
                                         vp, i64, vp, ctypes.c_size_t, vp]
    lib.gmp_edge_softmax_uv_fwd.argtypes = [_P(GmpAdj), _P(GmpCoo), _P(GmpSched), c_int, vp, i64,
                                            vp, i64, i32, vp, i64, vp, ctypes.c_size_t, vp]
    lib.gmp_edge_softmax_bwd.argtypes = [_P(GmpAdj), _P(GmpCoo), _P(GmpSched), c_int, vp, i64, vp,
                                         i64, i32, vp, i64, vp, ctypes.c_size_t, vp]
    lib.gmp_route_extrema.argtypes = [i64, i32, c_int, vp, vp, i64, vp, i64, vp]
    lib.gmp_extrema_bwd_workspace_size.argtypes = [i64, i32]
    lib.gmp_extrema_bwd_workspace_size.restype = ctypes.c_size_t
    lib.gmp_extrema_bwd_copy.argtypes = [i64, i32, c_int, vp, vp, i64, vp, i64, vp, i64, vp,
                                         ctypes.c_size_t, vp]
    lib.gmp_gather_rows.argtypes = [i64, i32, c_int, vp, vp, i64, vp, i64, vp]
    lib.gmp_gather_adj_workspace_size.argtypes = [_P(GmpAdj), _P(GmpSched), i32, c_int]
    lib.gmp_gather_adj_workspace_size.restype = ctypes.c_size_t
    lib.gmp_gather_adj.argtypes = [_P(GmpAdj), _P(GmpSched), i32, c_int, vp, i64, vp, i64, vp,
                                   ctypes.c_size_t, vp]
    lib.gmp_neighbor_sample.argtypes = [vp, i64, vp, i64, vp, ctypes.c_uint64, vp, vp, vp]
    lib.gmp_edge_softmax_uv_stats.argtypes = [_P(GmpAdj), _P(GmpSched), c_int, vp, i64, vp, i64,
                                              i32, vp, ctypes.c_size_t, vp]
    lib.gmp_gat_aggregate.argtypes = [_P(GmpAdj), _P(GmpSched), c_int, c_int, vp, i64, i32, vp,
                                      i64, vp, vp, i64, vp, i64, vp, _P(GmpTuning), vp]
    lib.gmp_pack_tiles.argtypes = [i64, i32, c_int, i32, vp, i64, vp, vp]
    lib.gmp_rowdot.argtypes = [i64, i32, c_int, vp, i64, c_int, vp, i64, vp, vp, i64, c_int, vp]
    lib.gmp_extrema_bwd_binary.argtypes = [_P(GmpCoo), i64, i32, c_int, vp, vp, i64, c_int, c_int,
                                           _P(GmpOperand), _P(GmpOperand), vp, i64, i32, i64, vp,
                                           ctypes.c_size_t, vp]
    lib.gmp_unpack_tiles.argtypes = [i64, i32, c_int, i32, vp, vp, i64, vp]
    lib.gmp_probe_l2_gather.argtypes = [vp, i64, i32, i64, vp, vp]
    lib.gmp_gspmm_ring_workspace_size.argtypes = [_P(GmpAdj), _P(GmpSched)]
    lib.gmp_gspmm_ring_workspace_size.restype = ctypes.c_size_t
    lib.gmp_gspmm_ring_prepare.argtypes = [_P(GmpAdj), _P(GmpSched), vp, ctypes.c_size_t, vp]
    lib.gmp_gspmm_ring.argtypes = [_P(GmpAdj), _P(GmpSched), c_int, c_int, c_int,
                                   _P(GmpOperand), _P(GmpOperand), i64, vp, i64, i32, vp,
                                   ctypes.c_size_t, vp]
    lib.gmp_last_error.restype = ctypes.c_char_p
    lib.gmp_strerror.argtypes = [c_int]
    lib.gmp_strerror.restype = ctypes.c_char_p
    lib.gmp_launch_count.restype = ctypes.c_uint64
    for name in ("gmp_build_schedule", "gmp_gspmm", "gmp_gspmm_staged", "gmp_gsddmm", "gmp_edge_softmax_fwd",
                 "gmp_edge_softmax_uv_fwd",
                 "gmp_edge_softmax_bwd", "gmp_route_extrema", "gmp_extrema_bwd_copy",
                 "gmp_gather_rows", "gmp_neighbor_sample", "gmp_edge_softmax_uv_stats",
                 "gmp_gat_aggregate", "gmp_pack_tiles", "gmp_unpack_tiles",
                 "gmp_extrema_bwd_binary", "gmp_rowdot", "gmp_version", "gmp_probe_l2_gather",
                 "gmp_gspmm_ring_prepare", "gmp_gspmm_ring", "gmp_gather_adj"):
        getattr(lib, name).restype = c_int


def load():
    """The loaded library; raises ImportError if libgmp.so was never built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            path = os.environ.get("GMP_LIB", str(LIB_PATH))
            if not Path(path).exists():
                raise ImportError(
                    "libgmp.so not found at %s: build it with `python -c \"import "
                    "__graft_entry__ as g; g.build()\"` (no CPU fallback exists)" % path)
            lib = ctypes.CDLL(path)
            _declare(lib)
            _lib = lib
    return _lib


def check(status, what):
    if status != GMP_OK:
        lib = load()
        detail = lib.gmp_last_error().decode(errors="replace")
        raise GmpError("%s failed (%s): %s" % (
            what, lib.gmp_strerror(status).decode(), detail))


def launch_count():
    return int(load().gmp_launch_count())
