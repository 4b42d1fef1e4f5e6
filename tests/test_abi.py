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
