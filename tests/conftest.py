"""Shared fixtures: the gpu marker, golden-fixture access, oracle helpers.

`-m "not gpu"` tests run on CPU (oracle vs golden, host logic, ABI exports);
`-m gpu` tests are the parity tests proper and call the CUDA kernels through
the C-ABI. Only tests (and smoke/bench baselines) may import oracle/.
"""

import json
import sys
from functools import lru_cache
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libgmp.so")


def pytest_collection_modifyitems(config, items):
    import torch
    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@lru_cache(maxsize=1)
def golden():
    data = np.load(GOLDEN / "reference_cases.npz")
    return {k: data[k] for k in data.files}


@lru_cache(maxsize=1)
def golden_meta():
    return json.loads((GOLDEN / "reference_cases.json").read_text())


def golden_graph(prefix):
    gd = golden()
    return gd[prefix + "/src"], gd[prefix + "/dst"], int(gd[prefix + "/n"])


def case_operands(case):
    gd = golden()
    return {k: gd["c%d/%s" % (case, k)] for k in ("X", "Y", "W") if "c%d/%s" % (case, k) in gd}


def rel_err(got, want):
    """Reference's rel_err (conftest.py:111-117): max|diff| / max(1, max|want|)."""
    got = np.asarray(got, float)
    want = np.asarray(want, float)
    if got.size == 0:
        return 0.0
    return float(np.abs(got - want).max()) / max(1.0, float(np.abs(want).max()))


def to_np(x):
    if x is None:
        return None
    try:
        import torch
        if torch.is_tensor(x):
            return x.detach().cpu().numpy()
    except ImportError:
        pass
    return np.asarray(x)


# fp32 parity bound of the north star: elementwise rtol 1e-5 / atol 1e-6
RTOL32, ATOL32 = 1e-5, 1e-6


def assert_close32(got, want, what=""):
    got, want = to_np(got), np.asarray(want)
    assert got.shape == want.shape, (what, got.shape, want.shape)
    ok = np.isclose(got.astype(np.float64), want.astype(np.float64), rtol=RTOL32, atol=ATOL32)
    assert ok.all(), "%s: %d/%d cells outside rtol=1e-5 atol=1e-6, worst |d|=%g" % (
        what, (~ok).sum(), ok.size, np.abs(got.astype(np.float64) - want).max())
