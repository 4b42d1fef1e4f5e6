"""g-SpMM / g-SDDMM on B200: the reference's kernel-engine API over libgmp.so.

Drop-in for /root/reference/pkg/src/graphmp/kernels.py. Same names, same
argument meaning, same validation errors (ValueError texts of
kernels.py:86-97,217-251,692-701,748-759; ZeroDivisionError naming the edge,
kernels.py:263-268), same return shapes:

  gspmm(g, phi, rho, X, Y, W, ...) -> (Z, aux)   aux: None | counts | ArgExtrema
  gsddmm(g, phi, X, Y, W, ...)     -> M

Differences that are the point of the port:
  * every call is one launch of a hand-written sm_100a kernel through the
    C-ABI (include/gmp.h); there is no CPU path - a graph or operand that is
    not on a CUDA device raises;
  * results are torch tensors on the graph's device. Operand dtype is kept:
    float32 operands run the fp32 kernels, float64 (e.g. numpy defaults) the
    fp64 ones; mixed operands are promoted to float64 (the reference coerces
    everything to float64, kernels.py:216);
  * `strategy` / `fmt` keep their names and legality tables
    (kernels.py:47-65) and select a GPU schedule; every schedule returns
    identical results (deterministic, no float atomics). num_workers and
    block_edges are CPU-thread knobs and are accepted but unused.
"""

import ctypes
import os
import threading
from contextlib import contextmanager
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, accounting
from .graph import HEAVY_ROW_THRESHOLD, LIGHT_ROW_THRESHOLD

BLOCK_EDGES = 2048  # reference chunk size (kernels.py:39); device kernels need no host chunking

OPS = ("copy_lhs", "copy_rhs", "add", "sub", "mul", "div", "dot")
TARGETS = ("src", "dst", "edge")
REDUCERS = ("sum", "max", "min", "mean")

GSPMM_STRATEGIES = ("node_parallel", "edge_parallel", "edge_parallel_atomic",
                    "feature_parallel", "serial_reference")
GSDDMM_STRATEGIES = ("node_parallel", "edge_parallel", "feature_parallel",
                     "serial_reference")
_GSPMM_FORMATS = {
    "node_parallel": ("csc",),
    "edge_parallel": ("csc",),
    "edge_parallel_atomic": ("coo", "csr", "csc"),
    "feature_parallel": ("csc",),
    "serial_reference": ("coo",),
}
_GSDDMM_FORMATS = {
    "node_parallel": ("csr", "csc"),
    "edge_parallel": ("coo", "csr", "csc"),
    "feature_parallel": ("coo", "csr", "csc"),
    "serial_reference": ("coo",),
}
_INT32_MAX = 2 ** 31 - 1


# ----------------------------------------------------------------------------
# message function descriptors (kernels.py:72-144)


@dataclass(frozen=True)
class MessageFunc:
    """op plus the operand target(s) it reads; see kernels.py:72-104."""
    op: str
    lhs_target: str = None
    rhs_target: str = None

    def __post_init__(self):
        if self.op not in OPS:
            raise ValueError("unknown op %r" % (self.op,))
        if self.op == "copy_lhs":
            if self.lhs_target not in TARGETS or self.rhs_target is not None:
                raise ValueError("copy_lhs takes exactly one lhs target")
        elif self.op == "copy_rhs":
            if self.rhs_target not in TARGETS or self.lhs_target is not None:
                raise ValueError("copy_rhs takes exactly one rhs target")
        else:
            if self.lhs_target not in TARGETS or self.rhs_target not in TARGETS:
                raise ValueError("%s takes lhs and rhs targets" % self.op)
            if self.lhs_target == self.rhs_target:
                raise ValueError("binary op targets must differ")

    @property
    def targets(self):
        return tuple(t for t in (self.lhs_target, self.rhs_target) if t is not None)

    def describe(self):
        return "%s(%s)" % (self.op, ",".join(self.targets))


def copy(target):
    return MessageFunc("copy_lhs", lhs_target=target)


def copy_rhs(target):
    return MessageFunc("copy_rhs", rhs_target=target)


def add(lhs, rhs):
    return MessageFunc("add", lhs, rhs)


def sub(lhs, rhs):
    return MessageFunc("sub", lhs, rhs)


def mul(lhs, rhs):
    return MessageFunc("mul", lhs, rhs)


def div(lhs, rhs):
    return MessageFunc("div", lhs, rhs)


def dot(lhs, rhs):
    return MessageFunc("dot", lhs, rhs)


def builtin_message_funcs():
    """The 30 built-in phis in the reference's canonical order (kernels.py:136-144)."""
    out = [copy(t) for t in TARGETS]
    pairs = (("src", "dst"), ("dst", "src"), ("src", "edge"), ("edge", "src"),
             ("dst", "edge"), ("edge", "dst"))
    for op in ("add", "sub", "mul", "div"):
        out.extend(MessageFunc(op, a, b) for a, b in pairs)
    out.extend(dot(a, b) for a, b in (("src", "dst"), ("src", "edge"), ("dst", "edge")))
    return out


@dataclass
class ArgExtrema:
    """Winning edge id per max/min cell: int64 device tensor, -1 on empty rows."""
    arg_edge: torch.Tensor

    @property
    def empty_rows(self):
        return self.arg_edge[:, 0] < 0


# ----------------------------------------------------------------------------
# configuration (kernels.py:161-206)

_config = threading.local()


@contextmanager
def force_strategy(name):
    prev = getattr(_config, "strategy", None)
    _config.strategy = name
    try:
        yield
    finally:
        _config.strategy = prev


@contextmanager
def default_workers(n):
    prev = getattr(_config, "workers", 1)
    _config.workers = int(n)
    try:
        yield
    finally:
        _config.workers = prev


@contextmanager
def tuning(tile_cols=None, l2_budget_mb=None):
    """Thread-local override of the row kernels' column tile / L2 budget."""
    prev = getattr(_config, "tuning", None)
    _config.tuning = (tile_cols or 0, l2_budget_mb or 0)
    try:
        yield
    finally:
        _config.tuning = prev


def select_format(kernel, direction="forward"):
    """gspmm walks the in-adjacency (csc; its backward the reverse graph's csc
    == the forward csr); gsddmm walks the edge list (coo). kernels.py:193-206."""
    if kernel == "gspmm":
        return "csc"
    if kernel == "gsddmm":
        return "coo"
    raise ValueError("unknown kernel %r" % (kernel,))


# ----------------------------------------------------------------------------
# operand plumbing


def _require_cuda(g):
    if g.device.type != "cuda":
        raise RuntimeError(
            "paper_1909_01315_b200 kernels run only on a CUDA device (graph is on %s); "
            "there is no CPU fallback" % g.device)


def _to_tensor(name, M, device):
    if isinstance(M, torch.Tensor):
        t = M
        if not (t.dtype == torch.float32 or t.dtype == torch.float64):
            t = t.to(torch.float32 if t.is_floating_point() else torch.float64)
    else:
        a = np.asarray(M)
        if a.dtype != np.float32:
            a = a.astype(np.float64)
        t = torch.from_numpy(np.ascontiguousarray(a))
    if t.dim() != 2:
        raise ValueError("%s must be a 2-D matrix, got ndim=%d" % (name, t.dim()))
    if t.device != device:
        t = t.to(device)
    if t.shape[1] > 1 and t.stride(1) != 1:
        t = t.contiguous()
    return t


def _as_matrix(name, M, rows, device):
    if M is None:
        return None
    t = _to_tensor(name, M, device)
    if t.shape[0] != rows:
        raise ValueError("%s has %d rows, expected %d" % (name, t.shape[0], rows))
    return t


def _operands_for(g, phi, X, Y, W):
    """Validate presence and shapes (kernels.py:224-252); return X, Y, W, d_out."""
    needed = set(phi.targets)
    if "src" in needed and X is None:
        raise ValueError("phi %s needs X (source rows)" % phi.describe())
    if "dst" in needed and Y is None:
        raise ValueError("phi %s needs Y (destination rows)" % phi.describe())
    if "edge" in needed and W is None:
        raise ValueError("phi %s needs W (edge rows)" % phi.describe())
    dev = g.device
    X = _as_matrix("X", X, g.num_nodes, dev) if "src" in needed else None
    Y = _as_matrix("Y", Y, g.num_nodes, dev) if "dst" in needed else None
    W = _as_matrix("W", W, g.num_edges, dev) if "edge" in needed else None
    mats = {"src": X, "dst": Y, "edge": W}
    if any(m is not None and m.dtype == torch.float64 for m in mats.values()):
        mats = {k: (None if m is None else m.to(torch.float64)) for k, m in mats.items()}
    X, Y, W = mats["src"], mats["dst"], mats["edge"]

    def dim(t):
        return mats[t].shape[1]

    if phi.op in ("copy_lhs", "copy_rhs"):
        d_out = dim(phi.targets[0])
    elif phi.op == "dot":
        dl, dr = dim(phi.lhs_target), dim(phi.rhs_target)
        if dl != dr:
            raise ValueError("dot needs equal operand dims, got %d and %d" % (dl, dr))
        d_out = 1
    else:
        dl, dr = dim(phi.lhs_target), dim(phi.rhs_target)
        if dl != dr and 1 not in (dl, dr):
            raise ValueError("operand dims %d and %d are not broadcastable" % (dl, dr))
        d_out = max(dl, dr)
    return X, Y, W, d_out


def _dtype_code(t):
    return _lib.GMP_F64 if t.dtype == torch.float64 else _lib.GMP_F32


def _ld(t):
    return max(int(t.stride(0)), int(t.shape[1])) if t.shape[0] > 1 else int(t.shape[1])


_dummy = {}


def _data_ptr(t):
    """Device address of t; empty tensors get a valid dummy address (never read)."""
    if t.numel():
        return t.data_ptr()
    d = _dummy.get(t.device)
    if d is None:
        d = _dummy.setdefault(t.device, torch.zeros(4, dtype=torch.float64, device=t.device))
    return d.data_ptr()


def _operand(t, target):
    if t is None:
        return None
    return _lib.GmpOperand(_data_ptr(t), _ld(t), int(t.shape[1]), _lib.TARGETS[target])


def _phi_operands(phi, X, Y, W):
    mats = {"src": X, "dst": Y, "edge": W}
    lhs = _operand(mats[phi.lhs_target], phi.lhs_target) if phi.lhs_target else None
    rhs = _operand(mats[phi.rhs_target], phi.rhs_target) if phi.rhs_target else None
    return lhs, rhs


def _ptr(obj):
    return None if obj is None else ctypes.byref(obj)


def _stream(device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _adj_struct(adj):
    s = adj._extra.get("struct")
    if s is None:
        s = _lib.GmpAdj(adj.num_groups, adj.indices.numel(), adj.indptr.data_ptr(),
                        adj.indices.data_ptr(), adj.edge_ids.data_ptr())
        adj._extra["struct"] = s
    return s


class _Schedule:
    __slots__ = ("struct", "order", "n_heavy", "n_medium", "n_nonempty")


def _build_schedule(adj):
    """Degree-sorted row order + heavy-row count (gmp_build_schedule)."""
    lib = _lib.load()
    n = adj.num_groups
    dev = adj.indptr.device
    order = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    ws_bytes = int(lib.gmp_schedule_workspace_size(n))
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    sched = _lib.GmpSched()
    _lib.check(lib.gmp_build_schedule(ctypes.byref(_adj_struct(adj)), HEAVY_ROW_THRESHOLD,
                                      LIGHT_ROW_THRESHOLD, order.data_ptr(), ws.data_ptr(), ws_bytes,
                                      ctypes.byref(sched), _stream(dev)), "gmp_build_schedule")
    out = _Schedule()
    out.struct, out.order = sched, order
    out.n_heavy, out.n_nonempty = int(sched.n_heavy), int(sched.n_nonempty)
    out.n_medium = int(sched.n_medium)
    return out


def _tuning_struct(strategy):
    tc, l2 = getattr(_config, "tuning", None) or (0, 0)
    if strategy == "feature_parallel" and not tc:
        tc = 32  # the reference's column split, one 128 B line per row slice
    if not tc and not l2:
        return None
    return _lib.GmpTuning(int(tc), 0, int(l2))


def _err_slot(device):
    return torch.full((1,), _INT32_MAX, dtype=torch.int32, device=device)


def _raise_div_zero(eid):
    raise ZeroDivisionError("division by zero in edge message at edge id %d" % int(eid))


# ----------------------------------------------------------------------------
# g-SpMM (kernels.py:685-725)


def _resolve_strategy(kind, strategy, fmt):
    if kind == "gspmm":
        strategy = strategy or getattr(_config, "strategy", None) or "node_parallel"
        if strategy not in GSPMM_STRATEGIES:
            raise ValueError("unknown gspmm strategy %r" % (strategy,))
        allowed = _GSPMM_FORMATS[strategy]
    else:
        if strategy == "edge_parallel_atomic":
            raise ValueError("gsddmm writes disjoint rows; it has no atomic variant")
        forced = getattr(_config, "strategy", None)
        if forced == "edge_parallel_atomic":
            forced = "edge_parallel"
        strategy = strategy or forced or "edge_parallel"
        if strategy not in GSDDMM_STRATEGIES:
            raise ValueError("unknown gsddmm strategy %r" % (strategy,))
        allowed = _GSDDMM_FORMATS[strategy]
    fmt = fmt or allowed[0]
    if fmt not in allowed:
        raise ValueError("%s strategy %s cannot run on format %s" % (kind, strategy, fmt))
    return strategy, fmt


def gspmm(g, phi, rho, X=None, Y=None, W=None, strategy=None, num_workers=None,
          fmt=None, block_edges=None):
    """Reduce per-edge messages into one row per destination: (Z, aux)."""
    if rho not in REDUCERS:
        raise ValueError("unknown reducer %r" % (rho,))
    X, Y, W, d_out = _operands_for(g, phi, X, Y, W)
    strategy, fmt = _resolve_strategy("gspmm", strategy, fmt)
    accounting.log_dispatch("gspmm", g.uid, phi.describe(), rho, strategy, g.num_nodes, d_out)
    _require_cuda(g)
    return _gspmm_launch(g, phi, rho, X, Y, W, d_out, _tuning_struct(strategy))


# column tiles for wide gathered operands: 256 B per row slice (64 fp32 / 32 fp64)
_TILE_BYTES = 256
_L2_BUDGET = 64 << 20


def _tile_cols(n_src, F, d_out):
    """Packed column-tile width: 256 B rows (the pipelined row kernel's
    shape). Rows narrower than that (d = 17..63 fp32) whose whole slice
    overflows the L2 budget are cut into 128 B or 64 B tiles (down to 64 B)
    until a tile's slice fits: C5 power-law / uniform n = 10^6, copy_u + sum
    d = 32: 1.47 / 1.20 -> 1.00 / 0.72 ms. Wider rows keep 256 B tiles even
    when a slice overflows: narrower tiles re-read the index arrays per tile
    and gather short runs (d = 128: 2.3 -> 4.0 ms with 64 B tiles)."""
    t = _TILE_BYTES // F
    if d_out >= t:
        return t
    while t * F > 64 and n_src * t * F > _L2_BUDGET:
        t //= 2
    return t


def _tiled_applies(phi, rho, X, W, d_out, n, tune):
    """Wide src-gathered aggregations whose column slices must be L2-tiled
    (the row kernel's rule) and whose rows are not already aligned 256 B runs:
    copy_u, or u_op_e with a per-edge scalar (the attention-weighted sum),
    under sum / mean. Packing the tiles makes every gather whole sectors read
    with 128-bit loads."""
    if tune is not None or rho not in ("sum", "mean") or X is None or n == 0:
        return False
    if phi.op == "copy_lhs":
        if phi.lhs_target != "src":
            return False
    elif phi.op in ("add", "sub", "mul", "div"):
        if (phi.lhs_target, phi.rhs_target) != ("src", "edge") or W is None or W.shape[1] != 1:
            return False
    else:
        return False
    if X.shape[1] != d_out:
        return False
    F = X.element_size()
    # the gathered slice is X's (source) rows - a row block of a partitioned
    # graph gathers more (or fewer) rows than it has destinations
    tile = _tile_cols(X.shape[0], F, d_out)
    if d_out <= tile or X.shape[0] * d_out * F <= _L2_BUDGET:
        return False
    if tile < _TILE_BYTES // F:
        return True  # narrower than one warp pass: the row kernel cannot split it in place
    aligned = _ld(X) % tile == 0 and X.data_ptr() % 16 == 0
    return not aligned


def _staged_call(lib, adj, sched, phi, rho, code, lhs, rhs, Z, ldz, d_out, err, tune, stream,
                 stage, col0=0):
    """gmp_gspmm, or gmp_gspmm_staged when `stage` = (acc fp64 tensor, mode,
    deg_full or None) is given (columns col0.. of acc for a column tile)."""
    if stage is None:
        return lib.gmp_gspmm(ctypes.byref(_adj_struct(adj)),
                             ctypes.byref(sched.struct) if sched is not None else None,
                             _lib.OPS[phi.op], _lib.RHOS[rho], code, _ptr(lhs), _ptr(rhs),
                             Z, ldz, d_out, None, None, err, _ptr(tune), stream)
    acc, mode, deg_full = stage
    return lib.gmp_gspmm_staged(ctypes.byref(_adj_struct(adj)),
                                ctypes.byref(sched.struct) if sched is not None else None,
                                _lib.OPS[phi.op], _lib.RHOS[rho], code, _ptr(lhs), _ptr(rhs),
                                acc.data_ptr() + col0 * 8, _ld(acc), mode,
                                deg_full.data_ptr() if deg_full is not None else None,
                                Z, ldz, d_out, err, _ptr(tune), stream)


# The heavy-row TMA gather4 ring (spmm_ring.cu) is opt-in (GMP_RING=1): it is
# correct and deterministic, but measured slower than the register-gather row
# kernel on the Reddit-shaped headline (copy_u d=602: 28.1 vs 23.8 ms; u_mul_e
# 41.0 vs 36.1 ms at 16 warps / SM; profiles/r02_tma_ring.json, DESIGN 3.1).
_RING_OFF = os.environ.get("GMP_RING", "0") in ("", "0")


def _ring_workspace(adj, sched, stream):
    """Workspace of the heavy-row TMA gather4 ring (gmp_gspmm_ring), prepared
    once per adjacency and cached with it; None when the schedule has no
    heavy rows or the ring is not enabled (GMP_RING=1)."""
    if _RING_OFF or sched.n_heavy <= 0:
        return None
    # one workspace per stream: calls on a stream are ordered; concurrent
    # callers on other streams get their own counter and partials
    key = ("ring_ws", stream.value)
    ws = adj._extra.get(key)
    if ws is None:
        lib = _lib.load()
        a, sc = ctypes.byref(_adj_struct(adj)), ctypes.byref(sched.struct)
        nbytes = int(lib.gmp_gspmm_ring_workspace_size(a, sc))
        ws = torch.empty(nbytes, dtype=torch.uint8, device=adj.indptr.device)
        _lib.check(lib.gmp_gspmm_ring_prepare(a, sc, ws.data_ptr(), nbytes, stream),
                   "gmp_gspmm_ring_prepare")
        adj._extra[key] = ws
    return ws


def _gspmm_tiled(g, phi, rho, X, W, Z, d_out, stage=None, events=None):
    """Aggregation over packed column tiles: gmp_pack_tiles, then one
    gmp_gspmm per 256 B tile (each tile's slice of X stays L2-resident while
    every destination row gathers it; a per-edge scalar is laid out in CSC
    order once and streamed by every tile) writing its columns of Z in place
    (16 B vectors stored as two 8 B halves when Z's rows are only 8 B
    aligned). `events` (measurement): a list that receives one (start, end)
    pair of CUDA events recorded around each tile launch."""
    lib = _lib.load()
    dev = g.device
    n = g.num_nodes
    F = X.element_size()
    tile = _tile_cols(X.shape[0], F, d_out)
    nt = -(-d_out // tile)
    code = _dtype_code(X)
    stream = _stream(dev)
    adj = g.to_csc()
    sched = adj.schedule()
    rhs = None
    err = None
    if phi.op != "copy_lhs":
        Wc = _gather_adj(adj, W.to(X.dtype))
        rhs = _lib.GmpOperand(_data_ptr(Wc), 1, 1, _lib.TARGETS["edge_pos"])
        if phi.op == "div":
            err = _err_slot(dev)
    n_src = X.shape[0]  # source rows: packed and gathered; Z has the n destination rows
    Xp = torch.empty((nt, n_src, tile), dtype=X.dtype, device=dev)
    _lib.check(lib.gmp_pack_tiles(n_src, d_out, code, tile, X.data_ptr(), _ld(X), Xp.data_ptr(),
                                  stream), "gmp_pack_tiles")
    ldz = _ld(Z)
    ring = _ring_workspace(adj, sched, stream) if (
        stage is None and F == 4 and phi.op in ("copy_lhs", "mul")) else None
    for t in range(nt):
        w = min(tile, d_out - t * tile)
        lhs = _lib.GmpOperand(Xp[t].data_ptr(), tile, w, _lib.TARGETS["src"])
        if events is not None:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record(torch.cuda.current_stream(dev))
        if ring is not None:
            _lib.check(lib.gmp_gspmm_ring(ctypes.byref(_adj_struct(adj)), ctypes.byref(sched.struct),
                                          _lib.OPS[phi.op], _lib.RHOS[rho], code, ctypes.byref(lhs),
                                          _ptr(rhs), n_src, Z.data_ptr() + t * tile * F, ldz, w,
                                          ring.data_ptr(), ring.numel(), stream), "gmp_gspmm_ring")
        else:
            _lib.check(_staged_call(lib, adj, sched, phi, rho, code, lhs, rhs,
                                    Z.data_ptr() + t * tile * F, ldz, w,
                                    err.data_ptr() if err is not None else None, None, stream,
                                    stage, col0=t * tile), "gmp_gspmm")
        if events is not None:
            ev[1].record(torch.cuda.current_stream(dev))
            events.append(ev)
    if err is not None:
        pos = int(err.item())
        if pos != _INT32_MAX:
            _raise_div_zero(adj.edge_ids[pos].item())


def _gspmm_launch(g, phi, rho, X, Y, W, d_out, tune=None, out=None, stage=None):
    """One g-SpMM launch on g's CSC. `stage` = (acc, mode, deg_full): a staged
    sum / mean (gmp_gspmm_staged) accumulating into the fp64 buffer acc;
    Z is written only by the STAGE_LAST launch."""
    lib = _lib.load()
    dev = g.device
    n = g.num_nodes
    ref = next(t for t in (X, Y, W) if t is not None)
    if stage is not None and (rho not in ("sum", "mean") or phi.op == "dot"):
        raise ValueError("staged g-SpMM takes sum / mean of non-dot messages")
    if _tiled_applies(phi, rho, X, W, d_out, n, tune):
        Z = out if out is not None else accounting.register(
            torch.empty((n, d_out), dtype=ref.dtype, device=dev))
        _gspmm_tiled(g, phi, rho, X, W, Z, d_out, stage)
        return Z, (g.to_csc().degrees().clone() if rho == "mean" else None)
    if (stage is None and tune is None and phi.op == "copy_lhs" and phi.lhs_target == "src"
            and rho in ("sum", "mean") and X.dtype == torch.float32 and 32 < d_out <= 64
            and n > 0 and _ld(X) == 64 and X.data_ptr() % 16 == 0):
        # already-packed 256 B source rows (a host-pipeline tile, or d = 64):
        # heavy rows over the TMA gather4 ring
        adj = g.to_csc()
        sched = adj.schedule()
        ring = _ring_workspace(adj, sched, _stream(dev))
        if ring is not None:
            Z = out if out is not None else accounting.register(
                torch.empty((n, d_out), dtype=ref.dtype, device=dev))
            lhs = _lib.GmpOperand(X.data_ptr(), 64, d_out, _lib.TARGETS["src"])
            _lib.check(lib.gmp_gspmm_ring(ctypes.byref(_adj_struct(adj)),
                                          ctypes.byref(sched.struct), _lib.OPS["copy_lhs"],
                                          _lib.RHOS[rho], _lib.GMP_F32, ctypes.byref(lhs), None,
                                          X.shape[0], Z.data_ptr(), _ld(Z), d_out, ring.data_ptr(),
                                          ring.numel(), _stream(dev)), "gmp_gspmm_ring")
            return Z, (adj.degrees().clone() if rho == "mean" else None)
    Z = out if out is not None else accounting.register(
        torch.empty((n, d_out), dtype=ref.dtype, device=dev))
    arg = None
    if rho in ("max", "min"):
        arg = accounting.register(torch.empty((n, d_out), dtype=torch.int64, device=dev))
    adj = g.to_csc()
    err = _err_slot(dev) if phi.op == "div" else None
    if (X is not None and phi.lhs_target == "src" and phi.op != "dot" and rho in ("sum", "mean")
            and X.dim() == 2 and X.shape[1] == d_out and d_out >= 8
            and g.num_edges >= 4 * max(n, 1)):
        X = _pad_rows16(X)  # 16 B gathers for widths that are not a multiple of 4
    lhs, rhs = _phi_operands(phi, X, Y, W)
    if W is not None and phi.op != "dot" and _permute_edge_scalar(W, d_out):
        # a per-edge scalar re-read by >= 3 column tiles: lay it out in CSC
        # order once so every tile streams it (gmp_gather_rows)
        Wc = _gather_adj(adj, W)
        op_w = _lib.GmpOperand(_data_ptr(Wc), 1, 1, _lib.TARGETS["edge_pos"])
        if phi.lhs_target == "edge":
            lhs = op_w
        else:
            rhs = op_w
    sched = adj.schedule() if n > 0 else None
    if stage is not None:
        _lib.check(_staged_call(lib, adj, sched, phi, rho, _dtype_code(ref), lhs, rhs,
                                _data_ptr(Z), _ld(Z) if Z.dim() == 2 and Z.shape[0] else
                                max(d_out, 1), d_out,
                                err.data_ptr() if err is not None else None, tune, _stream(dev),
                                stage), "gmp_gspmm_staged")
        if err is not None:
            pos = int(err.item())
            if pos != _INT32_MAX:
                _raise_div_zero(adj.edge_ids[pos].item())
        return Z, None
    st = lib.gmp_gspmm(ctypes.byref(_adj_struct(adj)),
                       ctypes.byref(sched.struct) if sched is not None else None,
                       _lib.OPS[phi.op], _lib.RHOS[rho], _dtype_code(ref),
                       _ptr(lhs), _ptr(rhs), _data_ptr(Z),
                       _ld(Z) if Z.dim() == 2 and Z.shape[0] else max(d_out, 1), d_out,
                       _data_ptr(arg) if arg is not None else None,
                       None, err.data_ptr() if err is not None else None,
                       _ptr(tune), _stream(dev))
    _lib.check(st, "gmp_gspmm")
    if err is not None:
        pos = int(err.item())
        if pos != _INT32_MAX:
            _raise_div_zero(adj.edge_ids[pos].item())
    if rho == "mean":
        return Z, adj.degrees().clone()
    if arg is not None:
        return Z, ArgExtrema(arg)
    return Z, None


def _permute_edge_scalar(W, d_out):
    if W.shape[1] != 1 or d_out <= 1 or W.shape[0] == 0:
        return False
    v = 4 if d_out % 4 == 0 else (2 if d_out % 2 == 0 else 1)
    if W.dtype == torch.float64:
        v = min(v, 2)
    return -(-d_out // (32 * v)) >= 3


# below this many edges the edge operand fits L2 and the plain gather is as good
_GATHER_ADJ_MIN_EDGES = 1 << 22


def _gather_adj(adj, M):
    """M's rows in adjacency order, out[p] = M[adj.edge_ids[p]]: the windowed
    gmp_gather_adj when the adjacency has heavy rows whose edge ids ascend
    (each window of edge ids is read from DRAM once), else gmp_gather_rows."""
    sched = adj.schedule() if adj.num_groups > 0 else None
    if (sched is None or sched.n_heavy == 0 or M.shape[0] < _GATHER_ADJ_MIN_EDGES
            or _sorted_eids(adj) is not adj.edge_ids):
        return _gather_rows(adj.edge_ids, M)
    lib = _lib.load()
    out = torch.empty((adj.edge_ids.numel(), M.shape[1]), dtype=M.dtype, device=M.device)
    sc = sched.struct
    saved = sc.sorted_eids
    sc.sorted_eids = adj.edge_ids.data_ptr()
    try:
        a = ctypes.byref(_adj_struct(adj))
        nbytes = int(lib.gmp_gather_adj_workspace_size(a, ctypes.byref(sc), M.shape[1],
                                                       _dtype_code(M)))
        ws = torch.empty(max(nbytes, 8), dtype=torch.uint8, device=M.device)
        _lib.check(lib.gmp_gather_adj(a, ctypes.byref(sc), M.shape[1], _dtype_code(M),
                                      M.data_ptr(), _ld(M), out.data_ptr(), M.shape[1],
                                      ws.data_ptr(), nbytes, _stream(M.device)),
                   "gmp_gather_adj")
    finally:
        sc.sorted_eids = saved
    return out


def _gather_rows(idx, M):
    """out[i] = M[idx[i]] on the device (gmp_gather_rows)."""
    out = torch.empty((idx.numel(), M.shape[1]), dtype=M.dtype, device=M.device)
    if out.numel():
        _lib.check(_lib.load().gmp_gather_rows(
            idx.numel(), M.shape[1], _dtype_code(M), idx.data_ptr(), M.data_ptr(), _ld(M),
            out.data_ptr(), M.shape[1], _stream(M.device)), "gmp_gather_rows")
    return out


# ----------------------------------------------------------------------------
# g-SDDMM (kernels.py:744-836)


def gsddmm(g, phi, X=None, Y=None, W=None, strategy=None, num_workers=None, fmt=None,
           block_edges=None):
    """Per-edge messages: one output row per edge, in edge-id order."""
    X, Y, W, d_out = _operands_for(g, phi, X, Y, W)
    strategy, fmt = _resolve_strategy("gsddmm", strategy, fmt)
    m = g.num_edges
    accounting.log_dispatch("gsddmm", g.uid, phi.describe(), "-", strategy, m, d_out)
    _require_cuda(g)
    return _gsddmm_launch(g, phi, X, Y, W, d_out)


def _gsddmm_launch(g, phi, X, Y, W, d_out, out=None):
    lib = _lib.load()
    dev = g.device
    m = g.num_edges
    ref = next(t for t in (X, Y, W) if t is not None)
    M = out if out is not None else accounting.register(
        torch.empty((m, d_out), dtype=ref.dtype, device=dev))
    err = _err_slot(dev) if phi.op == "div" else None
    lhs, rhs = _phi_operands(phi, X, Y, W)
    coo = _lib.GmpCoo(g.num_nodes, m, g.src.data_ptr(), g.dst.data_ptr())
    st = lib.gmp_gsddmm(ctypes.byref(coo), _lib.OPS[phi.op], _dtype_code(ref), _ptr(lhs),
                        _ptr(rhs), _data_ptr(M),
                        _ld(M) if M.shape[0] else max(d_out, 1), d_out,
                        err.data_ptr() if err is not None else None, _stream(dev))
    _lib.check(st, "gmp_gsddmm")
    if err is not None:
        e = int(err.item())
        if e != _INT32_MAX:
            _raise_div_zero(e)
    return M


# ----------------------------------------------------------------------------
# extrema gradient routing (kernels.py:843-857)


def route_extrema_grad(g, aux, dZ, d_out):
    """dM[arg[v,k], k] = dZ[v,k]: the (m, d_out) edge-keyed upstream of a max/min."""
    accounting.log_dispatch("gsddmm", g.uid, "argext_route", "-", "edge_parallel",
                            g.num_edges, d_out)
    _require_cuda(g)
    arg = aux.arg_edge
    dZ = _to_tensor("dZ", dZ, g.device)
    dM = accounting.register(torch.zeros((g.num_edges, d_out), dtype=dZ.dtype, device=g.device))
    if dM.numel():
        _lib.check(_lib.load().gmp_route_extrema(
            arg.shape[0], d_out, _dtype_code(dZ), arg.contiguous().data_ptr(), dZ.data_ptr(),
            _ld(dZ), dM.data_ptr(), d_out, _stream(g.device)), "gmp_route_extrema")
    return dM


def extrema_backward_copy(g, aux, dZ, target, rows):
    """Fused max/min backward of a copy message: scatter dZ straight into the
    copied operand's gradient (no (m, d) buffer). target 'src' -> dX (rows n),
    'edge' -> dW (rows m)."""
    _require_cuda(g)
    arg = aux.arg_edge.contiguous()
    dZ = _to_tensor("dZ", dZ, g.device)
    d = dZ.shape[1]
    out = accounting.register(torch.zeros((rows, d), dtype=dZ.dtype, device=g.device))
    tindex = g.src.data_ptr() if target == "src" else None
    if out.numel():
        lib = _lib.load()
        ws = _extrema_workspace(lib, arg.shape[0], d, g.device) if tindex else None
        _lib.check(lib.gmp_extrema_bwd_copy(
            arg.shape[0], d, _dtype_code(dZ), arg.data_ptr(), dZ.data_ptr(), _ld(dZ), tindex,
            rows, out.data_ptr(), d, ws.data_ptr() if ws is not None else None,
            ws.numel() if ws is not None else 0, _stream(g.device)), "gmp_extrema_bwd_copy")
    return out


def _extrema_workspace(lib, n, cells, device):
    """Scratch of the deterministic many-writer accumulation (sort-grouped
    fp64 sums) of the fused max/min backward."""
    return torch.empty(max(1, int(lib.gmp_extrema_bwd_workspace_size(n, cells))),
                       dtype=torch.uint8, device=device)


def rowdot(A, B, out, sub=None, pair=False):
    """out[v] = sum_c A[v,c] B[v,c] - sub[v] in fp64 (gmp_rowdot); out may be a
    strided column view (e.g. the w column of the attention pack); pair=True
    stores the fp64 value as hi in out[v] and lo in the next element."""
    n, d = A.shape
    if (B.shape != A.shape or out.shape[0] != n or out.dtype != A.dtype
            or B.dtype not in (A.dtype, torch.float64)):
        raise ValueError("rowdot: A, B (n, d) and out (n,) of one dtype (B may be float64)")
    if A.stride(-1) != 1 or B.stride(-1) != 1:
        raise ValueError("rowdot: rows must be contiguous")
    if sub is not None and (sub.dtype != torch.float64 or not sub.is_contiguous()):
        raise ValueError("rowdot: sub must be a contiguous float64 vector")
    _lib.check(_lib.load().gmp_rowdot(
        n, d, _dtype_code(A), A.data_ptr(), _ld(A) if n > 1 else d, _dtype_code(B), B.data_ptr(),
        _ld(B) if n > 1 else d, sub.data_ptr() if sub is not None else None, out.data_ptr(),
        int(out.stride(0)), 1 if pair else 0, _stream(A.device)), "gmp_rowdot")
    return out


def extrema_backward_binary(g, aux, dZ, phi, role, X, Y, W):
    """Fused max/min backward of a binary message: the gradient of phi's lhs
    (role 0) or rhs (role 1) operand from the winning edges, no (m, d)
    buffer (gmp_extrema_bwd_binary)."""
    _require_cuda(g)
    arg = aux.arg_edge.contiguous()
    dZ = _to_tensor("dZ", dZ, g.device)
    n, d = arg.shape
    mats = {"src": X, "dst": Y, "edge": W}
    own_t = phi.lhs_target if role == 0 else phi.rhs_target
    own = mats[own_t]
    rows = g.num_edges if own_t == "edge" else g.num_nodes
    own_dim = own.shape[1]
    out = accounting.register(torch.zeros((rows, own_dim), dtype=dZ.dtype, device=g.device))
    if out.numel() and n and d and g.num_edges:  # no edges: no winners, zero gradient
        lhs = _lib.GmpOperand(_data_ptr(mats[phi.lhs_target]), _ld(mats[phi.lhs_target]),
                              mats[phi.lhs_target].shape[1], _lib.TARGETS[phi.lhs_target])
        rhs = _lib.GmpOperand(_data_ptr(mats[phi.rhs_target]), _ld(mats[phi.rhs_target]),
                              mats[phi.rhs_target].shape[1], _lib.TARGETS[phi.rhs_target])
        coo = _lib.GmpCoo(g.num_nodes, g.num_edges, g.src.data_ptr(), g.dst.data_ptr())
        lib = _lib.load()
        many = own_t == "src" or (phi.op != "dot" and own_dim == 1)
        ws = _extrema_workspace(lib, n, own_dim if phi.op == "dot" else d, g.device) \
            if many else None
        _lib.check(lib.gmp_extrema_bwd_binary(
            ctypes.byref(coo), n, d, _dtype_code(dZ), arg.data_ptr(), dZ.data_ptr(), _ld(dZ),
            _lib.OPS[phi.op], role, ctypes.byref(lhs), ctypes.byref(rhs), out.data_ptr(),
            own_dim, own_dim, rows, ws.data_ptr() if ws is not None else None,
            ws.numel() if ws is not None else 0, _stream(g.device)), "gmp_extrema_bwd_binary")
    return out


# ----------------------------------------------------------------------------
# fused edge_softmax (replaces the 4-dispatch composition of messaging.py:105-126)


def _sorted_eids(adj):
    """The adjacency's edge ids with each row's ids ascending (cached): the
    edge ids themselves when they already ascend inside every row (CSC rows
    sorted by (source, edge id) over an edge list grouped by source), else a
    per-row sorted copy. Enables the windowed softmax statistics."""
    se = adj._extra.get("sorted_eids")
    if se is None:
        e = adj.edge_ids
        m, n = e.numel(), adj.num_groups
        se = e
        if m > 1:
            deg = adj.degrees()
            start = torch.zeros(m, dtype=torch.bool, device=e.device)
            start[adj.indptr[:-1][deg > 0]] = True
            if bool(((e[1:] < e[:-1]) & ~start[1:]).any()):
                row = torch.repeat_interleave(torch.arange(n, device=e.device), deg)
                key = row * m + e.to(torch.int64)
                se = e.index_select(0, torch.sort(key).indices)
        adj._extra["sorted_eids"] = se
    return se


# sub-steps per chunk of the segmented statistics pass (GMP_SEG_CHUNK_SUB, gmp.h)
_SEG_CHUNK_SUB = 16
# L2 bytes one window of score rows (both operands in the backward) may take
_SEG_WINDOW_MB = int(os.environ.get("GMP_SOFTMAX_SEG_MB", "64"))
# GMP_SOFTMAX_SEG=0 keeps the (window, row) work-item kernel (measurements)
_SEG_OFF = os.environ.get("GMP_SOFTMAX_SEG", "1") in ("", "0")
# the backward's statistics (two score arrays per edge) keep the (window, row)
# item kernel: measured Reddit H=8 3.68 ms vs 3.78 ms segmented (GMP_SOFTMAX_SEG_BWD=1)
_SEG_BWD_OFF = os.environ.get("GMP_SOFTMAX_SEG_BWD", "0") in ("", "0")
# below this many edges the score rows fit L2 and the row walk is as good
_SEG_MIN_EDGES = 1 << 22


class _Segplan:
    pass


def _softmax_lane_groups(H, itemsize, ld_ok=True):
    """Lane groups per warp of the softmax kernels for H heads (gmp_api.cu
    softmax_vec / pick_v with aligned operands): V elements per lane,
    next_pow2(H / V) lanes per score row."""
    if itemsize == 4 and H % 4 == 0:
        v = 4
    elif H % 2 == 0:
        v = 2
    else:
        v = 1
    lanes = 1
    while lanes < -(-H // v):
        lanes *= 2
    return 32 // min(lanes, 32)


def _softmax_segplan(adj, sched, win, group):
    """Window-major piece layout of the heavy rows' in-edges (gmp_segplan,
    gmp.h), cached per (window, lane groups). The heavy rows' edge ids sorted
    by (eid // win, heavy row index, eid), each (window, row) segment padded
    with -1 to a multiple of `group` positions (one warp sub-step); pieces =
    segments cut every _SEG_CHUNK_SUB sub-steps; row_pieces groups the piece
    ids by heavy row in ascending (= window) order. Built once with device
    sorts."""
    key = ("segplan", int(win), int(group))
    plan = adj._extra.get(key)
    if plan is not None:
        return plan
    R = sched.n_heavy
    dev = adj.indptr.device
    rows = sched.order[:R].to(torch.int64)
    first = adj.indptr.index_select(0, rows)
    deg = adj.indptr.index_select(0, rows + 1) - first
    n_edges = int(deg.sum())
    r_of = torch.repeat_interleave(torch.arange(R, device=dev), deg)
    base = torch.cumsum(deg, 0) - deg
    pos = torch.arange(n_edges, device=dev) - base.index_select(0, r_of) + first.index_select(0, r_of)
    eid = _sorted_eids(adj).index_select(0, pos)
    del pos, base
    wkey = torch.div(eid, int(win), rounding_mode="floor").to(torch.int64) * R + r_of
    del r_of
    wkey, idx = torch.sort(wkey, stable=True)
    eid = eid.index_select(0, idx)
    del idx
    # segments (runs of one (window, row)) and their padded extents
    seg_keys, seg_len = torch.unique_consecutive(wkey, return_counts=True)
    del wkey
    seg_sub = -(-seg_len // group)                      # sub-steps per segment
    seg_start = torch.cumsum(seg_len, 0) - seg_len      # unpadded first position
    seg_sub_start = torch.cumsum(seg_sub, 0) - seg_sub  # first sub-step
    n_sub = -(-int(seg_sub.sum()) // _SEG_CHUNK_SUB) * _SEG_CHUNK_SUB  # whole chunks
    n_pos = n_sub * group
    seg_of = torch.repeat_interleave(torch.arange(seg_keys.numel(), device=dev), seg_len)
    dest = (torch.arange(n_edges, device=dev) - seg_start.index_select(0, seg_of)
            + seg_sub_start.index_select(0, seg_of) * group)
    del seg_of, seg_start
    perm = torch.full((n_pos,), -1, dtype=torch.int32, device=dev)
    perm[dest] = eid
    del dest, eid
    # piece starts per sub-step: a segment's first sub-step or a chunk start
    new = torch.zeros(n_sub, dtype=torch.bool, device=dev)
    new[seg_sub_start] = True
    new[::_SEG_CHUNK_SUB] = True
    pid = torch.cumsum(new, 0)
    n_pieces = int(pid[-1])
    chunk_piece = (pid[::_SEG_CHUNK_SUB] - 1).to(torch.int32)
    sub_seg = torch.repeat_interleave(torch.arange(seg_keys.numel(), device=dev), seg_sub)
    tail = n_sub - sub_seg.numel()  # padding sub-steps of the last chunk: last segment's
    if tail:
        sub_seg = torch.cat([sub_seg, sub_seg[-1:].expand(tail)])
    piece_row = torch.remainder(seg_keys.index_select(0, sub_seg[new]), R)
    del pid, sub_seg
    row_pieces = torch.sort(piece_row, stable=True).indices.to(torch.int32)
    row_ptr = torch.zeros(R + 1, dtype=torch.int64, device=dev)
    torch.cumsum(torch.bincount(piece_row, minlength=R), 0, out=row_ptr[1:])
    nw = -(-n_sub // 32)
    bits = torch.zeros(nw * 32, dtype=torch.int64, device=dev)
    bits[:n_sub] = new.to(torch.int64)
    words = (bits.view(nw, 32) << torch.arange(32, device=dev)).sum(1)
    starts = torch.where(words >= 2 ** 31, words - 2 ** 32, words).to(torch.int32)
    plan = _Segplan()
    plan.tensors = (perm, starts, chunk_piece, row_ptr, row_pieces)
    plan.struct = _lib.GmpSegplan(n_pos, n_pieces, int(win), int(group), perm.data_ptr(),
                                  starts.data_ptr(), chunk_piece.data_ptr(), row_ptr.data_ptr(),
                                  row_pieces.data_ptr())
    adj._extra[key] = plan
    return plan


def _softmax_call(g, fn_name, S, G2, H, out, what):
    lib = _lib.load()
    adj = g.to_csc()
    sched = adj.schedule()
    if sched.n_heavy and g.num_edges >= (1 << 22) and not sched.struct.sorted_eids:
        sched.struct.sorted_eids = _sorted_eids(adj).data_ptr()
    sc = sched.struct
    if (sched.n_heavy and g.num_edges >= _SEG_MIN_EDGES and not _SEG_OFF
            and not (G2 is not None and _SEG_BWD_OFF)):
        row_bytes = H * S.element_size() * (2 if G2 is not None else 1)
        plan = _softmax_segplan(adj, sched, max(1 << 10, (_SEG_WINDOW_MB << 20) // row_bytes),
                                _softmax_lane_groups(H, S.element_size()))
        sc = _lib.GmpSched.from_buffer_copy(sched.struct)
        sc.segplan = ctypes.addressof(plan.struct)
    ws_bytes = int(lib.gmp_edge_softmax_workspace_size_ex(
        ctypes.byref(_adj_struct(adj)), ctypes.byref(sc), H, _dtype_code(S),
        1 if G2 is not None else 0))
    ws = torch.empty(max(ws_bytes, 8), dtype=torch.uint8, device=g.device)
    coo = _lib.GmpCoo(g.num_nodes, g.num_edges, g.src.data_ptr(), g.dst.data_ptr())
    args = [ctypes.byref(_adj_struct(adj)), ctypes.byref(coo), ctypes.byref(sc),
            _dtype_code(S), S.data_ptr(), _ld(S)]
    if G2 is not None:
        args += [G2.data_ptr(), _ld(G2)]
    args += [H, out.data_ptr(), H, ws.data_ptr(), ws_bytes, _stream(g.device)]
    _lib.check(getattr(lib, fn_name)(*args), what)


def edge_softmax_forward(g, scores):
    """alpha = per-destination softmax of (m, H) scores: a fused per-row
    statistics kernel plus an edge-order normalisation kernel."""
    _require_cuda(g)
    S = _as_matrix("scores", scores, g.num_edges, g.device)
    H = S.shape[1]
    accounting.log_dispatch("gspmm", g.uid, "edge_softmax", "softmax", "node_parallel",
                            g.num_edges, H)
    alpha = accounting.register(torch.empty((g.num_edges, H), dtype=S.dtype, device=g.device))
    if alpha.numel():
        _softmax_call(g, "gmp_edge_softmax_fwd", S, None, H, alpha, "gmp_edge_softmax_fwd")
    return alpha


def edge_softmax_backward(g, alpha, grad):
    """ds = alpha * (grad - sum_{in-edges} alpha * grad), fused."""
    _require_cuda(g)
    A = _as_matrix("alpha", alpha, g.num_edges, g.device)
    Gr = _as_matrix("grad", grad, g.num_edges, g.device).to(A.dtype)
    H = A.shape[1]
    accounting.log_dispatch("gspmm", g.uid, "edge_softmax_bwd", "softmax", "node_parallel",
                            g.num_edges, H)
    ds = accounting.register(torch.empty((g.num_edges, H), dtype=A.dtype, device=g.device))
    if ds.numel():
        _softmax_call(g, "gmp_edge_softmax_bwd", A, Gr, H, ds, "gmp_edge_softmax_bwd")
    return ds


def edge_softmax_uv_forward(g, el, er):
    """alpha = edge_softmax(el[src] + er[dst]) without materialising the
    scores (fused u_add_v g-SDDMM + edge_softmax, GAT layers.py:110-113)."""
    _require_cuda(g)
    L = _as_matrix("el", el, g.num_nodes, g.device)
    R = _as_matrix("er", er, g.num_nodes, g.device)
    if L.dtype != R.dtype:
        L, R = L.to(torch.float64), R.to(torch.float64)
    if L.shape[1] != R.shape[1]:
        raise ValueError("el and er need the same head count, got %d and %d"
                         % (L.shape[1], R.shape[1]))
    H = L.shape[1]
    accounting.log_dispatch("gspmm", g.uid, "edge_softmax(add(src,dst))", "softmax",
                            "node_parallel", g.num_edges, H)
    alpha = accounting.register(torch.empty((g.num_edges, H), dtype=L.dtype, device=g.device))
    if alpha.numel():
        lib = _lib.load()
        adj = g.to_csc()
        sched = adj.schedule()
        ws_bytes = int(lib.gmp_edge_softmax_workspace_size(g.num_nodes, H))
        ws = torch.empty(max(ws_bytes, 8), dtype=torch.uint8, device=g.device)
        coo = _lib.GmpCoo(g.num_nodes, g.num_edges, g.src.data_ptr(), g.dst.data_ptr())
        _lib.check(lib.gmp_edge_softmax_uv_fwd(
            ctypes.byref(_adj_struct(adj)), ctypes.byref(coo), ctypes.byref(sched.struct),
            _dtype_code(L), L.data_ptr(), _ld(L), R.data_ptr(), _ld(R), H, alpha.data_ptr(), H,
            ws.data_ptr(), ws_bytes, _stream(g.device)), "gmp_edge_softmax_uv_fwd")
    return alpha


# ----------------------------------------------------------------------------
# fused GAT attention (u_add_v -> edge_softmax -> u_mul_e + sum, layers.py:110-115)


def edge_softmax_uv_stats(g, el, er):
    """Per-destination statistics of the u_add_v scores el[src] + er[dst]:
    (n, 2H) = [max_h | 1/sum_h exp(s - max_h)]; zero rows for destinations
    without in-edges. The statistics pass of edge_softmax_uv_forward alone."""
    _require_cuda(g)
    L = _as_matrix("el", el, g.num_nodes, g.device)
    R = _as_matrix("er", er, g.num_nodes, g.device)
    if L.dtype != R.dtype or L.shape[1] != R.shape[1]:
        raise ValueError("el and er need the same dtype and head count")
    H = L.shape[1]
    stat = torch.zeros((g.num_nodes, 2 * H), dtype=L.dtype, device=g.device)
    if g.num_edges and H:
        lib = _lib.load()
        adj = g.to_csc()
        sched = adj.schedule()
        accounting.log_dispatch("gspmm", g.uid, "edge_softmax_stats(add(src,dst))", "softmax",
                                "node_parallel", g.num_edges, H)
        _lib.check(lib.gmp_edge_softmax_uv_stats(
            ctypes.byref(_adj_struct(adj)), ctypes.byref(sched.struct), _dtype_code(L),
            L.data_ptr(), _ld(L), R.data_ptr(), _ld(R), H, stat.data_ptr(),
            stat.numel() * stat.element_size(), _stream(g.device)), "gmp_edge_softmax_uv_stats")
    return stat


def pack_width(dtype):
    """Elements per 32-byte row of the fused attention's node pack (gmp.h):
    fp32 [er, max, inv_sum, w_hi, w_lo, 0, 0, 0], fp64 [er, max, inv_sum, w]."""
    return 4 if dtype == torch.float64 else 8


def _pad_rows16(X):
    """X itself when its rows are 16 B-aligned runs of whole float4s, else a
    copy with ld rounded up to a multiple of 4 (zero padding): a row width
    that is not a multiple of 4 (41 classes) then still gathers with 16 B
    loads, the last vector masked at the store (d=41: 4.2 -> 2.0 ms on
    Reddit for copy_u + sum)."""
    d = X.shape[1]
    if X.dtype != torch.float32 or d % 4 == 0 or d < 4 or X.shape[0] == 0:
        return X
    if _ld(X) % 4 == 0 and X.data_ptr() % 16 == 0:
        return X
    P = torch.zeros((X.shape[0], -(-d // 4) * 4), dtype=X.dtype, device=X.device)
    P[:, :d] = X
    return P[:, :d]


def gat_aggregate(g, X, el, pack, backward=False, z64=None):
    """One head of the fused attention aggregation (gmp_gat_aggregate).
    forward:  Z[v] = sum_{(u,e)->v} alpha_e X[u]   over g's in-adjacency
    backward: Z[u] = sum_{(v,e): u->v} alpha_e X[v] over reverse(g)'s, and
              t[u] = sum_{(v,e): u->v} alpha_e w[v] (fp64); returns (Z, t)
    with alpha_e = exp((el[u] + er[v]) - max[v]) * inv_sum[v] recomputed from
    el (n, 1) and pack (n, pack_width) = [er, max, inv_sum, w (hi, lo)]. z64 (optional (n, d)
    float64 view) also receives the unrounded rows."""
    from .graph import reverse
    _require_cuda(g)
    X = _as_matrix("X", X, g.num_nodes, g.device)
    d = X.shape[1]
    Z = accounting.register(torch.empty((g.num_nodes, d), dtype=X.dtype, device=g.device))
    t = torch.zeros(g.num_nodes if backward else 0, dtype=torch.float64, device=g.device)
    if not Z.numel():
        return (Z, t) if backward else Z
    if el.dtype != X.dtype or pack.dtype != X.dtype:
        raise ValueError("el / pack must have the feature dtype")
    if not (pack.is_contiguous() and pack.shape == (g.num_nodes, pack_width(X.dtype))):
        raise ValueError("pack must be a contiguous (n, %d) matrix" % pack_width(X.dtype))
    walk = reverse(g) if backward else g
    adj = walk.to_csc()
    sched = adj.schedule()
    accounting.log_dispatch("gspmm", walk.uid, "mul(src,edge_softmax(add(src,dst)))", "sum",
                            "node_parallel", g.num_nodes, d)
    lde = int(el.stride(0)) if el.shape[0] > 1 else 1
    X = _pad_rows16(X)
    _lib.check(_lib.load().gmp_gat_aggregate(
        ctypes.byref(_adj_struct(adj)), ctypes.byref(sched.struct), _dtype_code(X),
        1 if backward else 0, X.data_ptr(), _ld(X), d, el.data_ptr(), lde, pack.data_ptr(),
        Z.data_ptr(), _ld(Z), z64.data_ptr() if z64 is not None else None,
        _ld(z64) if z64 is not None else 0, t.data_ptr() if backward else None,
        _ptr(_tuning_struct(None)),
        _stream(g.device)), "gmp_gat_aggregate")
    return (Z, t) if backward else Z
