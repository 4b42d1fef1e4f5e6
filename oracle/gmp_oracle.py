"""CPU ORACLE - test infrastructure only.

A NumPy restatement of the reference's hot path (graphmp 0.1.0,
/root/reference/pkg/src/graphmp). Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import this module, and
only as the checker or the timed CPU baseline - never as the product path.
The product (paper_1909_01315_b200) never imports it.

Parity pinning: tests/golden/*.npz hold inputs and outputs produced by the
reference itself (tests/golden/make_golden.py imports /root/reference in the
build container); tests/test_oracle.py checks this restatement against every
fixture, including the reference's own frozen examples (test_kernels.py:16-65,
test_messaging.py:103-153, test_autodiff.py:107-171). Parity is pinned.

Arithmetic is float64 throughout, exactly like the reference (kernels.py:216).
"""

import os
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

BLOCK_EDGES = 2048      # kernels.py:39
_INT_MAX = np.iinfo(np.int64).max


# ---------------------------------------------------------------- graph ------

def build_adjacency(group, other, num_nodes):
    """(indptr int64, indices uint32, edge_ids uint32) grouped by `group`,
    neighbours ascending, ties by edge id (graph.py:35-44)."""
    group = np.asarray(group, dtype=np.int64)
    other = np.asarray(other, dtype=np.int64)
    eids = np.arange(group.size, dtype=np.int64)
    order = np.lexsort((eids, other, group))
    indptr = np.zeros(num_nodes + 1, dtype=np.int64)
    np.cumsum(np.bincount(group, minlength=num_nodes), out=indptr[1:])
    return indptr, other[order].astype(np.uint32), eids[order].astype(np.uint32)


def csc(src, dst, n):
    """In-adjacency (graph.py:137-139)."""
    return build_adjacency(dst, src, n)


def csr(src, dst, n):
    """Out-adjacency (graph.py:133-135)."""
    return build_adjacency(src, dst, n)


# ------------------------------------------------------------- messages ------

def _f64(a):
    return None if a is None else np.asarray(a, dtype=np.float64)


def out_dim(op, lhs_t, rhs_t, X, Y, W):
    """d_out rule of kernels.py:240-252."""
    mats = {"src": X, "dst": Y, "edge": W}
    if op in ("copy_lhs", "copy_rhs"):
        return mats[lhs_t or rhs_t].shape[1]
    if op == "dot":
        return 1
    return max(mats[lhs_t].shape[1], mats[rhs_t].shape[1])


def messages(op, lhs_t, rhs_t, X, Y, W, u, v, e):
    """Per-edge messages for edges (u, v, e) (kernels.py:255-296); returns
    (msgs, zero_row) where zero_row is the first row whose divisor has a 0."""
    mats = {"src": _f64(X), "dst": _f64(Y), "edge": _f64(W)}
    idx = {"src": u, "dst": v, "edge": e}

    def gather(t):
        return mats[t][np.asarray(idx[t], dtype=np.int64)]

    if op in ("copy_lhs", "copy_rhs"):
        return gather(lhs_t or rhs_t), None
    a, b = gather(lhs_t), gather(rhs_t)
    if op == "add":
        return a + b, None
    if op == "sub":
        return a - b, None
    if op == "mul":
        return a * b, None
    if op == "div":
        zero = (b == 0.0).any(axis=1)
        with np.errstate(divide="ignore", invalid="ignore"):
            out = a / b
        return out, (int(np.flatnonzero(zero)[0]) if zero.any() else None)
    return (a * b).sum(axis=1)[:, None], None


class DivByZero(ZeroDivisionError):
    def __init__(self, eid):
        super().__init__("division by zero in edge message at edge id %d" % eid)
        self.eid = eid


# ---------------------------------------------------------------- gspmm ------

def _reduce_rows(op, lhs_t, rhs_t, X, Y, W, indptr, indices, eids, rho, out, arg, lo, hi,
                 block):
    """Restates _GroupedWalk.run/_multi/_single (kernels.py:361-438): rows
    [lo, hi) in chunks of <= block edges, segment reductions by reduceat,
    max/min arg = smallest edge id among cells equal to the extremum."""
    ufunc = np.maximum if rho == "max" else np.minimum
    better = np.greater if rho == "max" else np.less
    counts = np.diff(indptr)
    cur = lo
    while cur < hi:
        p0 = indptr[cur]
        end = min(int(np.searchsorted(indptr, p0 + block, side="right")) - 1, hi)
        if end > cur:  # a run of whole rows (kernels.py:384-410)
            p1 = indptr[end]
            if p1 > p0:
                u = indices[p0:p1]
                e = eids[p0:p1]
                v = np.repeat(np.arange(cur, end), counts[cur:end])
                msgs, z = messages(op, lhs_t, rhs_t, X, Y, W, u, v, e)
                if z is not None:
                    raise DivByZero(int(e[z]))
                nz = np.flatnonzero(counts[cur:end] > 0)
                starts = (indptr[cur:end] - p0)[nz]
                res = np.zeros((end - cur, msgs.shape[1]))
                if rho in ("sum", "mean"):
                    res[nz] = np.add.reduceat(msgs, starts, axis=0)
                    out[cur:end] = res
                else:
                    res[nz] = ufunc.reduceat(msgs, starts, axis=0)
                    out[cur:end] = res
                    rep = np.repeat(res, counts[cur:end], axis=0)
                    masked = np.where(msgs == rep, e.astype(np.int64)[:, None], _INT_MAX)
                    a = np.full((end - cur, msgs.shape[1]), -1, dtype=np.int64)
                    a[nz] = np.minimum.reduceat(masked, starts, axis=0)
                    arg[cur:end] = a
            cur = end
            continue
        # one hub row longer than the block, folded with a carry (kernels.py:412-438)
        r0, r1 = indptr[cur], indptr[cur + 1]
        acc = acc_arg = None
        for q0 in range(r0, r1, block):
            q1 = min(q0 + block, r1)
            e = eids[q0:q1]
            msgs, z = messages(op, lhs_t, rhs_t, X, Y, W, indices[q0:q1],
                               np.full(q1 - q0, cur), e)
            if z is not None:
                raise DivByZero(int(e[z]))
            if rho in ("sum", "mean"):
                part = msgs.sum(axis=0)
                acc = part if acc is None else acc + part
            else:
                part = ufunc.reduce(msgs, axis=0)
                parg = np.where(msgs == part[None, :], e.astype(np.int64)[:, None],
                                _INT_MAX).min(axis=0)
                if acc is None:
                    acc, acc_arg = part, parg
                else:
                    gain, tie = better(part, acc), part == acc
                    acc_arg = np.where(gain, parg, np.where(tie, np.minimum(acc_arg, parg), acc_arg))
                    acc = ufunc(acc, part)
        if acc is not None:
            out[cur] = acc
            if acc_arg is not None:
                arg[cur] = acc_arg
        cur += 1


def gspmm(src, dst, n, op, lhs_t, rhs_t, rho, X=None, Y=None, W=None, workers=1,
          block=BLOCK_EDGES, adj=None):
    """Reference gspmm, default node_parallel strategy (kernels.py:473-482,
    685-725). Returns (Z, aux): aux None | counts int64 | arg int64."""
    indptr, indices, eids = adj if adj is not None else csc(src, dst, n)
    X, Y, W = _f64(X), _f64(Y), _f64(W)  # once, like kernels.py:216
    d_out = out_dim(op, lhs_t, rhs_t, X, Y, W)
    out = np.zeros((n, d_out))
    arg = np.full((n, d_out), -1, dtype=np.int64) if rho in ("max", "min") else None
    bounds = np.linspace(0, n, max(1, workers) + 1).astype(np.int64)
    parts = [(int(bounds[i]), int(bounds[i + 1])) for i in range(len(bounds) - 1)
             if bounds[i] < bounds[i + 1]]

    def run(lo, hi):
        _reduce_rows(op, lhs_t, rhs_t, X, Y, W, indptr, indices, eids, rho, out, arg, lo, hi,
                     block)

    if workers <= 1 or len(parts) <= 1:
        for p in parts:
            run(*p)
    else:
        with ThreadPoolExecutor(max_workers=workers) as pool:
            for f in [pool.submit(run, *p) for p in parts]:
                f.result()
    counts = np.diff(indptr)
    if rho == "mean":
        nz = counts > 0
        out[nz] /= counts[nz, None]
        return out, counts
    return out, arg


# --------------------------------------------------------------- gsddmm ------

def gsddmm(src, dst, n, op, lhs_t, rhs_t, X=None, Y=None, W=None, workers=1,
           block=BLOCK_EDGES):
    """Reference gsddmm, default edge_parallel over COO (kernels.py:744-836)."""
    m = len(src)
    X, Y, W = _f64(X), _f64(Y), _f64(W)
    d_out = out_dim(op, lhs_t, rhs_t, X, Y, W)
    out = np.empty((m, d_out))
    u_all = np.asarray(src, dtype=np.int64)
    v_all = np.asarray(dst, dtype=np.int64)
    bounds = np.linspace(0, m, max(1, workers) + 1).astype(np.int64)
    errors = []
    lock = threading.Lock()

    def run(q0, q1):
        for c0 in range(q0, q1, block):
            c1 = min(c0 + block, q1)
            e = np.arange(c0, c1)
            msgs, z = messages(op, lhs_t, rhs_t, X, Y, W, u_all[c0:c1], v_all[c0:c1], e)
            if z is not None:
                with lock:
                    errors.append(int(e[z]))
                return
            out[c0:c1] = msgs

    parts = [(int(bounds[i]), int(bounds[i + 1])) for i in range(len(bounds) - 1)
             if bounds[i] < bounds[i + 1]]
    if workers <= 1 or len(parts) <= 1:
        for p in parts:
            run(*p)
            if errors:
                break
    else:
        with ThreadPoolExecutor(max_workers=workers) as pool:
            for f in [pool.submit(run, *p) for p in parts]:
                f.result()
    if errors:
        raise DivByZero(min(errors))
    return out


# ---------------------------------------------------------- edge softmax ------

def edge_softmax(src, dst, n, scores):
    """messaging.py:105-126: max-shift, exp, per-destination sum, divide."""
    s = _f64(scores)
    peak, _ = gspmm(src, dst, n, "copy_rhs", None, "edge", "max", W=s)
    shifted = s - peak[np.asarray(dst, dtype=np.int64)]
    w = np.exp(shifted)
    total, _ = gspmm(src, dst, n, "copy_rhs", None, "edge", "sum", W=w)
    return w / total[np.asarray(dst, dtype=np.int64)]


def edge_softmax_backward(src, dst, n, alpha, grad):
    """Closed form of the composed backward: ds = a * (g - sum_{in} a * g)."""
    a, g = _f64(alpha), _f64(grad)
    tot, _ = gspmm(src, dst, n, "copy_rhs", None, "edge", "sum", W=a * g)
    return a * (g - tot[np.asarray(dst, dtype=np.int64)])


def route_extrema_grad(m, arg, dZ):
    """kernels.py:843-857: dM[arg[v,k], k] = dZ[v,k]."""
    arg = np.asarray(arg)
    dM = np.zeros((m, arg.shape[1]))
    vi, ci = np.nonzero(arg >= 0)
    dM[arg[vi, ci], ci] = _f64(dZ)[vi, ci]
    return dM


# ------------------------------------------------------------- backward ------

def gspmm_backward(src, dst, n, op, lhs_t, rhs_t, rho, X=None, Y=None, W=None, aux=None,
                   dZ=None):
    """Operand gradients of gspmm by an edge-loop formulation independent of the
    reference's routing code (checks Theorem 1, autodiff.py:289-412): per-edge
    upstream g_e from rho, per-edge partials of phi, scatter-add by target."""
    u = np.asarray(src, dtype=np.int64)
    v = np.asarray(dst, dtype=np.int64)
    m = u.size
    dZ = _f64(dZ)
    if rho == "sum":
        up = dZ[v]
    elif rho == "mean":
        cnt = np.asarray(aux, dtype=np.float64)
        scale = np.where(cnt > 0, 1.0 / np.where(cnt > 0, cnt, 1.0), 0.0)
        up = (dZ * scale[:, None])[v]
    else:
        up = route_extrema_grad(m, aux, dZ)
    return _edge_partials(op, lhs_t, rhs_t, X, Y, W, u, v, n, up)


def gsddmm_backward(src, dst, n, op, lhs_t, rhs_t, X=None, Y=None, W=None, dM=None):
    u = np.asarray(src, dtype=np.int64)
    v = np.asarray(dst, dtype=np.int64)
    return _edge_partials(op, lhs_t, rhs_t, X, Y, W, u, v, n, _f64(dM))


def _edge_partials(op, lhs_t, rhs_t, X, Y, W, u, v, n, up):
    m = u.size
    mats = {"src": _f64(X), "dst": _f64(Y), "edge": _f64(W)}
    idx = {"src": u, "dst": v, "edge": np.arange(m)}
    rows = {"src": n, "dst": n, "edge": m}

    def gather(t):
        return mats[t][idx[t]]

    def scatter(t, per_edge):
        width = mats[t].shape[1]
        if per_edge.shape[1] != width:  # a broadcast operand receives the row sum
            per_edge = per_edge.sum(axis=1, keepdims=True)
        out = np.zeros((rows[t], width))
        np.add.at(out, idx[t], per_edge)
        return out

    grads = {}
    if op in ("copy_lhs", "copy_rhs"):
        t = lhs_t or rhs_t
        grads[t] = scatter(t, up)
        return grads
    a, b = gather(lhs_t), gather(rhs_t)
    if op == "dot":
        da, db = up * b, up * a
    elif op == "add":
        da, db = up, up
    elif op == "sub":
        da, db = up, -up
    elif op == "mul":
        da, db = up * b, up * a
    else:
        with np.errstate(divide="ignore", invalid="ignore"):
            da = up / b
            db = -up * a / (b * b)
    grads[lhs_t] = scatter(lhs_t, np.broadcast_to(da, np.broadcast_shapes(da.shape, up.shape)))
    grads[rhs_t] = scatter(rhs_t, np.broadcast_to(db, np.broadcast_shapes(db.shape, up.shape)))
    return grads


def default_workers():
    return len(os.sched_getaffinity(0))
