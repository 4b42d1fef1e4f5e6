"""Backward of g-SpMM / g-SDDMM as g-SpMM / g-SDDMM (the paper's Theorem 1).

The gradient rules mirror /root/reference/pkg/src/graphmp/autodiff.py:273-418:
  * the gradient w.r.t. X (source rows) is a g-SpMM on reverse(g) - whose CSC
    is the forward CSR through the shared cache pair, so the backward runs the
    same deterministic row kernel with no atomics and no index rebuild;
  * w.r.t. Y (destination rows) a g-SpMM on g itself;
  * w.r.t. W (edge rows) a g-SDDMM on g;
  * mean scales the upstream by 1/in-degree first; max/min first route the
    upstream to each cell's winning edge (kernels.route_extrema_grad), and for
    plain copy messages that routing is fused with the scatter into the
    operand's gradient (no (m, d) buffer).
Dense glue (products, row sums, safe division) is elementwise torch on the
device.

The reference's Tape/Var is replaced by torch autograd: gspmm / gsddmm /
edge_softmax below are autograd Functions whose backward calls
gspmm_backward / gsddmm_backward (or the fused edge_softmax backward kernel).
"""

from dataclasses import dataclass

import torch

from . import accounting, kernels
from .graph import reverse


@dataclass
class GradBundle:
    dx: torch.Tensor = None
    dy: torch.Tensor = None
    dw: torch.Tensor = None


def _safe_div(a, b):
    """a / b where b != 0, else 0 (autodiff.py:280-283)."""
    if not torch.is_tensor(b):
        b = torch.as_tensor(b, dtype=a.dtype if torch.is_tensor(a) else torch.float64)
    if not torch.is_tensor(a):
        a = torch.as_tensor(a, dtype=b.dtype, device=b.device)
    nz = b != 0
    return torch.where(nz, a / torch.where(nz, b, torch.ones_like(b)), torch.zeros((), dtype=a.dtype, device=a.device))


_REV_SLOT = {"src": "dst", "dst": "src", "edge": "edge"}
_SLOT_KW = {"src": "X", "dst": "Y", "edge": "W"}


def _route(g, t, up, up_slot, kind, p_target=None, P=None, mode="ew"):
    """Sum up_e * factor_e over the edges keyed to target t (autodiff.py:289-336).

    kind 'one' (factor 1), 'val' (the operand at p_target) or 'inv' (its
    reciprocal); mode 'dot' row-reduces the product for a broadcast operand.
    """
    if kind != "one" and p_target == up_slot:
        comb = up * P if kind == "val" else _safe_div(up, P)
        if mode == "dot":
            comb = comb.sum(dim=1, keepdim=True)
        accounting.register(comb)
        return _route(g, t, comb, up_slot, "one")

    opname = None if kind == "one" else {"val": "mul" if mode == "ew" else "dot", "inv": "div"}[kind]
    if t == "edge":
        if up_slot == "edge":
            if kind == "one":
                return up
            phi = kernels.MessageFunc(opname, "edge", p_target)
            return kernels.gsddmm(g, phi, **{"W": up, _SLOT_KW[p_target]: P})
        if kind == "one":
            return kernels.gsddmm(g, kernels.copy("dst"), Y=up)
        phi = kernels.MessageFunc(opname, "dst", p_target)
        return kernels.gsddmm(g, phi, **{"Y": up, _SLOT_KW[p_target]: P})

    # node-keyed output: g-SpMM with sum; source-keyed gradients on reverse(g)
    if t == "dst":
        gg, smap = g, {"src": "src", "dst": "dst", "edge": "edge"}
    else:
        gg, smap = reverse(g), _REV_SLOT
    su = smap[up_slot]
    kw = {_SLOT_KW[su]: up}
    if kind == "one":
        phi = kernels.copy(su)
    else:
        sp = smap[p_target]
        phi = kernels.MessageFunc(opname, su, sp)
        kw[_SLOT_KW[sp]] = P
    Z, _ = kernels.gspmm(gg, phi, "sum", **kw)
    return Z


def _role_grad(g, phi, t, other_t, X, Y, W, up, up_slot):
    """Gradient w.r.t. the operand at target t (autodiff.py:339-372)."""
    vals = {"src": X, "dst": Y, "edge": W}
    own = vals[t]
    d_own, d_up = own.shape[1], up.shape[1]
    op = phi.op
    if op in ("copy_lhs", "copy_rhs", "add", "sub"):
        eff = up if d_own == d_up else accounting.register(up.sum(dim=1, keepdim=True))
        res = _route(g, t, eff, up_slot, "one")
        if op == "sub" and t == phi.rhs_target:
            res = -res
        return res
    other = vals[other_t]
    if op == "mul":
        mode = "dot" if (d_own == 1 and d_up > 1) else "ew"
        return _route(g, t, up, up_slot, "val", other_t, other, mode)
    if op == "dot":
        return _route(g, t, up, up_slot, "val", other_t, other, "ew")
    # div
    if t == phi.lhs_target:
        if d_own == 1 and d_up > 1:
            rec = accounting.register(_safe_div(1.0, other))
            return _route(g, t, up, up_slot, "val", other_t, rec, "dot")
        return _route(g, t, up, up_slot, "inv", other_t, other)
    mode = "dot" if (d_own == 1 and d_up > 1) else "ew"
    s = _route(g, t, up, up_slot, "val", other_t, other, mode)
    return accounting.register(-_safe_div(s, own * own))


def _edge_grads(g, phi, X, Y, W, up, up_slot, needs):
    if phi.op == "copy_lhs":
        roles = [(phi.lhs_target, None)]
    elif phi.op == "copy_rhs":
        roles = [(phi.rhs_target, None)]
    else:
        roles = [(phi.lhs_target, phi.rhs_target), (phi.rhs_target, phi.lhs_target)]
    slot_need = {"src": "x", "dst": "y", "edge": "w"}
    bundle = GradBundle()
    for t, other_t in roles:
        if slot_need[t] not in needs:
            continue
        res = _role_grad(g, phi, t, other_t, X, Y, W, up, up_slot)
        setattr(bundle, {"src": "dx", "dst": "dy", "edge": "dw"}[t], res)
    return bundle


def _dev_matrix(name, M, rows, g, dtype=None):
    if M is None:
        return None
    t = kernels._as_matrix(name, M, rows, g.device)
    return t if dtype is None else t.to(dtype)


def gspmm_backward(g, phi, rho, X=None, Y=None, W=None, Z=None, aux=None, dZ=None,
                   needs=("x", "y", "w")):
    """Operand gradients of gspmm(g, phi, rho) (autodiff.py:398-412)."""
    n, m = g.num_nodes, g.num_edges
    dZ = _dev_matrix("dZ", dZ, n, g)
    ops = [_dev_matrix("X", X, n, g), _dev_matrix("Y", Y, n, g), _dev_matrix("W", W, m, g)]
    dt = torch.float64 if any(o is not None and o.dtype == torch.float64
                              for o in ops + [dZ]) else torch.float32
    X, Y, W = [None if o is None else o.to(dt) for o in ops]
    dZ = dZ.to(dt)
    if rho == "sum":
        up, up_slot = dZ, "dst"
    elif rho == "mean":
        counts = torch.as_tensor(aux, device=g.device).to(dt)[:, None]
        up = accounting.register(_safe_div(dZ, counts))
        up_slot = "dst"
    elif rho in ("max", "min"):
        fused = _fused_extrema_copy(g, phi, aux, dZ, needs)
        if fused is not None:
            return fused
        if phi.op in ("add", "sub", "mul", "div", "dot"):
            return _fused_extrema_binary(g, phi, aux, dZ, X, Y, W, needs)
        up = kernels.route_extrema_grad(g, aux, dZ, dZ.shape[1])
        up_slot = "edge"
    else:
        raise ValueError("unknown reducer %r" % (rho,))
    return _edge_grads(g, phi, X, Y, W, up, up_slot, needs)


def _fused_extrema_binary(g, phi, aux, dZ, X, Y, W, needs):
    """add / sub / mul / div under max/min: one kernel per needed operand
    gradient straight from the winning edges (gmp_extrema_bwd_binary)."""
    slot = {"src": "x", "dst": "y", "edge": "w"}
    attr = {"src": "dx", "dst": "dy", "edge": "dw"}
    bundle = GradBundle()
    for role, t in ((0, phi.lhs_target), (1, phi.rhs_target)):
        if slot[t] not in needs:
            continue
        accounting.log_dispatch("gsddmm", g.uid, "argext_grad(%s,%d)" % (phi.describe(), role),
                                "-", "edge_parallel", g.num_edges, dZ.shape[1])
        res = kernels.extrema_backward_binary(g, aux, dZ, phi, role, X, Y, W)
        setattr(bundle, attr[t], res)
    return bundle


def _fused_extrema_copy(g, phi, aux, dZ, needs):
    """copy_lhs/copy_rhs of src or edge under max/min: one scatter kernel."""
    if phi.op not in ("copy_lhs", "copy_rhs"):
        return None
    t = phi.targets[0]
    if t == "dst":
        return None
    slot = {"src": "x", "edge": "w"}[t]
    bundle = GradBundle()
    if slot not in needs:
        return bundle
    accounting.log_dispatch("gsddmm", g.uid, "argext_route+scatter(%s)" % t, "-",
                            "edge_parallel", g.num_edges, dZ.shape[1])
    rows = g.num_nodes if t == "src" else g.num_edges
    res = kernels.extrema_backward_copy(g, aux, dZ, t, rows)
    setattr(bundle, "dx" if t == "src" else "dw", res)
    return bundle


def gsddmm_backward(g, phi, X=None, Y=None, W=None, M=None, dM=None, needs=("x", "y", "w")):
    """Operand gradients of gsddmm(g, phi) (autodiff.py:415-418)."""
    n, m = g.num_nodes, g.num_edges
    dM = _dev_matrix("dM", dM, m, g)
    ops = [_dev_matrix("X", X, n, g), _dev_matrix("Y", Y, n, g), _dev_matrix("W", W, m, g)]
    dt = torch.float64 if any(o is not None and o.dtype == torch.float64
                              for o in ops + [dM]) else torch.float32
    X, Y, W = [None if o is None else o.to(dt) for o in ops]
    return _edge_grads(g, phi, X, Y, W, dM.to(dt), "edge", needs)


# ----------------------------------------------------------------------------
# autograd Functions (replace the taped wrappers of autodiff.py:425-460)


def _needs(X, Y, W):
    return tuple(k for k, v in (("x", X), ("y", Y), ("w", W))
                 if torch.is_tensor(v) and v.requires_grad)


def _match(grad, like):
    if grad is None or like is None or not torch.is_tensor(like):
        return None
    if grad.shape != like.shape:
        grad = grad.reshape(like.shape)
    return grad.to(dtype=like.dtype, device=like.device)


class _GSpMM(torch.autograd.Function):
    @staticmethod
    def forward(ctx, g, phi, rho, kernel_kw, X, Y, W):
        Z, aux = kernels.gspmm(g, phi, rho, X=X, Y=Y, W=W, **kernel_kw)
        ctx.g, ctx.phi, ctx.rho, ctx.aux = g, phi, rho, aux
        ctx.needs = _needs(X, Y, W)
        ctx.save_for_backward(*(t if torch.is_tensor(t) else None for t in (X, Y, W)))
        ctx.host = tuple(None if torch.is_tensor(t) else t for t in (X, Y, W))
        return Z

    @staticmethod
    def backward(ctx, dZ):
        X, Y, W = (s if s is not None else h for s, h in zip(ctx.saved_tensors, ctx.host))
        b = gspmm_backward(ctx.g, ctx.phi, ctx.rho, X=X, Y=Y, W=W, aux=ctx.aux,
                           dZ=dZ.contiguous(), needs=ctx.needs)
        return (None, None, None, None, _match(b.dx, X), _match(b.dy, Y), _match(b.dw, W))


class _GSDDMM(torch.autograd.Function):
    @staticmethod
    def forward(ctx, g, phi, kernel_kw, X, Y, W):
        M = kernels.gsddmm(g, phi, X=X, Y=Y, W=W, **kernel_kw)
        ctx.g, ctx.phi = g, phi
        ctx.needs = _needs(X, Y, W)
        ctx.save_for_backward(*(t if torch.is_tensor(t) else None for t in (X, Y, W)))
        ctx.host = tuple(None if torch.is_tensor(t) else t for t in (X, Y, W))
        return M

    @staticmethod
    def backward(ctx, dM):
        X, Y, W = (s if s is not None else h for s, h in zip(ctx.saved_tensors, ctx.host))
        b = gsddmm_backward(ctx.g, ctx.phi, X=X, Y=Y, W=W, dM=dM.contiguous(), needs=ctx.needs)
        return (None, None, None, _match(b.dx, X), _match(b.dy, Y), _match(b.dw, W))


class _EdgeSoftmax(torch.autograd.Function):
    @staticmethod
    def forward(ctx, g, scores):
        alpha = kernels.edge_softmax_forward(g, scores)
        ctx.g = g
        ctx.save_for_backward(alpha)
        ctx.like = scores
        return alpha

    @staticmethod
    def backward(ctx, grad):
        (alpha,) = ctx.saved_tensors
        ds = kernels.edge_softmax_backward(ctx.g, alpha, grad.contiguous())
        return None, _match(ds, ctx.like)


class _EdgeSoftmaxUV(torch.autograd.Function):
    """alpha = edge_softmax(u_add_v(el, er)); backward = fused softmax backward
    then the u_add_v g-SDDMM backward (Theorem 1: d el on reverse(g), d er on g)."""

    @staticmethod
    def forward(ctx, g, el, er):
        alpha = kernels.edge_softmax_uv_forward(g, el, er)
        ctx.g = g
        ctx.save_for_backward(alpha, el, er)
        return alpha

    @staticmethod
    def backward(ctx, grad):
        alpha, el, er = ctx.saved_tensors
        ds = kernels.edge_softmax_backward(ctx.g, alpha, grad.contiguous())
        needs = tuple(k for k, need in (("x", ctx.needs_input_grad[1]),
                                        ("y", ctx.needs_input_grad[2])) if need)
        b = gsddmm_backward(ctx.g, kernels.add("src", "dst"), X=el, Y=er, dM=ds, needs=needs)
        return None, _match(b.dx, el), _match(b.dy, er)


def edge_softmax_uv(g, el, er):
    """Differentiable edge_softmax of u_add_v(el, er), scores never materialised."""
    if _grad_enabled(el, er):
        return _EdgeSoftmaxUV.apply(g, el, er)
    return kernels.edge_softmax_uv_forward(g, el, er)


class _GATAttention(torch.autograd.Function):
    """All heads of the reference GAT aggregation (layers.py:110-115):
    out[:, h] = sum_{(u,e)->v} alpha_{e,h} X_h[u], alpha = edge_softmax(el[u] + er[v]),
    with X_h = X (shared) or the h-th column block of X. The attention weights
    are recomputed in the row kernels from el / er / per-destination stats
    and never stored. Backward (Theorem 1 composed by hand):
      dX_h[u]  = sum_{u->v} alpha_e dZ_h[v]                 (reverse-graph rows)
      d el[u]  = sum_{u->v} alpha_e (g_e - S_v)  with g_e = dZ_h[v] . X_h[u],
                 S_v = sum_{e'->v} alpha_e' g_e' = dZ_h[v] . Z_h[v]
               = X_h[u] . dX_h[u] - sum_{u->v} alpha_e S_v
      d er[v]  = S_v (1 - sum_{e->v} alpha_e) = 0   (softmax is shift-invariant)
    S_v rides in the 4th column of the per-node pack the kernel gathers
    anyway; the reverse-graph kernel returns t[u] = sum_{u->v} alpha_e S_v.
    For fp32 features both row dots read the kernels' unrounded fp64 rows
    (Z64, dX64): S_v and X.dX - t cancel, and a dot of an fp32-rounded row
    would carry |row| 2^-24 per term into the difference."""

    @staticmethod
    def forward(ctx, g, el, er, X, shared):
        H = el.shape[1]
        d = X.shape[1] if shared else X.shape[1] // H
        stat = kernels.edge_softmax_uv_stats(g, el, er)
        pack = torch.zeros((H, g.num_nodes, kernels.pack_width(X.dtype)), dtype=X.dtype,
                           device=X.device)
        pack[:, :, 0] = er.t()
        pack[:, :, 1] = stat[:, :H].t()
        pack[:, :, 2] = stat[:, H:].t()
        outs = []
        z64 = None
        if X.dtype != torch.float64 and not isinstance(ctx, _NoCtx):
            z64 = torch.empty((g.num_nodes, H * d), dtype=torch.float64, device=X.device)
        for h in range(H):
            Xh = X if shared else X[:, h * d:(h + 1) * d]
            outs.append(kernels.gat_aggregate(
                g, Xh, el[:, h:h + 1], pack[h],
                z64=z64[:, h * d:(h + 1) * d] if z64 is not None else None))
        out = outs[0] if H == 1 else torch.cat(outs, dim=1)
        ctx.g, ctx.shared, ctx.d = g, shared, d
        ctx.save_for_backward(el, er, X, pack, out if z64 is None else z64)
        return out

    @staticmethod
    def backward(ctx, dout):
        el, er, X, pack = ctx.saved_tensors[:4]
        out = ctx.saved_tensors[4]
        g, shared, d = ctx.g, ctx.shared, ctx.d
        H = el.shape[1]
        dout = dout.to(X.dtype)
        if dout.stride(-1) != 1:
            dout = dout.contiguous()
        dX_parts = []
        dEl = torch.empty(el.shape, dtype=X.dtype, device=X.device)
        dx64 = None
        if X.dtype != torch.float64:
            dx64 = torch.empty((g.num_nodes, d), dtype=torch.float64, device=X.device)
        for h in range(H):
            dZh = dout[:, h * d:(h + 1) * d]
            Zh = out[:, h * d:(h + 1) * d]   # fp64 rows (Z64) for fp32 features
            # S_v = dZ[v].Z[v] (fp64) rides in the pack's 4th column;
            # t[u] = sum_{u->v} alpha_e S_v comes back from the kernel
            pk = pack[h].clone()
            kernels.rowdot(dZh, Zh, pk[:, 3], pair=X.dtype != torch.float64)
            dXh, t = kernels.gat_aggregate(g, dZh, el[:, h:h + 1], pk, backward=True, z64=dx64)
            Xh = X if shared else X[:, h * d:(h + 1) * d]
            kernels.rowdot(Xh, dXh if dx64 is None else dx64, dEl[:, h], sub=t)  # X.dX - t
            dX_parts.append(dXh)
        if shared:
            dX = dX_parts[0]
            for p in dX_parts[1:]:
                dX = dX + p
        else:
            dX = dX_parts[0] if H == 1 else torch.cat(dX_parts, dim=1)
        return None, _match(dEl, el), torch.zeros_like(er), _match(dX, X), None


def gat_attention(g, el, er, X, shared=False):
    """Differentiable fused GAT aggregation of every head (see _GATAttention):
    (n, H*d) with d = X's width (shared) or X's width / H."""
    if _grad_enabled(el, er, X):
        return _GATAttention.apply(g, el, er, X, shared)
    with torch.no_grad():
        return _GATAttention.forward(_NoCtx(), g, el, er, X, shared)


class _NoCtx:
    def save_for_backward(self, *a):
        pass


def _grad_enabled(*xs):
    return torch.is_grad_enabled() and any(torch.is_tensor(x) and x.requires_grad for x in xs)


def gspmm(g, phi, rho, X=None, Y=None, W=None, **kernel_kw):
    """Differentiable gspmm; returns Z (autodiff.py:425-442)."""
    if _grad_enabled(X, Y, W):
        return _GSpMM.apply(g, phi, rho, kernel_kw, X, Y, W)
    Z, _ = kernels.gspmm(g, phi, rho, X=X, Y=Y, W=W, **kernel_kw)
    return Z


def gsddmm(g, phi, X=None, Y=None, W=None, **kernel_kw):
    """Differentiable gsddmm; returns M (autodiff.py:445-460)."""
    if _grad_enabled(X, Y, W):
        return _GSDDMM.apply(g, phi, kernel_kw, X, Y, W)
    return kernels.gsddmm(g, phi, X=X, Y=Y, W=W, **kernel_kw)


def edge_softmax(g, scores):
    """Differentiable fused edge softmax (forward and backward one kernel each)."""
    if _grad_enabled(scores):
        return _EdgeSoftmax.apply(g, scores)
    return kernels.edge_softmax_forward(g, scores)
