"""GCN / GraphSAGE / GAT as thin torch callers of the g-SpMM / g-SDDMM kernels.

These exist to time and check the epoch configs (BASELINE.json configs 0-3);
they own no kernels. Semantics follow /root/reference/pkg/src/graphmp/layers.py:
  gcn_layer  act(mean_agg(X) @ W + b)          (layers.py:62-67; aggregate first)
  sage_layer act(X @ W_self + mean_agg(X) @ W_neigh)   (layers.py:76-81)
             (order="auto" aggregates the narrower side of W, as DGL's GraphConv
             does; order="aggregate_first" is the reference's literal order)
  gat_layer  per head: proj = X @ W; score_uv = a_l.proj_u + a_r.proj_v (u_add_v
             g-SDDMM, no LeakyReLU); alpha = edge_softmax; out = sum_u alpha*proj_u
             (u_mul_e g-SpMM); heads concatenated            (layers.py:96-116)
`aggregator="sum"` gives the copy_u+sum GCN named by BASELINE.json config 0.
Dense projections are torch matmuls (cuBLAS; fp32 with TF32 off by default so
parity tests compare against the reference's float64 numbers).
GAT (fused=True, default): el / er come from X (W a) without the projection;
a statistics kernel computes each destination's softmax max / sum of the
u_add_v scores, and the aggregation row kernels recompute every attention
weight from node-keyed data, forward (destination rows) and backward
(reverse-graph rows), so neither the (m, H) scores nor alpha are ever stored.
The aggregation runs on the narrower of the input and the projected features
(linearity: sum alpha (X W) = (sum alpha X) W).
"""

import contextlib
import threading
from dataclasses import dataclass

import numpy as np
import torch
import torch.nn.functional as F

from . import autodiff, kernels
from .graph import default_device

RELU_GAIN = float(np.sqrt(2.0))


def xavier_uniform(rng, fan_in, fan_out, gain=RELU_GAIN):
    """Uniform on [-a, a], a = gain * sqrt(6 / (fan_in + fan_out)) (layers.py:31-34)."""
    a = gain * np.sqrt(6.0 / (fan_in + fan_out))
    return rng.uniform(-a, a, size=(fan_in, fan_out))


def _act(h, name):
    if name == "relu":
        return torch.relu(h)
    if name in (None, "linear"):
        return h
    raise ValueError("unknown activation %r" % (name,))


def _check_rows(g, X):
    if X.shape[0] != g.num_nodes:
        raise ValueError("feature matrix has %d rows for a %d-node graph"
                         % (X.shape[0], g.num_nodes))


def _t(x, device, dtype):
    if torch.is_tensor(x):
        return x
    return torch.as_tensor(np.asarray(x), dtype=dtype, device=device)


_dense = threading.local()


@contextlib.contextmanager
def dense_precision(mode):
    """Precision of the layers' dense products (projections, attention
    vectors) for fp32 features: "fp32" (default: torch/cuBLAS fp32 GEMMs,
    TF32 off) or "fp64" (operands up-cast exactly, fp64 products and
    accumulation, rounded once to fp32 - the same numerics contract as the
    sparse kernels, so a whole layer matches the reference's float64 layer
    within north_star's rtol 1e-5 / atol 1e-6; the dense GEMMs are not part
    of the ported path). Thread-local, like the reference's kernel config
    (kernels.py:161)."""
    if mode not in ("fp32", "fp64"):
        raise ValueError("unknown dense precision %r" % (mode,))
    prev = getattr(_dense, "mode", "fp32")
    _dense.mode = mode
    try:
        yield
    finally:
        _dense.mode = prev


def _hi(t):
    """t in the dense-product precision (fp64 under dense_precision('fp64'))."""
    if getattr(_dense, "mode", "fp32") == "fp64" and t.dtype == torch.float32:
        return t.double()
    return t


def _mm(a, b):
    """a @ b in the dense-product precision, returned in a's dtype."""
    return (_hi(a) @ _hi(b)).to(a.dtype)


def aggregate(g, X, aggregator="mean", **kw):
    """copy_u g-SpMM with the given reducer (mean = in-degree normalised)."""
    return autodiff.gspmm(g, kernels.copy("src"), aggregator, X=X, **kw)


@dataclass
class GCNParams:
    W: torch.Tensor
    b: torch.Tensor


@dataclass
class SAGEParams:
    W_self: torch.Tensor
    W_neigh: torch.Tensor


@dataclass
class GATHead:
    W: torch.Tensor
    a_l: torch.Tensor
    a_r: torch.Tensor


@dataclass
class GATParams:
    heads: list


def _project_first(X, W, order):
    if order not in ("auto", "aggregate_first", "project_first"):
        raise ValueError("unknown layer order %r" % (order,))
    return order == "project_first" or (order == "auto" and W.shape[1] < W.shape[0])


def gcn_layer(g, X, params, act="relu", aggregator="mean", order="auto", **kw):
    """act(agg(X) @ W + b). The reference aggregates first (layers.py:62-67);
    agg is linear, so agg(X) @ W = agg(X @ W), and with order="auto" the
    aggregation runs on the narrower side (DGL GraphConv does the same when
    in_feats > out_feats). Same result up to fp rounding."""
    _check_rows(g, X)
    X = _t(X, g.device, torch.float64)
    W = _t(params.W, X.device, X.dtype)
    b = _t(params.b, X.device, X.dtype)
    if _project_first(X, W, order):
        return _act(aggregate(g, _mm(X, W), aggregator, **kw) + b, act)
    return _act(_mm(aggregate(g, X, aggregator, **kw), W) + b, act)


def sage_layer(g, X, params, act="relu", order="auto", **kw):
    """act(X @ W_self + mean_agg(X) @ W_neigh) (layers.py:76-81); the
    neighbour term aggregates the narrower side as in gcn_layer."""
    _check_rows(g, X)
    X = _t(X, g.device, torch.float64)
    Ws = _t(params.W_self, X.device, X.dtype)
    Wn = _t(params.W_neigh, X.device, X.dtype)
    if _project_first(X, Wn, order):
        return _act(_mm(X, Ws) + aggregate(g, _mm(X, Wn), "mean", **kw), act)
    return _act(_mm(X, Ws) + _mm(aggregate(g, X, "mean", **kw), Wn), act)


def gat_layer(g, X, params, num_heads=None, fused=True, **kw):
    """Heads concatenated column-wise; isolated destinations get zero rows.
    fused=True: the attention weights are recomputed inside the aggregation
    row kernels (gmp_gat_aggregate) and no (m, H) tensor exists in the forward
    or the backward; fused=False: the fused u_add_v + edge_softmax kernel pair
    writes alpha (m, H) and per-head u_mul_e g-SpMMs read it (the reference's
    composition, layers.py:110-115)."""
    _check_rows(g, X)
    heads = params.heads if num_heads is None else params.heads[:num_heads]
    if not heads:
        raise ValueError("head count must be >= 1")
    X = _t(X, g.device, torch.float64)
    dev, dt = X.device, X.dtype
    Wcat = torch.cat([_t(h.W, dev, dt) for h in heads], dim=1)           # (d_in, H*D)
    D = _t(heads[0].W, dev, dt).shape[1]
    H = len(heads)
    d_in = X.shape[1]
    al = torch.stack([_t(h.a_l, dev, dt)[:, 0] for h in heads])           # (H, D)
    ar = torch.stack([_t(h.a_r, dev, dt)[:, 0] for h in heads])
    # el = proj . a_l = X (W a_l): only (d_in, H) extra weights, no projection needed
    Wv = Wcat.view(d_in, H, D)
    el = _mm(X, (_hi(Wv) * _hi(al)).sum(-1)).contiguous()                # (n, H)
    er = _mm(X, (_hi(Wv) * _hi(ar)).sum(-1)).contiguous()
    if fused:
        if d_in < D:
            # sum_u alpha_uv (X_u W) = (sum_u alpha_uv X_u) W: aggregate the narrower side
            agg = autodiff.gat_attention(g, el, er, X, shared=True)       # (n, H*d_in)
            outs = [_mm(agg[:, h * d_in:(h + 1) * d_in], Wv[:, h, :]) for h in range(H)]
        else:
            return autodiff.gat_attention(g, el, er, _mm(X, Wcat), shared=False)
        return outs[0] if H == 1 else torch.cat(outs, dim=1)
    # u_add_v scores + edge_softmax fused: the (m, H) scores are never stored
    alpha = autodiff.edge_softmax_uv(g, el, er)                           # (m, H)
    if d_in < D:
        outs = [_mm(autodiff.gspmm(g, kernels.mul("src", "edge"), "sum", X=X,
                                   W=alpha[:, h:h + 1], **kw), Wv[:, h, :]) for h in range(H)]
    else:
        proj = _mm(X, Wcat)                                               # (n, H*D)
        outs = [autodiff.gspmm(g, kernels.mul("src", "edge"), "sum",
                               X=proj[:, h * D:(h + 1) * D], W=alpha[:, h:h + 1], **kw)
                for h in range(H)]
    return outs[0] if H == 1 else torch.cat(outs, dim=1)


def init_gcn(rng, d_in, d_out):
    return GCNParams(W=xavier_uniform(rng, d_in, d_out), b=np.zeros((1, d_out)))


def init_sage(rng, d_in, d_out):
    return SAGEParams(W_self=xavier_uniform(rng, d_in, d_out),
                      W_neigh=xavier_uniform(rng, d_in, d_out))


def init_gat(rng, d_in, d_head, num_heads):
    return GATParams(heads=[GATHead(W=xavier_uniform(rng, d_in, d_head),
                                    a_l=xavier_uniform(rng, d_head, 1),
                                    a_r=xavier_uniform(rng, d_head, 1))
                            for _ in range(num_heads)])


def _leaf(a, device, dtype):
    return torch.as_tensor(np.asarray(a), dtype=dtype, device=device).requires_grad_(True)


class GCNModel:
    """Stack of GCN layers (relu between, linear last); numpy-seeded init
    identical to the reference's GCNModel (layers.py:137-158)."""

    def __init__(self, dims, seed=0, aggregator="mean", device=None, dtype=torch.float32,
                 order="auto"):
        if len(dims) < 2:
            raise ValueError("need at least input and output dims")
        rng = np.random.default_rng(seed)
        device = device or default_device()
        self.aggregator = aggregator
        self.order = order
        self.layers = []
        self.out_dim = dims[-1]
        for a, b in zip(dims, dims[1:]):
            p = init_gcn(rng, a, b)
            self.layers.append(GCNParams(W=_leaf(p.W, device, dtype), b=_leaf(p.b, device, dtype)))

    def parameters(self):
        return [t for lp in self.layers for t in (lp.W, lp.b)]

    def layer(self, i, g, h, **kw):
        """Layer i on graph g (a full graph or a sampled block)."""
        return gcn_layer(g, h, self.layers[i], act="relu" if i < len(self.layers) - 1 else "linear",
                         aggregator=self.aggregator, order=self.order, **kw)

    def forward(self, g, x, **kw):
        h = x
        for i in range(len(self.layers)):
            h = self.layer(i, g, h, **kw)
        return h


class SAGEModel:
    """Stack of GraphSAGE-mean layers."""

    def __init__(self, dims, seed=0, device=None, dtype=torch.float32, order="auto"):
        rng = np.random.default_rng(seed)
        device = device or default_device()
        self.order = order
        self.layers = []
        self.out_dim = dims[-1]
        for a, b in zip(dims, dims[1:]):
            p = init_sage(rng, a, b)
            self.layers.append(SAGEParams(W_self=_leaf(p.W_self, device, dtype),
                                          W_neigh=_leaf(p.W_neigh, device, dtype)))

    def parameters(self):
        return [t for lp in self.layers for t in (lp.W_self, lp.W_neigh)]

    def layer(self, i, g, h, **kw):
        return sage_layer(g, h, self.layers[i],
                          act="relu" if i < len(self.layers) - 1 else "linear", order=self.order,
                          **kw)

    def forward(self, g, x, **kw):
        h = x
        for i in range(len(self.layers)):
            h = self.layer(i, g, h, **kw)
        return h


class GATModel:
    """Stack of GAT layers (heads concatenated, relu between layers, linear
    last) - the Reddit GAT epoch of the paper is 3 layers x 16 hidden x 1 head
    (PAPER.md:965-966); the reference only defines the single gat_layer."""

    def __init__(self, dims, heads=1, seed=0, device=None, dtype=torch.float32, fused=True):
        rng = np.random.default_rng(seed)
        device = device or default_device()
        self.fused = fused
        self.layers = []
        self.out_dim = dims[-1]
        if heads < 1:
            raise ValueError("head count must be >= 1")
        d_in = dims[0]
        for i, d_out in enumerate(dims[1:]):
            last = i == len(dims) - 2
            h = 1 if last else heads
            if d_out % h:
                raise ValueError("hidden width %d is not divisible by %d heads" % (d_out, h))
            p = init_gat(rng, d_in, d_out if last else d_out // h, h)
            for hp in p.heads:
                hp.W, hp.a_l, hp.a_r = (_leaf(a, device, dtype) for a in (hp.W, hp.a_l, hp.a_r))
            self.layers.append(p)
            d_in = d_out

    def parameters(self):
        return [t for p in self.layers for hp in p.heads for t in (hp.W, hp.a_l, hp.a_r)]

    def layer(self, i, g, h, **kw):
        h = gat_layer(g, h, self.layers[i], fused=self.fused, **kw)
        return torch.relu(h) if i < len(self.layers) - 1 else h

    def forward(self, g, x, **kw):
        h = x
        for i in range(len(self.layers)):
            h = self.layer(i, g, h, **kw)
        return h


@dataclass
class TrainConfig:
    lr: float = 0.05
    epochs: int = 100
    seed: int = 0
    strategy: str = None

    def __post_init__(self):
        if self.lr < 0:
            raise ValueError("learning rate must be non-negative")
        if self.epochs < 1:
            raise ValueError("epochs must be >= 1")


def xent_loss(logits, labels):
    """Mean cross-entropy of row-softmax probabilities (autodiff.py:228-246)."""
    return F.cross_entropy(logits, labels)


def train_epoch(g, x, labels, model, lr):
    """One full-graph gradient-descent step; returns the loss tensor (on device)."""
    params = model.parameters()
    loss = xent_loss(model.forward(g, x), labels)
    grads = torch.autograd.grad(loss, params)
    with torch.no_grad():
        for p, gr in zip(params, grads):
            p.sub_(lr * gr)
    return loss.detach()


def train(g, features, labels, model, cfg):
    """Full-graph gradient descent; per-epoch losses (layers.py:175-202)."""
    params = model.parameters()
    dev, dt = params[0].device, params[0].dtype
    x = features if torch.is_tensor(features) else torch.as_tensor(
        np.asarray(features), dtype=dt, device=dev)
    labels = torch.as_tensor(np.asarray(labels.cpu() if torch.is_tensor(labels) else labels),
                             dtype=torch.int64, device=dev)
    # the model's output width (GATModel's last parameter is a_r, (D, 1))
    n_classes = getattr(model, "out_dim", None) or params[-1].shape[1]
    if int(labels.min()) < 0 or int(labels.max()) >= n_classes:
        raise ValueError("label out of range [0, %d)" % n_classes)
    losses = []
    for _ in range(cfg.epochs):
        if cfg.strategy is not None:
            with kernels.force_strategy(cfg.strategy):
                loss = train_epoch(g, x, labels, model, cfg.lr)
        else:
            loss = train_epoch(g, x, labels, model, cfg.lr)
        losses.append(loss)
    return [float(v) for v in torch.stack(losses).cpu()]
