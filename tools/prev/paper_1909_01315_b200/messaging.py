"""Graph-centric message passing over named features.

Mirror of /root/reference/pkg/src/graphmp/messaging.py:32-126:
  update_all(g, msg('mul', src('h'), edge('w')), 'sum', ndata, edata, out='z')
      -> ONE g-SpMM launch, stored as ndata[out]
  apply_edges(g, msg('dot', src('p'), dst('p')), ndata, edata, out='s')
      -> ONE g-SDDMM launch, stored as edata[out]
  edge_softmax(g, scores, edata=None, out=None)
      -> ONE fused row kernel (the reference composes 4 kernels + exp; its
         dispatch-sequence test test_messaging.py:180-185 is superseded, see
         DESIGN.md). Differentiable through a fused backward kernel.
The degree-bucketed UDF path (update_all_udf, messaging.py:137-185) is out of
this round's hot-path scope.
"""

from dataclasses import dataclass

from . import autodiff, kernels


@dataclass(frozen=True)
class Field:
    target: str  # 'src' | 'dst' | 'edge'
    name: str


def src(name):
    """The named node feature, read at each edge's source."""
    return Field("src", name)


def dst(name):
    """The named node feature, read at each edge's destination."""
    return Field("dst", name)


def edge(name):
    """The named edge feature."""
    return Field("edge", name)


@dataclass(frozen=True)
class NamedMessage:
    op: str
    lhs: Field = None
    rhs: Field = None


def msg(op, lhs=None, rhs=None):
    """Message recipe over named features; 'copy' aliases copy_lhs and a lone
    field given to copy_rhs is its rhs (messaging.py:60-70)."""
    if op == "copy":
        op = "copy_lhs"
    if op == "copy_rhs" and rhs is None and lhs is not None:
        lhs, rhs = None, lhs
    return NamedMessage(op, lhs, rhs)


def _resolve(g, ndata, edata, recipe):
    phi = kernels.MessageFunc(recipe.op, recipe.lhs.target if recipe.lhs else None,
                              recipe.rhs.target if recipe.rhs else None)
    operands = {"X": None, "Y": None, "W": None}
    slot = {"src": "X", "dst": "Y", "edge": "W"}
    for f in (recipe.lhs, recipe.rhs):
        if f is not None:
            operands[slot[f.target]] = (edata if f.target == "edge" else ndata)[f.name]
    return phi, operands


def update_all(g, recipe, rho, ndata, edata=None, *, out, **kernel_kw):
    """One fused g-SpMM over named features; result stored as ndata[out]."""
    phi, ops = _resolve(g, ndata, edata, recipe)
    z = autodiff.gspmm(g, phi, rho, **ops, **kernel_kw)
    ndata[out] = z
    return z


def apply_edges(g, recipe, ndata=None, edata=None, *, out, **kernel_kw):
    """One fused g-SDDMM over named features; result stored as edata[out]."""
    if edata is None:
        raise ValueError("apply_edges stores per-edge output; pass the edata dict")
    phi, ops = _resolve(g, ndata, edata, recipe)
    m = autodiff.gsddmm(g, phi, **ops, **kernel_kw)
    edata[out] = m
    return m


def edge_softmax(g, scores, edata=None, out=None):
    """Per-destination softmax of per-edge scores (every column independent,
    always max-shifted); scores is a matrix or a name in edata."""
    if isinstance(scores, str):
        if edata is None:
            raise ValueError("named scores need the edata dict")
        scores = edata[scores]
    alpha = autodiff.edge_softmax(g, scores)
    if out is not None:
        if edata is None:
            raise ValueError("storing under a name needs the edata dict")
        edata[out] = alpha
    return alpha
