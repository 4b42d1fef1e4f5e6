"""Device-resident immutable multigraph with shared, lazily built adjacencies.

Mirrors the reference's graph core (/root/reference/pkg/src/graphmp/graph.py):
  * a Graph is (src, dst) over dense edge ids 0..m-1 (graph.py:62-100);
  * to_csc() groups edges by destination (the in-adjacency the g-SpMM row
    kernel walks, graph.py:137-139), to_csr() by source (graph.py:133-135);
    inside a group neighbours ascend and parallel edges break ties by edge id
    (graph.py:35-44), so index arrays compare bit-exactly with the reference;
  * the CSC/CSR pair is shared with reverse(g) (graph.py:203-215), so
    reverse(g).to_csc() IS g.to_csr() and the backward of a g-SpMM (which
    runs on the reverse graph, Theorem 1) never rebuilds an index;
  * caches are built under a double-checked lock and counted
    (adjacency_build_count, graph.py:116-131,141-143).

B200 layout: src/dst/indices/edge_ids are int32 device tensors, indptr int64
(graph.py:25-32 uses uint32/int64; m and n must stay below 2**31). The build is
a stable device sort of the composite key group * n + neighbour in edge-id
order, which reproduces np.lexsort((eids, other, group)) exactly. Each
adjacency also caches its degree-binned row schedule (gmp_build_schedule),
built on first kernel use.
"""

import itertools
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

_uid = itertools.count(1)
_INT32_LIMIT = 2 ** 31 - 1

# rows with more in-edges than this are reduced by a whole CTA (gmp_sched);
# rows with at most LIGHT_ROW_THRESHOLD in-edges share a warp (one per lane group)
HEAVY_ROW_THRESHOLD = 2048
LIGHT_ROW_THRESHOLD = 32


def default_device():
    return torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu")


@dataclass(frozen=True)
class Adjacency:
    """One grouped index: indptr (n+1, int64), indices / edge_ids (m, int32)."""
    indptr: torch.Tensor
    indices: torch.Tensor
    edge_ids: torch.Tensor
    _extra: dict = field(default_factory=dict, compare=False, repr=False)

    @property
    def num_groups(self):
        return self.indptr.numel() - 1

    def degrees(self):
        d = self._extra.get("degrees")
        if d is None:
            d = self.indptr[1:] - self.indptr[:-1]
            self._extra["degrees"] = d
        return d

    def numpy(self):
        """(indptr int64, indices uint32, edge_ids uint32) host copies, reference dtypes."""
        return (self.indptr.cpu().numpy(),
                self.indices.cpu().numpy().astype(np.uint32),
                self.edge_ids.cpu().numpy().astype(np.uint32))

    def schedule(self):
        """Cached degree-binned schedule (ctypes GmpSched + keep-alive tensors)."""
        s = self._extra.get("sched")
        if s is None:
            with self._extra.setdefault("lock", threading.Lock()):
                s = self._extra.get("sched")
                if s is None:
                    from . import kernels
                    s = kernels._build_schedule(self)
                    self._extra["sched"] = s
        return s


def _build_adjacency(group, other, num_nodes):
    m = group.numel()
    dev = group.device
    if m == 0:
        empty = torch.zeros(0, dtype=torch.int32, device=dev)
        return Adjacency(torch.zeros(num_nodes + 1, dtype=torch.int64, device=dev), empty, empty)
    key = group.to(torch.int64) * max(num_nodes, 1) + other.to(torch.int64)
    _, order = torch.sort(key, stable=True)
    indices = other.index_select(0, order).to(torch.int32)
    edge_ids = order.to(torch.int32)
    counts = torch.bincount(group.to(torch.int64), minlength=num_nodes)
    indptr = torch.zeros(num_nodes + 1, dtype=torch.int64, device=dev)
    torch.cumsum(counts, 0, out=indptr[1:])
    return Adjacency(indptr, indices, edge_ids)


class _CachePair:
    """Adjacencies shared by a graph and its reverse view, keyed on the base
    orientation (graph.py:47-59)."""
    __slots__ = ("by_src", "by_dst", "build_count", "lock")

    def __init__(self):
        self.by_src = None
        self.by_dst = None
        self.build_count = 0
        self.lock = threading.Lock()


def _as_ids(a, device):
    if isinstance(a, torch.Tensor):
        t = a.detach()
        if t.is_floating_point() or t.is_complex():
            raise ValueError("node ids must be integers")
        return t.to(device=device, dtype=torch.int64)
    arr = np.asarray(a)
    if arr.size and not np.issubdtype(arr.dtype, np.integer):
        raise ValueError("node ids must be integers")
    return torch.from_numpy(np.ascontiguousarray(arr, dtype=np.int64)).to(device)


class Graph:
    """Directed multigraph over dense int32 node ids; structure only."""

    def __init__(self, src, dst, num_nodes, device=None, _caches=None, _flipped=False):
        device = torch.device(device) if device is not None else (
            src.device if isinstance(src, torch.Tensor) else default_device())
        s = _as_ids(src, device)
        d = _as_ids(dst, device)
        if s.dim() != 1 or d.dim() != 1 or s.shape != d.shape:
            raise ValueError("src and dst must be 1-D arrays of equal length")
        num_nodes = int(num_nodes)
        if num_nodes < 0 or num_nodes > _INT32_LIMIT:
            raise ValueError("num_nodes out of range for int32 ids")
        if s.numel() > _INT32_LIMIT:
            raise ValueError("edge count exceeds the int32 edge-id range")
        if s.numel():
            bad = (s < 0) | (d < 0) | (s >= num_nodes) | (d >= num_nodes)
            if bool(bad.any()):
                i = int(torch.nonzero(bad)[0, 0])
                raise ValueError("edge %d has endpoint (%d, %d) outside [0, %d)"
                                 % (i, int(s[i]), int(d[i]), num_nodes))
        self._src = s.to(torch.int32)
        self._dst = d.to(torch.int32)
        self._num_nodes = num_nodes
        self._caches = _caches if _caches is not None else _CachePair()
        self._flipped = _flipped
        self._reverse_view = None
        self._eids = None
        self.uid = next(_uid)

    # -- queries --------------------------------------------------------------
    @property
    def device(self):
        return self._src.device

    @property
    def num_nodes(self):
        return self._num_nodes

    @property
    def num_edges(self):
        return self._src.numel()

    @property
    def src(self):
        return self._src

    @property
    def dst(self):
        return self._dst

    def edge_ids(self):
        if self._eids is None:
            self._eids = torch.arange(self.num_edges, dtype=torch.int32, device=self.device)
        return self._eids

    def coo(self):
        """(src, dst, edge_ids) device tensors in edge-id order (graph.py:98-100)."""
        return self._src, self._dst, self.edge_ids()

    def coo_numpy(self):
        """Host copy of coo() with the reference's uint32 dtypes."""
        return (self._src.cpu().numpy().astype(np.uint32), self._dst.cpu().numpy().astype(np.uint32),
                np.arange(self.num_edges, dtype=np.uint32))

    def to(self, device):
        """Same structure on another device (a new graph: caches are per device)."""
        return Graph(self._src.to(device), self._dst.to(device), self._num_nodes)

    def __repr__(self):
        return "Graph(num_nodes=%d, num_edges=%d, uid=%d, device=%s)" % (
            self.num_nodes, self.num_edges, self.uid, self.device)

    # -- grouped indexes --------------------------------------------------------
    def _slot(self, name):
        caches = self._caches
        adj = getattr(caches, name)
        if adj is None:
            with caches.lock:
                adj = getattr(caches, name)
                if adj is None:
                    base_src, base_dst = ((self._dst, self._src) if self._flipped
                                          else (self._src, self._dst))
                    if name == "by_src":
                        adj = _build_adjacency(base_src, base_dst, self._num_nodes)
                    else:
                        adj = _build_adjacency(base_dst, base_src, self._num_nodes)
                    setattr(caches, name, adj)
                    caches.build_count += 1
        return adj

    def to_csr(self):
        """Out-adjacency: edges grouped by source node."""
        return self._slot("by_dst" if self._flipped else "by_src")

    def to_csc(self):
        """In-adjacency: edges grouped by destination node."""
        return self._slot("by_src" if self._flipped else "by_dst")

    @property
    def adjacency_build_count(self):
        return self._caches.build_count

    # -- degrees ----------------------------------------------------------------
    def _degrees(self, keys, cached, nodes):
        if cached is not None:
            degs = cached.degrees()
        else:
            degs = torch.bincount(keys.to(torch.int64), minlength=self._num_nodes)
        if nodes is None:
            return degs
        idx = _as_ids(nodes, self.device)
        if idx.numel() and (int(idx.min()) < 0 or int(idx.max()) >= self._num_nodes):
            raise IndexError("node id out of range")
        return degs[idx]

    def in_degrees(self, nodes=None):
        cached = self._caches.by_src if self._flipped else self._caches.by_dst
        return self._degrees(self._dst, cached, nodes)

    def out_degrees(self, nodes=None):
        cached = self._caches.by_dst if self._flipped else self._caches.by_src
        return self._degrees(self._src, cached, nodes)


def build_graph(num_nodes, edges, device=None):
    """Graph from (u, v) pairs or a (src, dst) pair of arrays; ids in input order."""
    if isinstance(edges, tuple) and len(edges) == 2 and hasattr(edges[0], "__len__") and \
            not np.isscalar(edges[0]) and np.ndim(edges[0]) == 1:
        src, dst = edges
    else:
        arr = np.asarray(edges, dtype=np.int64)
        if arr.size == 0:
            arr = arr.reshape(0, 2)
        src, dst = arr[:, 0], arr[:, 1]
    s = _as_ids(src, torch.device("cpu")) if not isinstance(src, torch.Tensor) else src
    d = _as_ids(dst, torch.device("cpu")) if not isinstance(dst, torch.Tensor) else dst
    if s.numel() and (bool((s < 0).any()) or bool((d < 0).any())):
        i = int(torch.nonzero((s < 0) | (d < 0))[0, 0])
        raise ValueError("edge %d has a negative endpoint" % i)
    return Graph(s, d, num_nodes, device=device if device is not None else (
        src.device if isinstance(src, torch.Tensor) else None))


def from_arrays(src, dst, num_nodes=None, device=None):
    """Graph from endpoint arrays; num_nodes defaults to max id + 1."""
    if num_nodes is None:
        s = np.asarray(src.cpu() if isinstance(src, torch.Tensor) else src)
        d = np.asarray(dst.cpu() if isinstance(dst, torch.Tensor) else dst)
        num_nodes = int(max(s.max(initial=0), d.max(initial=0))) + 1 if s.size else 0
    return Graph(src, dst, num_nodes, device=device)


def reverse(g):
    """Edge-for-edge reversed view sharing g's adjacency pair (graph.py:203-215)."""
    if g._reverse_view is not None:
        return g._reverse_view
    rev = Graph.__new__(Graph)
    rev._src, rev._dst = g._dst, g._src
    rev._num_nodes = g._num_nodes
    rev._caches = g._caches
    rev._flipped = not g._flipped
    rev._reverse_view = g
    rev._eids = g._eids
    rev.uid = next(_uid)
    g._reverse_view = rev
    return rev


@dataclass(frozen=True)
class Subgraph:
    """A compactly relabelled induced piece of a parent graph (graph.py:218-228):
    row i of a parent node feature matrix sliced by parent_node_ids is the
    feature of subgraph node i; parent_edge_ids does the same for edges.
    Both are int64 device tensors."""
    graph: "Graph"
    parent_node_ids: torch.Tensor
    parent_edge_ids: torch.Tensor


def neighbor_sample(g, seeds, fanout, rng_seed):
    """Sample up to `fanout` in-edges per seed without replacement
    (graph.py:231-286). Seeds come first in the relabelling (first-occurrence
    order), then newly reached predecessors in ascending parent id; each
    seed's picks are in ascending in-adjacency position. The draw runs on the
    device (gmp_neighbor_sample): uniform over k-subsets like the reference's
    partial Fisher-Yates, from a counter-based generator, so a sample is fully
    determined by rng_seed (the reference's numpy stream is not reproduced;
    with fanout >= in-degree the result is identical to the reference's)."""
    from . import _lib
    fanout = int(fanout)
    if fanout < 1:
        raise ValueError("fanout must be at least 1")
    s = np.asarray(seeds.cpu() if isinstance(seeds, torch.Tensor) else seeds, dtype=np.int64)
    s = s.reshape(-1)
    if s.size and (s.min() < 0 or s.max() >= g.num_nodes):
        raise IndexError("seed node id out of range")
    if g.device.type != "cuda":
        raise RuntimeError("neighbor_sample: graph is on %s; libgmp has no CPU fallback" % g.device)
    _, first = np.unique(s, return_index=True)
    keep = s[np.sort(first)]                      # first-occurrence order
    dev = g.device
    seeds_d = torch.from_numpy(keep).to(dev)
    adj = g.to_csc()
    deg = adj.indptr.index_select(0, seeds_d + 1) - adj.indptr.index_select(0, seeds_d)
    k = torch.clamp(deg, max=fanout)
    off = torch.zeros(keep.size + 1, dtype=torch.int64, device=dev)
    torch.cumsum(k, 0, out=off[1:])
    total = int(off[-1]) if keep.size else 0
    pos = torch.empty(total, dtype=torch.int64, device=dev)
    if total:
        scratch = torch.empty(total, dtype=torch.int64, device=dev)
        stream = torch.cuda.current_stream(dev).cuda_stream
        _lib.check(_lib.load().gmp_neighbor_sample(
            adj.indptr.data_ptr(), adj.num_groups, seeds_d.data_ptr(), keep.size, off.data_ptr(),
            int(rng_seed) & (2 ** 64 - 1), scratch.data_ptr(), pos.data_ptr(), stream),
            "gmp_neighbor_sample")
    peids = adj.edge_ids.index_select(0, pos).to(torch.int64)
    psrc = g.src.index_select(0, peids).to(torch.int64)
    pdst = g.dst.index_select(0, peids).to(torch.int64)
    mark = torch.zeros(g.num_nodes, dtype=torch.bool, device=dev)
    mark[psrc] = True
    mark[seeds_d] = False
    node_ids = torch.cat([seeds_d, torch.nonzero(mark).reshape(-1)])
    relabel = torch.full((g.num_nodes,), -1, dtype=torch.int64, device=dev)
    relabel[node_ids] = torch.arange(node_ids.numel(), dtype=torch.int64, device=dev)
    sub = Graph(relabel.index_select(0, psrc), relabel.index_select(0, pdst), node_ids.numel(),
                device=dev)
    return Subgraph(sub, node_ids, peids)
