"""paper_1909_01315_b200: B200-native g-SpMM / g-SDDMM / edge_softmax.

A drop-in for the message-passing hot path of the reference package graphmp
(/root/reference/pkg/src/graphmp/__init__.py:19-48): the same Graph /
gspmm / gsddmm / update_all / apply_edges / edge_softmax surface, backed by
hand-written sm_100a CUDA kernels in libgmp.so (include/gmp.h) called through
ctypes. Tensors live on the GPU; there is no CPU fallback.

Out of this package's scope: the reference's Tape/Var and
dense ops (torch autograd replaces them), the UDF bucketing path, neighbour
sampling, graph IO and the CLI bench.
"""

from .accounting import (AllocationMeter, MemoryCapExceeded, capture_dispatch,
                         track_allocations)
from .autodiff import GradBundle, gsddmm_backward, gspmm_backward
from .features import FeatureDict, as_feature_matrix, slice_rows
from .generators import (GenSpec, chain, constant_indegree, erdos_renyi, generate,
                         power_law, rmat)
from .graph import Adjacency, Graph, build_graph, from_arrays, reverse
from .kernels import (ArgExtrema, MessageFunc, builtin_message_funcs, force_strategy,
                      gsddmm, gspmm, select_format)
from .messaging import apply_edges, dst, edge, edge_softmax, msg, src, update_all
from . import layers

__version__ = "0.1.0"

__all__ = [
    "Adjacency", "AllocationMeter", "ArgExtrema", "FeatureDict", "GenSpec", "GradBundle",
    "Graph", "MemoryCapExceeded", "MessageFunc", "apply_edges", "as_feature_matrix",
    "build_graph", "builtin_message_funcs", "capture_dispatch", "chain", "constant_indegree",
    "dst", "edge", "edge_softmax", "erdos_renyi", "force_strategy", "from_arrays", "generate",
    "gsddmm", "gsddmm_backward", "gspmm", "gspmm_backward", "layers", "msg", "power_law",
    "reverse", "rmat", "select_format", "slice_rows", "src", "track_allocations",
    "update_all",
]
