"""Graph and feature files, loaded straight into device tensors.

Same formats and function names as the reference's graphio
(/root/reference/pkg/src/graphmp/graphio.py:1-170), so a dataset written by
either side loads in the other:

* edge-list text: one ``u<TAB>v`` per line, 0-based ids, ``#`` comments, an
  optional ``nodes=N`` line pins the node count (else max id + 1);
* ``GRF1`` binary graph: magic, little-endian u64 num_nodes, u64 num_edges,
  then src[m] and dst[m] as u32 (graphio.py:58-79);
* dense features: headerless CSV, or ``FMX1`` binary: magic, u64 rows,
  u64 cols, f64 row-major (graphio.py:82-113);
* loss curves: CSV ``epoch,loss``.

The binary readers map the file (np.memmap: no parse, no Python loop) and copy
it to the device once through pinned host memory; the id arrays land as the
int32 device tensors the kernels use, the feature matrix as fp32 by default
(dtype=torch.float64 keeps the file's precision). Validation errors carry the
reference's messages (bad magic, truncated arrays, malformed lines).
"""

import csv
import struct

import numpy as np
import torch

from .graph import Graph, default_device

GRAPH_MAGIC = b"GRF1"
MATRIX_MAGIC = b"FMX1"
_HEADER = struct.Struct("<4sQQ")


def _to_device(arr, device, dtype):
    host = torch.from_numpy(np.ascontiguousarray(arr))
    if device.type == "cuda":
        host = host.pin_memory()
    return host.to(device=device, dtype=dtype, non_blocking=device.type == "cuda")


def _header(path, magic):
    with open(path, "rb") as f:
        raw = f.read(_HEADER.size)
    if len(raw) < 4 or raw[:4] != magic:
        raise ValueError("%s: bad magic %r, expected %r" % (path, raw[:4], magic))
    if len(raw) < _HEADER.size:
        raise ValueError("%s: truncated header" % path)
    _, a, b = _HEADER.unpack(raw)
    return a, b


def read_graph_binary(path, device=None):
    """GRF1 file -> Graph on `device` (default: cuda when present)."""
    device = torch.device(device) if device is not None else default_device()
    n, m = _header(path, GRAPH_MAGIC)
    body = np.memmap(path, dtype="<u4", mode="c", offset=_HEADER.size) if m else \
        np.zeros(0, dtype="<u4")
    if body.size < 2 * m:
        raise ValueError("%s: truncated edge arrays" % path)
    ids = _to_device(body[:2 * m].view(np.int32), device, torch.int32)
    return Graph(ids[:m], ids[m:], int(n), device=device)


def write_graph_binary(path, g):
    s, d = g.src.cpu().numpy(), g.dst.cpu().numpy()
    with open(path, "wb") as f:
        f.write(_HEADER.pack(GRAPH_MAGIC, g.num_nodes, g.num_edges))
        f.write(s.astype("<u4").tobytes())
        f.write(d.astype("<u4").tobytes())


def read_features_binary(path, device=None, dtype=torch.float32):
    """FMX1 file -> (rows, cols) tensor on `device`."""
    device = torch.device(device) if device is not None else default_device()
    rows, cols = _header(path, MATRIX_MAGIC)
    body = np.memmap(path, dtype="<f8", mode="c", offset=_HEADER.size) if rows * cols else \
        np.zeros(0)
    if body.size < rows * cols:
        raise ValueError("%s: truncated matrix data" % path)
    mat = np.asarray(body[:rows * cols]).reshape(rows, cols)
    return _to_device(mat, device, torch.float64).to(dtype)


def write_features_binary(path, matrix):
    mat = _host_matrix(matrix)
    with open(path, "wb") as f:
        f.write(_HEADER.pack(MATRIX_MAGIC, mat.shape[0], mat.shape[1]))
        f.write(mat.astype("<f8").tobytes())


def _host_matrix(matrix):
    if isinstance(matrix, torch.Tensor):
        matrix = matrix.detach().cpu().numpy()
    mat = np.asarray(matrix, dtype=np.float64)
    if mat.ndim == 1:
        mat = mat.reshape(-1, 1)
    if mat.ndim != 2:
        raise ValueError("feature matrix must be 1-D or 2-D")
    return mat


def read_edge_list(path, device=None):
    """Text edge list -> Graph (node count from a ``nodes=N`` line, else max id + 1)."""
    device = torch.device(device) if device is not None else default_device()
    pairs = []
    num_nodes = None
    with open(path) as f:
        for lineno, raw in enumerate(f, 1):
            line = raw.partition("#")[0].strip()
            if not line:
                continue
            if line.startswith("nodes="):
                num_nodes = int(line[6:])
                continue
            tok = line.split()
            if len(tok) != 2:
                raise ValueError("%s:%d: expected 'u<TAB>v', got %r" % (path, lineno, raw.rstrip()))
            pairs.append((int(tok[0]), int(tok[1])))
    e = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    if num_nodes is None:
        num_nodes = int(e.max()) + 1 if e.size else 0
    return Graph(e[:, 0], e[:, 1], num_nodes, device=device)


def write_edge_list(path, g, header=True):
    s, d = g.src.cpu().numpy(), g.dst.cpu().numpy()
    with open(path, "w") as f:
        if header:
            f.write("nodes=%d\n" % g.num_nodes)
        f.writelines("%d\t%d\n" % (u, v) for u, v in zip(s.tolist(), d.tolist()))


def read_features_csv(path, device=None, dtype=torch.float32):
    device = torch.device(device) if device is not None else default_device()
    with open(path) as f:
        rows = [[float(x) for x in r] for r in csv.reader(f) if r]
    mat = np.asarray(rows, dtype=np.float64)
    if mat.ndim == 1:
        mat = mat.reshape(-1, 1) if mat.size else mat.reshape(0, 0)
    return _to_device(mat, device, torch.float64).to(dtype)


def write_features_csv(path, matrix):
    mat = _host_matrix(matrix)
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        for row in mat:
            w.writerow([repr(float(x)) for x in row])


def write_loss_curve(path, losses):
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["epoch", "loss"])
        for i, v in enumerate(losses):
            w.writerow([i, repr(float(v))])


def read_loss_curve(path):
    with open(path) as f:
        r = csv.reader(f)
        next(r, None)
        return [float(row[1]) for row in r if row]
