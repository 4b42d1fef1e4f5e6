"""g-SpMM from host buffers with transfers overlapped tile by tile.

`gspmm_host` is the end-to-end entry point for features that live in host
memory (the reference's whole world is host memory: kernels.py:216 works on
NumPy arrays). A column tile of the output only needs the same column tile of
the source features (the row kernel's tiling, spmm_rows.cuh), so the work is
split into column tiles and pipelined over three CUDA streams:

    H2D copy of X[:, tile t+1]  |  row kernel on tile t  |  D2H copy of Z[:, tile t-1]

Each copy is one pitched 2-D DMA (cudaMemcpy2DAsync) of the tile's columns.
The kernel, the tiling and the numerics are exactly those of kernels.gspmm;
only the transfers overlap.
"""

import ctypes

import torch

from . import kernels

_cudart = None
_H2D, _D2H = 1, 2


def _rt():
    global _cudart
    if _cudart is None:
        lib = ctypes.CDLL("libcudart.so.12")
        lib.cudaMemcpy2DAsync.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                                          ctypes.c_size_t, ctypes.c_size_t, ctypes.c_size_t,
                                          ctypes.c_int, ctypes.c_void_p]
        lib.cudaMemcpy2DAsync.restype = ctypes.c_int
        _cudart = lib
    return _cudart


def _copy2d(dst, dpitch, src, spitch, width, height, kind, stream):
    rc = _rt().cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, kind,
                                 ctypes.c_void_p(stream.cuda_stream))
    if rc != 0:
        raise RuntimeError("cudaMemcpy2DAsync failed with %d" % rc)


def tile_bounds(d, elem_bytes, tile_bytes=256):
    """Column tiles of 256 B per row (64 fp32 / 32 fp64 columns) - the row
    kernel's packed tile width (kernels._gspmm_tiled)."""
    w = max(1, tile_bytes // elem_bytes)
    return [(c, min(d, c + w)) for c in range(0, d, w)], w


class HostPipeline:
    """Reusable device buffers and streams for repeated gspmm_host calls."""

    def __init__(self, device):
        self.device = torch.device(device)
        self.h2d = torch.cuda.Stream(self.device)
        self.d2h = torch.cuda.Stream(self.device)
        self.buffers = {}

    def buffer(self, name, shape, dtype, zero=False):
        b = self.buffers.get(name)
        if b is None or tuple(b.shape) != tuple(shape) or b.dtype != dtype:
            b = (torch.zeros if zero else torch.empty)(shape, dtype=dtype, device=self.device)
            self.buffers[name] = b
        return b


def gspmm_host(g, X_host, Z_host, rho="sum", pipe=None):
    """Z_host = gspmm(g, copy_lhs(src), rho, X_host) with pinned host X_host /
    Z_host (n, d), copies overlapped with the kernel per column tile.
    The H2D copy of tile t lands packed (n, 64) on the device - the aligned
    layout the row kernel gathers with 128-bit loads - and the D2H copy
    scatters the packed output tile back into Z_host's columns, so the tile
    packing costs no extra pass. Returns Z_host after the copies complete."""
    if rho not in ("sum", "mean"):
        raise ValueError("gspmm_host pipelines copy_u with sum / mean")
    if not (X_host.is_pinned() and Z_host.is_pinned()):
        raise ValueError("gspmm_host needs pinned host tensors")
    if X_host.dim() != 2 or not X_host.is_contiguous() or not Z_host.is_contiguous():
        raise ValueError("host tensors must be contiguous 2-D")
    n, d = X_host.shape
    if n != g.num_nodes or tuple(Z_host.shape) != (n, d) or Z_host.dtype != X_host.dtype:
        raise ValueError("X_host / Z_host must be (%d, d) of one dtype" % g.num_nodes)
    kernels._require_cuda(g)
    pipe = pipe or HostPipeline(g.device)
    comp = torch.cuda.current_stream(g.device)
    es = X_host.element_size()
    tiles, tw = tile_bounds(d, es)
    vec = max(1, 16 // es)
    # zero-initialised once: the pad columns of the last tile stay zero
    Xd = pipe.buffer("X", (len(tiles), n, tw), X_host.dtype, zero=True)
    Zd = pipe.buffer("Z", (len(tiles), n, tw), X_host.dtype)
    pitch = d * es
    h2d_done, comp_done = [], []
    pipe.h2d.wait_stream(comp)  # buffers are free once earlier work on comp is done
    for t, (c0, c1) in enumerate(tiles):
        with torch.cuda.stream(pipe.h2d):
            _copy2d(Xd[t].data_ptr(), tw * es, X_host.data_ptr() + c0 * es, pitch,
                    (c1 - c0) * es, n, _H2D, pipe.h2d)
            ev = torch.cuda.Event()
            ev.record(pipe.h2d)
            h2d_done.append(ev)
    phi = kernels.copy("src")
    for t, ((c0, c1), ev) in enumerate(zip(tiles, h2d_done)):
        comp.wait_event(ev)
        w = -(-(c1 - c0) // vec) * vec
        kernels._gspmm_launch(g, phi, rho, Xd[t][:, :w], None, None, w, out=Zd[t][:, :w])
        ce = torch.cuda.Event()
        ce.record(comp)
        comp_done.append(ce)
    for t, ((c0, c1), ce) in enumerate(zip(tiles, comp_done)):
        pipe.d2h.wait_event(ce)
        _copy2d(Z_host.data_ptr() + c0 * es, pitch, Zd[t].data_ptr(), tw * es,
                (c1 - c0) * es, n, _D2H, pipe.d2h)
    comp.wait_stream(pipe.d2h)
    return Z_host
