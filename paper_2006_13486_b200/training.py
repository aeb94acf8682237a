"""Training direction of the RBGP4 product (the paper trains with fixed
masks).  For O = W x I with W an RBGP4 chain matrix:

* input gradient   dI = W^T x dO  -- W^T is itself an RBGP4 chain matrix: the chain of the
  transposed factors (a Kronecker product of transposes; biregular factors stay biregular)
  with the values permuted into its sorted-column order.  It runs on the same product kernels.
* weight gradient  dW = (dO x I^T) restricted to the pattern -- `rbgp4_sddmm`, returned in the
  (rows, row_nnz) layout of RcubsMatrix.values, so the gradient never leaves the succinct format.

`SparseLinearFunction` wires both into torch.autograd for a layer y = x W^T whose values are a
trainable fp32 / fp64 tensor (the pattern stays fixed).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .device import chain_fields, device_format, dtype_code, resolve_device, stream_handle, torch
from .errors import InvalidArgumentError, ShapeError
from .graphs import BipartiteGraph
from .products import RbgpChain
from .rcubs import RcubsMatrix
from .sdmm import make_desc


def transpose_graph(g: BipartiteGraph) -> BipartiteGraph:
    """The transposed bipartite graph: right vertices become left ones, neighbours sorted."""
    rows = [[] for _ in range(g.num_right)]
    for u, nbrs in enumerate(g.adjacency):
        for v in nbrs:
            rows[v].append(u)
    return BipartiteGraph(g.num_right, g.num_left, tuple(tuple(sorted(r)) for r in rows))


def transpose_permutation(w) -> np.ndarray:
    """perm with values_T.flat = values.flat[perm] (W^T's rows in sorted-column order)."""
    csr = w.to_unstructured()
    rows = np.repeat(np.arange(w.rows, dtype=np.int64), w.row_nnz)
    return np.lexsort((rows, csr.indices.astype(np.int64)))


def transpose(w) -> RcubsMatrix:
    """W^T as an RcubsMatrix of the transposed chain (exact: a permutation of the values)."""
    chain_t = RbgpChain(tuple(transpose_graph(g) for g in w.chain.graphs))
    vals = np.asarray(w.values).reshape(-1)[transpose_permutation(w)]
    return RcubsMatrix(chain_t, vals.reshape(chain_t.num_left, chain_t.row_nnz))


def sddmm(w, d_out, inp, values_out=None):
    """grad[u, j] = sum_n d_out[u, n] * inp[c(u, j), n] over W's stored slots (CUDA tensors).

    `w` supplies the pattern (its values are not read).  d_out is (rows, N), inp (cols, N), both
    f32 or f64 CUDA tensors with unit column stride; returns (rows, row_nnz) of the same dtype.
    """
    t = torch()
    if w.chain.k != 4:
        raise InvalidArgumentError("sddmm needs a four-factor chain")
    if d_out.dim() != 2 or inp.dim() != 2 or d_out.shape[0] != w.rows or inp.shape[0] != w.cols \
            or d_out.shape[1] != inp.shape[1]:
        raise ShapeError(f"sddmm: d_out {tuple(d_out.shape)} / inp {tuple(inp.shape)} do not match "
                         f"W ({w.rows} x {w.cols})")
    if d_out.dtype != inp.dtype or d_out.dtype not in (t.float32, t.float64):
        raise ShapeError("sddmm: d_out and inp must share an f32 / f64 dtype")
    dev = resolve_device(d_out.device)
    d_out = d_out if d_out.stride(1) == 1 else d_out.contiguous()
    inp = inp if inp.stride(1) == 1 else inp.contiguous()
    fmt = device_format(w, dev, d_out.dtype)
    res = values_out if values_out is not None else t.empty((w.rows, w.row_nnz), dtype=d_out.dtype, device=dev)
    desc = make_desc(fmt.desc_fields, d_out.shape[1], d_out.shape[1], d_out.shape[1])
    _native.check(_native.lib().rbgp4_sddmm(
        ctypes.byref(desc), dtype_code(d_out.dtype), fmt.adj_o.data_ptr(), fmt.adj_i.data_ptr(),
        d_out.data_ptr(), d_out.stride(0), inp.data_ptr(), inp.stride(0), res.data_ptr(),
        stream_handle(dev)), "rbgp4_sddmm")
    return res


class _Pattern:
    """Fixed pattern of a trainable layer: forward and transposed device formats (adjacency only)."""

    def __init__(self, w, device):
        t = torch()
        self.w, self.wt = w, transpose(w)
        self.perm = t.from_numpy(transpose_permutation(w)).to(device)
        self.fmt = device_format(w, device, t.float64 if w.dtype == np.float64 else t.float32)
        self.fmt_t = device_format(self.wt, device, self.fmt.values.dtype)


def _product(fmt, values, inp, compute):
    """O = W x I with W's values given as a device tensor (the trainable parameter).

    The kernel reads `values` and `inp` in ONE element type (rbgp4_sdmm's in_dtype), so a
    mismatch would reinterpret bytes; it is rejected here before any launch.
    """
    t = torch()
    if values.dtype != inp.dtype or values.dtype != fmt.values.dtype:
        raise ShapeError(f"sparse linear: activations ({inp.dtype}), values ({values.dtype}) and the "
                         f"pattern's format ({fmt.values.dtype}) must share one dtype")
    if values.device != inp.device:
        raise ShapeError(f"sparse linear: values on {values.device}, activations on {inp.device}")
    out = t.empty((fmt.desc_fields["rows"], inp.shape[1]), dtype=inp.dtype, device=inp.device)
    desc = make_desc(fmt.desc_fields, inp.shape[1], inp.stride(0), out.stride(0))
    code = dtype_code(inp.dtype)
    _native.check(_native.lib().rbgp4_sdmm(
        ctypes.byref(desc), _native.COMPUTE[compute], code, code, values.data_ptr(), fmt.adj_o.data_ptr(),
        fmt.adj_i.data_ptr(), inp.data_ptr(), out.data_ptr(), None, 0, stream_handle(inp.device)),
        f"rbgp4_sdmm(compute={compute})")
    return out


def make_sparse_linear_function():
    t = torch()

    class SparseLinearFunction(t.autograd.Function):
        """y = x W^T for W = (pattern, values); grads for x and for the stored values."""

        @staticmethod
        def forward(ctx, x, values, pattern, compute):
            xt = x.t().contiguous()
            ctx.save_for_backward(xt, values)
            ctx.pattern, ctx.compute = pattern, compute
            return _product(pattern.fmt, values.contiguous(), xt, compute).t()

        @staticmethod
        def backward(ctx, dy):
            xt, values = ctx.saved_tensors
            pat = ctx.pattern
            d_out = dy.t().contiguous()                       # dO (rows x N)
            grad_x = grad_v = None
            if ctx.needs_input_grad[0]:
                vals_t = values.reshape(-1)[pat.perm].reshape(pat.wt.rows, pat.wt.row_nnz).contiguous()
                grad_x = _product(pat.fmt_t, vals_t, d_out, ctx.compute).t()   # (W^T dO)^T
            if ctx.needs_input_grad[1]:
                grad_v = sddmm(pat.w, d_out, xt)
            return grad_x, grad_v, None, None

    return SparseLinearFunction


class TrainableSparseLinear:
    """y = x W^T with a fixed RBGP4 pattern and trainable stored values (fp32 or fp64)."""

    def __init__(self, w, device="cuda", compute="ffma"):
        t = torch()
        if compute not in ("exact", "ffma"):
            raise InvalidArgumentError("trainable layer computes in 'exact' or 'ffma' (f32 / f64)")
        dev = resolve_device(device)
        self.pattern = _Pattern(w, dev)
        self.values = t.nn.Parameter(t.from_numpy(np.array(w.values)).to(dev))
        self.compute = compute
        self._fn = make_sparse_linear_function()

    def __call__(self, x):
        return self._fn.apply(x, self.values, self.pattern, self.compute)
