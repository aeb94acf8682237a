"""Training direction of the RBGP4 product (the paper trains with fixed
masks).  For O = W x I with W an RBGP4 chain matrix:

* input gradient   dI = W^T x dO  -- W^T is itself an RBGP4 chain matrix: the chain of the
  transposed factors (a Kronecker product of transposes; biregular factors stay biregular)
  with the values permuted into its sorted-column order.  It runs on the same product kernels.
* weight gradient  dW = (dO x I^T) restricted to the pattern -- `rbgp4_sddmm`, returned in the
  (rows, row_nnz) layout of RcubsMatrix.values, so the gradient never leaves the succinct format.

`SparseLinearFunction` wires both into torch.autograd for a layer y = x W^T whose values are a
trainable fp32 / fp64 tensor (the pattern stays fixed).

compute="bf16" runs all three products on the tensor cores: the forward and W^T x dO on the
streamed / gathered kernels (K5 / K4) of the bf16 values (fp32 master values cast per step; the
layer owns its prepared buffers and refreshes only their value copies, `rbgp4_prepare_values`),
and dW on K7 (`rbgp4_sddmm` with bf16 operands, fp32 gradient), fp32 accumulation throughout.
The forward and W^T x dO take the nn.Linear layout as it is: x (N x in) is an NHWC tensor of N
one-pixel images, so the product is a 1 x 1 streamed convolution whose NHWC output is y (N x out)
-- no transposes (`_PatternBF16.product_nk`; shapes the streamed conv does not take fall back to
the product on transposed operands); dW reads dO^T and I^T as MN-major operands (`sddmm_nk`).
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


def sddmm_nk(w, d_out_nk, inp_nk):
    """The bf16 pattern gradient from batch-major operands (the nn.Linear layout): d_out_nk
    (N, rows) = dO^T and inp_nk (N, cols) = I^T, bf16 CUDA tensors with unit column stride; K7
    reads them as MN-major MMA operands (`rbgp4_sddmm_nk`) -- bit-identical to
    sddmm(w, d_out_nk.t(), inp_nk.t()) without the transposed copies.  Returns (rows, row_nnz) f32."""
    t = torch()
    if w.chain.k != 4:
        raise InvalidArgumentError("sddmm needs a four-factor chain")
    if d_out_nk.dim() != 2 or inp_nk.dim() != 2 or d_out_nk.shape[1] != w.rows or inp_nk.shape[1] != w.cols \
            or d_out_nk.shape[0] != inp_nk.shape[0]:
        raise ShapeError(f"sddmm_nk: d_out {tuple(d_out_nk.shape)} / inp {tuple(inp_nk.shape)} do not match "
                         f"W^T ({w.cols} x {w.rows})")
    if d_out_nk.dtype != t.bfloat16 or inp_nk.dtype != t.bfloat16:
        raise ShapeError("sddmm_nk: bf16 operands")
    dev = resolve_device(d_out_nk.device)
    d_out_nk = d_out_nk if d_out_nk.stride(1) == 1 else d_out_nk.contiguous()
    inp_nk = inp_nk if inp_nk.stride(1) == 1 else inp_nk.contiguous()
    fmt = device_format(w, dev, t.bfloat16)
    res = t.empty((w.rows, w.row_nnz), dtype=t.float32, device=dev)
    n = d_out_nk.shape[0]
    desc = make_desc(fmt.desc_fields, n, n, n)
    _native.check(_native.lib().rbgp4_sddmm_nk(
        ctypes.byref(desc), fmt.adj_o.data_ptr(), fmt.adj_i.data_ptr(), d_out_nk.data_ptr(), d_out_nk.stride(0),
        inp_nk.data_ptr(), inp_nk.stride(0), res.data_ptr(), stream_handle(dev)), "rbgp4_sddmm_nk")
    return res


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
    if d_out.dtype != inp.dtype or d_out.dtype not in (t.float32, t.float64, t.bfloat16):
        raise ShapeError("sddmm: d_out and inp must share an f32 / f64 / bf16 dtype")
    dev = resolve_device(d_out.device)
    d_out = d_out if d_out.stride(1) == 1 else d_out.contiguous()
    inp = inp if inp.stride(1) == 1 else inp.contiguous()
    fmt = device_format(w, dev, d_out.dtype)
    # bf16 operands: tensor cores, f32 gradient
    gdt = t.float32 if d_out.dtype == t.bfloat16 else d_out.dtype
    res = values_out if values_out is not None else t.empty((w.rows, w.row_nnz), dtype=gdt, device=dev)
    if res.dtype != gdt or tuple(res.shape) != (w.rows, w.row_nnz) or not res.is_contiguous() or res.device != dev:
        raise ShapeError(f"sddmm: values_out must be a contiguous ({w.rows}, {w.row_nnz}) {gdt} tensor on {dev}")
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


class _PatternBF16:
    """Fixed pattern of a bf16 (tensor-core) trainable layer: device formats of W and W^T, and
    prepared buffers OWNED by the layer (their relayout copies follow the trainable values; the
    matrix's shared cached buffers are never mutated)."""

    def __init__(self, w, device):
        t = torch()
        self.w, self.wt = w, transpose(w)
        self.perm = t.from_numpy(transpose_permutation(w)).to(device)
        self.fmt = device_format(w, device, t.bfloat16)
        self.fmt_t = device_format(self.wt, device, t.bfloat16)
        self._prep = {}

    def _prepared(self, fmt, values, desc, device, stream):
        """The layer's prepared buffer for `fmt` (built once; its value copies refreshed from
        `values` on every later call -- they follow the trainable values)."""
        t = torch()
        lib = _native.lib()
        code = _native.COMPUTE["bf16"]
        nbytes = lib.rbgp4_prepare_size(ctypes.byref(desc), code)
        prep = None
        if nbytes:
            key = (id(fmt), nbytes)
            prep = self._prep.get(key)
            if prep is None:
                prep = t.empty(nbytes, dtype=t.uint8, device=device)
                _native.check(lib.rbgp4_prepare(ctypes.byref(desc), code, values.data_ptr(), fmt.adj_o.data_ptr(),
                                                fmt.adj_i.data_ptr(), prep.data_ptr(), nbytes, stream),
                              "rbgp4_prepare")
                self._prep[key] = prep
            else:
                _native.check(lib.rbgp4_prepare_values(ctypes.byref(desc), code, values.data_ptr(),
                                                       prep.data_ptr(), nbytes, stream), "rbgp4_prepare_values")
        return prep

    def product_nk(self, fmt, values, inp_nk, out_dtype):
        """The same product with both operands in the nn.Linear layout: inp_nk (N x cols) bf16 in,
        (N x rows) out -- the chain as a 1 x 1 convolution over N one-pixel images (NHWC = row
        major), so neither the input nor the output is transposed.  None when the streamed conv
        does not take the shape (the caller then uses `product` on transposed operands)."""
        t = torch()
        lib = _native.lib()
        n, cols = inp_nk.shape
        rows = fmt.desc_fields["rows"]
        if n == 0 or cols % 64 or inp_nk.data_ptr() % 16:
            return None
        out = t.empty((n, rows), dtype=out_dtype, device=inp_nk.device)
        desc = make_desc(fmt.desc_fields, n, n, n)
        cv = _native.ConvDesc(n, 1, 1, cols, 1, 1, 0, 1, 0)
        stream = stream_handle(inp_nk.device)
        prep = self._prepared(fmt, values, desc, inp_nk.device, stream)
        need = lib.rbgp4_conv2d_workspace_size(ctypes.byref(desc), ctypes.byref(cv))
        from .sdmm import workspace
        ws = workspace(inp_nk.device, need, stream) if need else None
        rc = lib.rbgp4_conv2d(ctypes.byref(desc), ctypes.byref(cv), dtype_code(out_dtype), values.data_ptr(),
                              fmt.adj_o.data_ptr(), fmt.adj_i.data_ptr(), prep.data_ptr() if prep is not None else None,
                              inp_nk.data_ptr(), out.data_ptr(), ws.data_ptr() if ws is not None else None, need,
                              stream)
        if rc == _native.EUNSUPPORTED:
            return None
        _native.check(rc, "rbgp4_conv2d (1 x 1, trainable layer)")
        return out

    def product(self, fmt, values, inp, out_dtype):
        """O = W x I on the tensor cores with the given bf16 values (the layer's own prep)."""
        t = torch()
        lib = _native.lib()
        out = t.empty((fmt.desc_fields["rows"], inp.shape[1]), dtype=out_dtype, device=inp.device)
        if inp.shape[1] == 0:
            return out
        desc = make_desc(fmt.desc_fields, inp.shape[1], inp.stride(0), out.stride(0))
        code = _native.COMPUTE["bf16"]
        stream = stream_handle(inp.device)
        prep = self._prepared(fmt, values, desc, inp.device, stream)
        need = lib.rbgp4_workspace_size(ctypes.byref(desc), code, _native.BF16)
        from .sdmm import workspace
        ws = workspace(inp.device, need, stream) if need else None
        _native.check(lib.rbgp4_sdmm_prepared(
            ctypes.byref(desc), code, _native.BF16, dtype_code(out_dtype), values.data_ptr(), fmt.adj_o.data_ptr(),
            fmt.adj_i.data_ptr(), prep.data_ptr() if prep is not None else None, inp.data_ptr(), out.data_ptr(),
            ws.data_ptr() if ws is not None else None, need, stream), "rbgp4_sdmm(compute=bf16)")
        return out


def make_sparse_linear_function_bf16():
    t = torch()

    class SparseLinearBF16(t.autograd.Function):
        """y = x W^T on the tensor cores: bf16 operands, fp32 accumulation, fp32 outputs and
        gradients; W = (pattern, fp32 master values)."""

        @staticmethod
        def forward(ctx, x, values, pattern):
            vb = values.detach().to(t.bfloat16).contiguous()
            xb = x.detach().to(t.bfloat16).contiguous()           # (N x in), no transpose
            ctx.save_for_backward(xb, vb)
            ctx.pattern = pattern
            # y (N x out) straight from the N-major operand (the 1 x 1 conv view); else the
            # product on transposed operands
            y = pattern.product_nk(pattern.fmt, vb, xb, t.float32)
            return y if y is not None else pattern.product(pattern.fmt, vb, xb.t().contiguous(), t.float32).t()

        @staticmethod
        def backward(ctx, dy):
            xb, vb = ctx.saved_tensors
            pat = ctx.pattern
            dyb = dy.to(t.bfloat16).contiguous()                  # dO^T (N x out), bf16
            grad_x = grad_v = None
            if ctx.needs_input_grad[0]:
                vt = vb.reshape(-1)[pat.perm].reshape(pat.wt.rows, pat.wt.row_nnz).contiguous()
                grad_x = pat.product_nk(pat.fmt_t, vt, dyb, t.float32)    # (W^T dO)^T, N x in
                if grad_x is None:
                    grad_x = pat.product(pat.fmt_t, vt, dyb.t().contiguous(), t.float32).t()
            if ctx.needs_input_grad[1]:
                # K7 on the batch-major operands as they are (MN-major MMA operands), f32
                grad_v = sddmm_nk(pat.w, dyb, xb)
            return grad_x, grad_v, None

    return SparseLinearBF16


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
    """y = x W^T with a fixed RBGP4 pattern and trainable stored values.

    compute "exact" / "ffma": SIMT kernels in the values' dtype (fp32 or fp64).  compute "bf16":
    tensor cores (K5/K4 products, K7 gradient) with fp32 master values, bf16 operands, fp32
    accumulation and fp32 outputs / gradients."""

    def __init__(self, w, device="cuda", compute="ffma"):
        t = torch()
        if compute not in ("exact", "ffma", "bf16"):
            raise InvalidArgumentError("trainable layer computes in 'exact', 'ffma' (f32 / f64) or 'bf16'")
        dev = resolve_device(device)
        self.compute = compute
        if compute == "bf16":
            self.pattern = _PatternBF16(w, dev)
            self.values = t.nn.Parameter(t.from_numpy(np.asarray(w.values, dtype=np.float32)).to(dev))
            self._fn = make_sparse_linear_function_bf16()
        else:
            self.pattern = _Pattern(w, dev)
            self.values = t.nn.Parameter(t.from_numpy(np.array(w.values)).to(dev))
            self._fn = make_sparse_linear_function()

    def __call__(self, x):
        if self.compute == "bf16":
            return self._fn.apply(x, self.values, self.pattern)
        return self._fn.apply(x, self.values, self.pattern, self.compute)
