"""Sparse convolution and linear layers on the RBGP4 product.

The reference represents convolutions only as an SDMM over an im2col'd input
(reference SPEC.md:9); here the im2col is never materialised.  A convolution
weight is a chain matrix with rows = output channels and columns in tap-major
im2col order, column = (i*kw + j)*c_in + c for conv weight[c_out, c, i, j], and
`sparse_conv2d` runs the implicit-im2col tcgen05 kernel (`rbgp4_conv2d`): each
pipeline step TMA-loads the tap-shifted NHWC window of the input directly
(out-of-bounds = zero padding).  Activations are NHWC bf16, outputs NHWC
(bf16 or f32), with an optional fused ReLU.

`SparseLinear` maps y = x W^T to the product's O = W x I with I = x^T.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .device import device_format, resolve_device, stream_handle, torch
from .errors import InvalidArgumentError, ShapeError, UnsupportedChainError
from .sdmm import make_desc, prepared, rbgp4mm, tiling_for_chain, workspace


def conv_weight_to_columns(weight: np.ndarray) -> np.ndarray:
    """(c_out, c_in, kh, kw) conv weight -> dense (c_out, kh*kw*c_in) in tap-major order."""
    c_out, c_in, kh, kw = weight.shape
    return np.ascontiguousarray(weight.transpose(0, 2, 3, 1).reshape(c_out, kh * kw * c_in))


def columns_to_conv_weight(dense: np.ndarray, c_in: int, kh: int, kw: int) -> np.ndarray:
    """Inverse of `conv_weight_to_columns`."""
    c_out = dense.shape[0]
    return np.ascontiguousarray(dense.reshape(c_out, kh, kw, c_in).transpose(0, 3, 1, 2))


def conv_out_hw(height: int, width: int, k: int, stride: int):
    """Output map of a 'same'-padded (pad = (k-1)/2) k x k convolution of stride 1 or 2."""
    pad = (k - 1) // 2
    return (height + 2 * pad - k) // stride + 1, (width + 2 * pad - k) // stride + 1


def sparse_conv2d(w, x, kernel_size: int = 3, *, stride: int = 1, relu: bool = False, out=None,
                  out_dtype=None, pool: bool = False, residual=None, relu_copy: bool = False):
    """NHWC conv of `x` (batch, H, W, c_in) with chain matrix `w`, 'same' padding, stride 1 or 2.

    Returns an NHWC (batch, H', W', c_out) CUDA tensor.  `x` must be a CUDA bf16 tensor
    (contiguous NHWC); the weight values are converted to bf16 once and cached.  Stride 2 is
    read by strided TMA boxes (every other input pixel); 1 x 1 kernels have no padding.
    pool=True also applies the 2x2 / stride-2 max pool (bf16 output (batch, H'/2, W'/2, c_out)):
    fused into the streamed kernel's epilogue where its pixel tiles hold whole windows, else
    the separate NHWC pool kernel.
    residual=R (an NHWC tensor shaped and typed like the output; relu and pool off) returns
    conv(x) + R, and relu_copy=True returns (conv(x) + R, relu(conv(x) + R)) -- the WRN block
    tail, fused into the streamed kernel's epilogue (`rbgp4_conv2d_residual`) and bit-identical to
    the conv followed by the torch add; shapes the streamed kernel does not take run the add
    separately.
    """
    t = torch()
    if w.chain.k != 4:
        raise UnsupportedChainError(f"sparse conv needs a 4-factor chain, got {w.chain.k}")
    if not (isinstance(x, t.Tensor) and x.is_cuda and x.dim() == 4):
        raise ShapeError("x must be a 4-D NHWC CUDA tensor")
    if x.dtype != t.bfloat16:
        raise ShapeError(f"x must be bf16, got {x.dtype}")
    batch, height, width, c_in = x.shape
    kh = kw = int(kernel_size)
    if w.cols != kh * kw * c_in:
        raise ShapeError(f"weight has {w.cols} columns, conv needs kh*kw*c_in = {kh * kw * c_in}")
    if kh % 2 != 1:
        raise InvalidArgumentError("only odd kernel sizes ('same' padding) are supported")
    if stride not in (1, 2):
        raise InvalidArgumentError(f"stride must be 1 or 2, got {stride}")
    x = x.contiguous()
    dev = resolve_device(x.device)
    res_dt = out_dtype if out_dtype is not None else t.bfloat16
    if res_dt not in (t.bfloat16, t.float32):
        raise InvalidArgumentError(f"conv writes bf16 or f32, got {res_dt}")
    oh, ow = conv_out_hw(height, width, kh, stride)
    if residual is not None:
        if relu or pool:
            raise InvalidArgumentError("residual=... adds before any ReLU / pool (relu and pool must be off)")
        if (not isinstance(residual, t.Tensor) or residual.device != x.device or residual.dtype != res_dt
                or tuple(residual.shape) != (batch, oh, ow, w.rows) or not residual.is_contiguous()):
            raise ShapeError(f"residual must be a contiguous NHWC ({batch}, {oh}, {ow}, {w.rows}) {res_dt} tensor "
                             f"on {x.device}")
    elif relu_copy:
        raise InvalidArgumentError("relu_copy=True needs residual=...")
    if pool:
        if res_dt != t.bfloat16 or oh % 2 or ow % 2:
            raise InvalidArgumentError("pool=True needs a bf16 output with an even output map")
        if out is not None:
            raise InvalidArgumentError("pool=True allocates its own output")
    with t.cuda.device(dev):
        fmt = device_format(w, dev, t.bfloat16)
        n_cols = batch * oh * ow
        desc = make_desc(fmt.desc_fields, n_cols, n_cols, n_cols)
        cv = _native.ConvDesc(batch, height, width, c_in, kh, kw, (kh - 1) // 2, stride,
                              int(bool(relu)) | (_native.CONV_POOL2 if pool else 0))
        if pool:
            res = t.empty((batch, oh // 2, ow // 2, w.rows), dtype=res_dt, device=dev)
        elif out is None:
            res = t.empty((batch, oh, ow, w.rows), dtype=res_dt, device=dev)
        else:
            res = out
            if (not isinstance(res, t.Tensor) or res.device != dev
                    or res.dtype not in (t.bfloat16, t.float32)
                    or tuple(res.shape) != (batch, oh, ow, w.rows) or not res.is_contiguous()):
                raise ShapeError(f"out must be a contiguous NHWC ({batch}, {oh}, {ow}, {w.rows}) bf16 or "
                                 f"f32 tensor on {dev}")
        res_relu = t.empty_like(res) if relu_copy else None
        if n_cols == 0:
            return (res, res_relu) if relu_copy else res
        lib = _native.lib()
        prep = prepared(fmt, "bf16", dev, desc)
        need = lib.rbgp4_conv2d_workspace_size(ctypes.byref(desc), ctypes.byref(cv))
        ws = workspace(dev, need, stream_handle(dev)) if need else None
        code = {t.bfloat16: _native.BF16, t.float32: _native.F32}[res.dtype]
        args = (fmt.values.data_ptr(), fmt.adj_o.data_ptr(), fmt.adj_i.data_ptr(),
                prep.data_ptr() if prep is not None else None, x.data_ptr())
        tail = (ws.data_ptr() if ws is not None else None, need, stream_handle(dev))
        if residual is not None:
            rc = lib.rbgp4_conv2d_residual(
                ctypes.byref(desc), ctypes.byref(cv), code, *args, residual.data_ptr(), res.data_ptr(),
                res_relu.data_ptr() if res_relu is not None else None, *tail)
            if rc == _native.EUNSUPPORTED:
                # no streamed plan for this shape: the conv, then the add on the device
                y = sparse_conv2d(w, x, kernel_size, stride=stride, out=res, out_dtype=res_dt)
                y.add_(residual)
                return (y, t.relu(y)) if relu_copy else y
            _native.check(rc, "rbgp4_conv2d_residual")
            return (res, res_relu) if relu_copy else res
        rc = lib.rbgp4_conv2d(ctypes.byref(desc), ctypes.byref(cv), code, *args, res.data_ptr(), *tail)
        if pool and rc == _native.EUNSUPPORTED:
            # no fused window layout for this shape: conv, then the NHWC pool kernel
            from .vgg import maxpool2x2
            return maxpool2x2(sparse_conv2d(w, x, kernel_size, stride=stride, relu=relu))
        _native.check(rc, "rbgp4_conv2d")
    return res


class SparseConv2d:
    """k x k 'same' convolution (stride 1 or 2) with an RBGP4-patterned weight (NHWC bf16)."""

    def __init__(self, w, kernel_size: int = 3, relu: bool = True, stride: int = 1):
        self.w, self.kernel_size, self.relu, self.stride = w, kernel_size, relu, stride

    def __call__(self, x, pool: bool = False):
        return sparse_conv2d(self.w, x, self.kernel_size, stride=self.stride, relu=self.relu, pool=pool)


class SparseLinear:
    """y = x W^T for a chain matrix W (out_features x in_features); x is (batch, in)."""

    def __init__(self, w, compute: str = "bf16"):
        self.w, self.compute = w, compute
        self.params = tiling_for_chain(w.chain, tn=1, rn=1, bn=1)

    def __call__(self, x):
        t = torch()
        xt = x.t().contiguous()
        if self.compute == "bf16" and xt.dtype != t.bfloat16:
            xt = xt.to(t.bfloat16)
        y, _ = rbgp4mm(self.w, xt, self.params, compute=self.compute)
        return y.t()
