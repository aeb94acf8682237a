"""WideResNet-40-4 for CIFAR-10 with RBGP4-sparse convolutions -- inference (BASELINE config 3).

Pre-activation WRN (depth 40 -> 6 blocks per group, widen 4 -> widths 64 / 128 / 256; groups
at 32x32, 16x16 (stride 2), 8x8 (stride 2)).  The paper's setup: the first
convolution and the classifier stay dense, every other convolution -- 36 3x3 and 3 1x1
shortcuts -- is RBGP4 sparse.  Batch norm is folded away and biases are omitted (synthetic,
random-init weights), so a block is

    o = relu(x);  y = conv3x3(o, stride s) -> relu;  y = conv3x3(y);  x = y + shortcut(o | x)

Two compute paths over the same RcubsMatrix weights:

* ``compute="bf16"`` -- NHWC bf16 activations; layers with >= 64 input channels run the
  implicit-im2col tcgen05 convolution (``sparse_conv2d``, stride 1 or 2, ReLU fused); the two
  16-input-channel layers of the first block run the tcgen05 SDMM on a materialised im2col;
* ``compute="ffma"`` -- fp32 activations, every sparse layer as im2col + the FFMA SIMT kernel
  (``rbgp4mm(compute="ffma")``), the reference's fp32 arithmetic on the GPU.

The block tail -- the residual add and the next block's pre-activation ReLU -- is written by
conv_b's epilogue (``sparse_conv2d(residual=..., relu_copy=True)`` on the streamed kernel, or the
im2col path's transpose ``rbgp4_nc_to_nhwc_residual``), bit-identical to the unfused torch ops
(``forward(fuse=False)``); the final pooling is plain torch.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .conv import columns_to_conv_weight, conv_out_hw, sparse_conv2d
from . import _native
from .device import stream_handle, torch
from .errors import GenerationExhaustedError, InvalidArgumentError, ShapeError
from .rcubs import init_random
from .sdmm import rbgp4mm, tiling_for_chain
from .vgg import _factor
from .graphs import complete_graph
from .products import RbgpChain

WIDTHS = (64, 128, 256)
STRIDES = (1, 2, 2)
BLOCKS = 6


def wrn_layer_chain(c_out: int, c_in: int, sparsity: float, k: int, seed: int = 0) -> RbgpChain:
    """RBGP4 chain of a (c_out, k*k*c_in) conv weight, tap-major columns.

    Tiles are up to 128 x 128 (128 x 64 when c_in = 64, a whole tap of c_in when c_in < 64);
    g_o takes 50 % when it has >= 4 tile-rows, g_i the rest, with the widest dense g_b block
    (16, 8, 4, 2, 1) the split allows -- every factor a certified Ramanujan lift chain.
    """
    tm = min(128, c_out)
    tk = 128 if c_in % 128 == 0 else 64 if c_in % 64 == 0 else c_in
    if c_out % tm or (k * k * c_in) % tk:
        raise InvalidArgumentError(f"unsupported conv shape {c_out}x{c_in}")
    u_o, v_o = c_out // tm, k * k * c_in // tk
    sp_o = 0.5 if u_o >= 4 else 0.0
    sp_i = 1.0 - (1.0 - sparsity) / (1.0 - sp_o)
    last = None
    for b in (16, 8, 4, 2, 1):
        if tm % b or tk % b:
            continue
        u_i, v_i = tm // b, tk // b
        d_i, d_r = v_i * (1 - sp_i), u_i * (1 - sp_i)
        if d_i < 2 or d_r < 2 or abs(d_i - round(d_i)) > 1e-9 or abs(d_r - round(d_r)) > 1e-9:
            continue
        try:
            return RbgpChain((_factor((u_o, v_o), sp_o, seed), complete_graph(1, 1),
                              _factor((u_i, v_i), sp_i, seed + 1), complete_graph(b, b)))
        except GenerationExhaustedError as exc:
            last = exc
    raise InvalidArgumentError(f"no RBGP4 factorisation for {c_out}x{c_in}x{k}x{k} at {sparsity}: {last}")


def im2col(x_nhwc, k: int, stride: int):
    """(B, H, W, C) -> (k*k*C, B*H'*W') in tap-major row order (the chain's column order).

    One pass of the library's NHWC im2col kernel (`rbgp4_im2col_nhwc`: 32 x 32 shared-memory
    transposes, zero padding); torch's pad / stack / permute / contiguous chain cost ~3 ms per
    64-channel 32x32 layer at batch 512 against 0.42 ms for the product itself.
    """
    t = torch()
    b, h, w, c = x_nhwc.shape
    oh, ow = conv_out_hw(h, w, k, stride)
    x_nhwc = x_nhwc.contiguous()
    cols = t.empty((k * k * c, b * oh * ow), dtype=x_nhwc.dtype, device=x_nhwc.device)
    code = {t.float32: _native.F32, t.bfloat16: _native.BF16}[x_nhwc.dtype]
    _native.check(_native.lib().rbgp4_im2col_nhwc(code, x_nhwc.data_ptr(), cols.data_ptr(), b, h, w, c, k, stride,
                                                  stream_handle(x_nhwc.device)), "rbgp4_im2col_nhwc")
    return cols, (b, oh, ow)


def to_nhwc(y, b, oh, ow, relu: bool, residual=None, relu_copy: bool = False):
    """The product's (C, B*H'*W') output -> NHWC (B, H', W', C), ReLU fused (`rbgp4_nc_to_nhwc`).

    residual=R: returns y^T + R (the WRN block tail, `rbgp4_nc_to_nhwc_residual`, rounded like the
    unfused add); with relu_copy=True also relu(y^T + R) as a second tensor.
    """
    t = torch()
    out = t.empty((b, oh, ow, y.shape[0]), dtype=y.dtype, device=y.device)
    code = {t.float32: _native.F32, t.bfloat16: _native.BF16}[y.dtype]
    if residual is None:
        _native.check(_native.lib().rbgp4_nc_to_nhwc(code, y.data_ptr(), out.data_ptr(), y.shape[0], y.shape[1],
                                                     int(bool(relu)), stream_handle(y.device)), "rbgp4_nc_to_nhwc")
        return out
    if relu or residual.shape != out.shape or residual.dtype != y.dtype or not residual.is_contiguous():
        raise ShapeError("to_nhwc: residual must match the NHWC output (and relu must be off)")
    out_relu = t.empty_like(out) if relu_copy else None
    _native.check(_native.lib().rbgp4_nc_to_nhwc_residual(
        code, y.data_ptr(), residual.data_ptr(), out.data_ptr(), out_relu.data_ptr() if relu_copy else None,
        y.shape[0], y.shape[1], stream_handle(y.device)), "rbgp4_nc_to_nhwc_residual")
    return (out, out_relu) if relu_copy else out


@dataclass
class _Conv:
    w: object
    c_in: int
    c_out: int
    k: int
    stride: int


@dataclass
class WRN40_4Sparse:
    """Inference-only WideResNet-40-4 (CIFAR-10) with RBGP4 sparse convolutions."""

    sparsity: float = 0.875
    num_classes: int = 10
    seed: int = 0
    device: str = "cuda"

    def __post_init__(self):
        t = torch()
        gen = t.Generator().manual_seed(self.seed)
        self.conv1 = (t.randn(16, 3, 3, 3, generator=gen) * (2.0 / 27) ** 0.5).to(self.device)
        self.blocks = []  # (conv_a, conv_b, shortcut | None)
        idx, c_in = 0, 16

        def make(c_o, c_i, k, stride):
            nonlocal idx
            chain = wrn_layer_chain(c_o, c_i, self.sparsity, k, seed=self.seed * 1000 + 10 * idx)
            w = init_random(chain, self.seed * 1000 + 10 * idx + 5, precision="f32")
            idx += 1
            return _Conv(w, c_i, c_o, k, stride)

        for width, stride in zip(WIDTHS, STRIDES):
            for b in range(BLOCKS):
                s = stride if b == 0 else 1
                conv_a = make(width, c_in, 3, s)
                conv_b = make(width, width, 3, 1)
                short = make(width, c_in, 1, s) if (b == 0) else None
                self.blocks.append((conv_a, conv_b, short))
                c_in = width
        self.fc = (t.randn(self.num_classes, 256, generator=gen) / 16.0).to(self.device)

    @property
    def sparse_convs(self):
        return [c for blk in self.blocks for c in blk if c is not None]

    # ---------------------------------------------------------------- one sparse layer
    def _conv(self, layer: _Conv, x, relu: bool, compute: str, residual=None):
        """One RBGP4 conv; with residual=R it returns (conv(x) + R, relu(conv(x) + R)): the block's
        sum and the ReLU the next block starts with, both written by the same epilogue."""
        if compute == "bf16" and layer.c_in % 64 == 0:
            return sparse_conv2d(layer.w, x, layer.k, stride=layer.stride, relu=relu, residual=residual,
                                 relu_copy=residual is not None)
        # materialised im2col + the product kernel (tcgen05 bf16 or SIMT fp32 FFMA)
        cols, (b, oh, ow) = im2col(x, layer.k, layer.stride)
        params = tiling_for_chain(layer.w.chain, tn=1, rn=1, bn=1)
        y, _ = rbgp4mm(layer.w, cols, params, compute=compute)
        return to_nhwc(y, b, oh, ow, relu, residual=residual, relu_copy=residual is not None)

    def forward(self, x_nhwc, compute: str = "bf16", fuse: bool = True):
        """x: (batch, 32, 32, 3) CUDA tensor -> (batch, num_classes) logits.

        fuse=True (default): every block's residual add and the next block's ReLU are written by
        conv_b's epilogue; fuse=False runs them as separate torch ops (bit-identical results).
        """
        t = torch()
        if compute not in ("bf16", "ffma"):
            raise InvalidArgumentError(f"compute must be 'bf16' or 'ffma', got {compute!r}")
        act_dt = t.bfloat16 if compute == "bf16" else t.float32
        x = t.nn.functional.conv2d(x_nhwc.permute(0, 3, 1, 2).float(), self.conv1, padding=1)
        x = x.permute(0, 2, 3, 1).contiguous().to(act_dt)
        o = t.relu(x)
        for conv_a, conv_b, short in self.blocks:
            if not fuse:
                o = t.relu(x)
            y = self._conv(conv_a, o, True, compute)
            r = self._conv(short, o, False, compute) if short is not None else x
            if fuse:
                x, o = self._conv(conv_b, y, False, compute, residual=r)
            else:
                x = self._conv(conv_b, y, False, compute) + r
        x = (o if fuse else t.relu(x)).float().mean(dim=(1, 2))
        return x @ self.fc.t()

    __call__ = forward

    def reference_forward(self, x_nhwc, round_bf16: bool = False):
        """Same network with dense fp32 weights via torch convolutions (test oracle); with
        round_bf16 the weights and every conv input are rounded to bf16 like the bf16 path."""
        t = torch()
        rb = (lambda v: v.to(t.bfloat16).float()) if round_bf16 else (lambda v: v)
        x = t.nn.functional.conv2d(x_nhwc.permute(0, 3, 1, 2).float(), self.conv1, padding=1)
        x = rb(x)

        def conv(layer, v):
            dense = layer.w.to_dense().astype(np.float32)
            wgt = t.from_numpy(columns_to_conv_weight(dense, layer.c_in, layer.k, layer.k)).to(v.device)
            return t.nn.functional.conv2d(rb(v), rb(wgt), padding=(layer.k - 1) // 2, stride=layer.stride)

        for conv_a, conv_b, short in self.blocks:
            o = t.relu(x)
            y = rb(t.relu(conv(conv_a, o)))
            y = rb(conv(conv_b, y))
            x = y + (rb(conv(short, o)) if short is not None else x)
            x = rb(x)
        x = t.relu(x).mean(dim=(2, 3))
        return x @ self.fc.t()

    def compulsory_bytes(self, batch: int, elt: int) -> float:
        """Roofline bytes of the 39 RBGP4 convolutions: each layer reads its input activation
        (batch * H * W * c_in) and its stored values once and writes its output once, in the
        activation element size `elt` (implicit im2col: no 9x inflation)."""
        total, hw = 0.0, 32
        for conv_a, conv_b, short in self.blocks:
            out = hw // conv_a.stride
            for layer, h_in in ((conv_a, hw), (conv_b, out), (short, hw)):
                if layer is not None:
                    total += elt * (batch * h_in * h_in * layer.c_in + layer.w.nnz
                                    + batch * out * out * layer.c_out)
            hw = out
        return total

    def sparse_flops(self, batch: int) -> float:
        """2 * nnz * output pixels over the 39 RBGP4 convolutions (the BASELINE metric)."""
        total, hw = 0.0, 32
        for conv_a, conv_b, short in self.blocks:
            out = hw // conv_a.stride
            for layer in (conv_a, conv_b, short):
                if layer is not None:
                    total += 2.0 * layer.w.nnz * batch * out * out
            hw = out
        return total
