"""VGG19 for CIFAR with RBGP4-sparse convolutions -- inference.

The paper's setup: every 3x3 convolution except the first is RBGP4
sparse; the first convolution and the classifier stay dense.  Here:

* sparse convs run `sparse_conv2d` (implicit-im2col tcgen05 kernel, NHWC bf16, ReLU fused);
* 2x2 max pooling runs `rbgp4_maxpool2x2_nhwc`;
* the dense first conv and the 512 -> classes classifier are plain library calls
  (cuDNN / cuBLAS through torch), as the reference's dense baseline is BLAS;
* batch norm is folded away and biases are omitted (synthetic, random-init weights).

Factorisations are chosen per layer (`layer_chain`): tiles of up to 128 x 128 built from
dense g_b = (b, b) element blocks (b = 16 when the sparsity split allows it -- whole MMA
operands for the gathered-block kernel -- else 8 / 4 / 2),
g_r = (1,1), g_o carrying up to 50 % when it has >= 4 tile-rows, g_i the rest.  Every factor
is a certified Ramanujan lift chain from the reference's generator.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .conv import SparseConv2d
from .device import stream_handle, torch
from .errors import GenerationExhaustedError, InvalidArgumentError
from .generate import LiftChainSpec, generate_ramanujan
from .graphs import complete_graph
from .products import RbgpChain
from .rcubs import init_random

#: VGG19 feature config (channels; "M" = 2x2 max pool)
VGG19 = [64, 64, "M", 128, 128, "M", 256, 256, 256, 256, "M", 512, 512, 512, 512, "M",
         512, 512, 512, 512, "M"]


def _factor(shape, sp, seed):
    if sp == 0.0:
        return complete_graph(*shape)
    return generate_ramanujan(LiftChainSpec(shape[0], shape[1], sp, rng_seed=seed, max_attempts=200)).graph


def layer_chain(c_out: int, c_in: int, sparsity: float, seed: int = 0, k: int = 3) -> RbgpChain:
    """A tensor-core-friendly RBGP4 chain for a (c_out, k*k*c_in) conv weight."""
    tm = min(128, c_out)
    tk = 128 if c_in % 128 == 0 else 64
    if c_in % tk or c_out % tm:
        raise InvalidArgumentError(f"unsupported conv shape {c_out}x{c_in}")
    u_o, v_o = c_out // tm, k * k * c_in // tk
    sp_o = 0.5 if u_o >= 4 else 0.0
    sp_i = 1.0 - (1.0 - sparsity) / (1.0 - sp_o)
    last = None
    for b in (16, 8, 4, 2):
        u_i, v_i = tm // b, tk // b
        d_i, d_r = v_i * (1 - sp_i), u_i * (1 - sp_i)
        if d_i < 2 or d_r < 2 or d_i != int(d_i) or d_r != int(d_r):
            continue
        try:
            return RbgpChain((_factor((u_o, v_o), sp_o, seed), complete_graph(1, 1),
                              _factor((u_i, v_i), sp_i, seed + 1), complete_graph(b, b)))
        except GenerationExhaustedError as exc:
            last = exc
    raise InvalidArgumentError(f"no RBGP4 factorisation for {c_out}x{c_in} at {sparsity}: {last}")


def _dense_conv_relu(x, w):
    """The dense first conv (3 -> 64, a library call as in the paper) with its ReLU fused by cuDNN
    (conv + separate relu_ measured 4.72 ms at batch 32768, fused 3.40 ms: the ReLU pass re-read
    and re-wrote the 4.3 GB activation)."""
    t = torch()
    fused = getattr(t.ops.aten, "cudnn_convolution_relu", None)
    if fused is not None and x.is_cuda:
        return fused(x, w, None, [1, 1], [1, 1], [1, 1], 1)
    return t.nn.functional.conv2d(x, w, padding=1).relu_()


def dense_conv1_relu(x_nhwc, w_cols):
    """The dense first conv (3 -> 64, 3x3 'same') with its ReLU on the library's own tcgen05 kernel
    (`rbgp4_dense_conv3x3_c3`, K8): NHWC bf16 in and out, w_cols the bf16 (64, 32) weight matrix
    from `conv1_columns`.  HBM-write-bound (4.3 GB out at batch 32768); cuDNN's fused conv + ReLU
    took 2.6-3.6 ms there."""
    t = torch()
    if not (x_nhwc.is_cuda and x_nhwc.dtype == t.bfloat16 and x_nhwc.dim() == 4 and x_nhwc.shape[3] == 3):
        raise InvalidArgumentError("dense_conv1_relu: x must be a CUDA bf16 NHWC tensor with 3 channels")
    x_nhwc = x_nhwc.contiguous()
    b, h, w, _ = x_nhwc.shape
    out = t.empty((b, h, w, w_cols.shape[0]), dtype=t.bfloat16, device=x_nhwc.device)
    _native.check(_native.lib().rbgp4_dense_conv3x3_c3(x_nhwc.data_ptr(), w_cols.data_ptr(), out.data_ptr(), b, h, w,
                                                       w_cols.shape[0], stream_handle(x_nhwc.device)),
                  "rbgp4_dense_conv3x3_c3")
    return out


def conv1_columns(weight):
    """(64, 3, 3, 3) conv weight -> the bf16 (64, 32) matrix K8 reads: column (i*3 + j)*3 + c, zeros
    past 27."""
    t = torch()
    c_out = weight.shape[0]
    cols = t.zeros((c_out, 32), dtype=t.bfloat16, device=weight.device)
    cols[:, :27] = weight.permute(0, 2, 3, 1).reshape(c_out, 27).to(t.bfloat16)
    return cols.contiguous()


def maxpool2x2(x):
    t = torch()
    b, h, w, c = x.shape
    y = t.empty((b, h // 2, w // 2, c), dtype=x.dtype, device=x.device)
    _native.check(_native.lib().rbgp4_maxpool2x2_nhwc(x.data_ptr(), y.data_ptr(), b, h, w, c,
                                                      stream_handle(x.device)), "rbgp4_maxpool2x2_nhwc")
    return y


@dataclass
class VGG19Sparse:
    """Inference-only VGG19-CIFAR with RBGP4 sparse convolutions (NHWC bf16 activations)."""

    sparsity: float = 0.875
    num_classes: int = 100
    seed: int = 0
    device: str = "cuda"

    def __post_init__(self):
        t = torch()
        gen = t.Generator().manual_seed(self.seed)
        # dense first conv (3 -> 64), channels-last bf16
        self.conv1 = (t.randn(64, 3, 3, 3, generator=gen) * (2.0 / 27) ** 0.5).to(
            self.device, t.bfloat16).to(memory_format=t.channels_last)
        self.conv1_cols = conv1_columns(self.conv1)
        self.layers = []   # ("conv", SparseConv2d) | ("pool", None)
        self.chains = []
        c_in, idx = 64, 0
        for v in VGG19[1:]:
            if v == "M":
                self.layers.append(("pool", None))
                continue
            chain = layer_chain(v, c_in, self.sparsity, seed=self.seed * 1000 + 10 * idx)
            w = init_random(chain, self.seed * 1000 + 10 * idx + 5, precision="f32")
            self.layers.append(("conv", SparseConv2d(w, 3, relu=True)))
            self.chains.append(chain)
            c_in, idx = v, idx + 1
        self.fc = (t.randn(self.num_classes, 512, generator=gen) / 512 ** 0.5).to(self.device, t.bfloat16)

    def forward(self, x_nhwc, dense: str = "native"):
        """x: (batch, 32, 32, 3) bf16 CUDA tensor -> (batch, num_classes) logits.

        dense: the first (dense) conv on the library's K8 kernel ("native") or cuDNN ("cudnn")."""
        t = torch()
        if dense == "native":
            x = dense_conv1_relu(x_nhwc, self.conv1_cols)
        else:
            x = x_nhwc.permute(0, 3, 1, 2)  # NCHW view of channels-last memory
            x = _dense_conv_relu(x, self.conv1)
            x = x.permute(0, 2, 3, 1).contiguous()  # NHWC (a view: cuDNN wrote channels-last)
        i = 0
        while i < len(self.layers):
            kind, layer = self.layers[i]
            if kind == "conv" and i + 1 < len(self.layers) and self.layers[i + 1][0] == "pool":
                x = layer(x, pool=True)  # conv + ReLU + 2x2 max pool in one epilogue
                i += 2
                continue
            x = maxpool2x2(x) if kind == "pool" else layer(x)
            i += 1
        return x.reshape(x.shape[0], -1) @ self.fc.t()

    __call__ = forward

    def reference_forward(self, x_nhwc):
        """Same network with dense fp32 weights via torch (test oracle for the float path)."""
        t = torch()
        from .conv import columns_to_conv_weight
        x = x_nhwc.permute(0, 3, 1, 2).float()
        x = t.nn.functional.conv2d(x, self.conv1.float(), padding=1).relu()
        c_in = 64
        for kind, layer in self.layers:
            if kind == "pool":
                x = t.nn.functional.max_pool2d(x, 2)
                continue
            dense = layer.w.to_dense().astype(np.float32)
            wgt = t.from_numpy(columns_to_conv_weight(dense, c_in, 3, 3)).to(x.device)
            # mirror the bf16 rounding of weights and activations of the product path
            wgt = wgt.to(t.bfloat16).float()
            x = t.nn.functional.conv2d(x.to(t.bfloat16).float(), wgt, padding=1).relu()
            c_in = layer.w.rows
        x = x.to(t.bfloat16).float().reshape(x.shape[0], -1)
        return x @ self.fc.float().t()

    @property
    def sparse_flops_per_image(self) -> float:
        """2 * nnz * pixels over the sparse convolutions (the RBGP4 metric)."""
        total, hw, i = 0.0, 32 * 32, 0
        for kind, layer in self.layers:
            if kind == "pool":
                hw //= 4
            else:
                total += 2.0 * layer.w.nnz * hw
        return total
