"""WideResNet-40-4 RBGP4 inference (BASELINE config 3).

CPU: every one of the 39 sparse layers gets a certified factorisation at the paper's
sparsities; the torch im2col used for the 16-channel layers matches the numpy oracle's
tap-major order.  GPU: the bf16 tcgen05 forward matches a dense torch forward with the same
bf16 roundings, and the fp32 FFMA forward matches the dense fp32 torch forward.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2006_13486_b200.wrn import BLOCKS, STRIDES, WIDTHS, im2col, wrn_layer_chain

from test_conv import im2col_nhwc


@pytest.mark.parametrize("sparsity", [0.75, 0.875])
def test_layer_factorisations(sparsity):
    c_in, n = 16, 0
    for width, stride in zip(WIDTHS, STRIDES):
        for b in range(BLOCKS):
            for c_o, c_i, k in ((width, c_in, 3), (width, width, 3)) + (((width, c_in, 1),) if b == 0 else ()):
                chain = wrn_layer_chain(c_o, c_i, sparsity, k, seed=n)
                assert chain.num_left == c_o and chain.num_right == k * k * c_i
                assert abs(chain.sparsity - sparsity) < 1e-12
                assert chain.graphs[1].is_complete() and chain.graphs[3].is_complete()
                n += 1
            c_in = width
    assert n == 39


@pytest.mark.gpu
def test_wrn_forward_bf16_and_ffma():
    from paper_2006_13486_b200.wrn import WRN40_4Sparse
    net = WRN40_4Sparse(sparsity=0.875, seed=2)
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(4, 32, 32, 3, device="cuda", generator=g)
    y16 = net(x, compute="bf16").float()
    ref16 = net.reference_forward(x, round_bf16=True)
    assert y16.shape == (4, 10)
    assert float((y16 - ref16).norm() / ref16.norm()) < 3e-3  # measured 4.0e-4 / 6.3e-4 (seeds 2, 3)
    y32 = net(x, compute="ffma")
    tf32 = torch.backends.cudnn.allow_tf32
    torch.backends.cudnn.allow_tf32 = False  # the fp32 reference must not round to tf32
    try:
        ref32 = net.reference_forward(x)
    finally:
        torch.backends.cudnn.allow_tf32 = tf32
    assert float((y32 - ref32).norm() / ref32.norm()) < 1e-4


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("b,h,w,c,k,stride", [(2, 5, 7, 16, 3, 1), (3, 8, 8, 64, 3, 2), (2, 6, 6, 48, 1, 2),
                                              (1, 32, 32, 16, 3, 1)])
def test_native_im2col_and_transpose_are_exact(dtype, b, h, w, c, k, stride):
    """rbgp4_im2col_nhwc == the numpy im2col oracle and rbgp4_nc_to_nhwc == transpose + ReLU, bit for
    bit (pure data movement)."""
    import torch
    from test_conv import im2col_nhwc
    from paper_2006_13486_b200 import wrn
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    x = torch.randn(b, h, w, c).to(tdt)
    cols, (bb, oh, ow) = wrn.im2col(x.cuda(), k, stride)
    want = im2col_nhwc(x.float().numpy(), k, stride)
    assert cols.shape == want.shape and np.array_equal(cols.float().cpu().numpy(), want)
    y = torch.randn(24, bb * oh * ow).to(tdt)
    got = wrn.to_nhwc(y.cuda(), bb, oh, ow, relu=True).cpu()
    assert torch.equal(got, y.t().reshape(bb, oh, ow, 24).relu())
