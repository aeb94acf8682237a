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


@pytest.mark.gpu
@pytest.mark.parametrize("c,hw,k,stride,out_dt,kern", [
    (64, 32, 3, 1, torch.bfloat16, "K5 halo+res"),    # WRN group 1 conv_b: halo strips
    (128, 16, 3, 1, torch.bfloat16, "K5 halo+res"),   # group 2
    (256, 8, 3, 1, torch.bfloat16, "K5 conv+res"),    # group 3: tap-shifted boxes (8x8 maps)
    (64, 32, 3, 1, torch.float32, "K5 halo"),         # f32 output: unfused fallback (conv, then add)
    (128, 16, 1, 1, torch.bfloat16, "K5 conv+res"),   # 1x1
])
def test_conv_residual_epilogue_bit_identical(c, hw, k, stride, out_dt, kern):
    """sparse_conv2d(residual=R, relu_copy=True) == (conv + R, relu(conv + R)) computed unfused (the
    conv, then the torch add), bit for bit: the epilogue rounds the conv, adds in f32 and rounds
    again exactly as the separate ops do."""
    from paper_2006_13486_b200 import _native
    from paper_2006_13486_b200.conv import sparse_conv2d
    from paper_2006_13486_b200.rcubs import init_random
    w = init_random(wrn_layer_chain(c, c, 0.875, k, seed=7), 3, precision="f32")
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(4, hw, hw, c, device="cuda", generator=g).to(torch.bfloat16)
    r = torch.randn(4, hw // stride, hw // stride, c, device="cuda", generator=g).to(out_dt)
    y, yr = sparse_conv2d(w, x, k, stride=stride, out_dtype=out_dt, residual=r, relu_copy=True)
    assert _native.last_kernel() == kern
    z = sparse_conv2d(w, x, k, stride=stride, out_dtype=out_dt)
    want = z + r
    torch.cuda.synchronize()
    assert torch.equal(y, want) and torch.equal(yr, want.relu())
    y2 = sparse_conv2d(w, x, k, stride=stride, out_dtype=out_dt, residual=r)  # no relu copy
    assert torch.equal(y2, want)


@pytest.mark.gpu
@pytest.mark.parametrize("compute", ["bf16", "ffma"])
def test_wrn_fused_block_tail_matches_unfused(compute):
    """The fused WRN forward (residual add + next ReLU in conv_b's epilogue) is bit-identical to the
    forward with separate torch ops."""
    from paper_2006_13486_b200.wrn import WRN40_4Sparse
    net = WRN40_4Sparse(sparsity=0.875, seed=4)
    g = torch.Generator(device="cuda").manual_seed(2)
    x = torch.randn(8, 32, 32, 3, device="cuda", generator=g)
    assert torch.equal(net(x, compute=compute, fuse=True), net(x, compute=compute, fuse=False))


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_transpose_residual_is_exact(dtype):
    """rbgp4_nc_to_nhwc_residual == transpose + torch add (+ relu copy), bit for bit."""
    from paper_2006_13486_b200 import wrn
    y = torch.randn(48, 2 * 6 * 5).to(dtype).cuda()
    r = torch.randn(2, 6, 5, 48).to(dtype).cuda()
    s, sr = wrn.to_nhwc(y, 2, 6, 5, relu=False, residual=r, relu_copy=True)
    want = y.t().reshape(2, 6, 5, 48) + r
    assert torch.equal(s, want) and torch.equal(sr, want.relu())


@pytest.mark.gpu
def test_conv_residual_argument_errors():
    """residual= with relu / pool, a mismatched residual, or relu_copy without a residual: the
    reference-style errors, before any device work."""
    from paper_2006_13486_b200.conv import sparse_conv2d
    from paper_2006_13486_b200.errors import InvalidArgumentError, ShapeError
    from paper_2006_13486_b200.rcubs import init_random
    w = init_random(wrn_layer_chain(64, 64, 0.875, 3, seed=1), 2, precision="f32")
    x = torch.randn(2, 8, 8, 64, device="cuda").to(torch.bfloat16)
    r = torch.randn(2, 8, 8, 64, device="cuda").to(torch.bfloat16)
    with pytest.raises(InvalidArgumentError):
        sparse_conv2d(w, x, 3, relu=True, residual=r)
    with pytest.raises(InvalidArgumentError):
        sparse_conv2d(w, x, 3, relu_copy=True)
    with pytest.raises(ShapeError):
        sparse_conv2d(w, x, 3, residual=r[:, :4])
    with pytest.raises(ShapeError):
        sparse_conv2d(w, x, 3, residual=r.float())
