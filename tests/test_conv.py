"""Implicit-im2col sparse convolution vs an f64 im2col oracle (numpy, test-only)."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2006_13486_b200 as ks
from paper_2006_13486_b200 import conv
from paper_2006_13486_b200 import workloads as wl

from conftest import ring_graph


def conv_chain(c_out, c_in, k=3, sp_i=0.5, seed=0):
    """TC-friendly factorisation of a (c_out, k*k*c_in) conv weight: 128x128 tiles of 8x8
    blocks, G_o complete over the k*k*c_in/128 tap-channel blocks."""
    cfg = wl.SweepConfig("conv", (c_out // 128, k * k * c_in // 128), 0.0, (1, 1), (16, 16), sp_i,
                         (8, 8), n_cols=1, seed=seed)
    return wl.build_chain(cfg)


def im2col_nhwc(x, k, stride=1):
    """(B, H, W, C) -> (k*k*C, B*H'*W'), tap-major rows, 'same' zero padding, stride 1 or 2."""
    b, h, w, c = x.shape
    p = k // 2
    oh, ow = (h + 2 * p - k) // stride + 1, (w + 2 * p - k) // stride + 1
    xp = np.zeros((b, h + 2 * p, w + 2 * p, c), dtype=x.dtype)
    xp[:, p:p + h, p:p + w] = x
    rows = []
    for i in range(k):
        for j in range(k):
            rows.append(xp[:, i:i + stride * oh:stride, j:j + stride * ow:stride, :].reshape(b * oh * ow, c).T)
    return np.concatenate(rows, axis=0)


def test_weight_layout_round_trip():
    wgt = np.random.default_rng(0).standard_normal((8, 4, 3, 3))
    cols = conv.conv_weight_to_columns(wgt)
    assert cols.shape == (8, 36)
    assert np.array_equal(conv.columns_to_conv_weight(cols, 4, 3, 3), wgt)
    # tap-major: column (i*3+j)*c_in + c
    assert cols[5, (2 * 3 + 1) * 4 + 3] == wgt[5, 3, 2, 1]


def test_im2col_oracle_matches_direct_conv():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((2, 5, 4, 3))
    wgt = rng.standard_normal((6, 3, 3, 3))
    cols = conv.conv_weight_to_columns(wgt)
    got = (cols @ im2col_nhwc(x, 3)).T.reshape(2, 5, 4, 6)
    # direct loop conv, 'same' padding
    xp = np.pad(x, ((0, 0), (1, 1), (1, 1), (0, 0)))
    want = np.zeros((2, 5, 4, 6))
    for i in range(3):
        for j in range(3):
            want += np.einsum("bhwc,oc->bhwo", xp[:, i:i + 5, j:j + 4, :], wgt[:, :, i, j])
    assert np.allclose(got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("c_out,c_in,hw,batch", [(128, 128, 4, 2), (256, 128, 8, 3), (128, 256, 2, 5),
                                                 (128, 128, 16, 1)])
@pytest.mark.parametrize("relu", [False, True])
@pytest.mark.parametrize("persistent", [False, True])
def test_sparse_conv_matches_oracle(c_out, c_in, hw, batch, relu, persistent, plan_options):
    import torch
    if persistent:  # persistent tile loop (chosen by itself for many-wave grids)
        plan_options("persistent", 1)
        plan_options("relayout", 0)
    chain = conv_chain(c_out, c_in, seed=c_out + c_in + hw)
    w = ks.init_random(chain, 7, precision="f32")
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, (batch, hw, hw, c_in)).astype(np.float32)
    xb = torch.from_numpy(x).to(torch.bfloat16)
    got = conv.sparse_conv2d(w, xb.cuda(), 3, relu=relu, out_dtype=torch.float32).cpu().numpy()
    xr = xb.float().numpy().astype(np.float64)  # oracle sees the same bf16-rounded inputs
    w64 = ks.RcubsMatrix(chain, w.values.astype(np.float64))
    ref = oracle.reference_product(w64, np.ascontiguousarray(im2col_nhwc(xr, 3)), threads=8)
    ref = ref.T.reshape(batch, hw, hw, c_out)
    if relu:
        ref = np.maximum(ref, 0)
    err = oracle.rel_l2(got, ref)
    assert err < 1e-2, err


@pytest.mark.gpu
def test_sparse_linear_matches_oracle():
    import torch
    chain = conv_chain(128, 128, k=1, seed=5)  # (128 x 128) weight
    w = ks.init_random(chain, 2, precision="f32")
    lin = conv.SparseLinear(w, compute="bf16")
    x = torch.randn(64, 128)
    y = lin(x.cuda()).float().cpu().numpy()
    xb = x.to(torch.bfloat16).float().numpy().astype(np.float64)
    want = (w.to_dense().astype(np.float64) @ xb.T).T
    assert oracle.rel_l2(y, want) < 1e-2


def test_im2col_oracle_stride2_matches_direct_conv():
    rng = np.random.default_rng(4)
    x = rng.standard_normal((2, 6, 8, 3))
    wgt = rng.standard_normal((5, 3, 3, 3))
    got = (conv.conv_weight_to_columns(wgt) @ im2col_nhwc(x, 3, 2)).T.reshape(2, 3, 4, 5)
    xp = np.pad(x, ((0, 0), (1, 1), (1, 1), (0, 0)))
    want = np.zeros((2, 3, 4, 5))
    for i in range(3):
        for j in range(3):
            want += np.einsum("bhwc,oc->bhwo", xp[:, i:i + 6:2, j:j + 8:2, :], wgt[:, :, i, j])
    assert np.allclose(got, want)
    assert conv.conv_out_hw(32, 32, 3, 2) == (16, 16) and conv.conv_out_hw(32, 32, 1, 2) == (16, 16)


STRIDED = [  # (c_out, c_in, k, stride, hw, batch, g_b)
    (128, 128, 3, 2, 16, 2, (8, 8)), (128, 128, 1, 1, 8, 2, (8, 8)), (128, 128, 1, 2, 16, 4, (8, 8)),
    (128, 128, 3, 2, 16, 2, (16, 16)), (128, 128, 1, 2, 8, 16, (16, 16)), (256, 128, 3, 2, 32, 1, (16, 16)),
]


@pytest.mark.gpu
@pytest.mark.parametrize("c_out,c_in,k,stride,hw,batch,g_b", STRIDED)
def test_strided_and_pointwise_conv_match_oracle(c_out, c_in, k, stride, hw, batch, g_b):
    import torch
    v_o = k * k * c_in // 128
    g_i = (128 // g_b[0], 128 // g_b[1])
    cfg = wl.SweepConfig("sconv", (c_out // 128, v_o), 0.0, (1, 1), g_i, 0.75 if g_b == (16, 16) else 0.5,
                         g_b, n_cols=1, seed=c_out + k + stride + hw)
    chain = wl.build_chain(cfg)
    w = ks.init_random(chain, 9, precision="f32")
    x = np.random.default_rng(5).uniform(-1, 1, (batch, hw, hw, c_in)).astype(np.float32)
    xb = torch.from_numpy(x).to(torch.bfloat16)
    got = conv.sparse_conv2d(w, xb.cuda(), k, stride=stride, out_dtype=torch.float32).cpu().numpy()
    oh = (hw + 2 * (k // 2) - k) // stride + 1
    w64 = ks.RcubsMatrix(chain, torch.from_numpy(w.values.astype(np.float32)).to(torch.bfloat16)
                         .double().numpy())
    ref = oracle.reference_product(w64, np.ascontiguousarray(im2col_nhwc(xb.float().numpy().astype(np.float64),
                                                                          k, stride)), threads=8)
    ref = ref.T.reshape(batch, oh, oh, c_out)
    assert got.shape == ref.shape
    assert oracle.rel_l2(got, ref) < 1e-5



@pytest.mark.gpu
def test_sparse_conv_out_checked_before_launch():
    """A caller-provided `out` on the wrong device or of an unsupported dtype is refused with
    ShapeError before its pointer reaches the TMA-store kernel."""
    import torch
    chain = conv_chain(128, 128, seed=3)
    w = ks.init_random(chain, 7, precision="f32")
    x = torch.zeros((2, 4, 4, 128), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ks.ShapeError):
        conv.sparse_conv2d(w, x, 3, out=torch.empty((2, 4, 4, 128), dtype=torch.bfloat16))
    with pytest.raises(ks.ShapeError):
        conv.sparse_conv2d(w, x, 3, out=torch.empty((2, 4, 4, 128), dtype=torch.float16, device="cuda"))
