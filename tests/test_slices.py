"""K5 on the slice relayout (csrc/sdmm_stream.cu) vs the f64 oracle: SDMM and implicit-im2col
convolution for element blocks narrower than 16 (the 8 x 8 / 4 x 4 blocks of the small-channel
VGG19 layers) and the TC16 convolution.

The slice relayout cuts a step's K range into K16 slices and multiplies each by the union of
the tile rows with a nonzero there (zero-padded to the MMA N); every output row sums at most
two partials.  Bar: rel-L2 <= 1e-2 with bf16 outputs (the output rounding is ~2e-3), <= 1e-5
with f32 outputs, against the f64 oracle on the same bf16-rounded operands (north star), and
the launch is the K5 kernel (rbgp4_last_kernel).  Shapes the slices cannot take (more than two
partials per row: g_i degree 8 with 8 x 8 blocks) still run, on the densify kernel K2.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2006_13486_b200 as ks
from paper_2006_13486_b200 import _native, conv
from paper_2006_13486_b200 import workloads as wl
from paper_2006_13486_b200.vgg import layer_chain

from test_conv import im2col_nhwc

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16)


def _w64(w):
    wb = _bf16(np.asarray(w.values, dtype=np.float32)).double().numpy()
    return ks.RcubsMatrix(w.chain, wb)


SDMM_CASES = [
    # (g_o, sp_o, g_i, sp_i, g_b, n_cols, kernel, what)
    ((4, 36), 0.5, (16, 16), 0.875, (8, 8), 4096, "K5 stream", "8x8 blocks, 128x128 tiles (VGG conv3-8 shape)"),
    ((4, 36), 0.5, (16, 16), 0.875, (8, 8), 1024, "K5 stream", "8x8 blocks, fewer tiles than SMs"),
    ((1, 9), 0.0, (16, 16), 0.875, (4, 4), 4096, "K5 stream", "4x4 blocks, 64x64 tiles (VGG conv0 shape)"),
    ((1, 9), 0.0, (32, 16), 0.875, (4, 4), 2048, "K5 stream", "4x4 blocks, 128x64 tiles, N = 64 slices"),
    ((2, 18), 0.0, (16, 16), 0.875, (8, 8), 65536, "K5 stream", "persistent, merged tile-row pairs (g_o complete)"),
    ((4, 18), 0.0, (8, 8), 0.75, (16, 16), 8192, "K5 stream", "TC16 with g_o complete: merged pairs, N = 64"),
    ((2, 9), 0.0, (16, 16), 0.875, (8, 8), 1024, "K5 stream", "merged pairs, one unit per CTA"),
    ((2, 9), 0.0, (16, 16), 0.875, (8, 8), 4160, "K5 stream", "merged pairs, ragged last column tile (N % 128 = 64)"),
    ((4, 36), 0.5, (16, 16), 0.875, (8, 8), 4160, "K5 stream", "8x8 slices, ragged last column tile"),
    ((4, 36), 0.5, (16, 16), 0.75, (8, 8), 4096, "K5 stream", "g_i degree 4 (8x8 blocks): four partials, N = 64"),
    ((2, 18), 0.0, (8, 8), 0.5, (16, 16), 8192, "K5 stream", "TC16 blocks, g_i degree 4 (50 %): four partials"),
    ((4, 36), 0.5, (16, 16), 0.5, (8, 8), 1024, "K2 tc", "g_i degree 8: too many partials -> densify K2"),
]


@pytest.mark.parametrize("g_o,sp_o,g_i,sp_i,g_b,n,kernel,what", SDMM_CASES, ids=[c[-1] for c in SDMM_CASES])
@pytest.mark.parametrize("out_dtype", ["bf16", "f32"])
def test_slice_sdmm_matches_oracle(g_o, sp_o, g_i, sp_i, g_b, n, kernel, what, out_dtype):
    cfg = wl.SweepConfig("slice", g_o, sp_o, (1, 1), g_i, sp_i, g_b, n_cols=n, seed=11)
    chain = wl.build_chain(cfg)
    rng = ks.make_rng(5)
    w = ks.init_random(chain, rng, precision="f32")
    x = rng.uniform(-1.0, 1.0, size=(w.cols, n)).astype(np.float32)
    xb = _bf16(x)
    p = ks.tiling_for_chain(chain, tn=1, rn=1, bn=1)
    odt = torch.bfloat16 if out_dtype == "bf16" else torch.float32
    y, _ = ks.rbgp4mm(w, xb.cuda(), p, compute="bf16", out_dtype=odt)
    torch.cuda.synchronize()
    assert _native.last_kernel() == kernel, (what, _native.last_kernel())
    got = y.float().cpu().numpy()
    # columns are independent (reference sdmm.py:167): sample 512 spread over every column tile
    cols = np.unique(np.linspace(0, n - 1, min(n, 512)).astype(int))
    ref = oracle.reference_product(_w64(w), np.ascontiguousarray(xb.double().numpy()[:, cols]), threads=8)
    tol = 1e-2 if out_dtype == "bf16" else 1e-5
    assert _rel(got[:, cols], ref) <= tol, what


@pytest.mark.parametrize("g_i,sp_i,g_b", [((8, 8), 0.75, (16, 16)), ((16, 16), 0.875, (8, 8))])
def test_merged_pairs_match_unmerged(g_i, sp_i, g_b):
    """Tile-row merging (option merge) changes only which MMA computes a partial: f32 outputs
    agree with the unmerged kernel to fp32 rounding."""
    cfg = wl.SweepConfig("merge", (2, 18), 0.0, (1, 1), g_i, sp_i, g_b, n_cols=4096, seed=21)
    chain = wl.build_chain(cfg)
    rng = ks.make_rng(4)
    w = ks.init_random(chain, rng, precision="f32")
    xb = _bf16(rng.uniform(-1.0, 1.0, size=(w.cols, 4096))).cuda()
    p = ks.tiling_for_chain(chain, tn=1, rn=1, bn=1)
    a, _ = ks.rbgp4mm(w, xb, p, compute="bf16", out_dtype=torch.float32)
    with _native.options(merge=0):
        b, _ = ks.rbgp4mm(w, xb, p, compute="bf16", out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert _rel(a.cpu().numpy(), b.cpu().numpy()) < 1e-6


def test_slice_sdmm_deterministic():
    cfg = wl.SweepConfig("slice", (4, 36), 0.5, (1, 1), (16, 16), 0.875, (8, 8), n_cols=4096, seed=3)
    chain = wl.build_chain(cfg)
    rng = ks.make_rng(9)
    w = ks.init_random(chain, rng, precision="f32")
    xb = _bf16(rng.uniform(-1.0, 1.0, size=(w.cols, 4096))).cuda()
    p = ks.tiling_for_chain(chain, tn=1, rn=1, bn=1)
    a, _ = ks.rbgp4mm(w, xb, p, compute="bf16", out_dtype=torch.float32)
    b, _ = ks.rbgp4mm(w, xb, p, compute="bf16", out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


CONV_CASES = [
    # (c_out, c_in, hw, batch, stride, kernel, what)
    (64, 64, 32, 2, 1, "K5 halo", "VGG conv0: 4x4 blocks, 64x64 tiles, halo strips"),
    (128, 64, 16, 3, 1, "K5 halo", "VGG conv2: 4x4 blocks, N = 64 slices, halo strips"),
    (128, 128, 16, 2, 1, "K5 halo", "VGG conv3: 8x8 blocks, halo strips"),
    (64, 64, 16, 3, 1, "K5 halo", "one strip column per image row (16 x 16 map, 64 channels)"),
    (256, 128, 8, 5, 1, "K5 conv", "VGG conv5: two images per tile"),
    (512, 256, 4, 16, 1, "K5 conv", "VGG conv10: TC16, eight images per tile"),
    (512, 512, 2, 64, 1, "K5 conv", "VGG conv15: TC16, 32 images per tile"),
    (128, 64, 32, 2, 2, "K5 conv", "stride 2 (WRN group transition)"),
]


@pytest.mark.parametrize("c_out,c_in,hw,batch,stride,kernel,what", CONV_CASES, ids=[c[-1] for c in CONV_CASES])
@pytest.mark.parametrize("relu", [False, True])
@pytest.mark.parametrize("out_dtype", ["bf16", "f32"])
def test_slice_conv_matches_oracle(c_out, c_in, hw, batch, stride, kernel, what, relu, out_dtype):
    _conv_case(c_out, c_in, hw, batch, stride, kernel, what, relu, out_dtype)


@pytest.mark.parametrize("c_out,c_in,hw,batch,stride,kernel,what", CONV_CASES[:4], ids=[c[-1] for c in CONV_CASES[:4]])
def test_tap_conv_matches_oracle(c_out, c_in, hw, batch, stride, kernel, what):
    """The same layers with the halo strips off (option halo=0): tap-shifted boxes per step."""
    with _native.options(halo=0):
        _conv_case(c_out, c_in, hw, batch, stride, "K5 conv", what, True, "bf16")


def _conv_case(c_out, c_in, hw, batch, stride, kernel, what, relu, out_dtype):
    chain = layer_chain(c_out, c_in, 0.875, seed=c_out + c_in + hw)
    w = ks.init_random(chain, 7, precision="f32")
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, (batch, hw, hw, c_in)).astype(np.float32)
    xb = _bf16(x)
    odt = torch.bfloat16 if out_dtype == "bf16" else torch.float32
    got = conv.sparse_conv2d(w, xb.cuda(), 3, stride=stride, relu=relu, out_dtype=odt)
    torch.cuda.synchronize()
    assert _native.last_kernel() == kernel, (what, _native.last_kernel())
    got = got.float().cpu().numpy()
    xr = xb.double().numpy()
    cols_i = im2col_nhwc(xr, 3, stride)
    ref = oracle.reference_product(_w64(w), np.ascontiguousarray(cols_i), threads=8)
    oh = (hw + 2 - 3) // stride + 1
    ref = ref.T.reshape(batch, oh, oh, c_out)
    if relu:
        ref = np.maximum(ref, 0.0)
    tol = 1e-2 if out_dtype == "bf16" else 1e-5
    assert _rel(got, ref) <= tol, what


POOL_CASES = [
    # (c_out, c_in, hw, batch, kernel)
    (64, 64, 32, 2, "K5 halo+pool"),      # VGG conv0 -> pool1 (halo strips: window rows ^8)
    (128, 128, 16, 2, "K5 halo+pool"),    # VGG conv3 -> pool4
    (256, 256, 8, 5, "K5 conv+pool"),     # VGG conv8 -> pool9 (two images per tile: rows ^8)
    (512, 512, 4, 16, "K5 conv+pool"),    # VGG conv13 -> pool14 (rows ^4)
    (512, 512, 2, 64, "K5 conv+pool"),    # VGG conv18 -> pool19 (one window per image)
    (256, 64, 32, 2, "K5 conv"),          # 32-wide non-halo map: no fused layout, separate pool
]


@pytest.mark.parametrize("c_out,c_in,hw,batch,kernel", POOL_CASES, ids=[f"{c[0]}x{c[1]}@{c[2]}" for c in POOL_CASES])
def test_fused_pool_is_conv_then_pool(c_out, c_in, hw, batch, kernel):
    """conv + ReLU + 2x2 max pool in one epilogue == the conv followed by the NHWC pool kernel,
    bit for bit (rounding to bf16 is monotonic, so max and rounding commute)."""
    from paper_2006_13486_b200.vgg import maxpool2x2
    chain = layer_chain(c_out, c_in, 0.875, seed=c_out + 3 * c_in + hw)
    w = ks.init_random(chain, 9, precision="f32")
    x = _bf16(np.random.default_rng(4).uniform(-1, 1, (batch, hw, hw, c_in))).cuda()
    fused = conv.sparse_conv2d(w, x, 3, relu=True, pool=True)
    torch.cuda.synchronize()
    got_kernel = _native.last_kernel()
    ref = maxpool2x2(conv.sparse_conv2d(w, x, 3, relu=True))
    torch.cuda.synchronize()
    assert fused.shape == (batch, hw // 2, hw // 2, c_out)
    assert got_kernel == kernel, got_kernel
    assert torch.equal(fused, ref)
