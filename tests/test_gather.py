"""K4, the gathered-block tcgen05 kernel (no densification), vs the f64 oracle.

Taken for compute="bf16" when the dense element blocks g_b are >= 16 x 16 (g_r = (1,1)).
Bar: rel-L2 <= 1e-2 against the f64 oracle on the same bf16-rounded operands (north star),
plus agreement with the densify kernel (K2, option dense=1) on the same inputs.
Covers: the VGG TC16 factorisation, split-K clusters (small N), f32 outputs, 32 x 32 blocks
(two K=16 MMAs per block), 64-row tile-rows, and the implicit-im2col convolution.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2006_13486_b200 as ks
from paper_2006_13486_b200 import _native, conv
from paper_2006_13486_b200 import workloads as wl

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def chain_of(g_o, sp_o, g_i, sp_i, g_b, seed=0):
    cfg = wl.SweepConfig("k4", g_o, sp_o, (1, 1), g_i, sp_i, g_b, n_cols=1, seed=seed)
    return wl.build_chain(cfg)


def run(w, x, compute="bf16", out_dtype=None, dense=False, relayout=False, persistent=False, msplit=False,
        direct=False, rl_persistent=False, rl_split=False):
    """dense: force K2 (densify); relayout: K4 on the prepared column-block relayout for any
    shape (by itself only where its immediate-offset loop applies, e.g. the VGG TC16 shape);
    direct / persistent / msplit: K4 on the compressed values as stored (no relayout).

    The prepared buffer is cached per matrix and its layout follows the mode, so non-default
    modes run on a fresh RcubsMatrix copy."""
    p = ks.tiling_for_chain(w.chain, tn=1, rn=1, bn=1)
    opt = {"stream": 0}  # K4 itself (K5 would take the prepared TC16 shape; tests/test_stream.py)
    if dense:
        opt["dense"] = 1
    if relayout:
        opt["relayout"] = 1
    if direct or persistent or msplit:
        opt["relayout"] = 0
    if rl_split:  # the TC16 relayout in the one-tile-per-CTA kernel (split-K clusters)
        opt["persistent"] = 0
    if relayout or direct or persistent or msplit or rl_persistent or rl_split:
        w = ks.RcubsMatrix(w.chain, np.array(w.values))
    if persistent or rl_persistent:  # rl_persistent: the persistent kernel on the TC16 relayout
        opt["persistent"] = 1
    if msplit:
        opt["msplit"] = 1
    with _native.options(**opt):
        y, _ = ks.rbgp4mm(w, x, p, compute=compute, out_dtype=out_dtype)
        torch.cuda.synchronize()
    return y.float().cpu().numpy()


def f64_ref(w, xb):
    w64 = ks.RcubsMatrix(w.chain, w.values.astype(np.float32).astype(np.float64))
    wb = torch.from_numpy(w.values.astype(np.float32)).to(torch.bfloat16).double().numpy()
    w64 = ks.RcubsMatrix(w.chain, wb)
    return oracle.reference_product(w64, xb.astype(np.float64), threads=8)


CASES = [
    # (g_o, sp_o, g_i, sp_i, g_b, n_cols)
    ((4, 36), 0.5, (8, 8), 0.75, (16, 16), 512),    # VGG conv10 TC16 shape, 4 column tiles
    ((4, 18), 0.5, (8, 8), 0.75, (16, 16), 128),    # one column tile: split-K cluster of 8
    ((4, 36), 0.5, (8, 8), 0.5, (16, 16), 384),     # 75 %: d_t = 64 (128-byte W rows)
    ((2, 8), 0.0, (4, 4), 0.5, (32, 32), 256),      # 32 x 32 blocks: 2 MMAs per block
    ((8, 16), 0.5, (4, 4), 0.5, (16, 16), 640),     # 64-row tile-rows (TMEM 64 columns)
    ((4, 12), 0.5, (8, 8), 0.75, (16, 16), 320),    # ragged last column tile (2.5 x 128)
]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}-{c[2]}-{c[4]}-n{c[5]}" for c in CASES])
def test_gather_sdmm_matches_oracle(case):
    g_o, sp_o, g_i, sp_i, g_b, n = case
    chain = chain_of(g_o, sp_o, g_i, sp_i, g_b, seed=n)
    w = ks.init_random(chain, 3, precision="f32")
    rng = np.random.default_rng(n)
    x = torch.from_numpy(rng.uniform(-1, 1, (w.cols, n)).astype(np.float32)).to(torch.bfloat16)
    ref = f64_ref(w, x.float().numpy())
    got = run(w, x.cuda())
    err = oracle.rel_l2(got, ref)
    assert err < 1e-2, err
    # output rounding is the only bf16 error left: the products are exact in fp32
    assert err < 4e-3, err
    dense = run(w, x.cuda(), dense=True)
    assert oracle.rel_l2(got, dense) < 4e-3
    relaid = run(w, x.cuda(), relayout=True)
    assert oracle.rel_l2(relaid, ref) < 4e-3
    direct = run(w, x.cuda(), direct=True)
    assert oracle.rel_l2(direct, ref) < 4e-3
    # persistent tile loop (taken by itself only for many-wave grids; forced here)
    pers = run(w, x.cuda(), persistent=True)
    assert oracle.rel_l2(pers, ref) < 4e-3
    pers_rl = run(w, x.cuda(), rl_persistent=True)
    assert oracle.rel_l2(pers_rl, ref) < 4e-3
    split_rl = run(w, x.cuda(), rl_split=True)
    assert oracle.rel_l2(split_rl, ref) < 4e-3
    # M-split (two row halves per tile, multicast slabs; taken by itself near half a wave)
    if w.chain.graphs[2].num_left % 2 == 0:
        ms = run(w, x.cuda(), msplit=True)
        assert oracle.rel_l2(ms, ref) < 4e-3


def test_gather_f32_output_and_host_tensors():
    chain = chain_of((4, 36), 0.5, (8, 8), 0.75, (16, 16), seed=9)
    w = ks.init_random(chain, 5, precision="f32")
    x = torch.from_numpy(np.random.default_rng(2).uniform(-1, 1, (w.cols, 256)).astype(np.float32))
    xb = x.to(torch.bfloat16)
    ref = f64_ref(w, xb.float().numpy())
    got = run(w, xb.cuda(), out_dtype=torch.float32)
    # f32 out: fp32 accumulation over exact bf16 products
    assert oracle.rel_l2(got, ref) < 1e-5
    host = run(w, xb.pin_memory())
    assert oracle.rel_l2(host, ref) < 4e-3


def test_gather_deterministic():
    chain = chain_of((4, 18), 0.5, (8, 8), 0.75, (16, 16), seed=4)
    w = ks.init_random(chain, 1, precision="f32")
    x = torch.rand((w.cols, 128), device="cuda").to(torch.bfloat16)
    a, b = run(w, x), run(w, x)
    assert np.array_equal(a, b)


CONV_CASES = [(128, 128, 4, 9), (256, 128, 8, 3), (128, 256, 16, 1), (128, 128, 2, 40),
              (128, 128, 32, 1)]


@pytest.mark.parametrize("c_out,c_in,hw,batch", CONV_CASES)
@pytest.mark.parametrize("relu", [False, True])
@pytest.mark.parametrize("mode", ["default", "direct", "persistent", "persistent_rl", "split_rl", "msplit"])
def test_gather_conv_matches_oracle(c_out, c_in, hw, batch, relu, mode):
    from test_conv import im2col_nhwc
    cfg = wl.SweepConfig("conv16", (c_out // 128, 9 * c_in // 128), 0.0, (1, 1), (8, 8), 0.75,
                         (16, 16), n_cols=1, seed=c_out + c_in + hw)
    chain = wl.build_chain(cfg)
    w = ks.init_random(chain, 7, precision="f32")
    x = np.random.default_rng(3).uniform(-1, 1, (batch, hw, hw, c_in)).astype(np.float32)
    xb = torch.from_numpy(x).to(torch.bfloat16)
    # default: the TC16 relayout (immediate-offset MMA loop); the other modes run on the
    # compressed values as stored
    opt = {"persistent": dict(persistent=1, relayout=0), "msplit": dict(msplit=1, relayout=0),
           "direct": dict(relayout=0), "persistent_rl": dict(persistent=1),
           "split_rl": dict(persistent=0)}.get(mode, {})
    with _native.options(**opt):
        got = conv.sparse_conv2d(w, xb.cuda(), 3, relu=relu, out_dtype=torch.float32).cpu().numpy()
    ref = f64_ref(w, np.ascontiguousarray(im2col_nhwc(xb.float().numpy(), 3)))
    ref = ref.T.reshape(batch, hw, hw, c_out)
    if relu:
        ref = np.maximum(ref, 0)
    assert oracle.rel_l2(got, ref) < 1e-5


def test_gather_persistent_many_waves():
    """A grid of 512 tiles (4 tile-rows x 128 column blocks) takes the persistent loop."""
    chain = chain_of((4, 4), 0.5, (8, 8), 0.75, (16, 16), seed=21)
    w = ks.init_random(chain, 6, precision="f32")
    x = torch.from_numpy(np.random.default_rng(8).uniform(-1, 1, (w.cols, 16384)).astype(np.float32))
    xb = x.to(torch.bfloat16)
    ref = f64_ref(w, xb.float().numpy())
    got = run(w, xb.cuda())
    assert oracle.rel_l2(got, ref) < 4e-3
    got32 = run(w, xb.cuda(), out_dtype=torch.float32)
    assert oracle.rel_l2(got32, ref) < 1e-5
    direct = run(w, xb.cuda(), direct=True)  # the persistent loop on the values as stored
    assert oracle.rel_l2(direct, ref) < 4e-3


def test_gather_persistent_ragged_last_tile():
    """Persistent loop on the TC16 relayout with a half-filled last column tile (N = 128k + 64)."""
    chain = chain_of((4, 4), 0.5, (8, 8), 0.75, (16, 16), seed=22)
    w = ks.init_random(chain, 7, precision="f32")
    n = 128 * 160 + 64
    x = torch.from_numpy(np.random.default_rng(9).uniform(-1, 1, (w.cols, n)).astype(np.float32))
    xb = x.to(torch.bfloat16)
    ref = f64_ref(w, xb.float().numpy())
    got = run(w, xb.cuda())
    assert oracle.rel_l2(got, ref) < 4e-3
    assert oracle.rel_l2(got[:, -64:], ref[:, -64:]) < 4e-3

