"""K5, the streamed TC16 SDMM (csrc/sdmm_stream.cu), vs the f64 oracle.

K5 is the default for compute="bf16" on the prepared TC16 factorisation (g_r = (1,1),
g_i (8,8) of degree 2, g_b = (16,16)): whole 128 x 128 tiles in a persistent loop when the
tiles fill the SMs, row groups of G = 4 / 2 / 1 row blocks (16-row slab pieces) below that.
Bar: rel-L2 <= 1e-2 against the f64 oracle on the same bf16-rounded operands (north star;
~2e-3 is the bf16 output rounding), <= 1e-5 with f32 outputs; and K5 agrees with K4 (option
stream=0) on the same inputs.  Columns are independent (reference sdmm.py:167): the oracle
runs on a column sample covering every column tile when N is large.

Covers: one unit per CTA and the persistent multi-unit loop (double-buffered accumulator,
direct-store epilogue for all but the last unit), every row-group size, ragged last column
tile (N % 128 == 64), bf16 and f32 outputs.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2006_13486_b200 as ks
from paper_2006_13486_b200 import _native
from paper_2006_13486_b200 import workloads as wl

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _operands(g_o, n, seed):
    cfg = wl.SweepConfig("k5", g_o, 0.5, (1, 1), (8, 8), 0.75, (16, 16), n_cols=n, seed=seed)
    chain = wl.build_chain(cfg)
    rng = ks.make_rng(np.random.SeedSequence([seed, 1]).generate_state(1)[0])
    w = ks.init_random(chain, rng, precision="f32")
    x = rng.uniform(-1.0, 1.0, size=(w.cols, n)).astype(np.float32)
    return w, x


def _product(w, xb, out_dtype, **opt):
    p = ks.tiling_for_chain(w.chain, tn=1, rn=1, bn=1)
    with _native.options(**opt):
        y, _ = ks.rbgp4mm(w, xb.cuda(), p, compute="bf16", out_dtype=out_dtype)
        torch.cuda.synchronize()
    return y.float().cpu().numpy()


def _oracle(w, xb, cols):
    wb = torch.from_numpy(np.asarray(w.values, dtype=np.float32)).to(torch.bfloat16).double().numpy()
    return oracle.reference_product(ks.RcubsMatrix(w.chain, wb),
                                    np.ascontiguousarray(xb.double().numpy()[:, cols]), threads=8)


CASES = [
    # (g_o, n_cols, stream_g [0 = auto], what)
    ((4, 36), 4096, 0, "conv10: whole tiles, one unit per CTA"),
    ((4, 18), 4096, 0, "conv9: whole tiles"),
    ((4, 36), 1024, 0, "conv13: row groups of 2 (auto)"),
    ((4, 36), 2048, 0, "row groups of 4 (auto)"),
    ((4, 36), 256, 0, "row groups of 1 (auto)"),
    ((4, 36), 16384, 0, "whole tiles, persistent (4 units per CTA)"),
    ((4, 36), 4096, 2, "row groups of 2, persistent (4 units per CTA)"),
    ((4, 36), 1088, 0, "ragged last column tile, row groups"),
    ((4, 36), 4160, 8, "ragged last column tile, whole tiles, persistent"),
    ((8, 36), 2048, 8, "8 tile-rows, whole tiles, 128 units"),
]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0][0]}x{c[0][1]}-n{c[1]}-g{c[2]}" for c in CASES])
@pytest.mark.parametrize("out_dtype", ["bf16", "f32"])
def test_stream_matches_oracle(case, out_dtype):
    g_o, n, g, _ = case
    w, x = _operands(g_o, n, seed=n + g)
    xb = torch.from_numpy(x).to(torch.bfloat16)
    od = torch.bfloat16 if out_dtype == "bf16" else torch.float32
    opt = {"stream_g": g} if g else {}
    got = _product(w, xb, od, **opt)
    cols = np.unique(np.linspace(0, n - 1, min(n, 640)).astype(np.int64))
    ref = _oracle(w, xb, cols)
    err = oracle.rel_l2(got[:, cols], ref)
    assert err <= (1e-2 if out_dtype == "bf16" else 1e-5), err
    # every column written (the sample may miss a ragged tail)
    assert np.isfinite(got).all()
    tail = np.arange(max(0, n - 64), n)
    err_tail = oracle.rel_l2(got[:, tail], _oracle(w, xb, tail))
    assert err_tail <= (1e-2 if out_dtype == "bf16" else 1e-5), err_tail


@pytest.mark.parametrize("n,g", [(4096, 0), (1024, 0), (2048, 4)])
def test_stream_agrees_with_k4(n, g):
    w, x = _operands((4, 36), n, seed=7)
    xb = torch.from_numpy(x).to(torch.bfloat16)
    a = _product(w, xb, torch.float32, **({"stream_g": g} if g else {}))
    w2 = ks.RcubsMatrix(w.chain, np.array(w.values))  # fresh prepared cache
    b = _product(w2, xb, torch.float32, stream=0)
    assert oracle.rel_l2(a, b) <= 1e-5


def test_stream_is_deterministic():
    w, x = _operands((4, 36), 1024, seed=3)
    xb = torch.from_numpy(x).to(torch.bfloat16)
    a = _product(w, xb, torch.float32)
    b = _product(w, xb, torch.float32)
    assert np.array_equal(a, b)
