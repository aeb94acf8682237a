"""Training direction: W^T via the transposed chain, the pattern-restricted
weight gradient (rbgp4_sddmm), and autograd through a trainable RBGP4 layer -- against dense
numpy / torch float64 references."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2006_13486_b200 as ks
from paper_2006_13486_b200 import training
from paper_2006_13486_b200 import workloads as wl

CHAINS = [wl.C1A, wl.C1B,
          wl.SweepConfig("tc", (4, 6), 0.5, (1, 1), (16, 16), 0.75, (8, 8), n_cols=1, seed=3),
          wl.SweepConfig("tc16", (4, 4), 0.5, (1, 1), (8, 8), 0.75, (16, 16), n_cols=1, seed=4)]


@pytest.mark.parametrize("cfg", CHAINS, ids=[c.config_id for c in CHAINS])
def test_transpose_is_exact(cfg):
    chain = wl.build_chain(cfg)
    w = ks.init_random(chain, 1, precision="f64")
    wt = training.transpose(w)
    assert wt.rows == w.cols and wt.cols == w.rows and wt.nnz == w.nnz
    assert np.array_equal(wt.to_dense(), w.to_dense().T)
    assert np.array_equal(training.transpose(wt).to_dense(), w.to_dense())


def _pattern_grad(w, d_out, inp):
    csr = w.to_unstructured()
    rows = np.repeat(np.arange(w.rows), w.row_nnz)
    return np.einsum("kn,kn->k", d_out[rows], inp[csr.indices]).reshape(w.rows, w.row_nnz)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", CHAINS, ids=[c.config_id for c in CHAINS])
@pytest.mark.parametrize("precision,tol", [("f64", 1e-12), ("f32", 1e-5)])
def test_sddmm_matches_dense(cfg, precision, tol):
    import torch
    import oracle
    chain = wl.build_chain(cfg)
    w = ks.init_random(chain, 1, precision=precision)
    rng = np.random.default_rng(7)
    dt = np.float64 if precision == "f64" else np.float32
    n = 200
    d_out = rng.standard_normal((w.rows, n)).astype(dt)
    inp = rng.standard_normal((w.cols, n)).astype(dt)
    got = training.sddmm(w, torch.from_numpy(d_out).cuda(), torch.from_numpy(inp).cuda()).cpu().numpy()
    ref = _pattern_grad(w, d_out.astype(np.float64), inp.astype(np.float64))
    assert oracle.rel_l2(got, ref) < tol


@pytest.mark.gpu
def test_autograd_trainable_layer():
    import torch
    cfg = CHAINS[2]
    chain = wl.build_chain(cfg)
    w = ks.init_random(chain, 2, precision="f64")
    layer = training.TrainableSparseLinear(w, compute="ffma")
    g = torch.Generator().manual_seed(0)
    x = torch.randn(64, w.cols, generator=g, dtype=torch.float64).cuda().requires_grad_(True)
    gy = torch.randn(64, w.rows, generator=g, dtype=torch.float64).cuda()
    y = layer(x)
    (y * gy).sum().backward()
    dense = torch.from_numpy(w.to_dense()).cuda()
    assert torch.allclose(y, x @ dense.t(), rtol=1e-10, atol=1e-10)
    assert torch.allclose(x.grad, gy @ dense, rtol=1e-10, atol=1e-10)
    want = _pattern_grad(w, gy.t().cpu().numpy(), x.detach().t().cpu().numpy())
    assert np.allclose(layer.values.grad.cpu().numpy(), want, rtol=1e-10, atol=1e-10)
    # one SGD step keeps the pattern: only stored slots move
    with torch.no_grad():
        layer.values -= 0.1 * layer.values.grad
    assert layer.values.shape == (w.rows, w.row_nnz)


@pytest.mark.gpu
def test_trainable_layer_rejects_mixed_dtypes():
    """The kernel reads values and activations in one element type: f32 activations against
    f64 trainable values (init_random's default) must raise, not reinterpret bytes."""
    import torch
    chain = wl.build_chain(CHAINS[2])
    w = ks.init_random(chain, 2, precision="f64")
    layer = training.TrainableSparseLinear(w, compute="ffma")
    x = torch.randn(8, w.cols, dtype=torch.float32).cuda()
    with pytest.raises(ks.ShapeError, match="dtype"):
        layer(x)


# ---------------------------------------------------------------- tensor-core training (bf16)
TC_CHAINS = [
    wl.SweepConfig("tc16", (4, 8), 0.5, (1, 1), (8, 8), 0.75, (16, 16), n_cols=1, seed=4),        # K5 TC16
    wl.SweepConfig("slice8", (4, 8), 0.5, (1, 1), (16, 16), 0.875, (8, 8), n_cols=1, seed=5),     # K5 slices
    wl.SweepConfig("tc", (4, 6), 0.5, (1, 1), (16, 16), 0.75, (8, 8), n_cols=1, seed=3),          # K5, 4 partials
    wl.SweepConfig("merged", (2, 6), 0.0, (1, 1), (8, 8), 0.75, (16, 16), n_cols=1, seed=6),      # merged pairs
    wl.SweepConfig("tc16-d4", (4, 8), 0.5, (1, 1), (8, 8), 0.5, (16, 16), n_cols=1, seed=7),      # TC16, 4 partials
]


def _bf16_round(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16).double().numpy()


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", TC_CHAINS, ids=[c.config_id for c in TC_CHAINS])
@pytest.mark.parametrize("n", [256, 200])
def test_sddmm_bf16_tensor_cores(cfg, n):
    """K7: bf16 dO / I, f32 gradient == the f64 pattern gradient of the same bf16-rounded
    operands (fp32 accumulation: rel-L2 <= 1e-5)."""
    import torch
    import oracle
    from paper_2006_13486_b200 import _native
    chain = wl.build_chain(cfg)
    w = ks.init_random(chain, 1, precision="f32")
    rng = np.random.default_rng(9)
    d_out = rng.standard_normal((w.rows, n)).astype(np.float32)
    inp = rng.standard_normal((w.cols, n)).astype(np.float32)
    db, ib = torch.from_numpy(d_out).to(torch.bfloat16), torch.from_numpy(inp).to(torch.bfloat16)
    got = training.sddmm(w, db.cuda(), ib.cuda())
    torch.cuda.synchronize()
    assert got.dtype == torch.float32 and _native.last_kernel() == "K7 sddmm"
    ref = _pattern_grad(w, db.double().numpy(), ib.double().numpy())
    assert oracle.rel_l2(got.cpu().numpy(), ref) < 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", TC_CHAINS, ids=[c.config_id for c in TC_CHAINS])
def test_autograd_trainable_layer_bf16(cfg):
    """Forward, input gradient and weight gradient of a bf16 tensor-core layer against f64
    references on the same bf16-rounded operands; then two SGD steps (the layer's prepared value
    copies follow the trainable values) still match."""
    import torch
    chain = wl.build_chain(cfg)
    w = ks.init_random(chain, 2, precision="f32")
    layer = training.TrainableSparseLinear(w, compute="bf16")
    g = torch.Generator().manual_seed(0)
    x = torch.randn(256, w.cols, generator=g).cuda().requires_grad_(True)
    gy = torch.randn(256, w.rows, generator=g).cuda()
    for step in range(3):
        x.grad = None
        layer.values.grad = None
        y = layer(x)
        (y * gy).sum().backward()
        wb = _bf16_round(layer.values.detach().cpu().numpy())
        dense = ks.RcubsMatrix(w.chain, wb).to_dense()
        xb = _bf16_round(x.detach().cpu().numpy())
        gb = _bf16_round(gy.cpu().numpy())
        rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)  # noqa: E731
        assert rel(y.detach().cpu().numpy(), xb @ dense.T) < 1e-5, step
        assert rel(x.grad.cpu().numpy(), gb @ dense) < 1e-5, step
        want = _pattern_grad(ks.RcubsMatrix(w.chain, wb), gb.T, xb.T)
        assert rel(layer.values.grad.cpu().numpy(), want) < 1e-5, step
        with torch.no_grad():
            layer.values -= 0.05 * layer.values.grad


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", TC_CHAINS, ids=[c.config_id for c in TC_CHAINS])
@pytest.mark.parametrize("n", [256, 200])
def test_sddmm_nk_bit_identical(cfg, n):
    """K7 on batch-major operands (dO^T, I^T as MN-major MMA operands) == K7 on the transposed
    copies, bit for bit (same MMAs, same batch order); ragged N included."""
    import torch
    from paper_2006_13486_b200 import _native
    chain = wl.build_chain(cfg)
    w = ks.init_random(chain, 3, precision="f32")
    g = torch.Generator(device="cuda").manual_seed(n)
    dnk = torch.randn(n, w.rows, device="cuda", generator=g).to(torch.bfloat16)
    xnk = torch.randn(n, w.cols, device="cuda", generator=g).to(torch.bfloat16)
    got = training.sddmm_nk(w, dnk, xnk)
    assert _native.last_kernel() == "K7 sddmm"
    want = training.sddmm(w, dnk.t().contiguous(), xnk.t().contiguous())
    torch.cuda.synchronize()
    assert torch.equal(got, want)
