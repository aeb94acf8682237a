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
