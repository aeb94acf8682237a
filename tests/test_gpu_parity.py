"""CUDA path vs the reference (golden hashes) and vs the pinned CPU oracle.

Bar (BASELINE north star):
  * compute="exact"  -> bit-identical to the reference rbgp4mm (f32 and f64)
  * sdmm_reference   -> bit-identical to the reference sdmm_reference
  * compute="ffma"   -> max-rel <= 1e-5 (f32) / 1e-12 (f64) vs the f64 oracle
  * tf32 / bf16      -> rel-L2 <= 1e-2 vs the f64 oracle
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2006_13486_b200 as ks
from paper_2006_13486_b200 import _native
from paper_2006_13486_b200 import workloads as wl

from conftest import case_config, corpus_chain, corpus_inputs, ring_graph, sha16

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def f64_oracle(w, inp):
    w64 = ks.RcubsMatrix(w.chain, np.asarray(w.values, dtype=np.float64))
    return oracle.reference_product(w64, np.asarray(inp, dtype=np.float64), threads=8)


def test_device_and_library_present():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    assert _native.lib().rbgp4_abi_version() == 3


@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_cases_exact_bit_identical(golden, precision):
    for cid, entry in golden["cases"].items():
        cfg = case_config(entry, precision, cid)
        chain, w, inp = wl.make_operands(cfg)
        p = ks.tiling_for_chain(chain, tn=cfg.tn, rn=cfg.rn, bn=cfg.bn, workers=4)
        out, rep = ks.rbgp4mm(w, inp, p)
        assert out.dtype == w.dtype and out.shape == (w.rows, cfg.n_cols)
        assert sha16(out) == entry[precision]["rbgp4mm"], cid
        assert rep.to_dict() == entry[precision]["report"], cid


@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_cases_sdmm_reference_bit_identical(golden, precision):
    for cid, entry in golden["cases"].items():
        chain, w, inp = wl.make_operands(case_config(entry, precision, cid))
        assert sha16(ks.sdmm_reference(w, inp)) == entry[precision]["sdmm_reference"], cid
        assert sha16(ks.sdmm_reference(w.to_unstructured(), inp)) == \
            entry[precision]["sdmm_reference"], cid


@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_corpus_exact_bit_identical(golden, precision):
    for rec in golden["corpus"]:
        chain = corpus_chain(rec)
        w, inp = corpus_inputs(rec, chain, precision)
        p = ks.tiling_for_chain(chain, tn=rec["tn"], rn=rec["rn"], bn=rec["bn"])
        out, rep = ks.rbgp4mm(w, inp, p)
        assert sha16(out) == rec[precision]["rbgp4mm"], rec
        assert rep.fma_count == rec[precision]["fma_count"]
        assert rep.steps_skipped_per_tile == rec[precision]["steps_skipped_per_tile"]


@pytest.mark.parametrize("precision,tol", [("f32", 1e-5), ("f64", 1e-12)])
def test_corpus_ffma_within_tolerance(golden, precision, tol):
    worst = 0.0
    for rec in golden["corpus"]:
        chain = corpus_chain(rec)
        w, inp = corpus_inputs(rec, chain, precision)
        p = ks.tiling_for_chain(chain, tn=rec["tn"], rn=rec["rn"], bn=rec["bn"])
        out, _ = ks.rbgp4mm(w, inp, p, compute="ffma")
        worst = max(worst, oracle.max_rel(out, f64_oracle(w, inp)))
    assert worst <= tol, worst


def test_identity_passthrough_bit_exact():
    chain = ks.RbgpChain((ring_graph(4, d=1), ks.complete_graph(1, 1), ks.complete_graph(1, 1),
                          ks.complete_graph(1, 1)))
    w = ks.RcubsMatrix(chain, np.ones((4, 1)))
    inp = np.random.default_rng(0).standard_normal((4, 8))
    out, rep = ks.rbgp4mm(w, inp, ks.tiling_for_chain(chain, tn=8, rn=1, bn=8, workers=2))
    assert np.array_equal(out, inp) and rep.steps_per_tile == 1


def test_ragged_and_strided_columns():
    """N not a multiple of 4, odd leading dimensions, column sub-views."""
    chain, w, _ = wl.make_operands(wl.C1A)
    p = ks.tiling_for_chain(chain, tn=1, rn=1, bn=1)
    rng = np.random.default_rng(3)
    for n in (1, 3, 5, 130):
        inp = rng.uniform(-1, 1, (w.cols, n)).astype(np.float32)
        out, _ = ks.rbgp4mm(w, inp, p)
        assert np.array_equal(out, oracle.tiled(w, inp, p)), n
    big = torch.from_numpy(rng.uniform(-1, 1, (w.cols, 301)).astype(np.float32)).cuda()
    view = big[:, 7:7 + 129]  # ld_in = 301, unaligned base
    out, _ = ks.rbgp4mm(w, view, p)
    assert out.is_cuda
    ref = oracle.tiled(w, view.cpu().numpy(), p)
    assert np.array_equal(out.cpu().numpy(), ref)


def test_zero_columns():
    chain, w, _ = wl.make_operands(wl.C1A)
    p = ks.tiling_for_chain(chain, tn=1, rn=1, bn=1)
    out, rep = ks.rbgp4mm(w, np.zeros((w.cols, 0), np.float32), p)
    assert out.shape == (w.rows, 0) and rep.fma_count == 0


def test_torch_tensors_stay_on_device_and_out_param():
    chain, w, inp = wl.make_operands(wl.C1A)
    p = ks.tiling_for_chain(chain)
    x = torch.from_numpy(inp).cuda()
    res = torch.empty((w.rows, inp.shape[1]), device="cuda", dtype=torch.float32)
    out, _ = ks.rbgp4mm(w, x, p, out=res)
    assert out is res
    assert sha16(res.cpu().numpy()) == "9fe440861f6f8868"
    pinned = torch.from_numpy(inp).pin_memory()
    host, _ = ks.rbgp4mm(w, pinned, p)
    assert not host.is_cuda and sha16(host.numpy()) == "9fe440861f6f8868"


def test_general_chain_reference_on_gpu():
    rng = np.random.default_rng(11)
    chain = ks.RbgpChain((ring_graph(8, 3), ks.complete_graph(2, 2), ring_graph(4, 2)))
    w = ks.init_random(chain, 4, precision="f32")
    inp = rng.uniform(-1, 1, (w.cols, 77)).astype(np.float32)
    got = ks.sdmm_reference(w, inp)
    assert np.array_equal(got, oracle.reference_product(w, inp))


@pytest.mark.parametrize("persistent", [False, True])
@pytest.mark.parametrize("compute,tol", [("tf32", 1e-2), ("bf16", 1e-2)])
def test_tensor_core_modes(golden, compute, tol, persistent, plan_options):
    if persistent:  # persistent tile loop of the tcgen05 kernels, forced (K4 on the stored values)
        plan_options("persistent", 1)
        plan_options("relayout", 0)
    lib = _native.lib()
    for cid in golden["cases"]:
        entry = golden["cases"][cid]
        chain, w, inp = wl.make_operands(case_config(entry, "f32", cid))
        p = ks.tiling_for_chain(chain, tn=entry["tn"], rn=entry["rn"], bn=entry["bn"])
        out, _ = ks.rbgp4mm(w, inp, p, compute=compute)
        err = oracle.rel_l2(out, f64_oracle(w, inp))
        assert err <= tol, (cid, compute, err)


@pytest.mark.parametrize("compute", ["bf16", "tf32"])
@pytest.mark.parametrize("n_cols", [5, 13, 67])
def test_tensor_core_modes_stage_unaligned_operands(compute, n_cols):
    """Any legal reference operand runs on the tensor cores: N not a multiple of the 16-byte
    TMA granule (tn = 1, reference sdmm.py:257-261 only needs N % tn == 0) is staged, not refused."""
    import torch
    chain, w, _ = wl.make_operands(wl.C1B)
    inp = np.random.default_rng(n_cols).uniform(-1, 1, (w.cols, n_cols)).astype(np.float32)
    p = ks.tiling_for_chain(chain, tn=1, rn=1, bn=1)
    x = torch.from_numpy(inp)
    if compute == "bf16":
        x = x.to(torch.bfloat16)
    out, _ = ks.rbgp4mm(w, x.cuda(), p, compute=compute, out_dtype=torch.float32)
    ref = f64_oracle(w, x.double().numpy())
    assert out.shape == (w.rows, n_cols)
    assert oracle.rel_l2(out.cpu().numpy(), ref) < 1e-2


@pytest.mark.parametrize("layer", [(64, 64), (128, 128), (256, 256), (64, 16)])
@pytest.mark.parametrize("n_cols", [1000, 4096])
def test_simt_wide_variants(layer, n_cols, plan_options):
    """K1's TMA-fed wide kernel at 16 / 8 / 4 rows per thread (VGG tc16 and WRN-40-4 G_b (8,8) /
    (4,4) factorisations), ragged N (zero-filled TMA boxes): exact mode bit-identical to the
    pinned C port of _tile_worker and to the generic K1 kernel; ffma within 1e-5 of f64."""
    from paper_2006_13486_b200.wrn import wrn_layer_chain
    chain = wrn_layer_chain(layer[0], layer[1], 0.875, 3)
    w = ks.init_random(chain, 5, precision="f32")
    inp = np.random.default_rng(n_cols).uniform(-1, 1, (w.cols, n_cols)).astype(np.float32)
    p = ks.tiling_for_chain(chain, tn=1, rn=1, bn=1)
    x = torch.from_numpy(inp).cuda()
    out, _ = ks.rbgp4mm(w, x, p)
    kern = _native.last_kernel()
    g = chain.graphs[3].num_left * chain.graphs[1].num_left
    assert kern == ("K1 simt wide" if g % 4 == 0 else "K1 simt"), (layer, kern)
    got = out.cpu().numpy()
    assert np.array_equal(got, oracle.tiled(w, inp, p, threads=8)), layer
    plan_options("simt_wide", 0)
    generic, _ = ks.rbgp4mm(w, x, p)
    assert _native.last_kernel() == "K1 simt"
    assert torch.equal(generic, out)
    plan_options("simt_wide", -1)
    fast, _ = ks.rbgp4mm(w, x, p, compute="ffma")
    assert oracle.max_rel(fast.cpu().numpy(), f64_oracle(w, inp)) <= 1e-5


@pytest.mark.parametrize("layer,n_cols", [((512, 512), 1024), ((64, 64), 256), ((256, 256), 1000)])
def test_simt_wide_ffma_split_pair(layer, n_cols, plan_options):
    """K1 wide ffma with the steps halved over a (1,1,2) cluster (grids short of the SMs): within
    1e-5 of the f64 oracle, deterministic (two runs bit-identical), and the unsplit plan agrees to
    fp32 reassociation; EXACT never splits."""
    from paper_2006_13486_b200.wrn import wrn_layer_chain
    chain = wrn_layer_chain(layer[0], layer[1], 0.875, 3)
    w = ks.init_random(chain, 9, precision="f32")
    inp = np.random.default_rng(n_cols + 1).uniform(-1, 1, (w.cols, n_cols)).astype(np.float32)
    p = ks.tiling_for_chain(chain, tn=1, rn=1, bn=1)
    x = torch.from_numpy(inp).cuda()
    plan_options("simt_ksplit", 2)
    a, _ = ks.rbgp4mm(w, x, p, compute="ffma")
    assert _native.last_kernel() == "K1 simt wide split"
    b, _ = ks.rbgp4mm(w, x, p, compute="ffma")
    assert torch.equal(a, b)
    assert oracle.max_rel(a.cpu().numpy(), f64_oracle(w, inp)) <= 1e-5
    e, _ = ks.rbgp4mm(w, x, p)  # exact: never split
    assert _native.last_kernel() == "K1 simt wide"
    assert np.array_equal(e.cpu().numpy(), oracle.tiled(w, inp, p, threads=8))
    plan_options("simt_ksplit", 1)
    c, _ = ks.rbgp4mm(w, x, p, compute="ffma")
    assert _native.last_kernel() == "K1 simt wide"
    assert float((a - c).norm() / c.norm()) < 1e-6


def test_acceptance_criteria_6_and_7_on_device(golden):
    """The reference's acceptance criteria 6 and 7 (test_acceptance.py:283-356) over the same
    108-config corpus, with the products on the B200: exact mode within 1e-12 (f64) / 1e-5 (f32) of
    the f64 oracle, bit-identical for workers 1, 2 and 8 (the GPU analogue of the reference's
    worker-count invariance, sdmm.py:18-20), and WorkReport's fma / skip counts equal to their
    closed forms."""
    worst = {"f64": 0.0, "f32": 0.0}
    n = 0
    for rec in golden["corpus"]:
        chain = corpus_chain(rec)
        for precision, tol in (("f64", 1e-12), ("f32", 1e-5)):
            w, inp = corpus_inputs(rec, chain, precision)
            p = ks.tiling_for_chain(chain, tn=rec["tn"], rn=rec["rn"], bn=rec["bn"], workers=1)
            outs = {nw: ks.rbgp4mm(w, inp, ks.with_workers(p, nw)) for nw in (1, 2, 8)}
            ref = f64_oracle(w, inp)
            rel = float(np.abs(outs[1][0] - ref).max() / np.abs(ref).max())
            worst[precision] = max(worst[precision], rel)
            assert rel <= tol, (rec, precision, rel)
            assert np.array_equal(outs[1][0], outs[2][0]) and np.array_equal(outs[1][0], outs[8][0])
            rep = outs[1][1]
            assert rep.fma_count == w.nnz * inp.shape[1]
            tiles_per_row = w.cols // p.tk
            g_o = chain.graphs[0]
            assert rep.steps_skipped_per_tile == tiles_per_row - len(g_o.adjacency[0])
            assert rep.steps_skipped_per_tile == g_o.sparsity * tiles_per_row
            n += 1
    assert n >= 200, n
