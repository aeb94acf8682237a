"""Pin the CPU oracle (oracle/rbgp4_oracle.c) to the reference's outputs.

Every golden hash below was produced by the reference kronsparse itself
(tests/golden/make_golden.py); the oracle must reproduce them bit-for-bit.
Only then is it trusted as the checker of the CUDA path.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2006_13486_b200 as ks
from paper_2006_13486_b200 import workloads as wl

from conftest import case_config, corpus_chain, corpus_inputs, sha16


def test_oracle_builds():
    assert oracle.build().endswith(".so")
    assert oracle.max_threads() >= 1


@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_cases_bit_exact(golden, precision):
    for cid, entry in golden["cases"].items():
        cfg = case_config(entry, precision, cid)
        chain, w, inp = wl.make_operands(cfg)
        p = ks.tiling_for_chain(chain, tn=cfg.tn, rn=cfg.rn, bn=cfg.bn)
        assert sha16(oracle.tiled(w, inp, p, threads=4)) == entry[precision]["rbgp4mm"], cid
        assert sha16(oracle.reference_product(w, inp, threads=4)) == \
            entry[precision]["sdmm_reference"], cid


@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_corpus_bit_exact(golden, precision):
    for rec in golden["corpus"]:
        chain = corpus_chain(rec)
        w, inp = corpus_inputs(rec, chain, precision)
        p = ks.tiling_for_chain(chain, tn=rec["tn"], rn=rec["rn"], bn=rec["bn"])
        assert sha16(inp) == rec[precision]["inp"]
        assert sha16(oracle.tiled(w, inp, p)) == rec[precision]["rbgp4mm"], rec
        assert sha16(oracle.reference_product(w, inp)) == rec[precision]["sdmm_reference"], rec


def test_worker_count_invariance():
    chain, w, inp = wl.make_operands(wl.C1A)
    p = ks.tiling_for_chain(chain)
    outs = [oracle.tiled(w, inp, p, threads=n) for n in (1, 2, 3, 8)]
    assert all(np.array_equal(outs[0], o) for o in outs[1:])


def test_tiled_close_to_f64_oracle(golden):
    entry = golden["cases"]["c1a"]
    chain, w, inp = wl.make_operands(case_config(entry, "f32"))
    p = ks.tiling_for_chain(chain)
    out = oracle.tiled(w, inp, p)
    w64 = ks.RcubsMatrix(chain, w.values.astype(np.float64))
    ref = oracle.reference_product(w64, inp.astype(np.float64))
    assert oracle.rel_l2(out, ref) == pytest.approx(entry["f32"]["rel_l2_vs_f64"], rel=1e-6)
