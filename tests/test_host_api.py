"""Host-side mirror of the reference API, pinned to the reference's own outputs.

Masks, index maps, values and synthetic inputs must be bit-identical to the
reference (golden hashes from tests/golden/make_golden.py, which imports
the reference itself).  Validation errors must be the reference's types.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

import paper_2006_13486_b200 as ks
from paper_2006_13486_b200 import workloads as wl

from conftest import case_config, corpus_chain, example_chain, ring_graph, sha16


class TestMasksBitExact:
    def test_generation_grid(self, golden):
        for rec in golden["masks"]:
            spec = ks.LiftChainSpec(rec["shape"][0], rec["shape"][1], rec["sparsity"],
                                    rng_seed=rec["seed"])
            res = ks.generate_ramanujan(spec)
            assert sha16(res.graph.adjacency_array()) == rec["adj"], rec
            assert res.attempts == rec["attempts"], rec
            assert res.report.sigma2 == pytest.approx(rec["sigma2"], abs=1e-9)

    def test_bench_recipe_cases(self, golden):
        for cid, entry in golden["cases"].items():
            for precision in ("f32", "f64"):
                chain, w, inp = wl.make_operands(case_config(entry, precision, cid))
                assert sha16(chain.graphs[0].adjacency_array()) == entry["adj_o"], cid
                assert sha16(chain.graphs[2].adjacency_array()) == entry["adj_i"], cid
                assert sha16(w.values) == entry[precision]["values"], cid
                assert sha16(inp) == entry[precision]["inp"], cid

    def test_corpus_chains(self, golden):
        for rec in golden["corpus"]:
            chain = corpus_chain(rec)
            assert sha16(chain.graphs[0].adjacency_array()) == rec["adj_o"]
            assert sha16(chain.graphs[2].adjacency_array()) == rec["adj_i"]

    def test_serialization_digest(self, golden):
        m = ks.init_random(example_chain(), 2024, precision="f32")
        assert hashlib.sha256(ks.serialize(m)).hexdigest() == \
            golden["digest"]["example_chain_seed2024_f32"]


class TestLifts:
    def test_identity_coins_make_disjoint_union(self):
        class Zeros:
            def integers(self, lo, hi, size=None, dtype=None):
                return np.zeros(size, dtype=dtype)
        g = ks.two_lift(ks.complete_graph(2, 2), Zeros())
        assert g.adjacency == ((0, 1), (0, 1), (2, 3), (2, 3))

    def test_crossover_pair(self):
        class Ones:
            def integers(self, lo, hi, size=None, dtype=None):
                return np.ones(size, dtype=dtype)
        g = ks.two_lift(ks.complete_graph(1, 1), Ones())
        assert g.adjacency == ((1,), (0,))

    def test_non_dyadic_rejected(self):
        with pytest.raises(ks.InvalidArgumentError):
            ks.LiftChainSpec(8, 8, 0.8)

    def test_exhaustion_reports_best(self):
        with pytest.raises(ks.GenerationExhaustedError) as info:
            ks.generate_ramanujan(ks.LiftChainSpec(8, 8, 0.875, max_attempts=3))
        assert info.value.attempts == 3 and info.value.best_lambda2 >= 1.0


class TestStorage:
    def test_neighbors_match_dense(self):
        chain = example_chain()
        w = ks.init_random(chain, 3)
        dense = w.to_dense()
        for u in range(chain.num_left):
            assert list(np.flatnonzero(dense[u])) == list(ks.neighbors(chain, u))

    def test_round_trip_dense(self):
        chain = wl.build_chain(wl.C1A)
        w = ks.init_random(chain, 5, precision="f32")
        back = ks.RcubsMatrix.from_dense(w.to_dense(), chain)
        assert np.array_equal(back.values, w.values)

    def test_off_pattern_rejected(self):
        chain = example_chain()
        dense = ks.init_random(chain, 1).to_dense()
        r, c = 0, int(np.flatnonzero(dense[0] == 0)[0])
        dense[r, c] = 1.0
        with pytest.raises(ks.PatternViolationError) as info:
            ks.RcubsMatrix.from_dense(dense, chain)
        assert (info.value.row, info.value.col) == (r, c)

    def test_csr_export(self):
        chain = example_chain()
        w = ks.init_random(chain, 2)
        csr = w.to_unstructured()
        assert csr.indptr[-1] == w.nnz and csr.indices.dtype == np.int32
        assert all(np.all(np.diff(csr.indices[i * w.row_nnz:(i + 1) * w.row_nnz]) > 0)
                   for i in range(w.rows))

    def test_serialize_round_trip_and_errors(self):
        w = ks.init_random(example_chain(), 9, precision="f32")
        blob = ks.serialize(w)
        back = ks.deserialize(blob)
        assert np.array_equal(back.values, w.values)
        with pytest.raises(ks.PrecisionMismatchError):
            ks.deserialize(blob, precision="f64")
        with pytest.raises(ks.BadMagicError):
            ks.deserialize(b"XXXX" + blob[4:])
        with pytest.raises(ks.TruncatedStreamError):
            ks.deserialize(blob[:-9])
        with pytest.raises(ks.ChecksumMismatchError):
            ks.deserialize(blob[:-1] + bytes([blob[-1] ^ 1]))

    def test_values_read_only_and_caller_untouched(self):
        chain = example_chain()
        vals = np.ones((chain.num_left, chain.row_nnz))
        w = ks.RcubsMatrix(chain, vals)
        assert not w.values.flags.writeable and vals.flags.writeable

    def test_memory_footprint(self):
        fp = ks.memory_footprint(ks.init_random(example_chain(), 1))
        assert fp.index_reduction_ratio == pytest.approx(512 / 22)


class TestTilingAndErrors:
    def test_c1a_tiling(self):
        params = ks.tiling_for_chain(wl.build_chain(wl.C1A))
        assert (params.tm, params.tk, params.tn, params.rm, params.rk, params.bm, params.bk,
                params.rn, params.bn, params.workers) == (64, 32, 128, 2, 1, 1, 1, 1, 32, 1)

    def test_all_violations_at_once(self):
        chain = wl.build_chain(wl.C1A)
        with pytest.raises(ks.ConfigurationError) as info:
            ks.tiling_for_chain(chain, tn=12, rn=5, bn=7, workers=0)
        assert "tn=12" in str(info.value) and "workers" in str(info.value)

    def test_incomplete_repeat_factor(self):
        chain = ks.RbgpChain((ring_graph(4), ring_graph(2, 1), ks.complete_graph(2, 2),
                              ks.complete_graph(1, 1)))
        with pytest.raises(ks.ConfigurationError, match="complete"):
            ks.tiling_for_chain(chain)

    def test_short_chain(self):
        with pytest.raises(ks.UnsupportedChainError):
            ks.tiling_for_chain(ks.RbgpChain((ks.complete_graph(2, 2),)))

    # error paths of rbgp4mm are raised before any device work, so they run on CPU
    def test_rbgp4mm_shape_dtype_columns_params(self):
        chain = wl.build_chain(wl.C1A)
        w = ks.init_random(chain, 1, precision="f32")
        p = ks.tiling_for_chain(chain)
        with pytest.raises(ks.ShapeError):
            ks.rbgp4mm(w, np.zeros((w.cols + 1, 128), np.float32), p)
        with pytest.raises(ks.ShapeError, match="dtype"):
            ks.rbgp4mm(w, np.zeros((w.cols, 128), np.float64), p)
        with pytest.raises(ks.ConfigurationError, match="columns"):
            ks.rbgp4mm(w, np.zeros((w.cols, 100), np.float32), p)
        from dataclasses import replace
        with pytest.raises(ks.ConfigurationError, match="tm"):
            ks.rbgp4mm(w, np.zeros((w.cols, 128), np.float32), replace(p, tm=p.tm + 1))
        with pytest.raises(ks.InvalidArgumentError):
            ks.rbgp4mm(w, np.zeros((w.cols, 128), np.float32), p, compute="fp8")
        import torch
        with pytest.raises(ks.InvalidArgumentError, match="bfloat16"):  # numpy cannot hold bf16
            ks.rbgp4mm(w, np.zeros((w.cols, 128), np.float32), p, compute="bf16",
                       out_dtype=torch.bfloat16)

    def test_general_chain_unsupported_by_tiled_product(self):
        chain = ks.RbgpChain((ks.complete_graph(4, 4), ks.complete_graph(2, 2)))
        w = ks.init_random(chain, 3)
        p = ks.tiling_for_chain(wl.build_chain(wl.C1A))
        with pytest.raises(ks.UnsupportedChainError):
            ks.rbgp4mm(w, np.zeros((w.cols, 128)), p)

    def test_work_report_closed_form(self, golden):
        from paper_2006_13486_b200.sdmm import work_report
        for cid, entry in golden["cases"].items():
            cfg = case_config(entry, "f32", cid)
            chain = wl.build_chain(cfg)
            w = ks.init_random(chain, 0, precision="f32")
            p = ks.tiling_for_chain(chain, tn=cfg.tn, rn=cfg.rn, bn=cfg.bn)
            assert work_report(w, cfg.n_cols, p).to_dict() == entry["f32"]["report"], cid

    def test_combined_sparsity(self):
        assert ks.combined_sparsity(0.5, 0.75) == 0.875
        assert ks.combined_sparsity(0.875, 0.5) == 0.9375
