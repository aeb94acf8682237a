"""Generate tests/golden/golden.json by running the REFERENCE (kronsparse).

Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Everything recorded is the sha256 prefix (16 hex digits) of raw
little-endian bytes, so the fixture stays small and the tests compare
bit-for-bit.  Inputs are regenerated in the tests from the same recipes
(seeded Philox / default_rng streams), and their hashes are recorded too so
a recipe drift is caught separately from a kernel mismatch.

Sections:
  masks    -- generate_ramanujan adjacency for a (shape, sparsity, seed) grid
  cases    -- bench-recipe configs (SweepConfig -> build_chain/init_random/
              uniform, reference bench.py:99-140): chain, W, I and the
              reference's rbgp4mm / sdmm_reference outputs (f32 and f64)
  corpus   -- the 108-config acceptance corpus (reference
              test_acceptance.py:235-323) with per-config seeded inputs
  digest   -- the reference's own golden serialisation digest
              (test_rcubs.py:29-31,220-222), re-derived here
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

import kronsparse as ks
from kronsparse import bench as kb

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")


def h(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


MASK_GRID = [
    ((8, 16), 0.5), ((16, 32), 0.5), ((32, 32), 0.5), ((32, 32), 0.75), ((32, 32), 0.875),
    ((32, 32), 0.9375), ((16, 16), 0.75), ((16, 16), 0.875), ((8, 8), 0.75), ((4, 8), 0.5),
    ((4, 16), 0.5), ((32, 64), 0.5), ((32, 64), 0.75), ((32, 64), 0.875), ((4, 72), 0.5),
    ((4, 36), 0.5), ((8, 72), 0.75), ((32, 128), 0.5), ((32, 128), 0.75), ((64, 64), 0.875),
    ((128, 128), 0.5), ((64, 256), 0.75),
]

# (config_id, g_o, sp_o, g_r, g_i, sp_i, g_b, n_cols, tn, rn, bn)
CASES = [
    ("c1a", (8, 16), 0.5, (2, 1), (32, 32), 0.5, (1, 1), 1024, 128, 1, 32),
    ("c1b", (4, 4), 0.5, (4, 1), (8, 8), 0.5, (4, 16), 1024, 128, 1, 32),
    ("desk-o50-i75", (16, 32), 0.5, (2, 1), (32, 32), 0.75, (1, 1), 256, 128, 1, 32),
    ("rep-r2b2", (8, 32), 0.5, (2, 1), (32, 16), 0.75, (2, 2), 256, 128, 2, 16),
    ("t2-o50-i50", (32, 128), 0.5, (4, 1), (32, 32), 0.5, (1, 1), 128, 128, 1, 32),
    ("t2-o0-i9375", (32, 128), 0.0, (4, 1), (32, 32), 0.9375, (1, 1), 128, 128, 1, 32),
    ("vgg-c10-875", (4, 72), 0.5, (4, 1), (32, 64), 0.75, (1, 1), 128, 128, 1, 32),
    ("vgg-c10-tc", (4, 36), 0.5, (1, 1), (16, 16), 0.75, (8, 8), 128, 128, 1, 32),
]

SPLIT_SHAPES = {
    (0.0, 0.75): [((2, 4), (8, 8)), ((4, 2), (8, 8)), ((4, 4), (8, 8))],
    (0.5, 0.5): [((4, 8), (4, 4)), ((8, 4), (8, 8)), ((4, 4), (4, 8))],
    (0.0, 0.875): [((2, 2), (16, 16)), ((4, 2), (16, 16)), ((2, 4), (16, 16))],
    (0.5, 0.75): [((4, 4), (8, 8)), ((4, 8), (8, 8)), ((8, 4), (8, 8))],
    (0.75, 0.5): [((8, 8), (4, 4)), ((8, 16), (4, 4)), ((16, 8), (4, 4))],
    (0.0, 0.9375): [((2, 2), (32, 32)), ((2, 4), (32, 32)), ((4, 2), (32, 32))],
    (0.5, 0.875): [((4, 4), (16, 16)), ((4, 8), (16, 16)), ((8, 4), (16, 16))],
    (0.75, 0.75): [((8, 8), (8, 8)), ((8, 16), (8, 8)), ((16, 8), (8, 8))],
    (0.875, 0.5): [((16, 16), (4, 4)), ((16, 32), (4, 4)), ((32, 16), (4, 4))],
}
VARIANTS = [
    ((1, 1), (1, 1), 16, 1, 8, 32),
    ((2, 1), (1, 1), 16, 2, 4, 64),
    ((2, 1), (2, 2), 32, 1, 16, 32),
    ((1, 1), (2, 1), 16, 1, 16, 64),
]


def corpus_configs():
    """The acceptance corpus enumeration (reference test_acceptance.py:257-272)."""
    out, seed = [], 0
    for (sp_o, sp_i), shapes in SPLIT_SHAPES.items():
        for go, gi in shapes:
            for g_r, g_b, tn, rn, bn, n_cols in VARIANTS:
                rows = go[0] * g_r[0] * gi[0] * g_b[0]
                cols = go[1] * g_r[1] * gi[1] * g_b[1]
                if rows > 512 or cols > 512:
                    continue
                seed += 1
                out.append(dict(sp_o=sp_o, sp_i=sp_i, g_o=go, g_i=gi, g_r=g_r, g_b=g_b, tn=tn,
                                rn=rn, bn=bn, n_cols=n_cols, seed=seed))
    return out


def factor(shape, sp, seed):
    if sp == 0.0:
        return ks.complete_graph(*shape)
    return ks.generate_ramanujan(ks.LiftChainSpec(shape[0], shape[1], sp, rng_seed=seed)).graph


def corpus_inputs(cfg, chain, precision):
    """Per-config seeded operands (the tests rebuild these with the same recipe)."""
    w = ks.init_random(chain, cfg["seed"], precision=precision)
    rng = np.random.default_rng(10_000 + cfg["seed"])
    inp = rng.uniform(-1, 1, size=(w.cols, cfg["n_cols"])).astype(w.dtype)
    return w, inp


def main():
    t0 = time.time()
    gold = {"generator": "kronsparse (reference) via tests/golden/make_golden.py",
            "masks": [], "cases": {}, "corpus": []}
    for (shape, sp) in MASK_GRID:
        for seed in (0, 1, 7):
            spec = ks.LiftChainSpec(shape[0], shape[1], sp, rng_seed=seed)
            try:
                res = ks.generate_ramanujan(spec)
                rec = {"shape": list(shape), "sparsity": sp, "seed": seed,
                       "adj": h(res.graph.adjacency_array()), "attempts": res.attempts,
                       "sigma2": res.report.sigma2}
            except ks.GenerationExhaustedError as exc:
                rec = {"shape": list(shape), "sparsity": sp, "seed": seed, "exhausted": True,
                       "best_lambda2": exc.best_lambda2}
            gold["masks"].append(rec)
    print(f"masks done {time.time() - t0:.1f}s", file=sys.stderr)

    for cid, g_o, sp_o, g_r, g_i, sp_i, g_b, n, tn, rn, bn in CASES:
        entry = {"g_o": list(g_o), "sp_o": sp_o, "g_r": list(g_r), "g_i": list(g_i),
                 "sp_i": sp_i, "g_b": list(g_b), "n_cols": n, "tn": tn, "rn": rn, "bn": bn}
        for precision in ("f32", "f64"):
            cfg = kb.SweepConfig(cid, g_o, sp_o, g_r, g_i, sp_i, g_b, n_cols=n, tn=tn, rn=rn,
                                 bn=bn, precision=precision, seed=0)
            chain = kb.build_chain(cfg)
            params = ks.tiling_for_chain(chain, tn=tn, rn=rn, bn=bn, workers=4)
            rng = ks.make_rng(np.random.SeedSequence([cfg.seed, 1]).generate_state(1)[0])
            w = ks.init_random(chain, rng, precision=precision)
            inp = rng.uniform(-1.0, 1.0, size=(w.cols, n)).astype(w.dtype)
            out, rep = ks.rbgp4mm(w, inp, params)
            ref = ks.sdmm_reference(w, inp)
            oracle64 = ks.sdmm_reference(ks.RcubsMatrix(chain, w.values.astype(np.float64)),
                                         inp.astype(np.float64))
            entry["adj_o"] = h(chain.graphs[0].adjacency_array())
            entry["adj_i"] = h(chain.graphs[2].adjacency_array())
            entry[precision] = {
                "values": h(w.values), "inp": h(inp), "rbgp4mm": h(out),
                "sdmm_reference": h(ref), "report": rep.to_dict(),
                "norm_f64": float(np.linalg.norm(oracle64)),
                "rel_l2_vs_f64": float(np.linalg.norm(out - oracle64) / np.linalg.norm(oracle64)),
            }
        gold["cases"][cid] = entry
        print(f"case {cid} done {time.time() - t0:.1f}s", file=sys.stderr)

    for cfg in corpus_configs():
        chain = ks.RbgpChain((factor(cfg["g_o"], cfg["sp_o"], cfg["seed"]),
                              ks.complete_graph(*cfg["g_r"]),
                              factor(cfg["g_i"], cfg["sp_i"], cfg["seed"] + 50000),
                              ks.complete_graph(*cfg["g_b"])))
        params = ks.tiling_for_chain(chain, tn=cfg["tn"], rn=cfg["rn"], bn=cfg["bn"], workers=1)
        rec = dict(cfg, g_o=list(cfg["g_o"]), g_i=list(cfg["g_i"]), g_r=list(cfg["g_r"]),
                   g_b=list(cfg["g_b"]), adj_o=h(chain.graphs[0].adjacency_array()),
                   adj_i=h(chain.graphs[2].adjacency_array()))
        for precision in ("f32", "f64"):
            w, inp = corpus_inputs(cfg, chain, precision)
            out, rep = ks.rbgp4mm(w, inp, params)
            rec[precision] = {"values": h(w.values), "inp": h(inp), "rbgp4mm": h(out),
                              "sdmm_reference": h(ks.sdmm_reference(w, inp)),
                              "fma_count": rep.fma_count,
                              "steps_skipped_per_tile": rep.steps_skipped_per_tile}
        gold["corpus"].append(rec)
    print(f"corpus ({len(gold['corpus'])}) done {time.time() - t0:.1f}s", file=sys.stderr)

    # reference test_rcubs.py:29-31 golden digest, re-derived from the reference
    sys.path.insert(0, "/root/reference/pkg/tests")
    from conftest import example_chain  # noqa: E402  (reference test fixture)
    m = ks.init_random(example_chain(), 2024, precision="f32")
    gold["digest"] = {"example_chain_seed2024_f32": hashlib.sha256(ks.serialize(m)).hexdigest()}

    with open(OUT, "w") as fh:
        json.dump(gold, fh, indent=1, sort_keys=True)
        fh.write("\n")
    print(f"wrote {OUT} in {time.time() - t0:.1f}s", file=sys.stderr)


if __name__ == "__main__":
    main()
