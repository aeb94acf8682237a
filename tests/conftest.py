"""Shared fixtures.  `-m gpu` tests need a B200 and the built CUDA library;
everything else runs on a CPU-only box.

The oracle (../oracle) is test infrastructure: tests use it as the checker,
never as the thing under test.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import paper_2006_13486_b200 as ks  # noqa: E402
from paper_2006_13486_b200 import workloads as wl  # noqa: E402

GOLDEN_PATH = os.path.join(ROOT, "tests", "golden", "golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device and the built library")


@pytest.fixture
def plan_options():
    """set_option(name, value) for this test's thread; every override is reset afterwards."""
    from paper_2006_13486_b200 import _native
    yield _native.set_option
    _native.lib().rbgp4_reset_options()


def sha16(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN_PATH) as fh:
        return json.load(fh)


def case_config(entry: dict, precision: str, cid: str = "case") -> wl.SweepConfig:
    return wl.SweepConfig(cid, tuple(entry["g_o"]), entry["sp_o"], tuple(entry["g_r"]),
                          tuple(entry["g_i"]), entry["sp_i"], tuple(entry["g_b"]),
                          n_cols=entry["n_cols"], tn=entry["tn"], rn=entry["rn"],
                          bn=entry["bn"], precision=precision, seed=0)


def factor(shape, sp, seed):
    if sp == 0.0:
        return ks.complete_graph(*shape)
    return ks.generate_ramanujan(ks.LiftChainSpec(shape[0], shape[1], sp, rng_seed=seed)).graph


def corpus_chain(rec: dict):
    """Chain of one acceptance-corpus record (make_golden.py / test_acceptance.py:292-297)."""
    return ks.RbgpChain((factor(rec["g_o"], rec["sp_o"], rec["seed"]),
                         ks.complete_graph(*rec["g_r"]),
                         factor(rec["g_i"], rec["sp_i"], rec["seed"] + 50000),
                         ks.complete_graph(*rec["g_b"])))


def corpus_inputs(rec: dict, chain, precision: str):
    w = ks.init_random(chain, rec["seed"], precision=precision)
    rng = np.random.default_rng(10_000 + rec["seed"])
    inp = rng.uniform(-1, 1, size=(w.cols, rec["n_cols"])).astype(w.dtype)
    return w, inp


def ring_graph(n, d=2):
    """Cyclic-diagonal biregular graph (same shape as the reference fixture)."""
    return ks.BipartiteGraph(n, n, tuple(tuple(sorted((u + j) % n for j in range(d)))
                                         for u in range(n)))


def example_chain():
    """The reference's four-factor example chain (512 edges, 22 stored)."""
    return ks.RbgpChain((ring_graph(4), ks.BipartiteGraph(2, 2, ((0,), (1,))), ring_graph(4),
                         ks.complete_graph(2, 2)))
