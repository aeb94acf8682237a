"""The reference's OWN tests of the hot path, against this package.

Two halves, because the GPU box has no /root/reference and this container has no GPU:

* CPU (this container): `/root/reference/pkg/tests/test_sdmm.py` runs UNMODIFIED with
  `kronsparse` resolved to `paper_2006_13486_b200` (a sys.modules alias installed by a pytest
  plugin).  Every test that needs no device -- tiling derivation, the validation errors and
  their messages, work accounting done before the launch, the dense baseline -- must pass;
  every other test must fail with DeviceError and nothing else (no silent CPU path).
* GPU: every product call those reference tests make, recorded on the reference itself by
  tests/golden/make_ref_suite.py (operands, tiling, result, WorkReport), is replayed through
  `rbgp4mm` / `sdmm_reference` here: results bit-identical, WorkReports equal.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys
import xml.etree.ElementTree as ET

import numpy as np
import pytest

import paper_2006_13486_b200 as ks

from conftest import ROOT

REF_TESTS = "/root/reference/pkg/tests"
GOLDEN = os.path.join(ROOT, "tests", "golden")

ALIAS_PLUGIN = r'''
import sys
import paper_2006_13486_b200 as _pkg
from paper_2006_13486_b200 import (errors, generate, graphs, products, rcubs, sdmm)
sys.modules["kronsparse"] = _pkg
for _name, _mod in dict(errors=errors, generate=generate, graphs=graphs, products=products,
                        rcubs=rcubs, sdmm=sdmm).items():
    sys.modules["kronsparse." + _name] = _mod
'''


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference tests not present (GPU box)")
def test_reference_test_sdmm_runs_unmodified_against_the_package(tmp_path):
    plug = tmp_path / "kronsparse_alias.py"
    plug.write_text(ALIAS_PLUGIN)
    junit = tmp_path / "junit.xml"
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(tmp_path), ROOT]), PYTHONDONTWRITEBYTECODE="1",
               CUDA_VISIBLE_DEVICES="")
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p", "kronsparse_alias",
           "--rootdir", REF_TESTS, f"--junitxml={junit}", os.path.join(REF_TESTS, "test_sdmm.py")]
    subprocess.run(cmd, env=env, cwd=str(tmp_path), capture_output=True, text=True, timeout=600)
    cases = ET.parse(junit).getroot().iter("testcase")
    passed, device_only, other = [], [], []
    for c in cases:
        name = c.get("name")
        fail = c.find("failure")
        err = c.find("error")
        bad = fail if fail is not None else err
        if bad is None:
            passed.append(name)
        elif "DeviceError" in (bad.get("message", "") + (bad.text or "")):
            device_only.append(name)
        else:
            other.append((name, bad.get("message", "")[:200]))
    assert not other, other
    # host-side contract of the reference's suite holds without a device
    for must in ("test_all_violations_reported_at_once", "test_incomplete_repeat_factor_rejected",
                 "test_short_chain_unsupported", "test_repetition_group_dimensions",
                 "test_fixed_tile_graph_shape", "test_shape_mismatch", "test_dtype_mismatch",
                 "test_columns_not_divisible_by_tn", "test_inconsistent_params_rejected",
                 "test_row_repetition_groups", "test_dense_gemm_shape_error"):
        assert must in passed, (must, passed)
    # and every product raises DeviceError on a box without a GPU (no fallback)
    assert "test_identity_passthrough_is_bit_exact" in device_only
    assert len(passed) + len(device_only) == 29


def _chain(graphs):
    return ks.RbgpChain(tuple(ks.BipartiteGraph(nl, nr, tuple(tuple(a) for a in adj))
                              for nl, nr, adj in graphs))


@pytest.fixture(scope="module")
def recorded():
    with open(os.path.join(GOLDEN, "ref_suite_calls.json")) as fh:
        meta = json.load(fh)
    return meta["calls"], np.load(os.path.join(GOLDEN, "ref_suite_calls.npz"))


def test_recording_covers_the_reference_kernel_tests(recorded):
    calls, _ = recorded
    tests = {c["test"].split("::")[-1] for c in calls}
    assert {"test_identity_passthrough_is_bit_exact", "test_bit_identical_across_worker_counts",
            "test_micro_block_factors_exercised", "test_fma_and_skip_counts_exact",
            "test_io_volume_monotone_in_outer_sparsity", "test_reference_accepts_csr_triple"} <= {
        t.split("[")[0] for t in tests}
    assert sum(c["fn"] == "rbgp4mm" for c in calls) >= 15


@pytest.mark.gpu
def test_reference_suite_calls_replay_bit_identical(recorded):
    """Each rbgp4mm / sdmm_reference call of the reference's test_sdmm.py, on the B200: the
    reference's own output bit for bit (exact mode) and its WorkReport field for field."""
    calls, arr = recorded
    for c in calls:
        inp = arr[c["inp"]]
        if c["fn"] == "rbgp4mm":
            w = ks.RcubsMatrix(_chain(c["graphs"]), arr[c["values"]])
            out, rep = ks.rbgp4mm(w, inp, ks.TilingParams(**c["params"]))
            assert np.array_equal(out, arr[c["out"]]), c["test"]
            got = {k: getattr(rep, k) for k in c["report"]}
            assert got == c["report"], (c["test"], got, c["report"])
        else:
            if c["kind"] == "chain":
                w = ks.RcubsMatrix(_chain(c["graphs"]), arr[c["values"]])
            else:
                w = ks.CsrMatrix(arr[c["indptr"]], arr[c["indices"]], arr[c["values"]], tuple(c["shape"]))
            out = ks.sdmm_reference(w, inp)
            assert np.array_equal(out, arr[c["out"]]), c["test"]


@pytest.mark.gpu
def test_worker_count_and_gpu_count_invariance(recorded):
    """Reference sdmm.py:18-20 (bit-identical for any worker count) -> identical for any
    `workers` knob and for any column split of the batch (what a GPU shard sees)."""
    calls, arr = recorded
    c = next(c for c in calls if "test_bit_identical_across_worker_counts" in c["test"])
    w = ks.RcubsMatrix(_chain(c["graphs"]), arr[c["values"]])
    inp = arr[c["inp"]]
    p = ks.TilingParams(**c["params"])
    full = ks.rbgp4mm(w, inp, p)[0]
    for n in (1, 2, 8):
        assert np.array_equal(ks.rbgp4mm(w, inp, ks.with_workers(p, n))[0], full)
    for shards in (2, 4):
        step = inp.shape[1] // shards
        parts = [ks.rbgp4mm(w, np.ascontiguousarray(inp[:, i * step:(i + 1) * step]), p)[0]
                 for i in range(shards)]
        assert np.array_equal(np.concatenate(parts, axis=1), full)


REF_OBJECTS = r'''
import sys
import numpy as np
sys.path.insert(0, "/root/reference/pkg/src")
import kronsparse as kr                     # the reference itself
import paper_2006_13486_b200 as ks          # this package (its own modules, no alias)
from paper_2006_13486_b200.errors import DeviceError
g = [kr.complete_graph(2, 4), kr.complete_graph(1, 1),
     kr.generate_ramanujan(kr.LiftChainSpec(8, 8, 0.75, rng_seed=3)).graph, kr.complete_graph(16, 16)]
chain = kr.RbgpChain(tuple(g))
w = kr.init_random(chain, kr.make_rng(5), precision="f32")
params = ks.tiling_for_chain(w.chain)                       # our tiling on the reference's chain
assert params == ks.TilingParams(**{f: getattr(kr.tiling_for_chain(w.chain), f)
                                    for f in ks.TilingParams.__dataclass_fields__})
inp = np.ones((w.cols, 256), dtype=np.float32)
try:
    ks.rbgp4mm(w, inp, params)                              # validation accepts it; no GPU here
except DeviceError:
    print("DEVICE-ONLY")
'''


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference not present (GPU box)")
def test_reference_built_objects_reach_the_device(tmp_path):
    """Route 1's claim: an RcubsMatrix / RbgpChain built by the reference itself
    goes through this package's tiling and rbgp4mm validation unchanged (duck-typed on
    .chain / .values) -- on this GPU-less host the call ends in DeviceError, i.e. at the device."""
    env = dict(os.environ, PYTHONPATH=ROOT, CUDA_VISIBLE_DEVICES="")
    res = subprocess.run([sys.executable, "-c", REF_OBJECTS], env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    assert "DEVICE-ONLY" in res.stdout
