"""Record every product call of the reference's OWN kernel tests, run on the REFERENCE.

Run in the build container, where the reference is importable:

    python tests/golden/make_ref_suite.py

It runs `/root/reference/pkg/tests/test_sdmm.py` (the reference's unit tests of the hot
path) under pytest with the real `kronsparse`, wrapping `kronsparse.rbgp4mm`
and `kronsparse.sdmm_reference` before the test module imports them.  Each call's operands
(chain factors, values, input, tiling), result and WorkReport go to
`tests/golden/ref_suite_calls.npz` (+ `ref_suite_calls.json`, the index), so the GPU box --
which has no /root/reference -- can replay exactly the calls the reference's tests make and
demand the reference's results bit for bit (tests/test_reference_suite.py).
"""

from __future__ import annotations

import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
OUT_NPZ = os.path.join(HERE, "ref_suite_calls.npz")
OUT_JSON = os.path.join(HERE, "ref_suite_calls.json")

PLUGIN = r'''
import json, os, sys
import numpy as np
import kronsparse

_calls, _arrays = [], {}

def _graphs(chain):
    return [[g.num_left, g.num_right, [list(a) for a in g.adjacency]] for g in chain.graphs]

def _store(name, a):
    key = f"a{len(_arrays)}"
    _arrays[key] = np.ascontiguousarray(a)
    return key

def _test_id():
    return os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0]

_rbgp4mm, _sdmm_reference = kronsparse.rbgp4mm, kronsparse.sdmm_reference

def rbgp4mm(w, inp, params):
    out, rep = _rbgp4mm(w, inp, params)
    _calls.append({"fn": "rbgp4mm", "test": _test_id(), "graphs": _graphs(w.chain),
                   "values": _store("v", w.values), "inp": _store("x", np.asarray(inp)),
                   "params": {k: getattr(params, k) for k in ("tm", "tk", "tn", "rm", "rk", "bm", "bk",
                                                           "rn", "bn", "workers")},
                   "out": _store("o", out),
                   "report": {k: int(getattr(rep, k)) for k in ("fma_count", "tiles", "steps_per_tile",
                              "steps_skipped_per_tile", "w_bytes_read", "i_bytes_read")}})
    return out, rep

def sdmm_reference(w, inp):
    out = _sdmm_reference(w, inp)
    rec = {"fn": "sdmm_reference", "test": _test_id(), "inp": _store("x", np.asarray(inp)),
           "out": _store("o", out)}
    if hasattr(w, "chain"):
        rec.update(kind="chain", graphs=_graphs(w.chain), values=_store("v", w.values))
    else:
        rec.update(kind="csr", shape=list(w.shape), indptr=_store("p", w.indptr),
                   indices=_store("i", w.indices), values=_store("v", w.values))
    _calls.append(rec)
    return out

kronsparse.rbgp4mm, kronsparse.sdmm_reference = rbgp4mm, sdmm_reference
import kronsparse.sdmm as _m
_m.rbgp4mm, _m.sdmm_reference = rbgp4mm, sdmm_reference

def pytest_sessionfinish(session, exitstatus):
    np.savez_compressed(os.environ["REF_SUITE_NPZ"], **_arrays)
    with open(os.environ["REF_SUITE_JSON"], "w") as fh:
        json.dump({"source": "reference pkg/tests/test_sdmm.py", "exitstatus": int(exitstatus),
                   "calls": _calls}, fh, indent=0)
'''


def main():
    plugdir = "/tmp/ref_suite_plugin"
    os.makedirs(plugdir, exist_ok=True)
    with open(os.path.join(plugdir, "ref_suite_recorder.py"), "w") as fh:
        fh.write(PLUGIN)
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([plugdir, REF_SRC]), PYTHONDONTWRITEBYTECODE="1",
               REF_SUITE_NPZ=OUT_NPZ, REF_SUITE_JSON=OUT_JSON)
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p", "ref_suite_recorder",
           "--rootdir", REF_TESTS, os.path.join(REF_TESTS, "test_sdmm.py")]
    res = subprocess.run(cmd, env=env, cwd=plugdir, capture_output=True, text=True)
    print(res.stdout[-2000:], res.stderr[-2000:])
    with open(OUT_JSON) as fh:
        meta = json.load(fh)
    print(f"recorded {len(meta['calls'])} calls, pytest exit {meta['exitstatus']}")
    if res.returncode != 0:
        raise SystemExit("the reference's own test_sdmm.py failed on the reference")


if __name__ == "__main__":
    main()
