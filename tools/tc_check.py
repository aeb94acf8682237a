"""Print rel-L2 of the tensor-core modes against the f64 oracle on every golden case."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import oracle  # noqa: E402
import paper_2006_13486_b200 as ks  # noqa: E402
from paper_2006_13486_b200 import workloads as wl  # noqa: E402
from conftest import case_config  # noqa: E402

g = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))
for cid, entry in g["cases"].items():
    chain, w, inp = wl.make_operands(case_config(entry, "f32", cid))
    p = ks.tiling_for_chain(chain, tn=entry["tn"], rn=entry["rn"], bn=entry["bn"])
    ref = oracle.reference_product(ks.RcubsMatrix(chain, w.values.astype(np.float64)),
                                   inp.astype(np.float64), threads=8)
    for comp in ("tf32", "bf16"):
        try:
            out, _ = ks.rbgp4mm(w, inp, p, compute=comp)
            torch.cuda.synchronize()
            print(cid, comp, p.tm, p.tk, "rel_l2=%.3e" % oracle.rel_l2(out, ref), flush=True)
        except Exception as e:  # report and continue
            print(cid, comp, p.tm, p.tk, "ERR", str(e)[:150], flush=True)
