import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_13486_b200 as ks
from paper_2006_13486_b200 import workloads as wl
cfg = wl.SweepConfig("k4", (4, 36), 0.5, (1, 1), (8, 8), 0.75, (16, 16), n_cols=1, seed=512)
w = ks.init_random(wl.build_chain(cfg), 3, precision="f32")
x = torch.rand((w.cols, int(sys.argv[1]) if len(sys.argv) > 1 else 512), device="cuda").to(torch.bfloat16)
p = ks.tiling_for_chain(w.chain, tn=1, rn=1, bn=1)
y, _ = ks.rbgp4mm(w, x, p, compute="bf16")
torch.cuda.synchronize()
print("ok", float(y.float().abs().sum()))
