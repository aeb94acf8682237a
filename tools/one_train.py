"""A few K7 (bf16 pattern weight gradient) launches on the conv10 shape (ncu target)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2006_13486_b200 as ks  # noqa: E402
from paper_2006_13486_b200 import training  # noqa: E402
from paper_2006_13486_b200 import workloads as wl  # noqa: E402

cfg = wl.vgg19_cifar_512_tc16(0.875)[1]
w = ks.init_random(wl.build_chain(cfg), 1, precision="f32")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
d_out = (torch.rand((w.rows, n), device="cuda") * 2 - 1).to(torch.bfloat16)
x = (torch.rand((w.cols, n), device="cuda") * 2 - 1).to(torch.bfloat16)
for _ in range(3):
    g = training.sddmm(w, d_out, x)
torch.cuda.synchronize()
print("ok", g.shape)
