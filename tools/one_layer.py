"""A few launches of one bench layer (the ncu --set full target):
    python tools/one_layer.py [layer] [n_cols] [reps] [compute]
layer: index into the tc16 VGG19 512-channel list (1 = conv10, 4 = conv13); compute: bf16
(default) or ffma / exact (f32 operands, K1)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2006_13486_b200 as ks  # noqa: E402
from paper_2006_13486_b200 import workloads as wl  # noqa: E402
from paper_2006_13486_b200.device import device_format  # noqa: E402
from paper_2006_13486_b200.sdmm import launch_sdmm  # noqa: E402

li = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
compute = sys.argv[4] if len(sys.argv) > 4 else "bf16"
dt = torch.bfloat16 if compute == "bf16" else torch.float32
dev = torch.device("cuda", 0)
cfg = wl.vgg19_cifar_512_tc16(0.875)[li]
w = ks.init_random(wl.build_chain(cfg), 1, precision="f32")
fmt = device_format(w, dev, dt)
x = (torch.rand((w.cols, n), device=dev) * 2 - 1).to(dt)
o = torch.empty((w.rows, n), device=dev, dtype=dt)
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
for _ in range(reps):
    flush.add_(1)
    launch_sdmm(fmt, compute, x, o, dev)
torch.cuda.synchronize()
print("ok", cfg.config_id, n)
