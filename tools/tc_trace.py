"""Per-step role timeline of CTA 0 for a VGG layer (RBGP4_TC_DEBUG bit 8).

usage: tc_trace.py [extra debug bits] [layer index]
"""
import ctypes
import os
import sys

import numpy as np
import torch

extra = int(sys.argv[1]) if len(sys.argv) > 1 else 0
li = int(sys.argv[2]) if len(sys.argv) > 2 else 1
os.environ["RBGP4_TC_DEBUG"] = str(extra if extra & 4096 else 8 | extra)
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2006_13486_b200 as ks  # noqa: E402
from paper_2006_13486_b200 import _native, workloads as wl  # noqa: E402
from paper_2006_13486_b200.device import device_format  # noqa: E402
from paper_2006_13486_b200.sdmm import launch_sdmm  # noqa: E402

cfg = (wl.vgg19_cifar_512_tc if os.environ.get("FACT") == "tc" else wl.vgg19_cifar_512)(0.875)[li]
w = ks.init_random(wl.build_chain(cfg), 1, precision="f32")
dev = torch.device("cuda", 0)
x = torch.rand((w.cols, cfg.n_cols), device=dev).to(torch.bfloat16)
o = torch.empty((w.rows, cfg.n_cols), device=dev, dtype=torch.bfloat16)
flush = torch.ones(128 << 20, dtype=torch.float32, device=dev)
fmt = device_format(w, dev, torch.bfloat16)
for _ in range(3):
    launch_sdmm(fmt, "bf16", x, o, dev)
flush.sum()
launch_sdmm(fmt, "bf16", x, o, dev)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (10 * 512))()
_native.lib().rbgp4_debug_trace(buf, 10 * 512)
t = np.frombuffer(buf, dtype=np.uint64).reshape(10, 512).astype(np.int64)
e0 = t[6, 3]
print("entry->table", t[6, 4] - e0, "entry->tmem", t[6, 5] - e0, "entry->setup", t[6, 0] - e0,
      "setup->epi", t[6, 1] - t[6, 0], "epi", t[6, 2] - t[6, 1])
print("MMA-warp totals over all steps: waits %d issue %d" % tuple(t[9, :2]))
d = int(os.environ.get("STEPS", str(min(36, cfg.g_o[1] // 2))))
print("step  B_iss  B_full(mma)  B_lat   A_ready(mma)  dens_s  dens_e  mma_e   W_iss(g) W_full(g)")
for s in range(d):
    print(f"{s:4d} {t[0, s]-e0:7d} {t[7, s]-e0:9d} {t[7, s]-t[0, s]:7d} {t[4, s]-e0:11d} "
          f"{t[2, s]-e0:8d} {t[3, s]-e0:7d} {t[5, s]-e0:7d} {t[1, s]-e0 if s < 10 else 0:9d} "
          f"{t[8, s]-e0 if s < 10 else 0:9d}")
