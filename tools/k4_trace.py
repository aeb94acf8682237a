"""Per-step timeline of K4 (gathered-block kernel) CTA 0, cold L2: RBGP4_TC_DEBUG bit 8."""
import ctypes
import os
import sys

import numpy as np
import torch

os.environ["RBGP4_TC_DEBUG"] = str(8 | int(os.environ.get("EXTRA", "0")))
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2006_13486_b200 as ks  # noqa: E402
from paper_2006_13486_b200 import _native, workloads as wl  # noqa: E402
from paper_2006_13486_b200.device import device_format  # noqa: E402
from paper_2006_13486_b200.sdmm import launch_sdmm  # noqa: E402

li = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
cfg = wl.vgg19_cifar_512_tc16(0.875)[li]
w = ks.init_random(wl.build_chain(cfg), 1, precision="f32")
dev = torch.device("cuda", 0)
x = torch.rand((w.cols, n), device=dev).to(torch.bfloat16)
o = torch.empty((w.rows, n), device=dev, dtype=torch.bfloat16)
flush = torch.ones(128 << 20, dtype=torch.float32, device=dev)
fmt = device_format(w, dev, torch.bfloat16)
for _ in range(3):
    launch_sdmm(fmt, "bf16", x, o, dev)
flush.sum()
launch_sdmm(fmt, "bf16", x, o, dev)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (4 * 256))()
_native.lib().rbgp4_debug_trace_gather(buf, 4 * 256)
t = np.frombuffer(buf, dtype=np.uint64).reshape(4, 256).astype(np.int64)
e0 = t[3, 0]
print("setup", t[3, 1] - e0, "tmem_full seen", t[3, 2] - e0, "epilogue done", t[3, 3] - e0)
print("epilogue marks (rel. tmem_full): barrier1", t[3, 4] - t[3, 2], "pushed", t[3, 5] - t[3, 2],
      "barrier2", t[3, 6] - t[3, 2], "staged", t[3, 7] - t[3, 2], "bar.sync", t[3, 8] - t[3, 2],
      "stored", t[3, 3] - t[3, 2], "| last chunk: rows loaded+reduced", t[3, 10] - t[3, 2])
print("step   issue   full   lat   mma_done")
for s in range(int(os.environ.get("STEPS", "18"))):
    print(f"{s:4d} {t[0, s]-e0:7d} {t[1, s]-e0:7d} {t[1, s]-t[0, s]:6d} {t[2, s]-e0:8d}")
