"""Per-CTA entry/exit timeline of one K4 launch (RBGP4_TC_DEBUG bit 512), cold L2.

Prints the launch window seen from the device: CTA entry skew, per-CTA lifetime percentiles,
exit tail, next to the event-timed duration of the same launch."""
import ctypes
import os
import sys

import numpy as np
import torch

os.environ["RBGP4_TC_DEBUG"] = str(512 | int(os.environ.get("EXTRA", "0")))
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2006_13486_b200 as ks  # noqa: E402
from paper_2006_13486_b200 import _native, workloads as wl  # noqa: E402
from paper_2006_13486_b200.device import device_format  # noqa: E402
from paper_2006_13486_b200.sdmm import launch_sdmm  # noqa: E402

li = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg = wl.vgg19_cifar_512_tc16(0.875)[li]
w = ks.init_random(wl.build_chain(cfg), 1, precision="f32")
dev = torch.device("cuda", 0)
n = cfg.n_cols
x = torch.rand((w.cols, n), device=dev).to(torch.bfloat16)
o = torch.empty((w.rows, n), device=dev, dtype=torch.bfloat16)
flush = torch.ones(64 << 20, dtype=torch.float32, device=dev)
fmt = device_format(w, dev, torch.bfloat16)
for _ in range(3):
    launch_sdmm(fmt, "bf16", x, o, dev)
flush.add_(1)
a, b = torch.cuda.Event(True), torch.cuda.Event(True)
a.record()
launch_sdmm(fmt, "bf16", x, o, dev)
b.record()
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (2 * 4096))()
_native.lib().rbgp4_debug_cta_stamps(buf, 2 * 4096)
st = np.frombuffer(buf, dtype=np.uint64).reshape(2, 4096).astype(np.int64)
ncta = int(np.count_nonzero(st[0]))
s0, s1 = st[0, :ncta], st[1, :ncta]
t0 = s0.min()
life = (s1 - s0) / 1e3
print(f"{cfg.config_id}: event-timed {a.elapsed_time(b) * 1e3:.2f} us, {ncta} CTAs")
print(f"  CTA entry skew: max {(s0.max() - t0) / 1e3:.2f} us, p50 {(np.median(s0) - t0) / 1e3:.2f} us")
print(f"  CTA lifetime us: min {life.min():.2f} p50 {np.median(life):.2f} p90 {np.percentile(life, 90):.2f} max {life.max():.2f}")
print(f"  first entry -> last exit: {(s1.max() - t0) / 1e3:.2f} us")
