"""Timeline of one K4 launch on a bench layer (debug library, option debug = 8 | 512), cold L2.

Prints the launch window seen from the device (CTA entry skew, lifetimes, exit tail, from
%globaltimer) next to the event-timed duration, and CTA 0's per-step trace in SM cycles:
producer TMA issue, MMA warp saw `full`, MMAs + commit issued; setup / epilogue marks.

    python tools/k4_timeline.py [layer index (1 = conv10)] [n_cols] [fact] [k=v plan options ...]
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_13486_b200 import _native, build  # noqa: E402

_native.use_library(build.build(debug=True))
import paper_2006_13486_b200 as ks  # noqa: E402
from paper_2006_13486_b200 import workloads as wl  # noqa: E402
from paper_2006_13486_b200.device import device_format  # noqa: E402
from paper_2006_13486_b200.sdmm import launch_sdmm  # noqa: E402

li = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
fact = sys.argv[3] if len(sys.argv) > 3 else "tc16"
for kv in sys.argv[4:]:
    k, v = kv.split("=")
    _native.set_option(k, int(v))
_native.set_option("debug", 8 | 512 | _native.get_option("debug"))
maker = {"tc16": wl.vgg19_cifar_512_tc16, "tc": wl.vgg19_cifar_512_tc}[fact]
cfg = maker(0.875)[li]
w = ks.init_random(wl.build_chain(cfg), 1, precision="f32")
dev = torch.device("cuda", 0)
x = (torch.rand((w.cols, n), device=dev) * 2 - 1).to(torch.bfloat16)
o = torch.empty((w.rows, n), device=dev, dtype=torch.bfloat16)
fmt = device_format(w, dev, torch.bfloat16)
flush = torch.empty(128 << 20, dtype=torch.float32, device=dev)
lib = _native.lib()
lib.rbgp4_debug_trace_gather.argtypes = [ctypes.c_void_p, ctypes.c_int]
lib.rbgp4_debug_cta_stamps.argtypes = [ctypes.c_void_p, ctypes.c_int]
for _ in range(3):
    launch_sdmm(fmt, "bf16", x, o, dev)
evs = []
for rep in range(5):
    flush.add_(1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    launch_sdmm(fmt, "bf16", x, o, dev)
    b.record()
    torch.cuda.synchronize()
    evs.append(a.elapsed_time(b) * 1e3)
tr = np.zeros(4 * 256, dtype=np.uint64)
lib.rbgp4_debug_trace_gather(tr.ctypes.data, tr.size)
tr = tr.reshape(4, 256).astype(np.int64)
st = np.zeros(2 * 4096, dtype=np.uint64)
lib.rbgp4_debug_cta_stamps(st.ctypes.data, st.size)
st = st.reshape(2, 4096).astype(np.int64)
used = np.nonzero(st[0])[0]
ent, ext = st[0][used], st[1][used]
t0 = ent.min()
print(f"layer {cfg.config_id} N={n}: event {np.median(evs):.2f} us (runs {', '.join(f'{e:.1f}' for e in evs)})")
print(f"CTAs {used.size}: entry skew {(ent.max() - t0) / 1e3:.2f} us, span {(ext.max() - t0) / 1e3:.2f} us, "
      f"lifetime p10/p50/p90 {np.percentile(ext - ent, 10) / 1e3:.2f}/{np.percentile(ext - ent, 50) / 1e3:.2f}/"
      f"{np.percentile(ext - ent, 90) / 1e3:.2f} us, exit p10/p90 {(np.percentile(ext, 10) - t0) / 1e3:.2f}/"
      f"{(np.percentile(ext, 90) - t0) / 1e3:.2f} us")
base = tr[3][0]
marks = {k: (tr[3][k] - base) if tr[3][k] else None for k in range(12)}
print("CTA0 marks (cycles from entry):", {k: v for k, v in marks.items() if v is not None})
steps = int(np.count_nonzero(tr[1]))
prev = None
for s in range(steps):
    iss, full, done = (tr[e][s] - base for e in range(3))
    print(f"step {s:3d}: issue {iss:7d}  full {full:7d}  mma-done {done:7d}  (lat {full - iss:6d}, "
          f"mma {done - full:5d}, period {'' if prev is None else full - prev})")
    prev = full
