"""Timeline of one K5 launch (csrc/sdmm_stream.cu) on a bench layer, cold L2 (debug library,
option debug = 512): CTA entry skew, lifetimes and exit tail from %globaltimer, next to the
event-timed duration, plus CTA 0's marks in SM cycles from its entry.

    python tools/k5_timeline.py [layer index (1 = conv10)] [n_cols] [k=v plan options ...]
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
for kv in sys.argv[3:]:
    k, v = kv.split("=")
    _native.set_option(k, int(v))
_native.set_option("debug", 512 | _native.get_option("debug"))
cfg = wl.vgg19_cifar_512_tc16(0.875)[li]
w = ks.init_random(wl.build_chain(cfg), 1, precision="f32")
dev = torch.device("cuda", 0)
x = (torch.rand((w.cols, n), device=dev) * 2 - 1).to(torch.bfloat16)
o = torch.empty((w.rows, n), device=dev, dtype=torch.bfloat16)
fmt = device_format(w, dev, torch.bfloat16)
flush = torch.empty(128 << 20, dtype=torch.float32, device=dev)
lib = _native.lib()
lib.rbgp4_debug_k5.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
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
# back-to-back launches (no flush; the second and later see their predecessor's tail)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(10):
        launch_sdmm(fmt, "bf16", x, o, dev)
g.replay()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
g.replay()
b.record()
torch.cuda.synchronize()
chain10 = a.elapsed_time(b) * 1e3 / 10
flush.add_(1)
launch_sdmm(fmt, "bf16", x, o, dev)
torch.cuda.synchronize()
st = np.zeros(2 * 4096, dtype=np.uint64)
mk = np.zeros(16, dtype=np.uint64)
assert lib.rbgp4_debug_k5(st.ctypes.data, st.size, mk.ctypes.data) == 0
st = st.reshape(2, 4096).astype(np.int64)
used = np.nonzero(st[0])[0]
ent, ext = st[0][used], st[1][used]
t0 = ent.min()
print(f"layer {cfg.config_id} N={n}: event {np.median(evs):.2f} us (runs {', '.join(f'{e:.1f}' for e in evs)}); "
      f"graph of 10 back-to-back (warm L2) {chain10:.2f} us each")
print(f"CTAs {used.size}: entry skew {(ent.max() - t0) / 1e3:.2f} us, span {(ext.max() - t0) / 1e3:.2f} us, "
      f"lifetime p10/p50/p90 {np.percentile(ext - ent, 10) / 1e3:.2f}/{np.percentile(ext - ent, 50) / 1e3:.2f}/"
      f"{np.percentile(ext - ent, 90) / 1e3:.2f} us, exit p10/p90 {(np.percentile(ext, 10) - t0) / 1e3:.2f}/"
      f"{(np.percentile(ext, 90) - t0) / 1e3:.2f} us")
names = {6: "steps loaded (I prod)", 7: "barriers init", 8: "after griddepcontrol.wait", 0: "first W issued",
         1: "first I issued", 2: "first full (MMA warp)", 3: "last acc ready", 11: "warp0 staged",
         4: "last stores issued", 5: "exit"}
print("CTA0 marks (cycles from entry): " + ", ".join(f"{nm} {int(mk[i])}" for i, nm in names.items()))
tr = np.zeros(208, dtype=np.uint64)
lib.rbgp4_debug_k5_trace.argtypes = [ctypes.c_void_p]
assert lib.rbgp4_debug_k5_trace(tr.ctypes.data) == 0
epi = tr[192:].astype(np.int64)
print("epilogue (warp 0, last unit): " + " ".join(str(int(v)) for v in epi if v))
tr = tr[:192].reshape(3, 64).astype(np.int64)
prev = None
for gidx in range(64):
    if tr[1][gidx] == 0 and gidx > 0:
        break
    print(f"  step {gidx:2d}: issued {tr[0][gidx]:6d}  full {tr[1][gidx]:6d}  mma-done {tr[2][gidx]:6d}  lat {tr[1][gidx] - tr[0][gidx]:6d}"
          f"  period {'' if prev is None else tr[1][gidx] - prev}")
    prev = tr[1][gidx]
