"""Device timeline of the bench headline step (the eight VGG19 512-channel layers as one CUDA
graph with PDL edges), K5 debug library (option debug = 2048): for every layer, when its CTAs
entered / exited relative to the step's first entry, and CTA 0's first I request, first full
stage, last accumulator ready and last store issue.  Shows what the step's time is made of:
per-layer startup, main loop, epilogue and the launch-to-launch gaps.

    python tools/step_timeline.py [k=v plan options ...]
"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_13486_b200 import _native, build  # noqa: E402

_native.use_library(build.build(debug=True))
import bench  # noqa: E402

args = bench.parse_args(["--steps", "20", "--warmup", "3"])
B = bench.Bench(args)
torch = B.torch
opts = {"debug": 2048}
for kv in sys.argv[1:]:
    k, v = kv.split("=")
    opts[k] = int(v)
with _native.options(**opts):
    layers = bench.build_layers(args.sparsity, args.batch, args.factorisation)
    st = B.setup(layers, "bf16")
flush = torch.empty(64 << 20, dtype=torch.float32, device=B.dev)
ms, _ = B.time_step(st, 20, 3)
flush.add_(1)
with torch.cuda.stream(B.stream):
    st["step"].replay()
torch.cuda.synchronize()
lib = _native.lib()
lib.rbgp4_debug_k5_seq.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
stamps = np.zeros(16 * 3 * 160, dtype=np.uint64)
marks = np.zeros(64, dtype=np.uint64)
assert lib.rbgp4_debug_k5_seq(stamps.ctypes.data, marks.ctypes.data) == 0
stamps = stamps.reshape(16, 3, 160).astype(np.int64)
marks = marks.reshape(16, 4).astype(np.int64)
# the step replay's launches: the n slots with the latest entries, in time order
n = len(layers)
used = [s for s in range(16) if (stamps[s][0] > 0).any()]
used.sort(key=lambda s: stamps[s][0][stamps[s][0] > 0].min())
slots = used[-n:]
t0 = min(stamps[s][0][stamps[s][0] > 0].min() for s in slots)
print(f"step {ms * 1e3:.1f} us (events, no flush); timeline of one replay after a 256 MB flush, us from first entry:")
for i, s in enumerate(slots):
    ent = stamps[s][0][stamps[s][0] > 0] - t0
    ext = stamps[s][1][stamps[s][1] > 0] - t0
    mk = [(m - t0) / 1e3 if m else float("nan") for m in marks[s]]
    print(f"  {layers[i]['name']:>6} CTAs {ent.size:3d}: entry {ent.min() / 1e3:6.2f}..{ent.max() / 1e3:6.2f}  "
          f"exit {ext.min() / 1e3:6.2f}..{ext.max() / 1e3:6.2f} | CTA0 first-I {mk[0]:6.2f} first-full {mk[1]:6.2f} "
          f"acc-ready {mk[2]:6.2f} stores {mk[3]:6.2f}")
    fi = stamps[s][2][: ent.size] - t0
    ok = stamps[s][2][: ent.size] > 0
    d = (fi[ok] - ent[ok]) / 1e3
    print(f"         first-I - entry p10/p50/p90 {np.percentile(d, 10):.2f}/{np.percentile(d, 50):.2f}/{np.percentile(d, 90):.2f} us; "
          f"first-I min/max {fi[ok].min() / 1e3:6.2f}/{fi[ok].max() / 1e3:6.2f}")
