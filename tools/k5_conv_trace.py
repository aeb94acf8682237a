"""Per-step trace of CTA 0 in one K5 conv launch (debug library, option debug = 512):
    python tools/k5_conv_trace.py [conv index] [batch]"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_13486_b200 import _native, build  # noqa: E402

_native.use_library(build.build(debug=True))
from paper_2006_13486_b200.vgg import VGG19Sparse  # noqa: E402

li = int(sys.argv[1]) if len(sys.argv) > 1 else 0
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
net = VGG19Sparse(sparsity=0.875)
convs = [l for k, l in net.layers if k == "conv"]
hw = [32, 16, 16, 8, 8, 8, 8, 4, 4, 4, 4, 2, 2, 2, 2]
layer = convs[li]
c_in = layer.w.cols // 9
x = (torch.rand((batch, hw[li], hw[li], c_in), device="cuda") * 2 - 1).to(torch.bfloat16)
layer(x)
torch.cuda.synchronize()
lib = _native.lib()
with _native.options(debug=512):
    layer(x)
    torch.cuda.synchronize()
print(_native.last_kernel())
mk = np.zeros(16, dtype=np.uint64)
st = np.zeros(2 * 4096, dtype=np.uint64)
lib.rbgp4_debug_k5.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
assert lib.rbgp4_debug_k5(st.ctypes.data, st.size, mk.ctypes.data) == 0
st = st.reshape(2, 4096).astype(np.int64)
used = np.nonzero(st[0])[0]
print(f"CTAs {used.size}, lifetime p50 {np.percentile(st[1][used] - st[0][used], 50) / 1e3:.1f} us")
print("marks:", [int(v) for v in mk])
tr = np.zeros(208, dtype=np.uint64)
lib.rbgp4_debug_k5_trace.argtypes = [ctypes.c_void_p]
assert lib.rbgp4_debug_k5_trace(tr.ctypes.data) == 0
epi = tr[192:].astype(np.int64).reshape(4, 4)
for u in range(4):
    print(f"  unit {u}: epilogue {epi[u][0]} .. {epi[u][1]} ({epi[u][1] - epi[u][0]} cycles); MMA acc_empty wait {epi[u][2]} .. {epi[u][3]}")
tr = tr[:192].reshape(3, 64).astype(np.int64)
prev = None
for g in range(64):
    if tr[1][g] == 0 and g > 0:
        break
    print(f"  step {g:2d}: issued {tr[0][g]:8d}  full {tr[1][g]:8d}  mma-done {tr[2][g]:8d}  lat {tr[1][g] - tr[0][g]:6d}"
          f"  period {'' if prev is None else tr[1][g] - prev}")
    prev = tr[1][g]
