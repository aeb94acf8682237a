"""A few launches of one VGG19 sparse conv layer (the ncu target, or a quick event timing):
    python tools/one_conv.py [conv index into VGG19Sparse.layers] [batch] [reps]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_13486_b200 import _native  # noqa: E402
from paper_2006_13486_b200.vgg import VGG19Sparse  # noqa: E402

li = int(sys.argv[1]) if len(sys.argv) > 1 else 0
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
net = VGG19Sparse(sparsity=0.875)
convs = [l for k, l in net.layers if k == "conv"]
hw = [32, 16, 16, 8, 8, 8, 8, 4, 4, 4, 4, 2, 2, 2, 2]
layer = convs[li]
c_in = layer.w.cols // 9
x = (torch.rand((batch, hw[li], hw[li], c_in), device="cuda") * 2 - 1).to(torch.bfloat16)
y = layer(x)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    y = layer(x)
b.record()
torch.cuda.synchronize()
print(f"conv{li}: {layer.w.rows}x{c_in} @{hw[li]}x{hw[li]} batch {batch}: {a.elapsed_time(b) / reps * 1e3:.1f} us/launch "
      f"({_native.last_kernel()})")
