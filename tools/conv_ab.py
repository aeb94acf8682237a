"""A/B of plan options on one VGG19 conv layer: python tools/conv_ab.py LAYER BATCH "opt=v,..." ..."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_13486_b200 import _native  # noqa: E402
from paper_2006_13486_b200.vgg import VGG19Sparse  # noqa: E402

li, batch = int(sys.argv[1]), int(sys.argv[2])
net = VGG19Sparse(sparsity=0.875)
convs = [l for k, l in net.layers if k == "conv"]
hw = [32, 16, 16, 8, 8, 8, 8, 4, 4, 4, 4, 2, 2, 2, 2]
layer = convs[li]
c_in = layer.w.cols // 9
x = (torch.rand((batch, hw[li], hw[li], c_in), device="cuda") * 2 - 1).to(torch.bfloat16)
for spec in sys.argv[3:] or [""]:
    opts = {k: int(v) for k, v in (kv.split("=") for kv in spec.split(",") if kv)}
    with _native.options(**opts):
        y = layer(x)
        torch.cuda.synchronize()
        kern = _native.last_kernel()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(10):
                y = layer(x)
        g.replay()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
    print(f"conv{li} {layer.w.rows}x{c_in}@{hw[li]} b={batch} [{spec or 'default'}]: {a.elapsed_time(b) / 10 * 1e3:8.1f} us ({kern})")
