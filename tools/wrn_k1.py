"""K1 (fp32 FFMA) on a WRN-40-4 layer's materialised im2col: python tools/wrn_k1.py [c_out c_in hw batch]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2006_13486_b200 as ks  # noqa: E402
from paper_2006_13486_b200 import _native  # noqa: E402
from paper_2006_13486_b200.device import device_format  # noqa: E402
from paper_2006_13486_b200.sdmm import launch_sdmm  # noqa: E402
from paper_2006_13486_b200.wrn import wrn_layer_chain  # noqa: E402

c_out, c_in, hw, batch = (int(a) for a in (sys.argv[1:5] if len(sys.argv) > 4 else (64, 64, 32, 512)))
chain = wrn_layer_chain(c_out, c_in, 0.875, 3)
w = ks.init_random(chain, 1, precision="f32")
dev = torch.device("cuda", 0)
fmt = device_format(w, dev, torch.float32)
n = batch * hw * hw
x = torch.rand((w.cols, n), device=dev) * 2 - 1
o = torch.empty((w.rows, n), device=dev)
for ct in (0, 8, 16, 32):
    with _native.options(simt_ct=ct):
        launch_sdmm(fmt, "ffma", x, o, dev)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        for _ in range(5):
            launch_sdmm(fmt, "ffma", x, o, dev)
        b.record()
        torch.cuda.synchronize()
    us = a.elapsed_time(b) / 5 * 1e3
    print(f"{c_out}x{c_in}@{hw} b={batch} (tm {chain.num_left // chain.graphs[0].num_left}, bm {chain.graphs[3].num_left}) "
          f"ct={ct}: {us:8.1f} us  {2 * w.nnz * n / us / 1e6:6.2f} TF/s  {x.numel() * 4 / us / 1e3:7.1f} GB/s of I  ({_native.last_kernel()})")
