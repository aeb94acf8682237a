"""K1 A/B on a bench layer: python tools/simt_ab.py [layer] [n_cols] -- ffma / exact, wide on / off."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2006_13486_b200 as ks  # noqa: E402
from paper_2006_13486_b200 import _native  # noqa: E402
from paper_2006_13486_b200 import workloads as wl  # noqa: E402
from paper_2006_13486_b200.device import device_format  # noqa: E402
from paper_2006_13486_b200.sdmm import launch_sdmm  # noqa: E402

li = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
dev = torch.device("cuda", 0)
cfg = wl.vgg19_cifar_512_tc16(0.875)[li]
w = ks.init_random(wl.build_chain(cfg), 1, precision="f32")
fmt = device_format(w, dev, torch.float32)
x = torch.rand((w.cols, n), device=dev) * 2 - 1
flops = 2.0 * w.nnz * n
for compute in ("ffma", "exact"):
    ref = None
    for wide, ct in ((-1, 0), (-1, 8), (-1, 16), (-1, 32), (0, 0)):
        with _native.options(simt_wide=wide, simt_ct=ct):
            o = torch.empty((w.rows, n), device=dev)
            launch_sdmm(fmt, compute, x, o, dev)
            torch.cuda.synchronize()
            kern = _native.last_kernel()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                launch_sdmm(fmt, compute, x, o, dev)
            b.record()
            torch.cuda.synchronize()
            us = a.elapsed_time(b) / 20 * 1e3
        same = "" if ref is None else f" bit-identical to wide={-1}: {torch.equal(ref, o)}"
        ref = o if ref is None else ref
        print(f"{cfg.config_id} N={n} {compute:5s} wide={wide:2d} ct={ct:2d}: {us:7.1f} us  {flops / us / 1e6:6.2f} TF/s  ({kern}){same}")
