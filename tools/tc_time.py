"""Device time of the tensor-core kernel on VGG layer shapes, cold L2.

Each sample: a read-only flush over 512 MB (evicts the operands without leaving
dirty lines), then CUDA events around ONE launch queued behind the flush, so the
GPU never idles waiting for the host.  Prints the median per shape.
Env knobs (RBGP4_TC_TN / RBGP4_TC_KSPLIT / RBGP4_TC_DEBUG) pass through.
"""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2006_13486_b200 as ks  # noqa: E402
from paper_2006_13486_b200 import workloads as wl  # noqa: E402
from paper_2006_13486_b200.device import device_format  # noqa: E402
from paper_2006_13486_b200.sdmm import launch_sdmm  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.ones(128 << 20, dtype=torch.float32, device=dev)  # 512 MB
layers = {"conv9": 0, "conv10": 1, "conv13": 4}
which = sys.argv[1:] or list(layers)
for name in which:
    maker = wl.vgg19_cifar_512_tc if os.environ.get("FACT") == "tc" else wl.vgg19_cifar_512
    cfg = maker(0.875)[layers[name]]
    w = ks.init_random(wl.build_chain(cfg), 1, precision="f32")
    x = (torch.rand((w.cols, cfg.n_cols), device=dev) * 2 - 1).to(torch.bfloat16)
    o = torch.empty((w.rows, cfg.n_cols), device=dev, dtype=torch.bfloat16)
    fmt = device_format(w, dev, torch.bfloat16)
    launch_sdmm(fmt, "bf16", x, o, dev)
    torch.cuda.synchronize()
    times = []
    for _ in range(15):
        flush.sum()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        launch_sdmm(fmt, "bf16", x, o, dev)
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e) * 1e3)
    med = statistics.median(times)
    byts = w.nnz * 2 + w.cols * cfg.n_cols * 2 + w.rows * cfg.n_cols * 2
    print(f"{name} (M,K,N)=({w.rows},{w.cols},{cfg.n_cols}) {med:7.2f} us  {byts / med / 1e3:7.1f} GB/s")
