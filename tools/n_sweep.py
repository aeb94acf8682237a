"""Kernel time vs N at a fixed chain (fixed-cost vs per-byte slope), cold L2.

usage: n_sweep.py [layer index (tc factorisation)] -- env knobs pass through
Each sample: read-only 512 MB flush, then events around one launch; mean of 40.
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

li = int(sys.argv[1]) if len(sys.argv) > 1 else 1
dev = torch.device("cuda", 0)
flush = torch.ones(128 << 20, dtype=torch.float32, device=dev)
cfg = {"tc": wl.vgg19_cifar_512_tc, "tc16": wl.vgg19_cifar_512_tc16}[os.environ.get("FACT", "tc")](0.875)[li]
w = ks.init_random(wl.build_chain(cfg), 1, precision="f32")
fmt = device_format(w, dev, torch.bfloat16)
for n in [int(v) for v in os.environ.get("NS", "128,512,1024,2048,4096,8192,16384").split(",")]:
    x = (torch.rand((w.cols, n), device=dev) * 2 - 1).to(torch.bfloat16)
    o = torch.empty((w.rows, n), device=dev, dtype=torch.bfloat16)
    g = torch.cuda.CUDAGraph()
    launch_sdmm(fmt, "bf16", x, o, dev)
    torch.cuda.synchronize()
    s_ = torch.cuda.Stream()
    with torch.cuda.stream(s_):
        launch_sdmm(fmt, "bf16", x, o, dev)
        s_.synchronize()
        with torch.cuda.graph(g, stream=s_):
            launch_sdmm(fmt, "bf16", x, o, dev)
    torch.cuda.synchronize()
    times = []
    for _ in range(int(os.environ.get("REPS", "40"))):
        if not os.environ.get("WARM"):
            flush.sum()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        g.replay()
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e) * 1e3)
    mean = statistics.mean(times)
    byts = w.nnz * 2 + w.cols * n * 2 + w.rows * n * 2
    print(f"N={n:6d} {mean:8.2f} us  {byts / mean / 1e3:8.1f} GB/s  ({byts/1e6:.1f} MB)")
