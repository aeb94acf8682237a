"""BASELINE config 4: sparsity / shape sweep of the RBGP4 product on one B200.

M = K in {1024, 4096, 8192}, N in {4096, 65536}, sparsity 50 / 75 / 87.5 / 93.75 / 96.875 %,
TC16 family (tile 128 x 128, G_b = (16,16), G_i = (8,8) @ .5 / .75, the rest of
the sparsity in G_o), plus the `tc` family (G_b = (8,8), G_i = (16,16) @ .875: the K5 slice
relayout) and the paper family (G_r = (4,1), G_i = (32,64), G_b = (1,1): K2) at M = K = 4096;
bf16 operands, fp32 accumulation, bf16 out, through `rbgp4mm`'s launcher.
Each point: mean of event-timed launches, L2 flushed (256 MB overwrite) before each launch.
Reports effective TFLOP/s (2 nnz N), the HBM and tensor-core roofline fractions (SURVEY §8(d):
T* = max(F / P, B / BW)), and the kernel taken.  Writes profiles/<tag>_sweep.json.

usage: python tools/sweep.py [tag]
"""
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2006_13486_b200 as ks  # noqa: E402
from paper_2006_13486_b200 import _native  # noqa: E402
from paper_2006_13486_b200 import workloads as wl  # noqa: E402
from paper_2006_13486_b200.device import device_format  # noqa: E402
from paper_2006_13486_b200.sdmm import launch_sdmm  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r01b"
with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
    peaks = json.load(fh)
BW, PTC = peaks["hbm_gbs"] * 1e9, peaks["bf16_tflops"] * 1e12
# sparsity -> (sp_o, sp_i)
# (75 %: all of it in g_i, so the point runs the TC16 relayout like 87.5-96.9 %; 50 % needs
# g_i degree 4 and runs the direct gather)
SPLITS = {0.5: (0.0, 0.5), 0.75: (0.0, 0.75), 0.875: (0.5, 0.75), 0.9375: (0.75, 0.75),
          0.96875: (0.875, 0.75)}
dev = torch.device("cuda", 0)
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
rows = []
POINTS = []
for mk in (1024, 4096, 8192):
    for sp, (sp_o, sp_i) in SPLITS.items():
        u = mk // 128
        if sp_o > 0 and u * (1 - sp_o) < 2:
            continue  # g_o right degree < 2: not generatable
        POINTS.append(("tc16", mk, sp, wl.SweepConfig(f"sweep-{mk}-{sp}", (u, u), sp_o, (1, 1), (8, 8), sp_i,
                                                        (16, 16), n_cols=1, seed=mk)))
for sp, sp_o in ((0.875, 0.0), (0.9375, 0.5)):
    POINTS.append(("tc", 4096, sp, wl.SweepConfig(f"sweep-tc-{sp}", (32, 32), sp_o, (1, 1), (16, 16), 0.875,
                                                  (8, 8), n_cols=1, seed=4096)))
for sp, sp_o in ((0.875, 0.5), (0.9375, 0.75)):
    POINTS.append(("paper", 4096, sp, wl.SweepConfig(f"sweep-paper-{sp}", (32, 64), sp_o, (4, 1), (32, 64), 0.75,
                                                     (1, 1), n_cols=1, seed=4096)))
for family, mk, sp, cfg in POINTS:
    if True:
        chain = wl.build_chain(cfg)
        w = ks.init_random(chain, 1, precision="f32")
        fmt = device_format(w, dev, torch.bfloat16)
        for n in (4096, 65536):
            x = (torch.rand((mk, n), device=dev) * 2 - 1).to(torch.bfloat16)
            o = torch.empty((mk, n), device=dev, dtype=torch.bfloat16)
            launch_sdmm(fmt, "bf16", x, o, dev)
            torch.cuda.synchronize()
            kern = _native.last_kernel()
            times = []
            for _ in range(10):
                flush.add_(1)
                a, b = torch.cuda.Event(True), torch.cuda.Event(True)
                a.record()
                launch_sdmm(fmt, "bf16", x, o, dev)
                b.record()
                torch.cuda.synchronize()
                times.append(a.elapsed_time(b) * 1e-3)
            t = statistics.mean(times)
            flops = 2.0 * w.nnz * n
            byts = w.nnz * 2 + 4 * (chain.graphs[0].num_left * len(chain.graphs[0].adjacency[0])
                                    + chain.graphs[2].num_left * len(chain.graphs[2].adjacency[0])) \
                + mk * n * 2 * 2
            t_star = max(flops / PTC, byts / BW)
            rows.append({"family": family, "kernel": kern, "M": mk, "K": mk, "N": n, "sparsity": sp, "us": t * 1e6,
                         "tflops_eff": flops / t / 1e12, "hbm_frac": byts / t / BW, "tc_frac": flops / t / PTC,
                         "roofline_frac": t_star / t, "bound": "tensor" if flops / PTC > byts / BW else "hbm"})
            r = rows[-1]
            print(f"{family:5s} M=K={mk:5d} N={n:6d} sp={sp:.5f}: {r['us']:9.1f} us {r['tflops_eff']:7.1f} TF/s  "
                  f"bound {r['bound']:6s} roofline {r['roofline_frac']:.3f}  ({kern})", flush=True)
            del x, o
        torch.cuda.empty_cache()
out = {"what": "BASELINE config 4 sweep, TC16 / tc / paper families, bf16, cold L2 per launch (kernel per point)",
       "peaks": {"hbm_gbs": peaks["hbm_gbs"], "bf16_tflops": peaks["bf16_tflops"]}, "points": rows}
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", f"{tag}_sweep.json"), "w") as fh:  # copied to profiles/
    json.dump(out, fh, indent=1)
