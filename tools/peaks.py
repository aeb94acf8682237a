"""Measure the two roofline denominators MEASURED_PEAKS.json lacks (the fp32 legs'
fractions rested on a derived 74.4 TF/s): fp32 FFMA (tools/ffma_peak.cu, our own kernel) and
tf32 tensor throughput (cuBLAS fp32 GEMM with TF32 enabled, 8192^3 -- the same method the
driver uses for the bf16 figure), with SM clocks sampled meanwhile.  Writes
profiles/measured_peaks_r02.json; bench.py reads it (falling back to derived figures).

    nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/ffma_peak.cu -o tools/ffma_peak.bin
    python tools/peaks.py
"""
import json
import os
import subprocess
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "measured_peaks_r02.json")


def tf32_tflops(n=8192, reps=10):
    torch.backends.cuda.matmul.allow_tf32 = True
    a = torch.randn(n, n, device="cuda")
    b = torch.randn(n, n, device="cuda")
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return 2 * n ** 3 / (best * 1e-3) / 1e12, best


def main():
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm", "--format=csv,noheader,nounits",
                            "-lms", "50"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    ffma = json.loads(subprocess.run([os.path.join(ROOT, "tools", "ffma_peak.bin")], capture_output=True,
                                     text=True, check=True).stdout)
    tf32, ms = tf32_tflops()
    smi.terminate()
    clocks = [float(line.split(",")[0]) for line in smi.stdout.read().splitlines() if line.strip()]
    res = {"ffma_tflops": ffma["ffma_tflops"], "tf32_tflops": tf32,
           "how": {"ffma": "tools/ffma_peak.cu: 592 CTAs x 512 threads x 8 independent fmaf chains, best of 5",
                   "tf32": f"torch.matmul fp32 8192^3 with allow_tf32 (cuBLAS), best of 10 ({ms:.2f} ms)"},
           "sm_mhz_samples_median": sorted(clocks)[len(clocks) // 2] if clocks else None,
           "gpu": torch.cuda.get_device_name(0)}
    with open(OUT, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    sys.exit(main())
