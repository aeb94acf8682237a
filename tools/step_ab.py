"""A/B of plan options on the bench headline step (BASELINE config 2: the eight VGG19-CIFAR
512-channel layers at batch 256, tc16 87.5 %), built exactly as bench.py builds it: one CUDA
graph per step (PDL edges between layers), device-resident inputs.

    python tools/step_ab.py "stages=2" "stages=3" "stream=0" ...

Each argument is a comma-separated list of k=v plan options ("" = defaults).  Prints the step
time (no flush, and with a 256 MB overwrite before each step) and the per-layer event times.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2006_13486_b200 import _native  # noqa: E402


def main():
    sets = sys.argv[1:] or [""]
    args = bench.parse_args(["--steps", "50", "--warmup", "5"])
    B = bench.Bench(args)
    torch = B.torch
    flush = torch.empty(64 << 20, dtype=torch.float32, device=B.dev)
    for spec in sets:
        opts = dict(kv.split("=") for kv in spec.split(",") if kv)
        with _native.options(**{k: int(v) for k, v in opts.items()}):
            layers = bench.build_layers(args.sparsity, args.batch, args.factorisation)
            st = B.setup(layers, "bf16")
        ms, _ = B.time_step(st, 50, 5)
        ms_cold, _ = B.time_step(st, 20, 3, flush=flush)
        lay = B.per_layer(st, 10)
        tf = st["flops"] / (ms * 1e-3) / 1e12
        print(f"[{spec or 'default'}] step {ms * 1e3:.1f} us ({tf:.1f} TF/s), cold step {ms_cold * 1e3:.1f} us; "
              f"layers " + " ".join(f"{v * 1e3:.1f}" for v in lay), flush=True)


if __name__ == "__main__":
    main()
