"""The VGG19 dense first conv at batch 32768: K8 (rbgp4_dense_conv3x3_c3) vs cuDNN's fused conv + ReLU,
events around 10 back-to-back calls each; HBM floor = (input + output bytes) / the measured copy bandwidth."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_13486_b200.vgg import _dense_conv_relu, conv1_columns, dense_conv1_relu  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
x = torch.randn(batch, 32, 32, 3, device="cuda").to(torch.bfloat16)
w = torch.randn(64, 3, 3, 3, device="cuda").to(torch.bfloat16).to(memory_format=torch.channels_last)
wc = conv1_columns(w)


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


t8 = timed(lambda: dense_conv1_relu(x, wc))
tc = timed(lambda: _dense_conv_relu(x.permute(0, 3, 1, 2), w))
nbytes = batch * 32 * 32 * (3 + 64) * 2
try:
    bw = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
except (OSError, KeyError, ValueError):
    bw = 6650.0
floor = nbytes / (bw * 1e9) * 1e3
print(f"batch {batch}: K8 {t8:.3f} ms, cuDNN fused {tc:.3f} ms; HBM floor {floor:.3f} ms "
      f"({nbytes / 1e9:.2f} GB); K8 at {floor / t8:.2f} of it")
