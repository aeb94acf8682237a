"""What the K5 conv epilogue's per-lane NHWC stores cost: VGG19 / WRN conv layers on the debug
library with and without them (option debug bit 4096 drops the conv output stores; ablation only),
and the staged TMA-store epilogue (default) against per-lane stores (option conv_ostage=0).

    python tools/conv_store_ab.py [batch]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_13486_b200 import _native, build  # noqa: E402

_native.use_library(build.build(debug=True))
from paper_2006_13486_b200.conv import sparse_conv2d  # noqa: E402
from paper_2006_13486_b200.rcubs import init_random  # noqa: E402
from paper_2006_13486_b200.vgg import layer_chain  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 32768


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for c_out, c_in, hw, pool in ((64, 64, 32, True), (128, 128, 16, False), (256, 256, 8, False), (512, 512, 4, False),
                              (256, 256, 8, True), (512, 512, 4, True)):
    w = init_random(layer_chain(c_out, c_in, 0.875, seed=11), 1, precision="f32")
    x = torch.randn(batch, hw, hw, c_in, device="cuda").to(torch.bfloat16)
    base = timed(lambda: sparse_conv2d(w, x, 3, relu=True, pool=pool))
    kern = _native.last_kernel()
    with _native.options(debug=4096):
        nost = timed(lambda: sparse_conv2d(w, x, 3, relu=True, pool=pool))
    with _native.options(conv_ostage=0):
        direct = timed(lambda: sparse_conv2d(w, x, 3, relu=True, pool=pool))
    out_mb = batch * (hw // (2 if pool else 1)) ** 2 * c_out * 2 / 1e6
    print(f"{c_out}x{c_in} @{hw}x{hw}{' +pool' if pool else ''} [{kern}]: {base:.3f} ms with stores, "
          f"{nost:.3f} ms without, {direct:.3f} ms with per-lane stores (conv_ostage=0) ({out_mb:.0f} MB out)",
          flush=True)
