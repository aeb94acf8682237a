"""A/B of the WRN block tail on one conv_b per group (batch from argv, bf16): the conv alone, the
conv + torch add + torch relu (unfused), and the residual epilogue (sparse_conv2d(residual=,
relu_copy=True)).  Events around 20 back-to-back repetitions of each.

    python tools/wrn_tail_ab.py [batch]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_13486_b200.conv import sparse_conv2d  # noqa: E402
from paper_2006_13486_b200 import _native  # noqa: E402
from paper_2006_13486_b200.rcubs import init_random  # noqa: E402
from paper_2006_13486_b200.wrn import wrn_layer_chain  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 512


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


for c, hw in ((64, 32), (128, 16), (256, 8)):
    w = init_random(wrn_layer_chain(c, c, 0.875, 3, seed=3), 1, precision="f32")
    x = torch.randn(batch, hw, hw, c, device="cuda").to(torch.bfloat16)
    r = torch.randn(batch, hw, hw, c, device="cuda").to(torch.bfloat16)
    t_conv = timed(lambda: sparse_conv2d(w, x, 3))
    kern = _native.last_kernel()
    t_add = timed(lambda: r + r)
    t_relu = timed(lambda: torch.relu(r))

    def unfused():
        y = sparse_conv2d(w, x, 3) + r
        return y, torch.relu(y)
    t_unf = timed(unfused)
    t_fus = timed(lambda: sparse_conv2d(w, x, 3, residual=r, relu_copy=True))
    kf = _native.last_kernel()
    t_res = timed(lambda: sparse_conv2d(w, x, 3, residual=r))
    mb = batch * hw * hw * c * 2 / 1e6
    print(f"{c}ch {hw}x{hw} ({mb:.0f} MB/act): conv {t_conv:.1f} us [{kern}], add {t_add:.1f}, relu {t_relu:.1f}; "
          f"unfused tail {t_unf:.1f}; fused res+relu {t_fus:.1f} [{kf}]; fused res only {t_res:.1f}", flush=True)
