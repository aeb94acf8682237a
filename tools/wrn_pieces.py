"""Split one WRN-40-4 fp32 layer into im2col / product / NHWC transpose (event-timed, 5 reps each)."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2006_13486_b200 as ks  # noqa: E402
from paper_2006_13486_b200 import wrn  # noqa: E402

c_out, c_in, hw, batch = (int(a) for a in (sys.argv[1:5] if len(sys.argv) > 4 else (64, 64, 32, 512)))
chain = wrn.wrn_layer_chain(c_out, c_in, 0.875, 3)
w = ks.init_random(chain, 1, precision="f32")
x = torch.randn(batch, hw, hw, c_in, device="cuda")
params = ks.tiling_for_chain(chain, tn=1, rn=1, bn=1)


def ev(f, reps=5):
    f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    t0 = time.perf_counter()
    a.record()
    for _ in range(reps):
        r = f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3, (time.perf_counter() - t0) / reps * 1e6, r


t1, h1, (cols, (b, oh, ow)) = ev(lambda: wrn.im2col(x, 3, 1))
t2, h2, (y, _) = ev(lambda: ks.rbgp4mm(w, cols, params, compute="ffma"))
t3, h3, _ = ev(lambda: wrn.to_nhwc(y, b, oh, ow, True))
t4, h4, _ = ev(lambda: ks.tiling_for_chain(chain, tn=1, rn=1, bn=1))
print(f"{c_out}x{c_in}@{hw} b={batch}: im2col {t1:.1f} us (host {h1:.0f}), rbgp4mm {t2:.1f} us (host {h2:.0f}), "
      f"to_nhwc {t3:.1f} us (host {h3:.0f}), tiling_for_chain host {h4:.0f} us")
