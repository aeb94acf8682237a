"""Per-layer time of the WRN-40-4 forward (bf16 tcgen05 or fp32 FFMA), batch from argv."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_13486_b200.wrn import WRN40_4Sparse, im2col  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 512
compute = sys.argv[2] if len(sys.argv) > 2 else "bf16"
net = WRN40_4Sparse()
x = torch.randn(batch, 32, 32, 3, device="cuda")
net(x, compute=compute)
torch.cuda.synchronize()
act = torch.bfloat16 if compute == "bf16" else torch.float32
h = torch.randn(batch, 32, 32, 16, device="cuda").to(act)
rows = {}
for bi, (a, b, sc) in enumerate(net.blocks):
    for name, layer, inp in (("a", a, h), ("b", b, None), ("s", sc, h)):
        if layer is None:
            continue
        if inp is None:
            oh = h.shape[1] // a.stride
            inp = torch.randn(batch, oh, oh, layer.c_in, device="cuda").to(act)
        for _ in range(2):
            net._conv(layer, inp, False, compute)
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        y = net._conv(layer, inp, False, compute)
        e.record()
        torch.cuda.synchronize()
        key = f"{layer.c_out}x{layer.c_in}x{layer.k}s{layer.stride}@{inp.shape[1]}"
        rows.setdefault(key, []).append(s.elapsed_time(e))
    h = torch.randn(batch, h.shape[1] // a.stride, h.shape[2] // a.stride, a.c_out, device="cuda").to(act)
tot = 0.0
for k, v in rows.items():
    tot += sum(v)
    print(f"{k:24s} x{len(v):2d}  {sum(v) / len(v) * 1e3:9.1f} us each  {sum(v):8.3f} ms")
print(f"sum of sparse convs {tot:.2f} ms ({compute}, batch {batch})")
