import os, sys, torch
sys.path.insert(0, "/root/repo")
from paper_2006_13486_b200.wrn import WRN40_4Sparse, im2col
from paper_2006_13486_b200.sdmm import rbgp4mm, tiling_for_chain
net = WRN40_4Sparse()
layer = net.blocks[0][2]  # 64x16 1x1 shortcut
x = torch.randn(512, 32, 32, 16, device="cuda").to(torch.bfloat16)
def t(f, n=3):
    f(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(n): r = f()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n * 1e3, r
us, (cols, shp) = t(lambda: im2col(x, 1, 1))
print("im2col", us, cols.shape, cols.dtype, cols.is_contiguous())
p = tiling_for_chain(layer.w.chain, tn=1, rn=1, bn=1)
us2, (y, _) = t(lambda: rbgp4mm(layer.w, cols, p, compute="bf16"))
print("rbgp4mm", us2, y.shape)
us3, _ = t(lambda: y.view(64, 512, 32, 32).permute(1, 2, 3, 0).contiguous())
print("permute", us3)
import paper_2006_13486_b200._native as nat
os.environ["RBGP4_TC_DEBUG"] = "8192"
rbgp4mm(layer.w, cols, p, compute="bf16"); torch.cuda.synchronize()
