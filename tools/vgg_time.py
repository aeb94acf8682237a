"""Time the full VGG19-CIFAR RBGP4 inference forward (CUDA graph, device events)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2006_13486_b200.vgg import VGG19Sparse

if len(sys.argv) > 3 and sys.argv[3] == "cudnn-benchmark":
    torch.backends.cudnn.benchmark = True

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
sp = float(sys.argv[2]) if len(sys.argv) > 2 else 0.875
net = VGG19Sparse(sparsity=sp)
x = torch.randn(batch, 32, 32, 3, device="cuda").to(torch.bfloat16)
for _ in range(3):
    net(x)
torch.cuda.synchronize()
# per-stage eager breakdown
ev = []
xx = x.permute(0, 3, 1, 2)
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
from paper_2006_13486_b200.vgg import _dense_conv_relu
s.record(); h = _dense_conv_relu(xx, net.conv1).permute(0, 2, 3, 1).contiguous(); e.record()
ev.append(("conv1+nhwc", s, e))
from paper_2006_13486_b200.vgg import maxpool2x2
for i, (kind, layer) in enumerate(net.layers):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); h = maxpool2x2(h) if kind == "pool" else layer(h); e.record()
    ev.append((f"{kind}{i} {tuple(h.shape[1:])}", s, e))
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record(); h = h.reshape(batch, -1) @ net.fc.t(); e.record(); ev.append(("fc", s, e))
torch.cuda.synchronize()
tot = 0
for name, s, e in ev:
    ms = s.elapsed_time(e); tot += ms
    print(f"{name:28s} {ms*1e3:9.1f} us")
print(f"sum {tot:.3f} ms")
g = torch.cuda.CUDAGraph()
st = torch.cuda.Stream()
st.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(st):
    net(x)
torch.cuda.current_stream().wait_stream(st)
with torch.cuda.graph(g):
    y = net(x)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
K = 10
s.record()
for _ in range(K):
    g.replay()
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / K
print(f"graph forward batch {batch}: {ms:.3f} ms  -> {batch/ms*1e3:.0f} img/s, "
      f"{net.sparse_flops_per_image*batch/ms/1e9:.1f} sparse TFLOP/s")
