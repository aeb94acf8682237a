"""Time the dominant VGG layer (conv10 shape) under RBGP4_TC_DEBUG ablations."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, torch, numpy as np
sys.path.insert(0, %r)
import paper_2006_13486_b200 as ks
from paper_2006_13486_b200 import workloads as wl
from paper_2006_13486_b200.device import device_format
from paper_2006_13486_b200.sdmm import launch_sdmm
cfg = wl.vgg19_cifar_512(0.875)[1]
chain = wl.build_chain(cfg)
w = ks.init_random(chain, 1, precision="f32")
dev = torch.device("cuda", 0)
x = torch.rand((w.cols, cfg.n_cols), device=dev).to(torch.bfloat16)
o = torch.empty((w.rows, cfg.n_cols), device=dev, dtype=torch.bfloat16)
fmt = device_format(w, dev, torch.bfloat16)
for _ in range(5): launch_sdmm(fmt, "bf16", x, o, dev)
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
for _ in range(50): launch_sdmm(fmt, "bf16", x, o, dev)
e.record(); torch.cuda.synchronize()
print("%%.2f us" %% (s.elapsed_time(e) / 50 * 1e3))
''' % ROOT
for mode in sys.argv[1:] or ["0", "1", "2", "4", "3", "7"]:
    if os.environ.get("RBGP4_TC_DEBUG") and len(sys.argv) > 1 and sys.argv[1] == "0":
        mode = os.environ["RBGP4_TC_DEBUG"]
    env = dict(os.environ, RBGP4_TC_DEBUG=mode)
    out = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
    print("debug", mode, out.stdout.strip(), out.stderr.strip()[-300:])
