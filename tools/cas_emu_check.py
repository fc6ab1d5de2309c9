"""Quick check of bench.cas_emulation on a reduced model (bounded run): python tools/cas_emu_check.py [layers] [world]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2605_28095_b200 as P
from sidp_inputs import MODELS, WORKLOADS

L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
W = int(sys.argv[2]) if len(sys.argv) > 2 else 8
model = sys.argv[3] if len(sys.argv) > 3 else None
wl = WORKLOADS["M2"]
m = MODELS[model or wl.model].with_layers(L)
class A: pass
a = A(); a.emulate_steps = 2; a.pool = "layer"
a.cas_batches = os.environ.get("CAS_BATCHES", "1,4,16")
ctx = int(os.environ.get("CAS_CTX", "256"))
torch.cuda.set_device(0)
t = time.time()
r = bench.cas_emulation(a, P, m, wl.seed, 0, W, ctx)
print(time.time() - t, "s", r, flush=True)
