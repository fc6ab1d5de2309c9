"""One context in CaS mode with world = 1 (it owns every layer and serves its own rows): the CaS
per-layer kernel chain without any cross-rank wait, so ncu can serialise it.  Used to compare the
owner chain's kernel durations with the standalone GEMM microbenchmarks.
    python tools/cas_d1_trace.py [--model qwen3-32b] [--layers 4] [--batch 16] [--ctx 1024] [--iters 3]"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2605_28095_b200 as P
from sidp_inputs import MODELS

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="qwen3-32b")
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--batch", type=int, default=16)
ap.add_argument("--ctx", type=int, default=1024)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--step", action="store_true", help="whole sidp_step calls (CUDA-graph replayed "
                "unless SIDP_GRAPH=0) instead of per-layer sidp_decode_layer")
a = ap.parse_args()
m = MODELS[a.model].with_layers(a.layers)
c = P.Context(m, rank=0, world=1, max_batch=a.batch, max_ctx=a.ctx + a.iters + 16, seed=7)
c.init_weights_synthetic()
kv = P.KVCache(m, a.batch, a.ctx + a.iters + 16)
kv.fill_synthetic(7, 0, a.batch, a.ctx)
kv.set_pos(np.full(a.batch, a.ctx))
c.set_batches([a.batch])
c.set_mode(1, 0)
x = (torch.randn(a.batch, m.hidden, device="cuda") * 0.5).to(torch.bfloat16)
s = torch.cuda.Stream()
from sidp_inputs import gen
tok = torch.from_numpy(gen.tokens(7, np.arange(a.batch), m.vocab)).to(torch.int32).cuda()


def one():
    if a.step:
        c.step(tok, tok, kv, batch=a.batch, stream=s, advance_pos=True)
    else:
        for l in range(m.num_layers):
            c.decode_layer(x, l, 1, kv, batch=a.batch, stream=s)


for it in range(a.iters):
    one()
s.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 5
e0.record(s)
for _ in range(n):
    one()
e1.record(s)
s.synchronize()
what = "sidp_step" if a.step else "decode_layer chain"
print(f"world=1 CaS {what}: {e0.elapsed_time(e1) * 1e3 / n / m.num_layers:.1f} us per layer "
      f"({e0.elapsed_time(e1) / n:.3f} ms per call-set), graph replays {c.stats()['graph_replays']}",
      flush=True)
c.destroy()
