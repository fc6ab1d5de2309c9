"""Device-ring diagnostics: rank 0 of an emulated d-rank WaS group (serve-only owners, as
bench.py --emulate-only) stepping with CUDA-graph replay; on a timeout, dumps the device fetch
trace and consume log so the stalled slot / epoch is visible.

    python tools/ring_diag.py [--layers 16] [--batch 256] [--ctx 1024] [--steps 6] [--pace 770]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2605_28095_b200 as P
from sidp_inputs import MODELS, gen

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="qwen3-32b")
ap.add_argument("--layers", type=int, default=16)
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--ctx", type=int, default=1024)
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--pace", type=float, default=770.0)
ap.add_argument("--sync-each", action="store_true")
ap.add_argument("--ce-share", type=float, default=0.0)
a = ap.parse_args()

m = MODELS[a.model].with_layers(a.layers)
seed, B, W = 20261017, a.batch, a.world
max_ctx = a.ctx + a.steps + 8
ctx0 = P.Context(m, rank=0, world=W, slots=2, max_batch=B, max_ctx=max_ctx, fetch_sms=16,
                 fetch_engine="sm", seed=seed, fetch_pace_gbps=a.pace, fetch_ce_share=a.ce_share)
peers = []
for r in range(1, W):
    c = P.Context(m, rank=r, world=W, max_batch=B, max_ctx=max_ctx, seed=seed, alloc=False)
    c.alloc_serve_only()
    peers.append(c)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    ctx0.init_weights_synthetic(stream=s)
    for c in peers:
        c.init_weights_synthetic(stream=s)
    kv = P.KVCache(m, B, max_ctx)
    kv.fill_synthetic(seed, 0, B, a.ctx, stream=s)
s.synchronize()
ctx0.import_handles([ctx0.export_handles()] + [c.export_handles() for c in peers])
kv.set_pos(np.full(B, a.ctx))
tok = torch.from_numpy(gen.tokens(seed, np.arange(B), m.vocab)).to(torch.int32).cuda()
print("plan", ctx0.plan(), "stats", {k: v for k, v in ctx0.stats().items()
                                      if k in ("fetch_sms_held", "compute_sms", "stagger_tick_ns")},
      flush=True)
err = None
t0 = time.time()
for i in range(a.steps):
    try:
        ctx0.step(tok, tok, kv, batch=B, stream=s, advance_pos=True)
        if a.sync_each:
            s.synchronize()
            print(f"step {i} ok {time.time() - t0:.2f}s", flush=True)
    except Exception as e:
        err = e
        print(f"step {i}: {e}", flush=True)
        break
try:
    s.synchronize()
except Exception as e:
    print("sync:", e)
print("elapsed", time.time() - t0, flush=True)
tr = ctx0.fetch_trace()
cl = ctx0.consume_log()
t_ref = min([r[5] for r in tr] + [r[4] for r in cl]) if (tr or cl) else 0
print(f"fetch trace ({len(tr)}): j layer slot owner epoch t_start_us t_end_us")
for r in tr[-40:]:
    print("  F", r[0], r[1], r[2], r[3], r[4], round((r[5] - t_ref) / 1e3, 1), round((r[6] - t_ref) / 1e3, 1))
print(f"consume log ({len(cl)}): layer slot tag epoch t_us")
for r in cl[-40:]:
    print("  C", r[0], r[1], r[2], r[3], round((r[4] - t_ref) / 1e3, 1))
print("stats", ctx0.stats())
