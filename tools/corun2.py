"""WaS fetch engines alone and beside compute: fetch GB/s per engine / CTA count
(local HBM, unpaced), then the gate/up GEMM (M = 1024) and a 2-layer Qwen3 step's kernel classes
(B = 1024, S_ctx = 384) alone and beside a long-running fetch on another stream.  The compute SM
budget comes from SIDP_SM_BUDGET (read once per process).  Usage:
  SIDP_SM_BUDGET=140 python tools/corun2.py [--fetch-only]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_28095_b200 as P
from sidp_inputs import MODELS, gen

lib = P._abi.lib()
budget = int(os.environ.get("SIDP_SM_BUDGET", "0"))
out = {"budget": budget}
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
nbytes = 1 << 30
src = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
dst = torch.empty_like(src)


def fetch(engine, ctas, n=nbytes, stream=sa):
    P._abi.check(lib.sidp_test_fetch(dst.data_ptr(), src.data_ptr(), n, ctas, engine,
                                     stream.cuda_stream), "fetch")


def timed(fn, reps=5, stream=sa):
    fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


res = {}
for eng, name, ctas_list in ((0, "bulk", (2, 4, 8, 16, 32)), (2, "ldg", (16, 48)), (1, "ce", (0,))):
    for c in ctas_list:
        ms = timed(lambda: fetch(eng, c))
        res[f"{name}_{c}"] = round(nbytes / (ms * 1e-3) / 1e9, 1)
out["fetch_copy_GBps_local"] = res
print(json.dumps(out), flush=True)
if "--fetch-only" in sys.argv:
    sys.exit(0)

M, N, K = 1024, 51200, 5120
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
w = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
y = torch.empty(M, N // 2, device="cuda", dtype=torch.bfloat16)


def gemm():
    P.test_gemm(x, w, y, M, N, K, 3, stream=sb)


def beside(bg, fn):
    """fn's time on sb while `bg` (a long kernel) runs on sa."""
    torch.cuda.synchronize()
    bg()
    t = timed(fn, reps=3, stream=sb)
    sa.synchronize()
    return round(t * 1e3, 1)


big = 8 << 30
big_src = torch.empty(big, dtype=torch.uint8, device="cuda")
big_dst = torch.empty_like(big_src)


def long_fetch(engine, ctas):
    def f():
        P._abi.check(lib.sidp_test_fetch(big_dst.data_ptr(), big_src.data_ptr(), big, ctas, engine,
                                         sa.cuda_stream), "fetch")
    return f


def sleeper():
    with torch.cuda.stream(sa):
        torch.cuda._sleep(2_000_000_000)


g = {"alone": round(timed(gemm, 3, sb) * 1e3, 1),
     "beside_1cta_sleep": beside(sleeper, gemm),
     "beside_bulk8": beside(long_fetch(0, 8), gemm),
     "beside_bulk16": beside(long_fetch(0, 16), gemm),
     "beside_ldg1": beside(long_fetch(2, 1), gemm),
     "beside_ce": beside(long_fetch(1, 0), gemm)}
out["gateup_M1024_us"] = g
print(json.dumps(out), flush=True)

# one 2-layer step's kernel classes
m = MODELS["qwen3-32b"].with_layers(2)
B, ctx_len = 1024, 384
ctx = P.Context(m, rank=0, world=1, max_batch=B, max_ctx=ctx_len + 64, seed=1)
ctx.init_weights_synthetic()
kv = P.KVCache(m, B, ctx_len + 64)
kv.fill_synthetic(1, 0, B, ctx_len)
kv.set_pos(np.full(B, ctx_len))
tok = torch.from_numpy(gen.tokens(1, np.arange(B), m.vocab)).to(torch.int32).cuda()
names = {1: "gate_up", 2: "attn", 4: "down", 5: "qkv", 6: "o", 7: "lm"}


def classes(bg=None):
    torch.cuda.synchronize()
    if bg:
        bg()
    ctx.set_timing(sum(1 << c for c in names))
    for _ in range(3):
        ctx.step(tok, tok, kv, batch=B, stream=sb)
    sb.synchronize()
    st = ctx.stats()
    sa.synchronize()
    return {names[c]: round(st["timed_ms"][c] * 1e3 / max(1, st["timed_launches"][c]), 1)
            for c in names}


out["step_classes_us"] = {"alone": classes(), "beside_bulk8": classes(long_fetch(0, 8)),
                          "beside_bulk16": classes(long_fetch(0, 16)),
                          "beside_ldg48": classes(long_fetch(2, 48)),
                          "beside_ce": classes(long_fetch(1, 0))}
ctx.destroy()
print(json.dumps(out), flush=True)
