import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_28095_b200 as P
from sidp_inputs import MODELS, gen
m = MODELS["tiny"].with_layers(int(os.environ.get("L", "4")))
B = [int(x) for x in os.environ.get("BATCHES", "3,5").split(",")]
d = len(B); mb = max(B); SEED = 1
ctxs, kvs, toks, nxts, streams = [], [], [], [], []
for r in range(d):
    c = P.Context(m, rank=r, world=d, max_batch=mb, max_ctx=80, seed=SEED, pool=os.environ.get("POOL", "layer"))
    c.init_weights_synthetic()
    kv = P.KVCache(m, mb, 80); kv.fill_synthetic(SEED, sum(B[:r]), mb, 80)
    bg = np.arange(sum(B[:r]), sum(B[:r]) + B[r]); kv.set_pos(gen.positions(SEED, bg, 0, 63) if B[r] else [0])
    toks.append(torch.from_numpy(gen.tokens(SEED, bg, m.vocab)).int().cuda()); nxts.append(torch.zeros(mb, dtype=torch.int32, device="cuda"))
    ctxs.append(c); kvs.append(kv); streams.append(torch.cuda.Stream())
blobs = [c.export_handles() for c in ctxs]
for c in ctxs: c.import_handles(blobs); c.set_batches(B); c.set_mode(1, 0)
torch.cuda.synchronize()
for r in range(d):
    with torch.cuda.stream(streams[r]):
        ctxs[r].step(toks[r], nxts[r], kvs[r], batch=B[r], stream=streams[r], logits=torch.zeros(mb, m.vocab, device="cuda"))
import time; time.sleep(float(os.environ.get("WAIT", "3")))
for r in range(d):
    arr = (C.c_uint64 * (d + 2))()
    P._abi.lib().sidp_debug_flags(ctxs[r].h, arr, d + 2)
    print("rank", r, "flags arrive/done/served:", list(arr))
torch.cuda.synchronize()
print("done", [c.stats()["timeouts"] for c in ctxs])
