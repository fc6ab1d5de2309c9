"""The WaS <-> CaS mode switch driven through the PRODUCT on a synthetic long-tail job (SURVEY.md
§8(f) NEXT-2): d computing virtual ranks on one GPU, each holding up
to `--bmax` live requests; a request finishes after a lognormal number of tokens and its slot is
refilled from the rank's queue until the queue is empty, so the per-rank batch decays into a
long tail.  Every step the product's ModeController observes all ranks' batches and issues the
collective-consistent directive (sidp_set_mode at the next step, sidp_set_batches); every rank
runs sidp_step.  Policies: WaS only, CaS only, controller-driven.  Job time = the sum of the
device-timed steps (events on every rank's stream around the step, max over ranks).

On one GPU the ranks' kernels share the SMs and HBM, so the absolute times are not a d-GPU
job's; what is measured is the product's switching path under a live, shrinking workload.
    python tools/longtail_run.py [--world 4] [--layers 8] [--bmax 64] [--requests 192]"""
import argparse
import json
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2605_28095_b200 as P
from paper_2605_28095_b200.orchestrator import CAS, WAS, ModeController, ModePolicy
from sidp_inputs import MODELS, gen

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="qwen3-32b")
ap.add_argument("--world", type=int, default=4)
ap.add_argument("--layers", type=int, default=8)
ap.add_argument("--bmax", type=int, default=64)
ap.add_argument("--requests", type=int, default=192, help="per rank")
ap.add_argument("--median-tokens", type=float, default=24.0)
ap.add_argument("--ctx", type=int, default=256)
ap.add_argument("--bth", type=float, default=24.0)
ap.add_argument("--window", type=int, default=8)
ap.add_argument("--dwell", type=int, default=16)
ap.add_argument("--pace", type=float, default=770.0)
ap.add_argument("--policies", default="was,cas,switch")
a = ap.parse_args()

m = MODELS[a.model].with_layers(a.layers)
d, seed = a.world, 20261017
rng = random.Random(7)
lengths = [[max(1, int(rng.lognormvariate(np.log(a.median_tokens), 0.9))) for _ in range(a.requests)]
           for _ in range(d)]


def job_steps():   # the schedule's step count (host replay of the refill rule)
    live = [list(l[:a.bmax]) for l in lengths]
    queue = [list(l[a.bmax:]) for l in lengths]
    n = 0
    while any(live):
        n += 1
        for r in range(d):
            nxt = [x - 1 for x in live[r] if x > 1]
            while len(nxt) < a.bmax and queue[r]:
                nxt.append(queue[r].pop(0))
            live[r] = nxt
    return n


max_steps = job_steps() + 8


def run(policy):
    ranks = []
    max_ctx = a.ctx + max_steps + 8
    for r in range(d):
        c = P.Context(m, rank=r, world=d, slots=2, max_batch=a.bmax, max_ctx=max_ctx, fetch_sms=8,
                      seed=seed, fetch_pace_gbps=a.pace)
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            c.init_weights_synthetic(stream=st)
            kv = P.KVCache(m, a.bmax, max_ctx)
            kv.fill_synthetic(seed, r * a.bmax, a.bmax, a.ctx, stream=st)
        st.synchronize()
        kv.set_pos(np.full(a.bmax, a.ctx))
        tok = torch.from_numpy(gen.tokens(seed, np.arange(r * a.bmax, (r + 1) * a.bmax), m.vocab)).to(torch.int32).cuda()
        ranks.append([c, st, kv, tok])
    blobs = [c.export_handles() for c, _, _, _ in ranks]
    for c, _, _, _ in ranks:
        c.import_handles(blobs)
    initial = CAS if policy == "cas" else WAS
    ctl = ModeController(ModePolicy(b_threshold=a.bth if policy == "switch" else (-1 if policy == "was" else 1e9),
                                    window=a.window, min_dwell=a.dwell), d, initial=initial)
    if initial == CAS:
        for c, _, _, _ in ranks:
            c.set_mode(CAS, 0)
    # per rank: remaining tokens of each live request, and the queue of waiting requests
    live = [[l for l in lengths[r][:a.bmax]] for r in range(d)]
    queue = [list(lengths[r][a.bmax:]) for r in range(d)]
    total_ms, steps, cas_steps, tokens, switches = 0.0, 0, 0, 0, 0
    mode = initial
    try:
        while any(live[r] for r in range(d)):
            batches = [len(live[r]) for r in range(d)]
            for c, _, _, _ in ranks:
                c.set_batches(batches)
            evs = []
            for r, (c, st, kv, tok) in enumerate(ranks):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                c.step(tok, tok, kv, batch=batches[r], stream=st, advance_pos=batches[r] > 0)
                e1.record(st)
                evs.append((e0, e1))
            torch.cuda.synchronize()
            total_ms += max(e0.elapsed_time(e1) for e0, e1 in evs)
            steps += 1
            cas_steps += mode == CAS
            tokens += sum(batches)
            # requests progress; finished ones are refilled from the queue
            for r in range(d):
                nxt = []
                for rem in live[r]:
                    if rem > 1:
                        nxt.append(rem - 1)
                while len(nxt) < a.bmax and queue[r]:
                    nxt.append(queue[r].pop(0))
                live[r] = nxt
            new = ctl.observe(batches)
            if new != mode:
                switches += 1
                for c, _, _, _ in ranks:
                    c.set_mode(new, c.stats()["steps"] + 0)   # effective at each rank's next step
                mode = new
        timeouts = sum(c.stats()["timeouts"] for c, _, _, _ in ranks)
    finally:
        for c, _, _, _ in ranks:
            c.destroy()
    return {"policy": policy, "world": d, "layers": a.layers, "model": m.name, "bmax": a.bmax,
            "requests_per_rank": a.requests, "steps": steps, "cas_share": round(cas_steps / steps, 3),
            "switches": switches, "job_ms": round(total_ms, 1), "tokens": tokens,
            "tokens_per_s": round(tokens / (total_ms / 1e3), 1), "timeouts": timeouts,
            "b_threshold": a.bth if policy == "switch" else None}


for pol in a.policies.split(","):
    print(json.dumps(run(pol)), flush=True)
    import gc
    gc.collect()
    torch.cuda.empty_cache()   # the KV caches' memory back to the driver for the next contexts
