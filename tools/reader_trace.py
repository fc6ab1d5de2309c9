"""Per-owner concurrent-reader trace ("peak shifting"):
d COMPUTING virtual ranks on one GPU, each with its own paced SM fetch, run WaS steps; every
rank's device fetch trace (layer, owner, first-claim and publish %globaltimer stamps) is merged
and, per owner, the number of ranks reading it at the same time is counted over the timed steps.

Schedules compared: EXEC order + the C-S7 start stagger (the default, S=2), lockstep EXEC (no
stagger, S=2) and the paper's rotated PAPER order with S = d-1.  On NVLink an owner read by k
ranks at once gives each about 1/k of its egress (PAPER.md:356 incast); here the owners are local
HBM and the pace is per reader, so the trace shows the schedule's reader structure, not its
slowdown.

    python tools/reader_trace.py [--world 4] [--layers 16] [--steps 4] [--model qwen3-32b]
Prints one JSON line per schedule."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2605_28095_b200 as P
from sidp_inputs import MODELS, gen

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="qwen3-32b")
ap.add_argument("--world", type=int, default=4)
ap.add_argument("--layers", type=int, default=16)
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--ctx", type=int, default=128)
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--fetch-sms", type=int, default=8)
ap.add_argument("--pace", type=float, default=770.0)
ap.add_argument("--schedules", default="stagger,lockstep,paper")
a = ap.parse_args()

m = MODELS[a.model].with_layers(a.layers)
d, B, seed = a.world, a.batch, 20261017


def run(schedule):
    order = "paper" if schedule == "paper" else "exec"
    slots = d - 1 if schedule == "paper" else 2
    ranks = []
    for r in range(d):
        c = P.Context(m, rank=r, world=d, slots=slots, order=order, max_batch=B,
                      max_ctx=a.ctx + a.steps + 8, fetch_sms=a.fetch_sms, seed=seed,
                      stagger=schedule == "stagger", fetch_pace_gbps=a.pace)
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            c.init_weights_synthetic(stream=st)
            kv = P.KVCache(m, B, a.ctx + a.steps + 8)
            kv.fill_synthetic(seed, r * B, B, a.ctx, stream=st)
        st.synchronize()
        kv.set_pos(np.full(B, a.ctx))
        tok = torch.from_numpy(gen.tokens(seed, np.arange(r * B, (r + 1) * B), m.vocab)).to(torch.int32).cuda()
        ranks.append((c, st, kv, tok))
    blobs = [c.export_handles() for c, _, _, _ in ranks]
    for c, _, _, _ in ranks:
        c.import_handles(blobs)
    try:
        for _ in range(a.steps + 1):   # step 0 warms up (and carries the stagger)
            for c, st, kv, tok in ranks:
                c.step(tok, tok, kv, batch=B, stream=st, advance_pos=True)
        torch.cuda.synchronize()
        ev = []   # (t_start, t_end, owner, rank)
        for r, (c, _, _, _) in enumerate(ranks):
            tr = c.fetch_trace()
            R = len(c.plan())
            for e in tr[R:]:    # skip the warm-up step's fetches
                ev.append((e[5], e[6], e[3], r))
        timeouts = sum(c.stats()["timeouts"] for c, _, _, _ in ranks)
    finally:
        for c, _, _, _ in ranks:
            c.destroy()
    # sweep: per owner, the number of concurrent readers; time-weighted histogram over the span
    t0 = min(e[0] for e in ev)
    t1 = max(e[1] for e in ev)
    hist = {}
    worst = 0
    for o in range(d):
        pts = sorted([(e[0], 1) for e in ev if e[2] == o] + [(e[1], -1) for e in ev if e[2] == o])
        cur, last = 0, None
        for t, dlt in pts:
            if last is not None and cur > 0:
                hist[cur] = hist.get(cur, 0.0) + (t - last)
            cur += dlt
            last = t
            worst = max(worst, cur)
    busy = sum(hist.values())
    return {"schedule": schedule, "order": order, "slots": slots, "world": d,
            "layers": a.layers, "model": m.name, "fetches": len(ev), "timeouts": timeouts,
            "span_ms": (t1 - t0) / 1e6,
            "owner_busy_time_share_by_readers": {str(k): round(v / busy, 4) for k, v in sorted(hist.items())},
            "max_concurrent_readers_per_owner": worst,
            "mean_readers_while_read": round(sum(k * v for k, v in hist.items()) / busy, 3)}


for sch in a.schedules.split(","):
    print(json.dumps(run(sch)), flush=True)
