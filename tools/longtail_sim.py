"""Job-level effect of the WaS <-> CaS mode switch (PAPER.md:228-232,
385-390) on a synthetic offline long-tail job, priced with step times MEASURED on one B200 by
this repo's single-GPU d=8 emulations (profiles/r1_was_emulation_sweep.jsonl and
profiles/r1_cas_was_crossover.txt, Qwen3-32B shape).  The directive comes from the product's
own ModeController (paper_2605_28095_b200/orchestrator.py), fed the per-rank batches every step.

This is a model, not a measurement: step cost(B, mode) is interpolated from the measured points
(WaS: fetch-bound, flat up to B = 256; CaS: all-live 8-rank emulation, which over-states CaS at
large B — DESIGN.md §8.1), the job keeps each rank's batch at min(256, live requests), and
requests finish after a long-tailed number of tokens.  Usage: python tools/longtail_sim.py
"""
from __future__ import annotations

import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_28095_b200.orchestrator import CAS, WAS, ModeController, ModePolicy  # noqa: E402

# measured step times (ms) at S_ctx = 256 (profiles/r1_cas_was_crossover.txt)
WAS_PTS = [(16, 70.86), (64, 70.88), (128, 70.99), (256, 71.14)]
CAS_PTS = [(1, 25.9), (16, 36.8), (32, 43.2), (64, 63.0), (128, 103.4), (256, 184.0)]  # 256: linear extrapolation


def interp(pts, b):
    if b <= pts[0][0]:
        return pts[0][1]
    for (b0, t0), (b1, t1) in zip(pts, pts[1:]):
        if b <= b1:
            return t0 + (t1 - t0) * (b - b0) / (b1 - b0)
    return pts[-1][1]


def step_ms(mode, batches):
    b = max(batches)   # every rank runs the same mode; the step waits for the busiest rank
    if b == 0:
        return 0.0
    return interp(WAS_PTS if mode == WAS else CAS_PTS, b)


def run(policy_mode, b_th=80.0, d=8, reqs_per_rank=8192, bmax=256, seed=7):
    rng = random.Random(seed)
    # long-tail output lengths (lognormal, median ~200 tokens, a few thousand-token stragglers)
    queues = [[max(1, int(rng.lognormvariate(5.3, 0.9))) for _ in range(reqs_per_rank)] for _ in range(d)]
    live = [[] for _ in range(d)]
    ctrl = ModeController(ModePolicy(b_threshold=b_th), d, initial=WAS)
    mode = WAS if policy_mode in ("was", "switch") else CAS
    t_ms, tokens, steps, cas_steps = 0.0, 0, 0, 0
    while any(queues) or any(live):
        for r in range(d):
            while len(live[r]) < bmax and queues[r]:
                live[r].append(queues[r].pop())
        batches = [len(l) for l in live]
        t_ms += step_ms(mode, batches)
        tokens += sum(batches)
        steps += 1
        cas_steps += mode == CAS
        for r in range(d):
            live[r] = [n - 1 for n in live[r] if n > 1]
        if policy_mode == "switch":
            mode = ctrl.observe(batches)
    return {"policy": policy_mode, "job_s": t_ms / 1e3, "tokens": tokens, "steps": steps,
            "cas_step_share": cas_steps / steps, "tok_s_group": tokens / (t_ms / 1e3)}


def main():
    res = [run("was"), run("cas"), run("switch")]
    base = res[0]["job_s"]
    for r in res:
        r["speedup_vs_was_only"] = base / r["job_s"]
    out = {"what": __doc__.strip().splitlines()[0], "b_threshold": 80.0, "results": res}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
