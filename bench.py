#!/usr/bin/env python
"""Decode-throughput benchmark of the B200-native SiDP WaS hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload M2]

N=1 runs configs[1] (Qwen3-32B shape, B=256/GPU, S_ctx=1024; 64 layers, bf16) on one GPU
(d=1: every layer owned; the WaS ring is idle).  N>1 (torchrun, one process per GPU, NCCL
for the control plane only) runs SiDP WaS over d=N ranks: each rank owns L/d layers and
streams the rest over NVLink into S=2 cache slots (EXEC order + C-S7 stagger).

One step = one full decode step of the whole hot path (embedding, L layers, LM head with
fused argmax) over B rows per GPU; tokens and positions are advanced on the device by the
library, so the timed loop launches only library kernels.  Prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode tokens/s at 1/2/4/8 B200 (WaS); fraction of per-layer roofline"
UNIT = "tokens/s"
CLS_NAMES = {1: "gate_up_gemm", 2: "attention", 3: "fetch", 4: "down_gemm", 5: "qkv_gemm",
             6: "o_gemm", 7: "lm_head_gemm"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="M2")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--ctx", type=int, default=None)
    ap.add_argument("--layers", type=int, default=None, help="override (marks config reduced)")
    ap.add_argument("--slots", type=int, default=None)
    ap.add_argument("--order", default="exec", choices=["exec", "paper"])
    ap.add_argument("--pool", default="layer", choices=["layer", "ffn"])
    ap.add_argument("--fetch", default="sm", choices=["sm", "ce"],
                    help="WaS fetch engine: the SM fetch kernel (default: TMA bulk copies on "
                         "--fetch-sms dedicated SMs, device epoch flags) or the copy engine + CUDA "
                         "events (the paper's mechanism, A/B baseline)")
    ap.add_argument("--fetch-sms", type=int, default=24)
    ap.add_argument("--slot-parts", type=int, default=0, choices=[0, 1, 2],
                    help="WaS cache granularity: 1 whole layers, 2 tiles (per-component flags); 0 = 1")
    ap.add_argument("--paged", action="store_true",
                    help="paged KV cache (16-token blocks in a shuffled pool, sidp_kv.block_table)")
    ap.add_argument("--no-stagger", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-rows", type=int, default=4,
                    help="rows of the oracle sample (cpu_baseline and --impl reference)")
    ap.add_argument("--emulate-world", type=int, default=8,
                    help="N=1 only: also time rank 0 of a d-rank WaS group on this GPU, the d-1 "
                         "owners being serve-only contexts in local HBM (0 = off)")
    ap.add_argument("--emulate-fetch-sms", type=int, default=24,
                    help="SMs the emulated rank's fetch kernel holds (the real-run default, 16)")
    ap.add_argument("--emulate-ce-share", type=float, default=0.0,
                    help="hybrid fetch of the emulated rank: share of each layer copied by the "
                         "copy engine (sidp_config.fetch_ce_share)")
    ap.add_argument("--emulate-pace-gbps", type=float, default=770.0,
                    help="the emulated rank's fetch kernel paces itself to this rate: the NVLink 5 "
                         "reader rate (B200_PROFILING.md measured peer copy); 0 = unpaced")
    ap.add_argument("--emulate-batch", type=int, default=None)
    ap.add_argument("--emulate-ctx", type=int, default=None)
    ap.add_argument("--emulate-steps", type=int, default=4)
    ap.add_argument("--alias-owners", action="store_true",
                    help="timing only: the d-1 serve-only owners share ONE arena "
                         "(sidp_alloc_serve_only_alias), so the KV cache of big points fits")
    ap.add_argument("--emulate-only", action="store_true",
                    help="skip the d=1 run (shapes whose weights do not fit one GPU, e.g. M3 "
                         "Llama-3.1-70B) and print only the WaS emulation line")
    ap.add_argument("--cas-emulate", type=int, default=1,
                    help="N=1 only: time CaS steps of --emulate-world virtual ranks on this GPU "
                         "(small-batch tail, SURVEY.md M5 analogue; 0 = off)")
    ap.add_argument("--cas-ctx", type=int, default=1024)
    ap.add_argument("--cas-batches", default="1,4,16",
                    help="all-live per-rank batches of the CaS emulation (B=16 also runs the "
                         "half-live and one-live dummy patterns)")
    ap.add_argument("--m3-emulate", type=int, default=1,
                    help="N=1 only: also time the north-star point — M3, Llama-3.1-70B WaS d=8 at "
                         "B=1024 / S_ctx=384 (the measured B_e, max KV with aliased owners) — in a "
                         "child process (0 = off)")
    ap.add_argument("--cas-only", action="store_true",
                    help="print only the CaS emulation (run as a child of the default bench)")
    ap.add_argument("--extra-timeout", type=int, default=240,
                    help="seconds each child measurement (WaS / CaS emulation) may take")
    ap.add_argument("--share-gpu", action="store_true",
                    help="all ranks on cuda:0 with a gloo control plane (functional multi-process "
                         "test of the IPC path on a 1-GPU box; not a scaling number)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampled every 200 ms during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.idx)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "power_w_max": max(power) if power else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ----------------------------------------------------------------------------- cpu oracle
def oracle_sample(m, seed, rows, ctx_len, timed_iters=1):
    """Time the fp64 oracle on a bounded sample: one decoder layer for `rows` rows at the
    workload's shapes and context, plus the LM head on a 1/16 vocab slice (scaled).  Returns
    (tokens/s extrapolated to the full L-layer step, description, cores)."""
    import numpy as np
    from oracle import model as OM
    from sidp_inputs import gen
    bg = np.arange(rows)
    p = gen.layer_params(seed, m, 0)
    T = ctx_len + 1
    K = gen.kv(seed, gen.KCACHE, 0, bg, range(T), m.n_kv_heads, m.head_dim)
    V = gen.kv(seed, gen.VCACHE, 0, bg, range(T), m.n_kv_heads, m.head_dim)
    x = gen.activations(seed, 0, bg, m.hidden)
    pos = np.full(rows, ctx_len)
    vs = max(1, m.vocab // 16)
    head = {"g_final": gen.gain(seed, gen.G_FINAL, 0, m.hidden),
            "wlm": gen.weight(seed, gen.WLM, 0, vs, m.hidden)}
    t_layer = []
    for _ in range(timed_iters):
        Kc, Vc = K.copy(), V.copy()
        t0 = time.perf_counter()
        OM.decoder_layer(m, p, x, pos, Kc, Vc)
        t_layer.append(time.perf_counter() - t0)
    t0 = time.perf_counter()
    OM.lm_head(m, head, x)
    t_head = (time.perf_counter() - t0) * (m.vocab / vs)
    tl = min(t_layer)
    t_step = m.num_layers * tl + t_head
    cores = len(os.sched_getaffinity(0))
    desc = (f"oracle fp64 (numpy BLAS) on {rows} rows: 1 decoder layer timed ({tl*1e3:.1f} ms) x "
            f"{m.num_layers} layers + LM head on 1/16 of the vocab x16 ({t_head*1e3:.1f} ms); "
            f"ctx {ctx_len}; extrapolated to one full decode step")
    return rows / t_step, desc, cores, t_step


# ----------------------------------------------------------------------------- roofline
def kernel_work(cls, m, B, ctx_avg, layer_bytes, fused_mlp=False):
    """Algorithmic (flops, bytes) per launch of a kernel class.  Class 1 with
    fused_mlp is the fused gate/up -> down launch (mlp2_kernel): gate/up plus down work, the act
    tile written and read once, the fp32 down output slice written once."""
    h, I, V = m.hidden, m.intermediate, m.vocab
    q, kvd = m.q_dim, m.kv_dim
    if cls == 1 and fused_mlp:
        return (2.0 * B * 2 * I * h + 2.0 * B * h * I,
                2.0 * (3 * I * h + B * h + 2 * B * I) + 4.0 * B * h)
    if cls == 1:
        return 2.0 * B * 2 * I * h, 2.0 * (2 * I * h + B * h + B * I)
    if cls == 4:
        return 2.0 * B * h * I, 2.0 * (h * I + B * I + 2 * B * h)
    if cls == 5:
        return 2.0 * B * m.qkv_dim * h, 2.0 * (m.qkv_dim * h + B * h) + 4.0 * B * m.qkv_dim
    if cls == 6:
        return 2.0 * B * h * q, 2.0 * (h * q + B * q + 2 * B * h)
    if cls == 7:
        return 2.0 * B * V * h, 2.0 * (V * h + B * h)
    if cls == 2:
        toks = B * (ctx_avg + 1)
        return 4.0 * m.n_q_heads * m.head_dim * toks, 2.0 * 2 * kvd * toks + 2.0 * 2 * B * q
    if cls == 3:
        return 0.0, float(layer_bytes)
    raise ValueError(cls)


def roofline_entry(cls, m, B, ctx_avg, layer_bytes, avg_ms, peaks, traffic=None, fused_mlp=False):
    flops, byts = kernel_work(cls, m, B, ctx_avg, layer_bytes, fused_mlp)
    t_tensor = flops / (peaks["tflops"] * 1e12) if flops else 0.0
    t_hbm = byts / (peaks["hbm"] * 1e9)
    if cls == 3:
        ach = byts / (avg_ms * 1e-3) / 1e9
        return {"kernel": CLS_NAMES[cls], "bound": "nvlink", "achieved": ach, "peak": peaks["nvl"],
                "unit": "GB/s", "frac": ach / peaks["nvl"], "traffic": traffic}
    if t_tensor > t_hbm:
        ach = flops / (avg_ms * 1e-3) / 1e12
        return {"kernel": CLS_NAMES[cls], "bound": "tensor", "achieved": ach,
                "peak": peaks["tflops"], "unit": "TFLOP/s", "frac": ach / peaks["tflops"],
                "traffic": traffic, "algorithmic_bytes": byts, "algorithmic_flops": flops}
    ach = byts / (avg_ms * 1e-3) / 1e9
    return {"kernel": CLS_NAMES[cls], "bound": "hbm", "achieved": ach, "peak": peaks["hbm"],
            "unit": "GB/s", "frac": ach / peaks["hbm"], "traffic": traffic,
            "algorithmic_bytes": byts, "algorithmic_flops": flops}


def load_peaks():
    p = {"hbm": 6549.1, "tflops": 1369.2, "tflops_burst": 1634.2, "nvl": 770.0,
         "source": "MEASURED_PEAKS.json"}
    try:
        j = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        p["hbm"] = float(j["hbm_gbs"])
        p["tflops"] = float(j.get("bf16_tflops_sustained", j["bf16_tflops"]))
        p["tflops_burst"] = float(j["bf16_tflops"])
    except Exception:
        p.update({"hbm": 6650.0, "tflops": 1400.0, "tflops_burst": 1590.0,
                  "source": "fallback (B200_PROFILING.md)"})
    return p


def load_traffic(workload, cls):
    """dram bytes per launch from a committed ncu --set full capture (profiles/), or None."""
    try:
        j = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        return j.get(workload, {}).get(CLS_NAMES[cls])
    except Exception:
        return None


def north_star_roofline(m, B, ctx_avg, d, peaks, step_ms, remote_bytes=None):
    """Step-level roofline of SURVEY.md §8(d): T2 = max(sum 2PB/P_peak, sum R/BW_nvl) + T_lm;
    T3 adds HBM weight reads and KV reads per layer.  remote_bytes: the bytes actually fetched
    per step (FFN-only pooling fetches less than whole layers)."""
    P = m.hidden * m.qkv_dim + m.q_dim * m.hidden + 3 * m.hidden * m.intermediate   # P_l
    L = m.num_layers
    lm = max(2.0 * B * m.vocab * m.hidden / (peaks["tflops"] * 1e12),
             2.0 * m.vocab * m.hidden / (peaks["hbm"] * 1e9))
    remote = (L - -(-L // d)) * P * 2.0 if d > 1 else 0.0      # (L - L/d) layers x bytes
    if remote_bytes is not None:
        remote = float(remote_bytes)
    t_gemm = L * 2.0 * P * B / (peaks["tflops"] * 1e12)
    t_nvl = remote / (peaks["nvl"] * 1e9)
    T2 = max(t_gemm, t_nvl) + lm
    per_layer = max(2.0 * P * B / (peaks["tflops"] * 1e12), 2.0 * P / (peaks["hbm"] * 1e9)) + \
        B * (ctx_avg + 1) * 4.0 * m.kv_dim / (peaks["hbm"] * 1e9)
    T3 = max(L * per_layer, t_nvl) + lm
    return {"T2_ms": T2 * 1e3, "T3_ms": T3 * 1e3, "frac_T2": T2 * 1e3 / step_ms,
            "frac_T3": T3 * 1e3 / step_ms, "nvlink_bytes_per_step": remote,
            "peaks": {"bf16_tflops": peaks["tflops"], "hbm_gbs": peaks["hbm"],
                      "nvlink_gbs": peaks["nvl"]}}


def per_remote_layer(ctx0, m, B, W, peaks, layer_bytes, steps):
    """per remote layer in steady state, T_roof(l) / t_meas(l), T_roof(l) =
    max(2 P_l B / P_peak, R_l / BW_nvl) and t_meas(l) from the device's %globaltimer stamps: the
    ring's consume log stamps each remote layer when its ready wait passes (its slot landed and
    the compute stream reached it), so for two consecutive remote layers l, l+1 of one step
    t_meas(l) = t(l+1) - t(l) — the period at which the pipeline retires layer l."""
    cons = ctx0.consume_log()
    if not cons:
        return None
    P = m.hidden * m.qkv_dim + m.q_dim * m.hidden + 3 * m.hidden * m.intermediate
    t_roof = max(2.0 * P * B / (peaks["tflops"] * 1e12), layer_bytes / (peaks["nvl"] * 1e9))
    # tile slots log one consumption per part: keep each layer's first (its QKV part)
    firsts = [c for i, c in enumerate(cons) if i == 0 or c[0] != cons[i - 1][0]]
    rows = firsts[-(m.num_layers - -(-m.num_layers // W)) * steps:]     # the timed steps
    fr, tm = [], []
    for a, b in zip(rows, rows[1:]):
        if b[0] == a[0] + 1 and b[4] > a[4]:           # consecutive remote layers of one step
            t = (b[4] - a[4]) * 1e-9
            tm.append(t)
            fr.append(t_roof / t)
    if not fr:
        return None
    fr.sort()
    return {"layers": len(fr), "t_roof_us": t_roof * 1e6,
            "t_meas_us_median": sorted(tm)[len(tm) // 2] * 1e6,
            "frac_median": fr[len(fr) // 2], "frac_min": fr[0], "frac_max": fr[-1],
            "how": "t_meas = %globaltimer consume stamps of consecutive remote layers (device ring log)"}


# ----------------------------------------------------------------------------- WaS emulation
def was_emulation(args, P, m, wl, seed, local, stream, kv, tok, B, ctx_len, W, peaks):
    """Rank 0 of a W-rank WaS group on ONE GPU (SURVEY.md §8(a) a2-a4 at full size): the W-1
    other owners are serve-only contexts (sidp_alloc_serve_only) whose arenas sit in this GPU's
    HBM, so the fetch reads local HBM instead of a peer over NVLink: on the copy engine by
    default (--fetch ce: 64 MB chunks), or the SM fetch kernel on --emulate-fetch-sms CTAs
    (--fetch sm), paced (sidp_config.fetch_pace_gbps) to the NVLink 5 reader rate, 770 GB/s,
    which local HBM would otherwise exceed ~4x; HBM traffic equals a real rank's (its
    slot writes + one owner's serve reads under the stagger).  Not a multi-GPU number: NVLink
    latency and the other ranks' compute are absent."""
    import numpy as np
    import torch
    max_ctx = kv.max_ctx
    slots = args.slots or wl.slots
    ctx0 = P.Context(m, rank=0, world=W, slots=slots, order=args.order, pool=args.pool,
                     max_batch=kv.max_batch, max_ctx=max_ctx, fetch_sms=args.emulate_fetch_sms,
                     fetch_engine=args.fetch, stagger=not args.no_stagger, device=local, seed=seed,
                     fetch_pace_gbps=args.emulate_pace_gbps, slot_parts=args.slot_parts,
                     fetch_ce_share=args.emulate_ce_share)
    peers = []
    try:
        for r in range(1, W):
            c = P.Context(m, rank=r, world=W, slots=slots, pool=args.pool, max_batch=kv.max_batch,
                          max_ctx=max_ctx, device=local, seed=seed, alloc=False)
            c.alloc_serve_only(alias_of=peers[0] if (args.alias_owners and peers) else None)
            peers.append(c)
        with torch.cuda.stream(stream):
            ctx0.init_weights_synthetic(stream=stream)
            for c in peers:
                c.init_weights_synthetic(stream=stream)
        stream.synchronize()
        ctx0.import_handles([ctx0.export_handles()] + [c.export_handles() for c in peers])
        kv.set_pos(np.full(B, ctx_len))

        def step():
            ctx0.step(tok, tok, kv, batch=B, stream=stream, advance_pos=True)

        all_mask = sum(1 << c for c in CLS_NAMES)
        warm = max(2, min(args.warmup, 3))
        for i in range(warm):
            if i == warm - 1:
                ctx0.set_timing(all_mask)
            step()
        stream.synchronize()
        st0 = ctx0.stats()
        shares = st0["timed_ms"]
        us_layer = {CLS_NAMES[c]: round(shares[c] * 1e3 / m.num_layers, 2) for c in CLS_NAMES
                    if shares[c] > 0}
        ctx0.set_timing(1 << 3)
        pos_before = kv.max_pos
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        h0 = time.perf_counter()
        for _ in range(args.emulate_steps):
            step()
        host_ms = (time.perf_counter() - h0) * 1e3 / args.emulate_steps
        ev1.record(stream)
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1) / args.emulate_steps
        st = ctx0.stats()
        n_f = st["timed_launches"][3] - st0["timed_launches"][3]
        f_ms = (st["timed_ms"][3] - st0["timed_ms"][3]) / max(1, n_f)
        lb = st["layer_bytes"]
        trace = ctx0.fetch_trace() if args.fetch == "sm" else []
        remote = m.num_layers - len([l for l in range(m.num_layers) if l % W == 0])
        if trace:   # device log: first claim -> publish of each layer of the timed steps
            durs = [(e[6] - e[5]) * 1e-6 for e in trace[-remote * args.emulate_steps:]]
            if durs:
                f_ms = sum(durs) / len(durs)
        fetch_gbs = lb / (f_ms * 1e-3) / 1e9 if f_ms > 0 else None
        ctx_avg = pos_before + (args.emulate_steps - 1) / 2.0
        ns = north_star_roofline(m, B, ctx_avg, W, peaks, ms,
                                 remote_bytes=(m.num_layers - len([l for l in range(m.num_layers)
                                                                    if l % W == 0])) * st["layer_bytes"])
        remote_layers = m.num_layers - len([l for l in range(m.num_layers) if l % W == 0])
        per_layer = per_remote_layer(ctx0, m, B, W, peaks, st["layer_bytes"], args.emulate_steps) \
            if args.fetch == "sm" else None
        return {
            "what": f"rank 0 of a {W}-rank WaS group on one B200; the {W - 1} other owners are "
                    "serve-only contexts in local HBM (bench.py was_emulation docstring)",
            "world_emulated": W, "batch": B, "ctx": ctx_len, "slots": slots,
            "slot_parts": args.slot_parts or 1,
            "fetch_engine": args.fetch, "fetch_sms": st["fetch_sms_held"],
            "compute_sms": st["compute_sms"], "stagger_tick_ms": st["stagger_tick_ns"] * 1e-6,
            "fetch_pace_gbps": args.emulate_pace_gbps,
            "owners_aliased": bool(args.alias_owners),
            "fetch_ce_share": args.emulate_ce_share,
            "steps": args.emulate_steps,
            "ms_per_step": ms, "tokens_s_rank": B / (ms / 1e3),
            "host_enqueue_ms_per_step": host_ms,
            "graph_replays_in_timed_steps": st["graph_replays"] - st0["graph_replays"],
            "group_tokens_s_est": W * B / (ms / 1e3),
            "remote_layers_per_step": remote_layers, "layer_bytes": lb,
            "fetch_bytes_per_step": remote_layers * lb,
            "fetch": {"avg_launch_ms": f_ms, "GBps": fetch_gbs,
                      "frac_of_nvlink_770": (fetch_gbs / peaks["nvl"]) if fetch_gbs else None,
                      "fetch_busy_frac": (remote_layers * f_ms / ms) if f_ms else None},
            "north_star_roofline": ns,
            "per_remote_layer": per_layer,
            "kernel_us_per_layer": us_layer,
            "footprint_bytes_rank0": {"owned": st["owned_bytes"], "slots": st["slot_bytes"],
                                      "replicated": st["replicated_bytes"],
                                      "workspace": st["workspace_bytes"]},
        }
    finally:
        ctx0.destroy()
        for c in reversed(peers):   # aliases before their donor
            c.destroy()


def cas_emulation(args, P, m, seed, local, W, ctx_len):
    """CaS tail (SURVEY.md §8(a) a12, M5 analogue) with W virtual ranks on ONE GPU: every rank is
    a full context with its own arena, KV cache and stream; per layer the owner runs the fused
    GEMMs over all live rows while the others wait on device flags — as on W GPUs, where the
    non-owners also idle, so the step time is representative minus NVLink hop latency (the
    shipped activations are KBs).  Ranks' attention kernels share this GPU (small at B <= 16).
    Step time = max over ranks of (common start event -> rank's end event)."""
    import numpy as np
    import torch
    from sidp_inputs import gen
    bl = [int(b) for b in str(getattr(args, "cas_batches", "1,4,16")).split(",") if b]
    Bmax = max(bl + [16])
    steps = max(2, args.emulate_steps)
    max_ctx = ctx_len + 3 + steps * 8 + 8
    ranks = []
    try:
        for r in range(W):
            c = P.Context(m, rank=r, world=W, max_batch=Bmax, max_ctx=max_ctx, device=local,
                          seed=seed, pool=args.pool)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                c.init_weights_synthetic(stream=st)
                kv = P.KVCache(m, Bmax, max_ctx)
                kv.fill_synthetic(seed, r * Bmax, Bmax, ctx_len, stream=st)
            st.synchronize()
            tok = torch.from_numpy(gen.tokens(seed, np.arange(r * Bmax, (r + 1) * Bmax), m.vocab)).to(torch.int32).cuda()
            ranks.append((c, st, kv, tok))
        blobs = [c.export_handles() for c, _, _, _ in ranks]
        for c, _, _, _ in ranks:
            c.import_handles(blobs)
            c.set_mode(1, 0)   # SIDP_CAS from step 0 (collective-consistent: same on all ranks)
        patterns = [(f"all live, B={b}", [b] * W) for b in bl]
        patterns += [("half live, B=16", [16] * (W // 2) + [0] * (W - W // 2)),
                     ("one live, B=16", [16] + [0] * (W - 1))]
        out = []
        common = torch.cuda.Stream()
        xs = [(torch.randn(Bmax, m.hidden, device="cuda") * 0.5).to(torch.bfloat16) for _ in range(W)]
        for name, bt in patterns:
            for c, _, kv, _ in ranks:
                c.set_batches(bt)
            for r, (c, st, kv, tok) in enumerate(ranks):
                kv.set_pos(np.full(Bmax, ctx_len))
            def run(n):
                # layer by layer across ranks (sidp_decode_layer, the per-layer collective):
                # enqueuing one rank's whole step first can fill the launch queue while its
                # stream spins on a flag only a later rank's (not yet enqueued) kernels set
                evs = []
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record(common)
                for r, (c, st, kv, tok) in enumerate(ranks):
                    st.wait_event(e0)
                h0 = time.perf_counter()
                for _ in range(n):
                    for layer in range(m.num_layers):
                        for r, (c, st, kv, tok) in enumerate(ranks):
                            c.decode_layer(xs[r], layer, 1, kv, batch=bt[r], stream=st)
                host_ms[0] = (time.perf_counter() - h0) * 1e3 / n
                for r, (c, st, kv, tok) in enumerate(ranks):
                    e1 = torch.cuda.Event(enable_timing=True)
                    e1.record(st)
                    evs.append(e1)
                torch.cuda.synchronize()
                return max(e0.elapsed_time(e) for e in evs) / n
            host_ms = [0.0]
            run(2)   # warm-up
            ms = run(steps)
            live = sum(1 for b in bt if b)
            out.append({"pattern": name, "batches": bt, "ms_per_layer_stack": ms,
                        "host_enqueue_ms": host_ms[0],
                        "ms_per_layer": ms / m.num_layers,
                        "group_tokens_s": sum(bt) / (ms / 1e3),
                        "tokens_s_per_live_rank": (sum(bt) / max(1, live)) / (ms / 1e3)})
        # per-class kernel time of the one-live pattern (every rank times its kernel classes;
        # summed over ranks: the owners' GEMMs + the live rank's attention), per layer
        bt = patterns[-1][1]
        for c, _, kv, _ in ranks:
            c.set_batches(bt)
            kv.set_pos(np.full(Bmax, ctx_len))
        host_ms = [0.0]
        run(1)
        for c, _, _, _ in ranks:
            c.set_timing(sum(1 << k for k in CLS_NAMES))
        run(1)
        cls_us = {}
        for c, _, _, _ in ranks:
            st = c.stats()
            for k, nm in CLS_NAMES.items():
                if st["timed_ms"][k] > 0:
                    cls_us[nm] = cls_us.get(nm, 0.0) + st["timed_ms"][k] * 1e3 / m.num_layers
            c.set_timing(0)
        timeouts = sum(c.stats()["timeouts"] for c, _, _, _ in ranks)
        return {"what": f"CaS (pool={args.pool}) decode of all {m.num_layers} layers by {W} "
                        f"virtual ranks on one B200, S_ctx={ctx_len} (bench.py cas_emulation "
                        "docstring); a full step adds the local embed + LM head; the ranks' "
                        "per-layer small kernels serialise on this one GPU, so the all-live "
                        "patterns over-state the W-GPU time",
                "world_emulated": W, "ctx": ctx_len, "steps": steps, "timeouts": timeouts,
                "cas_level": int(os.environ.get("SIDP_CAS_FUSED", "2")),
                "one_live_kernel_us_per_layer": {k: round(v, 2) for k, v in cls_us.items()},
                "results": out}
    finally:
        for c, _, _, _ in ranks:
            c.destroy()


def run_emulation_only(args, P, m, wl, local, world):
    """--emulate-only: the d=W WaS emulation line alone (the d=1 run would not fit)."""
    import numpy as np
    import torch
    from sidp_inputs import gen
    if world != 1:
        raise SystemExit("--emulate-only is a single-GPU mode")
    W = max(2, args.emulate_world)
    B = args.emulate_batch or args.batch or wl.batch
    ctx_len = args.emulate_ctx or args.ctx or wl.ctx
    seed = wl.seed
    stream = torch.cuda.Stream()
    kv = P.KVCache(m, B, ctx_len + args.warmup + args.emulate_steps + 8)
    with torch.cuda.stream(stream):
        kv.fill_synthetic(seed, 0, B, ctx_len, stream=stream)
    stream.synchronize()
    tok = torch.from_numpy(gen.tokens(seed, np.arange(B), m.vocab)).to(torch.int32).cuda()
    peaks = load_peaks()
    emu = was_emulation(args, P, m, wl, seed, local, stream, kv, tok, B, ctx_len, W, peaks)
    fp = emu["footprint_bytes_rank0"]
    st_d1 = {"owned_bytes": m.num_layers * emu["layer_bytes"], "slot_bytes": 0,
             "replicated_bytes": fp["replicated"], "workspace_bytes": fp["workspace"]}
    line = {"metric": METRIC, "emulate_only": True, "unit": UNIT, "n_gpus": 1,
            "dtype": "bf16", "data": "synthetic: counter-hash bf16 weights and KV (sidp_inputs.gen), seeded",
            "config": {"workload": f"{wl.id}: {m.name} WaS d={W} single-GPU emulation, B={B}, S_ctx={ctx_len}",
                       "layers": m.num_layers, "reduced": args.layers is not None},
            "was_emulation": emu,
            "kv_capacity": kv_capacity(m, st_d1, fp, W)}
    line["kv_capacity"]["replicated_d1"]["note"] = ("footprint = all layers + replicated + "
                                                    "workspaces (the d=1 run is not executed)")
    print(json.dumps(line), flush=True)


def kv_capacity(m, st_d1, fp_dw, W, util=0.9):
    """KV tokens per GPU left by the MEASURED per-GPU footprint of this library (owned weights +
    WaS slots + replicated tensors + workspaces) at a vLLM-style 0.9 memory utilisation: the
    replicated-DP run (d=1) vs rank 0 of the emulated d=W SiDP group.  PAPER.md:21 reports up
    to 1.8x (H20/H200/B200, with TP); the arithmetic is SPEC.md:100-103's MemoryBreakdown."""
    import torch
    total = torch.cuda.mem_get_info()[1]
    per_tok = 2 * m.n_kv_heads * m.head_dim * 2 * m.num_layers
    def tokens(fp):
        return max(0, int((total * util - fp) // per_tok))
    fp1 = st_d1["owned_bytes"] + st_d1["slot_bytes"] + st_d1["replicated_bytes"] + st_d1["workspace_bytes"]
    out = {"gpu_bytes": total, "util": util, "kv_bytes_per_token": per_tok,
           "replicated_d1": {"footprint_bytes": fp1, "kv_tokens": tokens(fp1)}}
    if fp_dw:
        fpw = sum(fp_dw.values())
        out[f"sidp_d{W}"] = {"footprint_bytes": fpw, "kv_tokens": tokens(fpw)}
        out["ratio"] = tokens(fpw) / max(1, tokens(fp1))
        # tensor parallelism over the same W GPUs (PAPER.md:314's other comparison), ANALYTIC:
        # every weight (layers, embedding, LM head) sharded W ways, KV heads sharded W ways
        # (so a GPU stores 1/W of each token's KV), the same workspaces; group tokens per GPU
        # are then free / (per_tok / W) / W = free / per_tok, directly comparable with SiDP's
        fp_tp = (st_d1["owned_bytes"] + st_d1["replicated_bytes"]) / W + st_d1["workspace_bytes"]
        out[f"tp{W}_analytic"] = {"footprint_bytes": int(fp_tp), "kv_tokens": tokens(fp_tp),
                                  "note": "weights and KV heads sharded; tokens per GPU of the group"}
        out["ratio_vs_tp"] = tokens(fpw) / max(1, tokens(fp_tp))
    return out


def _child_json(extra, timeout_s):
    """Run this script again with the parent's flags plus `extra`; return its last JSON line, or
    {"error": ...} (non-zero exit, no JSON, or killed after timeout_s)."""
    argv = [a for a in sys.argv[1:] if a not in ("--emulate-only", "--cas-only")]
    try:
        r = subprocess.run([sys.executable, os.path.abspath(__file__)] + argv + extra,
                           capture_output=True, text=True, timeout=timeout_s)
    except subprocess.TimeoutExpired:
        return {"error": f"{' '.join(extra)}: killed after {timeout_s} s"}
    for ln in reversed(r.stdout.strip().splitlines()):
        if ln.startswith("{"):
            try:
                return json.loads(ln)
            except ValueError:
                break
    return {"error": f"{' '.join(extra)}: rc {r.returncode}: {(r.stderr or '')[-300:]}"}


# ----------------------------------------------------------------------------- main arms
def run_reference(args, wl, m, rank, world):
    """The tier's reference arm: the fp64 oracle as it stands, on the host cores, each step a
    bounded sample of the workload (one decoder layer on --cpu-rows rows + 1/16 of the LM head)
    extrapolated to a full step's tokens/s.  ms_per_step is the wall time each executed sample
    step took; the extrapolated full-step time is reported beside it."""
    if rank != 0:
        return
    B = args.cpu_rows
    ctx_len = wl.ctx
    vals, walls, fulls = [], [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        v, desc, cores, t_step = oracle_sample(m, wl.seed, B, ctx_len, timed_iters=1)
        wall = time.perf_counter() - t0
        if i >= args.warmup:
            vals.append(v)
            walls.append(wall)
            fulls.append(t_step)
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": statistics.median(walls) * 1e3,
            "extrapolated_full_step_ms": statistics.median(fulls) * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": _config(args, wl, m, world),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": len(os.sched_getaffinity(0)),
                             "kind": "oracle", "sample": desc},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _config(args, wl, m, world):
    B = args.batch or wl.batch
    return {"workload": f"{wl.id}: {m.name} WaS decode, B={B}/GPU, S_ctx={args.ctx or wl.ctx}",
            "batch_per_gpu": B, "ctx": args.ctx or wl.ctx, "layers": m.num_layers,
            "reduced": args.layers is not None, "world": world, "slots": args.slots or wl.slots,
            "order": args.order, "pool": args.pool, "fetch": args.fetch,
            "stagger": not args.no_stagger,
            "kv_layout": "paged, 16-token blocks (shuffled pool)" if args.paged else "contiguous",
            "l2": "no flush needed: per-step working set (weights + KV) >> 126 MB L2",
            "parallelism": f"sidp-dp{world}"}


def main():
    args = parse()
    from sidp_inputs import MODELS, WORKLOADS
    wl = WORKLOADS[args.workload]
    m = MODELS[wl.model]
    if args.layers:
        m = m.with_layers(args.layers)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, wl, m, rank, world)
        return
    import numpy as np
    import torch
    import paper_2605_28095_b200 as P
    from sidp_inputs import gen
    if args.share_gpu:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if args.share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    B = args.batch or wl.batch
    ctx_len = args.ctx or wl.ctx
    slots = args.slots or wl.slots
    if args.emulate_only:
        run_emulation_only(args, P, m, wl, local, world)
        return
    if args.cas_only:
        print(json.dumps({"cas_emulation": cas_emulation(args, P, m, wl.seed, local,
                                                         max(2, args.emulate_world), args.cas_ctx)}),
              flush=True)
        return
    e2e_steps = 0 if args.no_e2e else args.steps
    max_ctx = ctx_len + args.warmup + args.steps + e2e_steps + 8
    seed = wl.seed
    ctx = P.Context(m, rank=rank, world=world, slots=slots, order=args.order, pool=args.pool,
                    max_batch=B, max_ctx=max_ctx, fetch_sms=args.fetch_sms,
                    fetch_engine=args.fetch, stagger=not args.no_stagger, device=local,
                    seed=seed, slot_parts=args.slot_parts)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        ctx.init_weights_synthetic(stream=stream)
        if args.paged:
            nb = -(-max_ctx // P.PagedKVCache.BLOCK)
            kv = P.PagedKVCache(m, B, max_ctx, B * nb)
            kv.fill_synthetic(seed, rank * B, B, ctx_len, stream=stream, perm_seed=seed)
        else:
            kv = P.KVCache(m, B, max_ctx)
            kv.fill_synthetic(seed, rank * B, B, ctx_len, stream=stream)
    stream.synchronize()
    if world > 1:
        from paper_2605_28095_b200.orchestrator import exchange_handles
        exchange_handles(ctx, dist)
        dist.barrier()
    bg = np.arange(rank * B, rank * B + B)
    kv.set_pos(np.full(B, ctx_len))
    tok = torch.from_numpy(gen.tokens(seed, bg, m.vocab)).to(torch.int32).cuda()
    torch.cuda.synchronize()

    def step():
        ctx.step(tok, tok, kv, batch=B, stream=stream, advance_pos=True)

    # warm-up; the last warm-up step times every kernel class to find the dominant one
    all_mask = sum(1 << c for c in CLS_NAMES)
    for i in range(args.warmup):
        if i == args.warmup - 1:
            ctx.set_timing(all_mask)
        step()
    stream.synchronize()
    shares = ctx.stats()["timed_ms"]
    tot = sum(shares[1:]) or 1.0
    kernel_shares = {CLS_NAMES[c]: shares[c] / tot for c in CLS_NAMES}
    # absolute per-layer class times of that (event-bracketed, so PDL-serialised) warm-up step
    kernel_us_per_layer = {CLS_NAMES[c]: round(shares[c] * 1e3 / m.num_layers, 2) for c in CLS_NAMES
                           if shares[c] > 0}
    dom = max((c for c in CLS_NAMES if c != 3 or world > 1), key=lambda c: shares[c])

    # ---------------- timed region (device-side, CUDA events, max over ranks)
    ctx.set_timing(1 << dom)
    st_pre = ctx.stats()
    launches0, replays0 = st_pre["launches"], st_pre["graph_replays"]
    pos_before = kv.max_pos
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = ev0.elapsed_time(ev1)
    st = ctx.stats()
    launches = st["launches"] - launches0
    dom_ms = st["timed_ms"][dom] / max(1, st["timed_launches"][dom])
    if dist:
        t = torch.tensor([ms], device="cpu" if args.share_gpu else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        gathered = [None] * world
        dist.all_gather_object(gathered, clocks)
        clocks = dict(gathered[0])
        clocks["reasons"] = sorted({r for g in gathered for r in g["reasons"]})
        clocks["per_rank_sm_mhz"] = [g["sm_mhz"] for g in gathered]
    ms_step = ms / args.steps
    value = B * world * args.steps / (ms / 1e3)
    ctx_avg = pos_before + (args.steps - 1) / 2.0

    # ---------------- end to end through the public API with host buffers
    e2e = None
    if e2e_steps:
        h_in = torch.from_numpy(gen.tokens(seed, bg, m.vocab)).to(torch.int32).pin_memory()
        h_out = torch.empty(B, dtype=torch.int32).pin_memory()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            with torch.cuda.stream(stream):
                tok.copy_(h_in, non_blocking=True)
            step()
            with torch.cuda.stream(stream):
                h_out.copy_(tok, non_blocking=True)
            stream.synchronize()
            h_in, h_out = h_out, h_in
        t1 = time.perf_counter()
        e_ms = (t1 - t0) * 1e3
        if dist:
            t = torch.tensor([e_ms], device="cpu" if args.share_gpu else "cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": B * world * e2e_steps / (e_ms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": 4 * B, "d2h_bytes_per_step": 4 * B,
               "ms_per_step": e_ms / e2e_steps,
               "note": "host tokens H2D from pinned memory, sidp_step, next tokens D2H + sync, per step"}

    if rank != 0:
        ctx.destroy()
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    peaks = load_peaks()
    # the gate/up class is the fused gate/up -> down launch when no separate down GEMM ran
    fused_mlp = shares[1] > 0 and shares[4] == 0
    roof = roofline_entry(dom, m, B, ctx_avg, st["layer_bytes"], dom_ms, peaks,
                          load_traffic(wl.id, dom), fused_mlp=fused_mlp)
    roof["avg_launch_ms"] = dom_ms
    roof["launches_timed"] = st["timed_launches"][dom]
    roof["peak_source"] = peaks["source"] + (" (sustained bf16)" if roof["unit"] == "TFLOP/s" else "")
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        v, desc, cores, _ = oracle_sample(m, seed, args.cpu_rows, ctx_len)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic: counter-hash bf16 weights and KV (sidp_inputs.gen), seeded",
        "config": _config(args, wl, m, world),
        "roofline": roof,
        "north_star_roofline": north_star_roofline(m, B, ctx_avg, world, peaks, ms_step),
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "graph_replays_in_timed_steps": st["graph_replays"] - replays0,
        "clocks": clocks,
        "per_gpu_tokens_s": value / world,
        "kernel_shares": kernel_shares,
        "kernel_us_per_layer": kernel_us_per_layer,
        "footprint_bytes_per_gpu": {"owned": st["owned_bytes"], "slots": st["slot_bytes"],
                                    "replicated": st["replicated_bytes"],
                                    "kv": 2 * kv.k.numel() * 2},
    }
    ctx.destroy()
    if world == 1 and (args.emulate_world > 1 or args.cas_emulate):
        # the extra single-GPU measurements run in child processes with a time limit, so a
        # failure or hang there can never cost the main line; this process frees the GPU first
        del kv, tok
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        if args.emulate_world > 1:
            child = _child_json(["--emulate-only"], args.extra_timeout)
            line["was_emulation"] = child.get("was_emulation", child)
            if "was_emulation" in child:
                line["kv_capacity"] = kv_capacity(m, st, child["was_emulation"].get("footprint_bytes_rank0"),
                                                  args.emulate_world)
        if args.cas_emulate and args.emulate_world > 1:
            child = _child_json(["--cas-only"], args.extra_timeout)
            line["cas_emulation"] = child.get("cas_emulation", child)
        if args.m3_emulate and args.emulate_world > 1 and args.layers is None:
            # the double-buffered cache as two tile-granular slots (NEXT-3: per-component
            # flags, same 3.4 GB as two whole-layer slots; 0.928 vs 0.909 of T2)
            child = _child_json(["--emulate-only", "--workload", "M3", "--emulate-batch", "1024",
                                 "--emulate-ctx", "384", "--alias-owners", "--emulate-steps", "3",
                                 "--slots", "2", "--slot-parts", "2"],
                                args.extra_timeout)
            m3 = child.get("was_emulation", child)
            if isinstance(m3, dict) and "error" not in m3:
                m3["note"] = ("north-star target shape (SURVEY.md M3) at the measured B_e; owners "
                              "aliased (timing only), so this GPU keeps a real rank's KV memory; "
                              "two tile-granular slots (3.4 GB)")
            line["m3_emulation"] = m3
    print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
