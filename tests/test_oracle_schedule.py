"""Pins for oracle/schedule.py, oracle/policy.py and oracle/accounting.py.

Pinned against: SPEC.md worked examples (tests/golden/spec_examples.json),
brute-force event replay (an independent discrete-event simulation), and
exhaustive enumeration.  None of these re-types the function under test.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

from oracle import accounting as A
from oracle import policy as P
from oracle import schedule as S
from sidp_inputs import MODELS

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ---------------------------------------------------------------- C-S1 owner map
def test_owner_of_examples():
    for ex in GOLD["owner_of"]:
        own = S.owner_map(ex["layer"] + 1, ex["d"])
        assert own[ex["layer"]] == ex["owner"], ex["cite"]


def test_owner_balance_and_uniqueness():
    ex = GOLD["owner_balance"]
    own = S.owner_map(ex["L"], ex["d"])
    assert [own.count(r) for r in range(ex["d"])] == [ex["per_rank"]] * ex["d"]
    for L, d in itertools.product(range(1, 40), range(1, 9)):
        own = S.owner_map(L, d)
        counts = [own.count(r) for r in range(d)]
        assert set(counts) <= {L // d, -(-L // d)}          # floor or ceil
        assert len(own) == L and all(0 <= o < d for o in own)  # exactly one owner each


def test_owner_map_rejects_bad_owner():
    with pytest.raises(ValueError):
        S.owner_map(4, 2, [0, 1, 2, 0])
    with pytest.raises(ValueError):
        S.owner_map(4, 2, [0, 1, 1])


# ---------------------------------------------------------------- C-S2 plans
def test_peak_shift_order_examples():
    for ex in GOLD["peak_shift_order"]:
        own = S.owner_map(ex["L"], ex["d"])
        assert S.peak_shift_order(ex["rank"], ex["c"], ex["d"], ex["L"], own) == ex["order"], ex["cite"]


def test_build_prefetch_plan_example():
    for ex in GOLD["build_prefetch_plan"]:
        own = S.owner_map(ex["L"], ex["d"])
        assert S.plan_paper(own, ex["d"], ex["rank"]) == ex["plan"], ex["cite"]


@pytest.mark.parametrize("order", ["exec", "paper"])
def test_plan_completeness(order):
    """Every non-owned layer exactly once per pass, never an owned one."""
    for d in range(1, 9):
        for L in range(d, 4 * d + 3):
            own = S.owner_map(L, d)
            for r in range(d):
                pl = S.plan(own, d, r, order)
                assert sorted(pl) == [l for l in range(L) if own[l] != r]


def test_paper_order_single_reader_per_cycle_step():
    """SPEC.md:376 / :390: at each in-cycle step k the ranks read pairwise distinct
    layers (hence distinct owners) — exhaustive over d in 2..8, L multiple of d."""
    for d in range(2, 9):
        for L in range(d, 8 * d + 1, d):
            own = S.owner_map(L, d)
            for c in range(0, L, d):
                orders = [S.peak_shift_order(r, c, d, L, own) for r in range(d)]
                for k in range(d - 1):
                    layers = [o[k] for o in orders]
                    assert len(set(layers)) == d
                    assert len({own[l] for l in layers}) == d


# ---------------------------------------------------------------- C-S4 / C-S5 / C-S6
def _replay_cases():
    for d in range(2, 7):
        for L in (d, 2 * d, 3 * d + 1):
            for slots in (1, 2, 3, d - 1, d):
                if slots < 1:
                    continue
                for order in ("exec", "paper"):
                    yield d, L, slots, order


def test_deadlock_rule_matches_event_replay():
    """C-S4: the replay completes iff max(p - q) < S (brute-force discrete events)."""
    for d, L, slots, order in _replay_cases():
        own = S.owner_map(L, d)
        for r in range(d):
            pl = S.plan(own, d, r, order)
            rep = S.event_replay(own, r, pl, slots, steps=3)
            assert rep.completed == S.deadlock_free(pl, slots), (d, L, slots, order, r)


def test_paper_order_needs_d_minus_1_slots():
    """C-S4: PAPER order is deadlock-free for every rank iff S >= d-1 (d | L, d >= 2)."""
    for d in range(2, 9):
        L = 2 * d
        own = S.owner_map(L, d)
        need = max(S.lag(S.plan_paper(own, d, r)) for r in range(d)) + 1
        assert need == max(1, d - 1)


def test_fifo_slot_recurrence_matches_event_replay_under_jitter():
    """C-S5: slot assignment is timing-independent; recurrence == replay for several timings."""
    for d, L, slots, order in _replay_cases():
        own = S.owner_map(L, d)
        for r in range(d):
            pl = S.plan(own, d, r, order)
            if not pl or not S.deadlock_free(pl, slots):
                continue
            rec = S.slot_schedule(pl, slots, steps=3)
            for ft, ct, jit, seed in [(1.0, 0.5, 0.0, 0), (0.1, 0.9, 3.0, 1), (2.0, 0.01, 2.0, 7)]:
                rep = S.event_replay(own, r, pl, slots, 3, ft, ct, jit, seed)
                assert rep.completed
                assert rep.assignments == rec
                assert rep.max_busy <= slots            # cache never exceeds S
                assert rep.transitions_ok and rep.consumed_tags_ok


def test_exec_order_is_ring():
    """C-S5: for EXEC order the FIFO recurrence reduces to slot = j mod S."""
    own = S.owner_map(16, 4)
    for r in range(4):
        pl = S.plan_exec(own, r)
        for slots in (1, 2, 3, 5):
            sched = S.slot_schedule(pl, slots, steps=4)
            assert [s for _, _, s in sched] == [j % slots for j in range(len(sched))]


def test_paper_order_slot_sequence_survey_examples():
    """C-S5 worked sequences printed in SURVEY.md §8(c) (PAPER d=8,S=7 and d=4,S=3, rank 1)."""
    own8 = S.owner_map(16, 8)
    s8 = [s for _, _, s in S.slot_schedule(S.plan_paper(own8, 8, 1), 7, 2)]
    assert s8[:14] == [0, 1, 2, 3, 4, 5, 6, 6, 0, 1, 2, 3, 4, 5]
    own4 = S.owner_map(12, 4)
    s4 = [s for _, _, s in S.slot_schedule(S.plan_paper(own4, 4, 1), 3, 2)]
    assert s4[:9] == [0, 1, 2, 2, 0, 1, 1, 2, 0]


# ---------------------------------------------------------------- C-S7 stagger
def test_stagger_single_reader_brute_force():
    """Latin-square property: with t_r = (-r) mod (d-1), owners read at every tick are
    pairwise distinct (d | L); lockstep start (all t_r = 0) violates it for d >= 3."""
    for d in range(3, 9):
        for L in range(d, 64 + 1, d):
            own = S.owner_map(L, d)
            plans = [S.plan_exec(own, r) for r in range(d)]
            offs = [S.stagger_ticks(d, r) for r in range(d)]
            assert S.single_reader_violations(own, d, 3 * len(plans[0]), plans, offs) == 0
            assert S.single_reader_violations(own, d, len(plans[0]), plans, [0] * d) > 0


def test_stagger_requires_d_divides_L():
    """the property can fail when d does not divide L."""
    bad = 0
    for d in range(3, 9):
        for L in range(d + 1, 40):
            if L % d == 0:
                continue
            own = S.owner_map(L, d)
            plans = [S.plan_exec(own, r) for r in range(d)]
            offs = [S.stagger_ticks(d, r) for r in range(d)]
            bad += S.single_reader_violations(own, d, 2 * len(plans[0]), plans, offs) > 0
    assert bad > 0


# ---------------------------------------------------------------- C-S8 mode policy
def test_policy_drained_window_goes_cas():
    """SPEC.md:457 window all zeros (job drained) -> CaS."""
    pol = P.ModePolicy(b_threshold=32, window=5, hysteresis=1.5, min_dwell=5)
    assert P.decide_mode(pol, [[0, 0]] * 5, P.WAS, dwell=10) == P.CAS
    assert P.decide_mode(pol, [[0, 0]] * 5, P.CAS, dwell=10) is None


def test_policy_oscillation_no_change():
    """SPEC.md:458 batches oscillating across b_threshold within one window -> no change."""
    pol = P.ModePolicy(b_threshold=32, window=4, hysteresis=1.5, min_dwell=1)
    win = [[20, 44], [44, 20], [20, 44], [44, 20]]
    assert P.decide_mode(pol, win, P.WAS, dwell=100) is None
    assert P.decide_mode(pol, win, P.CAS, dwell=100) is None


def test_policy_dwell_and_hysteresis_timeline():
    pol = P.ModePolicy(b_threshold=10, window=2, hysteresis=1.5, min_dwell=4)
    # long bulk phase, then a tail below threshold, then a burst above 1.5*B_th
    batches = [[100, 100]] * 6 + [[3, 0]] * 6 + [[12, 12]] * 4 + [[30, 0]] * 6
    modes = P.mode_timeline(pol, batches)
    assert modes[:6] == [P.WAS] * 6
    assert P.CAS in modes[6:16]
    i_cas = modes.index(P.CAS)
    assert i_cas % pol.window == 0                      # switches only at window boundaries
    assert modes[-1] == P.WAS                           # 30 > 15 re-enters WaS
    # 12 is within the hysteresis band (10, 15]: no flip back while in it
    for t in range(12, 16):
        if modes[t - 1] == P.CAS:
            assert modes[t] == P.CAS


# ---------------------------------------------------------------- accounting
def _stats(name):
    g = GOLD["model_stats"][name]
    return A.derive_model_stats(g["L"], g["h"], g["I"], g["n_kv"], g["hd"], g["V"],
                                n_q=g.get("n_q")), g


def test_model_stats_llama():
    st, g = _stats("llama-3.1-70b")
    assert abs(st.total_params - g["total_params_approx"]) / g["total_params_approx"] < 0.005
    assert abs(st.ffn_params - g["ffn_params_approx"]) / g["ffn_params_approx"] < 0.001
    assert st.kv_bytes_per_token == g["kv_bytes_per_token"]


def test_model_stats_qwen3_ffn_fraction():
    st, g = _stats("qwen3-32b")
    assert abs(st.ffn_fraction - g["ffn_fraction"]) <= g["ffn_fraction_tol"]


def test_unit_ffn():
    u = GOLD["unit_ffn"]
    st = A.derive_model_stats(u["L"], u["h"], u["I"], 1, 1, 1, n_q=1)
    assert st.ffn_params == u["ffn_params"]


def test_weight_footprint_and_slots():
    for ex in GOLD["weight_footprint"]:
        st, _ = _stats(ex["model"])
        got = A.weight_footprint(st, ex["mode"], d=ex["d"])
        assert abs(got - ex["bytes_approx"]) / ex["bytes_approx"] < ex["rel_tol"], ex["cite"]
    for ex in GOLD["slot_bytes"]:
        st, _ = _stats(ex["model"])
        got = A.slot_bytes(st, ex["slots"])
        assert abs(got - ex["bytes_approx"]) / ex["bytes_approx"] < ex["rel_tol"], ex["cite"]


def test_max_batch_and_capacity():
    for ex in GOLD["max_batch"]:
        assert A.max_batch(ex["tokens"], ex["S"]) == ex["batch"], ex["cite"]
    ex = GOLD["kv_capacity_infeasible"]
    st, _ = _stats(ex["model"])
    w = A.weight_footprint(st, "replicated", d=ex["d"])
    assert (A.kv_tokens(ex["M"], ex["util"], w, 0, 0, st.kv_bytes_per_token) > 0) == ex["feasible"]


def test_pooled_layer_params():
    g = GOLD["paper_layer_params"]
    for name in ("llama-3.1-70b", "qwen3-32b", "qwen2.5-72b"):
        assert A.pooled_params_per_layer(MODELS[name]) == g[name]


def test_remote_bytes_per_step():
    m = MODELS["llama-3.1-70b"]
    got = A.remote_bytes_per_step(m, 8)
    assert abs(got - 70 * 1.711e9) / (70 * 1.711e9) < 0.001    # 119.8 GB
    assert A.remote_bytes_per_step(m, 1) == 0


def test_kv_bytes_per_token_layer():
    """Pinned by SPEC.md:64's printed Llama-3.1-70B KV bytes per token (all 80 layers) and by
    the bytes of one cached token in the oracle's own cache layout (Kc and Vc rows of a layer)."""
    g = GOLD["model_stats"]["llama-3.1-70b"]
    m = MODELS["llama-3.1-70b"]
    assert A.kv_bytes_per_token_layer(m) * m.num_layers == g["kv_bytes_per_token"]
    t = MODELS["tiny"]
    from sidp_inputs import gen as G
    K = G.kv(1, G.KCACHE, 0, np.arange(1), range(1), t.n_kv_heads, t.head_dim)   # [1, 1, nkv, hd]
    assert A.kv_bytes_per_token_layer(t) == 2 * K[0, 0].size * 2                # K + V, bf16


def test_layer_flops_per_token_brute_force():
    """2 x (multiply-adds) of one decoded token through the oracle layer, counted on the actual
    parameter arrays (every linear's weight matrix) and by walking the attention loops of
    oracle.model.attend (scores q.K and values p.V over pos + 1 tokens per query head) — not
    the closed form under test.  Also the SURVEY.md §8(d) figures: 32,768 (S_ctx + 1) attention
    FLOPs for 64 x 128 heads and 2 P_l = 1.711 GFLOP for Llama-3.1-70B."""
    from sidp_inputs import gen as G
    for name in ("tiny", "tiny-qwen3", "tiny-qwen25"):
        m = MODELS[name]
        p = G.layer_params(3, m, 0)
        linear = sum(p[k].size for k in ("wq", "wk", "wv", "wo", "wgate", "wup", "wdown"))
        for ctx in (0, 5, 63):
            macs = linear
            for _ in range(m.n_q_heads):          # attend(): per head, scores then values
                macs += (ctx + 1) * m.head_dim    # s_t = q . K[t]
                macs += (ctx + 1) * m.head_dim    # o += p_t V[t]
            assert A.layer_flops_per_token(m, ctx) == 2 * macs, (name, ctx)
    ll = MODELS["llama-3.1-70b"]
    attn = A.layer_flops_per_token(ll, 100) - A.layer_flops_per_token(ll, 99)
    assert attn == 32768
    assert abs((A.layer_flops_per_token(ll, 0) - 32768) / 1.711e9 - 1) < 1e-3
