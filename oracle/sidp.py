"""SiDP execution over d simulated ranks (oracle; test infrastructure only).

Moves real arrays the way the paper's runtime moves weights and activations,
then computes with ``oracle.model``.  Used to pin the paper's invariant that
"the two modes are numerically equivalent" and that SiDP leaves
"numerics ... unchanged": WaS and CaS outputs must equal the
replicated-DP result exactly in fp64 (same function on identical arrays, up to
BLAS blocking for CaS, whose row count differs; see DESIGN.md C-N5 bound).

Pool scope (reading C-A2): ``layer`` pools QKV/O/gate/up/down (north_star);
``ffn`` pools only gate/up/down as the paper does.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import model as M
from . import schedule as S

ATTN_KEYS = ("wq", "wk", "wv", "wo", "g_attn", "g_q", "g_k", "bq", "bk", "bv")
FFN_KEYS = ("wgate", "wup", "wdown", "g_mlp")


def pooled_keys(pool: str, p: dict) -> list[str]:
    if pool == "layer":
        return list(p.keys())
    if pool == "ffn":
        return [k for k in p if k in FFN_KEYS]
    raise ValueError(pool)


@dataclass
class RankState:
    """One DP replica: its batch rows, positions and local KV caches (never pooled,
    PAPER.md:163)."""
    r: int
    tokens: np.ndarray                  # [B_r]
    pos: np.ndarray                     # [B_r] cached tokens
    caches: list                        # per layer (Kc [B_r,T,n_kv,hd], Vc)
    history: list = field(default_factory=list)   # per step: dict(next, logits, layer_inputs)

    @property
    def B(self) -> int:
        return int(self.tokens.shape[0])


def build_owned_arenas(layers: list[dict], owner: list[int], d: int, pool: str) -> list[dict]:
    """Owner-only placement: rank r holds copies of the pooled
    tensors of the layers it owns; other ranks hold nothing for them."""
    arenas = [dict() for _ in range(d)]
    for l, p in enumerate(layers):
        arenas[owner[l]][l] = {k: p[k].copy() for k in pooled_keys(pool, p)}
    return arenas


def local_tensors(layers: list[dict], pool: str) -> list[dict]:
    """Tensors every rank keeps locally (the un-pooled remainder; empty for layer scope)."""
    out = []
    for p in layers:
        pk = set(pooled_keys(pool, p))
        out.append({k: v for k, v in p.items() if k not in pk})
    return out


# ------------------------------------------------------------------------------------
# Replicated DP: every rank holds every layer (the baseline SiDP must reproduce).
# ------------------------------------------------------------------------------------
def run_replicated(m, layers, head, embed_fn, ranks: list[RankState], steps: int):
    for st in ranks:
        toks = st.tokens
        for t in range(steps):
            if st.B == 0:
                st.history.append(None)
                continue
            coll: list = []
            nxt, logits, _ = M.decode_step(m, layers, head, embed_fn, toks, st.pos + t,
                                           st.caches, collect=coll)
            st.history.append({"next": nxt, "logits": logits, "layer_inputs": coll})
            toks = nxt
    return ranks


# ------------------------------------------------------------------------------------
# WaS (§4.2): per rank, independently; remote layers are copied verbatim
# from the owner's arena into a cache slot chosen by the FIFO free-list (C-S5),
# compute reads only the slot, and the slot is released after the layer's last use.
# ------------------------------------------------------------------------------------
def run_was(m, layers, head, embed_fn, ranks: list[RankState], steps: int, d: int,
            owner: list[int], slots: int, order: str = "exec", pool: str = "layer",
            log: list | None = None):
    arenas = build_owned_arenas(layers, owner, d, pool)
    local = local_tensors(layers, pool)
    for st in ranks:
        r = st.r
        pl = S.plan(owner, d, r, order)
        sched = S.slot_schedule(pl, slots, steps) if pl else []
        slot_buf: list = [None] * slots      # (tag, tensors)
        slot_busy = [False] * slots          # filled and not yet released
        nf = 0

        def pump_fetches(need):
            """Issue fetches in plan order while the target slot is free; stop once
            `need` (t, l) is resident."""
            nonlocal nf
            while nf < len(sched):
                t_f, l_f, s_f = sched[nf]
                if slot_busy[s_f]:
                    break
                src = arenas[owner[l_f]][l_f]          # one-sided read of the owner's HBM
                slot_buf[s_f] = ((t_f, l_f), {k: v.copy() for k, v in src.items()})
                slot_busy[s_f] = True
                if log is not None:
                    log.append((r, t_f, l_f, s_f))
                nf += 1
                if (t_f, l_f) == need:
                    return

        toks = st.tokens
        for t in range(steps):
            if st.B == 0:
                st.history.append(None)
                # a dummy WaS rank still walks its plan (weights stream regardless)
            x = embed_fn(toks) if st.B else None
            coll: list = []
            for l in range(len(layers)):
                if owner[l] == r:
                    p = dict(local[l]); p.update(arenas[r][l])
                    s_used = None
                else:
                    pump_fetches((t, l))
                    hit = [s for s in range(slots)
                           if slot_busy[s] and slot_buf[s][0] == (t, l)]
                    if len(hit) != 1:
                        raise RuntimeError(f"rank {r}: layer {(t, l)} not resident (deadlock)")
                    s_used = hit[0]
                    p = dict(local[l]); p.update(slot_buf[s_used][1])
                if st.B:
                    coll.append(x.copy())
                    x = M.decoder_layer(m, p, x, st.pos + t, st.caches[l][0], st.caches[l][1])
                if s_used is not None:
                    slot_busy[s_used] = False        # housekeeper frees after compute
            if st.B:
                logits = M.lm_head(m, head, x)
                nxt = M.argmax_lowest(logits)
                st.history.append({"next": nxt, "logits": logits, "layer_inputs": coll})
                toks = nxt
    return ranks


# ------------------------------------------------------------------------------------
# CaS (§4.3): per layer, non-dummy ranks ship rows to the owner, which
# concatenates them in ascending rank order (reading C-A10), runs the pooled part
# once on the fused rows (GEMM fusion) and returns each slice.
# Dummy ranks send nothing and compute nothing; the owner serves
# even when it is itself dummy.
# ------------------------------------------------------------------------------------
def cas_offsets(batches: list[int]) -> list[int]:
    """Exclusive prefix sums of per-rank rows, dummy ranks counting 0 (C-A10)."""
    off, acc = [], 0
    for b in batches:
        off.append(acc)
        acc += b
    return off


def run_cas(m, layers, head, embed_fn, ranks: list[RankState], steps: int, d: int,
            owner: list[int], pool: str = "layer", traffic: list | None = None):
    arenas = build_owned_arenas(layers, owner, d, pool)
    local = local_tensors(layers, pool)
    toks = [st.tokens for st in ranks]
    for t in range(steps):
        live = [st for st in ranks if st.B > 0]
        Bs = [st.B for st in ranks]
        off = cas_offsets(Bs)
        xs = {st.r: embed_fn(toks[st.r]) for st in live}
        coll = {st.r: [] for st in live}
        for l in range(len(layers)):
            o = owner[l]
            W = arenas[o][l]                      # only the owner touches pooled weights

            def serve(parts, fn):
                """Owner: fuse rows of all live ranks in rank order, compute once, split."""
                if not parts:
                    return {}
                stage = {k: np.concatenate([parts[st.r][k] for st in live], axis=0)
                         for k in parts[live[0].r]}
                out = fn(stage)
                res = {st.r: out[off[st.r]:off[st.r] + st.B] for st in live}
                if traffic is not None:
                    traffic.append((t, l, o, [st.r for st in live]))
                return res

            for st in live:
                coll[st.r].append(xs[st.r].copy())
            if pool == "layer":
                p_loc = local[l]
                # RT1: send u, receive u W_qkv^T (+b)
                us = {st.r: {"u": M.attn_norm(m, {**p_loc, **W}, xs[st.r])} for st in live}
                qkv = serve(us, lambda s: M.qkv_proj(m, {**p_loc, **W}, s["u"]))
                os_ = {}
                for st in live:
                    pos = st.pos + t
                    q, k, v = M.qkv_post(m, {**p_loc, **W}, qkv[st.r], pos)
                    M.append_kv(st.caches[l][0], st.caches[l][1], k, v, pos)
                    os_[st.r] = {"o": M.attend(m, q, st.caches[l][0], st.caches[l][1], pos),
                                 "x": xs[st.r]}
                # RT2: send (o, x), receive out
                outs = serve(os_, lambda s: M.post_attn(m, {**p_loc, **W}, s["x"], s["o"]))
                for st in live:
                    xs[st.r] = outs[st.r]
            else:  # ffn scope: attention local, one round trip for the FFN
                p_loc = local[l]
                u2s, x2s = {}, {}
                for st in live:
                    pos = st.pos + t
                    u = M.attn_norm(m, p_loc, xs[st.r])
                    q, k, v = M.qkv_post(m, p_loc, M.qkv_proj(m, p_loc, u), pos)
                    M.append_kv(st.caches[l][0], st.caches[l][1], k, v, pos)
                    o_ = M.attend(m, q, st.caches[l][0], st.caches[l][1], pos)
                    x2s[st.r] = M.o_proj_residual(m, p_loc, xs[st.r], o_)
                    u2s[st.r] = {"u2": M.mlp_norm(m, W, x2s[st.r])}
                ys = serve(u2s, lambda s: M.down_proj(m, W, M.mlp_act(m, W, s["u2"])))
                for st in live:
                    xs[st.r] = x2s[st.r] + ys[st.r]
        for st in ranks:
            if st.B == 0:
                st.history.append(None)
                continue
            logits = M.lm_head(m, head, xs[st.r])
            nxt = M.argmax_lowest(logits)
            st.history.append({"next": nxt, "logits": logits, "layer_inputs": coll[st.r]})
            toks[st.r] = nxt
    return ranks
