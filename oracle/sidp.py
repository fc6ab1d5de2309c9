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


def cas_layer(m, W: dict, p_loc: dict, xs: dict, pos: dict, caches: dict, pool: str = "layer",
              on_serve=None) -> dict:
    """One layer in CaS mode for every live rank (§4.3).  W: the owner's pooled
    tensors of this layer (only the owner touches them); p_loc: the tensors every rank keeps.
    xs / pos / caches: per live rank r (ascending order) its layer input [B_r, h], positions
    [B_r] and this layer's (Kc, Vc), updated in place (the KV cache is local).
    Returns {r: layer output}.  Dummy ranks are simply absent."""
    live = sorted(xs)
    off, acc = {}, 0
    for r in live:                                 # exclusive prefix sums (C-A10)
        off[r] = acc
        acc += xs[r].shape[0]

    def serve(parts, fn):
        """Owner: fuse rows of all live ranks in rank order, compute once, split."""
        stage = {k: np.concatenate([parts[r][k] for r in live], axis=0) for k in parts[live[0]]}
        out = fn(stage)
        if on_serve is not None:
            on_serve(live)
        return {r: out[off[r]:off[r] + xs[r].shape[0]] for r in live}

    if not live:
        return {}
    if pool == "layer":
        P = {**p_loc, **W}
        # RT1: send u, receive u W_qkv^T (+b)
        qkv = serve({r: {"u": M.attn_norm(m, P, xs[r])} for r in live},
                    lambda s: M.qkv_proj(m, P, s["u"]))
        os_ = {}
        for r in live:
            q, k, v = M.qkv_post(m, P, qkv[r], pos[r])
            M.append_kv(caches[r][0], caches[r][1], k, v, pos[r])
            os_[r] = {"o": M.attend(m, q, caches[r][0], caches[r][1], pos[r]), "x": xs[r]}
        # RT2: send (o, x), receive out
        return serve(os_, lambda s: M.post_attn(m, P, s["x"], s["o"]))
    # ffn scope: attention local, one round trip for the FFN
    u2s, x2s = {}, {}
    for r in live:
        u = M.attn_norm(m, p_loc, xs[r])
        q, k, v = M.qkv_post(m, p_loc, M.qkv_proj(m, p_loc, u), pos[r])
        M.append_kv(caches[r][0], caches[r][1], k, v, pos[r])
        o_ = M.attend(m, q, caches[r][0], caches[r][1], pos[r])
        x2s[r] = M.o_proj_residual(m, p_loc, xs[r], o_)
        u2s[r] = {"u2": M.mlp_norm(m, W, x2s[r])}
    ys = serve(u2s, lambda s: M.down_proj(m, W, M.mlp_act(m, W, s["u2"])))
    return {r: x2s[r] + ys[r] for r in live}


def run_cas(m, layers, head, embed_fn, ranks: list[RankState], steps: int, d: int,
            owner: list[int], pool: str = "layer", traffic: list | None = None):
    arenas = build_owned_arenas(layers, owner, d, pool)
    local = local_tensors(layers, pool)
    toks = [st.tokens for st in ranks]
    for t in range(steps):
        live = [st for st in ranks if st.B > 0]
        xs = {st.r: embed_fn(toks[st.r]) for st in live}
        coll = {st.r: [] for st in live}
        for l in range(len(layers)):
            o = owner[l]
            for st in live:
                coll[st.r].append(xs[st.r].copy())
            xs = cas_layer(m, arenas[o][l], local[l], xs, {st.r: st.pos + t for st in live},
                           {st.r: st.caches[l] for st in live}, pool,
                           on_serve=None if traffic is None else
                           (lambda lv, t=t, l=l, o=o: traffic.append((t, l, o, list(lv)))))
        for st in ranks:
            if st.B == 0:
                st.history.append(None)
                continue
            logits = M.lm_head(m, head, xs[st.r])
            nxt = M.argmax_lowest(logits)
            st.history.append({"next": nxt, "logits": logits, "layer_inputs": coll[st.r]})
            toks[st.r] = nxt
    return ranks
