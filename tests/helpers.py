"""Shared test helpers: seeded inputs for both sides and the oracle-side reference runs.

Inputs come only from sidp_inputs (the shared generator).  Expected values come only from
oracle/.  Nothing here is computed by the CUDA path.
"""
from __future__ import annotations

import numpy as np

from oracle import model as OM
from oracle import schedule as OS
from oracle import sidp as OSD
from sidp_inputs import gen


class OracleModel:
    """fp64 parameters of a model (lazy per layer) for teacher-forced checks."""

    def __init__(self, m, seed):
        self.m, self.seed = m, seed
        self._layers = {}
        self._head = None
        self._embed = None

    def layer(self, l):
        if l not in self._layers:
            self._layers[l] = gen.layer_params(self.seed, self.m, l)
        return self._layers[l]

    @property
    def head(self):
        if self._head is None:
            self._head = gen.head_params(self.seed, self.m)
        return self._head

    def embed(self, toks):
        return gen.embed_rows(self.seed, np.asarray(toks), self.m.hidden)


def rank_inputs(m, seed, b0, B, ctx, span, T):
    """(b_global, tokens, pos, caches) of one rank: logical rows b0..b0+B-1."""
    bg = np.arange(b0, b0 + B)
    toks = gen.tokens(seed, bg, m.vocab)
    pos = gen.positions(seed, bg, ctx, span)
    caches = []
    for l in range(m.num_layers):
        K = gen.kv(seed, gen.KCACHE, l, bg, range(T), m.n_kv_heads, m.head_dim)
        V = gen.kv(seed, gen.VCACHE, l, bg, range(T), m.n_kv_heads, m.head_dim)
        caches.append((K, V))
    return bg, toks, pos, caches


def oracle_layer(om: OracleModel, l, x, pos, K, V):
    """Teacher-forced oracle layer on copies of the caches. Returns (out, k_new, v_new)."""
    Kc, Vc = K.copy(), V.copy()
    out = OM.decoder_layer(om.m, om.layer(l), x, pos, Kc, Vc)
    b = np.arange(x.shape[0])
    return out, Kc[b, pos], Vc[b, pos]


def rel_err(got, ref):
    return float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30))


def oracle_steps(m, seed, om, toks, pos, caches, steps):
    """Un-forced oracle decode of `steps` steps on one rank (fp64). Returns per-step logits."""
    cs = [(K.copy(), V.copy()) for K, V in caches]
    out = []
    t = toks
    for s in range(steps):
        nxt, logits, _ = OM.decode_step(m, [om.layer(l) for l in range(m.num_layers)], om.head,
                                        om.embed, t, pos + s, cs)
        out.append((nxt, logits))
        t = nxt
    return out


def cas_oracle_check(m, om: OracleModel, d, pool, dumps, logits, caches, pos, tol):
    """Teacher-forced CaS parity against the ORACLE's CaS layer (oracle/sidp.py cas_layer: the
    owner fuses the live ranks' rows in ascending rank order; dummy ranks are
    absent).  Per live rank r (keys of `dumps`): dumps[r] [L, B_r, h] the GPU's
    bf16 layer inputs, logits[r] [B_r, V], caches[r] = (K, V) [L, B_r, T, n_kv, hd] the GPU's KV
    state after the step, pos[r] the step's positions.  Each layer's oracle output must match the
    next dump, the GPU's newly written k/v, and (last layer) the logits, within tol * max|oracle|.
    Returns the largest relative error seen."""
    from oracle import sidp as OSD
    L = m.num_layers
    owner = OS.owner_map(L, d)
    layers = [om.layer(l) for l in range(L)]
    arenas = OSD.build_owned_arenas(layers, owner, d, pool)
    local = OSD.local_tensors(layers, pool)
    live = sorted(dumps)
    worst = 0.0
    out = None
    for l in range(L):
        xs = {r: dumps[r][l] for r in live}
        cs = {r: (caches[r][0][l].copy(), caches[r][1][l].copy()) for r in live}
        gk = {r: caches[r][0][l][np.arange(len(pos[r])), pos[r]] for r in live}
        gv = {r: caches[r][1][l][np.arange(len(pos[r])), pos[r]] for r in live}
        out = OSD.cas_layer(m, arenas[owner[l]][l], local[l], xs, pos, cs, pool)
        for r in live:
            b = np.arange(len(pos[r]))
            errs = [rel_err(gk[r], cs[r][0][b, pos[r]]), rel_err(gv[r], cs[r][1][b, pos[r]])]
            if l + 1 < L:
                errs.append(rel_err(dumps[r][l + 1], out[r]))
            worst = max(worst, *errs)
            assert max(errs) <= tol, (r, l, errs)
    for r in live:
        e = rel_err(logits[r], OM.lm_head(m, om.head, out[r]))
        worst = max(worst, e)
        assert e <= tol, (r, e)
    return worst


__all__ = ["cas_oracle_check", "OracleModel", "rank_inputs", "oracle_layer", "rel_err", "oracle_steps", "OS", "OSD"]
