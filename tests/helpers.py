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


__all__ = ["OracleModel", "rank_inputs", "oracle_layer", "rel_err", "oracle_steps", "OS", "OSD"]
