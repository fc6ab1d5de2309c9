"""Byte / capacity arithmetic (oracle; test infrastructure only).

PAPER.md:32-39 (§1): K = B*S; B ~ N(M-W)/S for DP and (NM-W)/S for MP.
Concrete formulas from SPEC.md catalog/capacity, whose worked
examples pin them (tests/golden/spec_examples.json).  pooled_params_per_layer
is this build's layer-scope pooling (reading C-A2).
"""
from __future__ import annotations

import math
from dataclasses import dataclass


@dataclass(frozen=True)
class ModelStats:
    total_params: int
    ffn_params: int
    ffn_fraction: float
    ffn_bytes_per_layer: float
    non_ffn_weight_bytes: float
    weight_bytes_total: float
    kv_bytes_per_token: int
    dtype_bytes: int = 2


def derive_model_stats(L, h, I, n_kv, hd, V, n_q=None, tied=False, dtype_bytes=2) -> ModelStats:
    """SPEC.md:58-64 derive_model_stats: ffn = L*3*h*I; attention = L*(2*h*q_dim + 2*h*kv_dim)
    (q_dim = h unless overridden); embeddings = V*h*(1 if tied else 2)."""
    q_dim = h if n_q is None else n_q * hd
    ffn = L * 3 * h * I
    attn = L * (2 * h * q_dim + 2 * h * n_kv * hd)
    emb = V * h * (1 if tied else 2)
    total = ffn + attn + emb
    return ModelStats(
        total_params=total,
        ffn_params=ffn,
        ffn_fraction=ffn / total,
        ffn_bytes_per_layer=ffn * dtype_bytes / L,
        non_ffn_weight_bytes=(total - ffn) * dtype_bytes,
        weight_bytes_total=total * dtype_bytes,
        kv_bytes_per_token=2 * n_kv * hd * dtype_bytes * L,
        dtype_bytes=dtype_bytes,
    )


def weight_footprint(st: ModelStats, mode: str, d: int = 1, tp: int = 1, pp: int = 1) -> float:
    """Replicated/TpShard -> W/(tp*pp); Fsdp/SiDP -> (non_ffn + ffn/d)/(tp*pp)."""
    if mode in ("replicated", "tpshard"):
        return st.weight_bytes_total / (tp * pp)
    if mode in ("fsdp", "sidp"):
        ffn_total = st.ffn_params * st.dtype_bytes
        return (st.non_ffn_weight_bytes + ffn_total / d) / (tp * pp)
    raise ValueError(mode)


def slot_bytes(st: ModelStats, was_slots: int, tp: int = 1, fraction: float = 1.0) -> float:
    """was_slot_count * ffn_bytes_per_layer / tp * granularity."""
    return was_slots * st.ffn_bytes_per_layer / tp * fraction


def kv_tokens(M_bytes, util, weights, slots, reserve, kv_per_token, tp=1) -> int:
    """SPEC.md:100-103 MemoryBreakdown: budget = max(0, M*util - W - slots - reserve);
    tokens = floor(budget / (kv_per_token/tp))."""
    budget = max(0.0, M_bytes * util - weights - slots - reserve)
    return int(budget // (kv_per_token / tp))


def max_batch(kv_tokens_node: int, S: int) -> int:
    """floor(kv_tokens / S)."""
    return kv_tokens_node // S


def pooled_params_per_layer(m) -> int:
    """Layer-scope pooled parameters P_l (SURVEY.md §8 notation): W_q, W_k, W_v, W_o,
    W_gate, W_up, W_down; biases and norm gains excluded (SPEC.md:82 ignores them; they
    add < 0.01% and are still fetched with the layer)."""
    return m.hidden * m.qkv_dim + m.q_dim * m.hidden + 3 * m.hidden * m.intermediate


def layer_flops_per_token(m, ctx: int) -> float:
    """Algorithmic FLOPs per decoded token per layer: 2*P_l for the linears plus
    4*n_q*hd*(ctx+1) for attention scores and values."""
    return 2.0 * pooled_params_per_layer(m) + 4.0 * m.n_q_heads * m.head_dim * (ctx + 1)


def kv_bytes_per_token_layer(m, dtype_bytes=2) -> int:
    return 2 * m.n_kv_heads * m.head_dim * dtype_bytes


def remote_bytes_per_step(m, d: int, dtype_bytes=2) -> float:
    """Per rank per step over NVLink: (L - L/d) layers x pooled bytes, independent of B."""
    remote_layers = m.num_layers - math.ceil(m.num_layers / d) if d > 1 else 0
    return remote_layers * pooled_params_per_layer(m) * dtype_bytes
