"""Plain fp64 definition of the decode computation (oracle; test infrastructure only).

PAPER.md:62-64 (§2.1) describes the block generically ("self-attention ... FFN,
usually a two-layer MLP and a non-linearity"); PAPER.md:164 says SiDP leaves
"model architecture and numerics ... unchanged".  The concrete block is therefore
the HF-Llama/Qwen decoder layer (reading C-A16), written
out step by step in that order.  All arithmetic is float64 with no rounding
points (the GPU's bf16 rounding points are listed in DESIGN.md, C-N3).

Shapes: x [B, h]; pos [B] = tokens already cached (the new token sits at pos);
caches Kc, Vc [B, T, n_kv, hd] valid on [0, pos_b).
"""
from __future__ import annotations

import numpy as np


def rmsnorm(x: np.ndarray, g: np.ndarray, eps: float) -> np.ndarray:
    """C-N2 step 1/8: x / sqrt(mean(x^2) + eps) * g (over the last axis)."""
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps) * g


def rope(x: np.ndarray, pos: np.ndarray, theta: float) -> np.ndarray:
    """C-N2 step 4, rotate-half RoPE: f_i = theta^(-2i/hd), a = pos*f_i;
    y[i] = x[i] cos a - x[i+hd/2] sin a;  y[i+hd/2] = x[i+hd/2] cos a + x[i] sin a.
    x [B, H, hd], pos [B]."""
    hd = x.shape[-1]
    half = hd // 2
    i = np.arange(half, dtype=np.float64)
    f = theta ** (-2.0 * i / hd)
    a = np.asarray(pos, dtype=np.float64)[:, None] * f[None, :]
    c = np.cos(a)[:, None, :]
    s = np.sin(a)[:, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def silu(z: np.ndarray) -> np.ndarray:
    """C-N2 step 9: SiLU(z) = z / (1 + e^-z)."""
    return z / (1.0 + np.exp(-z))


# ---- the layer, split at the cut points CaS needs (C-N6) ----------------------------

def attn_norm(m, p, x):
    """Step 1: u = RMSNorm(x) * g_attn."""
    return rmsnorm(x, p["g_attn"], m.rms_eps)


def qkv_proj(m, p, u):
    """Step 2: qkv = u W_qkv^T (+ b_qkv); rows of W_qkv are [W_q; W_k; W_v]."""
    qkv = np.concatenate([u @ p["wq"].T, u @ p["wk"].T, u @ p["wv"].T], axis=-1)
    if m.qkv_bias:
        qkv = qkv + np.concatenate([p["bq"], p["bk"], p["bv"]])
    return qkv


def qkv_post(m, p, qkv, pos):
    """Steps 3-4: split heads, optional per-head RMSNorm (Qwen3 qk_norm), RoPE on q and k."""
    B = qkv.shape[0]
    q = qkv[:, :m.q_dim].reshape(B, m.n_q_heads, m.head_dim)
    k = qkv[:, m.q_dim:m.q_dim + m.kv_dim].reshape(B, m.n_kv_heads, m.head_dim)
    v = qkv[:, m.q_dim + m.kv_dim:].reshape(B, m.n_kv_heads, m.head_dim)
    if m.qk_norm:
        q = rmsnorm(q, p["g_q"], m.rms_eps)
        k = rmsnorm(k, p["g_k"], m.rms_eps)
    q = rope(q, pos, m.rope_theta)
    k = rope(k, pos, m.rope_theta)
    return q, k, v


def attend(m, q, Kc, Vc, pos):
    """Steps 5-6 (after the append): for head j with group g = j // (n_q/n_kv),
    s_t = q_j . K[b,t,g] / sqrt(hd) for t in [0, pos_b]; p = softmax(s);
    o_j = sum_t p_t V[b,t,g].  Returns o [B, n_q*hd]."""
    B = q.shape[0]
    grp = m.n_q_heads // m.n_kv_heads
    o = np.zeros((B, m.n_q_heads, m.head_dim))
    for b in range(B):
        n = int(pos[b]) + 1
        for j in range(m.n_q_heads):
            g = j // grp
            s = Kc[b, :n, g, :] @ q[b, j] / np.sqrt(m.head_dim)
            s = s - s.max()
            w = np.exp(s)
            w = w / w.sum()
            o[b, j] = w @ Vc[b, :n, g, :]
    return o.reshape(B, m.q_dim)


def o_proj_residual(m, p, x, o):
    """Step 7: x2 = x + o W_o^T."""
    return x + o @ p["wo"].T


def mlp_norm(m, p, x2):
    """Step 8: u2 = RMSNorm(x2) * g_mlp."""
    return rmsnorm(x2, p["g_mlp"], m.rms_eps)


def mlp_act(m, p, u2):
    """Step 9: m = SiLU(u2 W_gate^T) * (u2 W_up^T)."""
    return silu(u2 @ p["wgate"].T) * (u2 @ p["wup"].T)


def down_proj(m, p, act):
    """Step 10 (without residual): act W_down^T."""
    return act @ p["wdown"].T


def post_attn(m, p, x, o):
    """Steps 7-10: out = x2 + SiLU(u2 W_g^T)*(u2 W_u^T) W_d^T with x2 = x + o W_o^T."""
    x2 = o_proj_residual(m, p, x, o)
    u2 = mlp_norm(m, p, x2)
    return x2 + down_proj(m, p, mlp_act(m, p, u2))


def append_kv(Kc, Vc, k, v, pos):
    """Step 5: Kc[b, pos_b] = k_b; Vc[b, pos_b] = v_b (in place)."""
    for b in range(k.shape[0]):
        Kc[b, int(pos[b])] = k[b]
        Vc[b, int(pos[b])] = v[b]


def decoder_layer(m, p, x, pos, Kc, Vc):
    """One decoder layer (C-N2 steps 1-10).  Updates Kc/Vc in place; returns out."""
    u = attn_norm(m, p, x)
    q, k, v = qkv_post(m, p, qkv_proj(m, p, u), pos)
    append_kv(Kc, Vc, k, v, pos)
    o = attend(m, q, Kc, Vc, pos)
    return post_attn(m, p, x, o)


def lm_head(m, head, x):
    """C-N7: logits = (RMSNorm(x) * g_final) W_lm^T."""
    return rmsnorm(x, head["g_final"], m.rms_eps) @ head["wlm"].T


def argmax_lowest(logits):
    """C-N7 / reading C-A21: argmax with ties broken by the lowest index
    (np.argmax returns the first maximal index)."""
    return np.argmax(logits, axis=-1)


def decode_step(m, layers, head, embed_fn, tokens, pos, caches, collect=None):
    """C-N7: x = E[tokens]; L layers; logits; next = argmax.
    layers: list of per-layer param dicts; caches: list of (Kc, Vc) per layer (updated).
    collect: optional list receiving each layer's input x (teacher-forcing dumps)."""
    x = embed_fn(tokens)
    for l, p in enumerate(layers):
        if collect is not None:
            collect.append(x.copy())
        x = decoder_layer(m, p, x, pos, caches[l][0], caches[l][1])
    logits = lm_head(m, head, x)
    return argmax_lowest(logits), logits, x
