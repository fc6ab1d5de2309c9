"""Counter-based synthetic value generator.

value(seed, tensor, layer, idx) is a pure function of LOGICAL coordinates:

    key = seed ^ (tensor << 56) ^ (layer << 44) ^ idx          (idx < 2**44)
    h   = splitmix64(key)
    lvl = (h >> 56) - 128                                        in [-128, 127]

* weights  W[N, K]: lvl * 2**-7 * 2**-floor(log2(K)/2)
* gains    g[n]   : 1 + ((h >> 60) - 8) * 2**-7
* biases   b[n]   : lvl * 2**-7 * 2**-3
* embed, activations, KV cache: lvl * 2**-7
* tokens          : h mod vocab

Every value is one of 256 levels times a power of two, so it is exactly
representable in bf16 and no rounding happens anywhere in generation.  The CUDA
side (K12, csrc/kernels/init.cu) implements the same function; tests compare the
two bit for bit.  Storage layout never enters a value, so packed/interleaved GPU
layouts are permutations of these logical arrays.
"""
from __future__ import annotations

import os

import numpy as np

# ---- tensor ids (logical tensors of the model and workload) ----
EMBED = 1
WQ = 2
WK = 3
WV = 4
WO = 5
WGATE = 6
WUP = 7
WDOWN = 8
G_ATTN = 9
G_MLP = 10
G_Q = 11
G_K = 12
BQ = 13
BK = 14
BV = 15
G_FINAL = 16
WLM = 17
KCACHE = 18
VCACHE = 19
TOKENS = 20
POS = 21
XACT = 22

# logical index stride of the context axis in KV / activation tensors
T_STRIDE = 1 << 17
IDX_LIMIT = 1 << 44

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on a uint64 array (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def hash_u64(seed: int, tensor: int, layer: int, idx) -> np.ndarray:
    idx = np.asarray(idx, dtype=np.uint64)
    if idx.size and int(idx.max()) >= IDX_LIMIT:
        raise ValueError("logical index exceeds 2**44")
    if not (0 <= layer < (1 << 12)):
        raise ValueError("layer out of range")
    key = (np.uint64(seed & 0xFFFFFFFFFFFFFFFF) ^ np.uint64(tensor << 56)
           ^ np.uint64(layer << 44))
    return splitmix64(key ^ idx)


def _levels(h: np.ndarray) -> np.ndarray:
    return ((h >> np.uint64(56)).astype(np.int64) - 128).astype(np.float64) * 2.0 ** -7


def weight_scale(K: int) -> float:
    return 2.0 ** -((int(K).bit_length() - 1) // 2)


def weight(seed: int, tensor: int, layer: int, n_rows: int, K: int, rows=None) -> np.ndarray:
    """Logical weight W[N, K] (row-major logical index n*K + k); optionally a row subset."""
    rows = np.arange(n_rows, dtype=np.uint64) if rows is None else np.asarray(rows, dtype=np.uint64)
    out = np.empty((rows.shape[0], K), dtype=np.float64)
    step = max(1, (1 << 20) // K)          # bounded temporaries for big layers
    cols = np.arange(K, dtype=np.uint64)[None, :]
    scale = weight_scale(K)

    def fill(i):
        idx = rows[i:i + step, None] * np.uint64(K) + cols
        out[i:i + step] = _levels(hash_u64(seed, tensor, layer, idx)) * scale

    starts = range(0, rows.shape[0], step)
    if rows.shape[0] * K >= (1 << 23):     # numpy ufuncs release the GIL: chunk over threads
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
            list(ex.map(fill, starts))
    else:
        for i in starts:
            fill(i)
    return out


def gain(seed: int, tensor: int, layer: int, n: int) -> np.ndarray:
    h = hash_u64(seed, tensor, layer, np.arange(n, dtype=np.uint64))
    return 1.0 + ((h >> np.uint64(60)).astype(np.int64) - 8).astype(np.float64) * 2.0 ** -7


def bias(seed: int, tensor: int, layer: int, n: int) -> np.ndarray:
    h = hash_u64(seed, tensor, layer, np.arange(n, dtype=np.uint64))
    return _levels(h) * 2.0 ** -3


def embed_rows(seed: int, token_ids, hidden: int) -> np.ndarray:
    t = np.asarray(token_ids, dtype=np.uint64)
    idx = t[:, None] * np.uint64(hidden) + np.arange(hidden, dtype=np.uint64)[None, :]
    return _levels(hash_u64(seed, EMBED, 0, idx))


def kv(seed: int, tensor: int, layer: int, b_global, t, n_kv: int, hd: int) -> np.ndarray:
    """KV cache values [len(b), len(t), n_kv, hd] (logical (b, t, g, d))."""
    b = np.asarray(b_global, dtype=np.uint64)[:, None, None, None]
    tt = np.asarray(t, dtype=np.uint64)[None, :, None, None]
    g = np.arange(n_kv, dtype=np.uint64)[None, None, :, None]
    d = np.arange(hd, dtype=np.uint64)[None, None, None, :]
    idx = ((b * np.uint64(T_STRIDE) + tt) * np.uint64(n_kv) + g) * np.uint64(hd) + d
    return _levels(hash_u64(seed, tensor, layer, idx))


def activations(seed: int, layer: int, b_global, hidden: int) -> np.ndarray:
    b = np.asarray(b_global, dtype=np.uint64)
    idx = b[:, None] * np.uint64(hidden) + np.arange(hidden, dtype=np.uint64)[None, :]
    return _levels(hash_u64(seed, XACT, layer, idx))


def tokens(seed: int, b_global, vocab: int, step: int = 0) -> np.ndarray:
    h = hash_u64(seed, TOKENS, step, np.asarray(b_global, dtype=np.uint64))
    return (h % np.uint64(vocab)).astype(np.int64)


def positions(seed: int, b_global, ctx: int, span: int = 0) -> np.ndarray:
    """Cached tokens per sequence: ctx, or ctx + (h mod (span+1)) for ragged contexts."""
    b = np.asarray(b_global, dtype=np.uint64)
    if span <= 0:
        return np.full(b.shape, ctx, dtype=np.int64)
    h = hash_u64(seed, POS, 0, b)
    return ctx + (h % np.uint64(span + 1)).astype(np.int64)


def layer_params(seed: int, m, layer: int) -> dict:
    """All logical tensors of decoder layer ``layer`` of model dims ``m`` (float64, exact)."""
    p = {
        "wq": weight(seed, WQ, layer, m.q_dim, m.hidden),
        "wk": weight(seed, WK, layer, m.kv_dim, m.hidden),
        "wv": weight(seed, WV, layer, m.kv_dim, m.hidden),
        "wo": weight(seed, WO, layer, m.hidden, m.q_dim),
        "wgate": weight(seed, WGATE, layer, m.intermediate, m.hidden),
        "wup": weight(seed, WUP, layer, m.intermediate, m.hidden),
        "wdown": weight(seed, WDOWN, layer, m.hidden, m.intermediate),
        "g_attn": gain(seed, G_ATTN, layer, m.hidden),
        "g_mlp": gain(seed, G_MLP, layer, m.hidden),
    }
    if m.qk_norm:
        p["g_q"] = gain(seed, G_Q, layer, m.head_dim)
        p["g_k"] = gain(seed, G_K, layer, m.head_dim)
    if m.qkv_bias:
        p["bq"] = bias(seed, BQ, layer, m.q_dim)
        p["bk"] = bias(seed, BK, layer, m.kv_dim)
        p["bv"] = bias(seed, BV, layer, m.kv_dim)
    return p


def head_params(seed: int, m) -> dict:
    """Replicated tensors: embedding, final norm gain, LM head."""
    return {
        "g_final": gain(seed, G_FINAL, 0, m.hidden),
        "wlm": weight(seed, WLM, 0, m.vocab, m.hidden),
    }
