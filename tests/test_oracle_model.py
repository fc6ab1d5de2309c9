"""Pins for oracle/model.py and oracle/sidp.py and the shared generator.

* library routines: HF ``transformers`` Llama/Qwen2/Qwen3 causal LMs in float64
  (full-sequence forward) and torch-CPU float64 functional ops;
* closed forms (C-P): W_o = W_down = 0 => out = x; pos = 0 => attention output = v;
  W_q = 0 => uniform weights => o = mean of V; constant-vector RMSNorm;
* invariants: WaS == replicated bitwise, CaS == replicated to BLAS
  rounding, dummy neutrality.
"""
import copy

import numpy as np
import pytest
import torch

from oracle import model as M
from oracle import schedule as S
from oracle import sidp as SD
from sidp_inputs import MODELS, gen

SEED = 20261017


def _model_params(m, seed=SEED):
    layers = [gen.layer_params(seed, m, l) for l in range(m.num_layers)]
    head = gen.head_params(seed, m)
    return layers, head


# --------------------------------------------------------------------- generator
def test_generator_exact_bf16_and_range():
    w = gen.weight(SEED, gen.WQ, 3, 64, 256)
    t = torch.from_numpy(w)
    assert torch.equal(t.to(torch.bfloat16).double(), t)          # exactly representable
    assert np.abs(w).max() <= 2.0 ** -4 and len(np.unique(w)) <= 256
    g = gen.gain(SEED, gen.G_ATTN, 0, 4096)
    assert torch.equal(torch.from_numpy(g).to(torch.bfloat16).double(), torch.from_numpy(g))
    assert g.min() >= 1 - 8 / 128 and g.max() <= 1 + 7 / 128
    kv = gen.kv(SEED, gen.KCACHE, 1, [0, 5], range(7), 2, 64)
    assert kv.shape == (2, 7, 2, 64)
    assert torch.equal(torch.from_numpy(kv).to(torch.bfloat16).double(), torch.from_numpy(kv))


def test_generator_logical_coordinates():
    """Row subsets and KV sub-ranges equal slices of the full tensor (layout-free values)."""
    full = gen.weight(SEED, gen.WUP, 2, 40, 128)
    np.testing.assert_array_equal(full[[3, 17, 39]], gen.weight(SEED, gen.WUP, 2, 40, 128, rows=[3, 17, 39]))
    a = gen.kv(SEED, gen.VCACHE, 0, [4, 9], range(10), 2, 64)
    b = gen.kv(SEED, gen.VCACHE, 0, [9], range(3, 8), 2, 64)
    np.testing.assert_array_equal(a[1:2, 3:8], b)
    assert not np.array_equal(gen.weight(SEED, gen.WQ, 0, 4, 64), gen.weight(SEED, gen.WK, 0, 4, 64))


def test_splitmix64_public_vector(golden_dir):
    import json, os
    gold = json.load(open(os.path.join(golden_dir, "spec_examples.json")))["splitmix64_seed0"]
    gamma = 0x9E3779B97F4A7C15
    got = [int(gen.splitmix64(np.array([(k * gamma) % 2**64], dtype=np.uint64))[0]) for k in range(3)]
    assert got == [int(x, 16) for x in gold["outputs"]]


# --------------------------------------------------------------------- HF pin
def _hf_model(m, layers, head, embed):
    from transformers import LlamaConfig, Qwen2Config, Qwen3Config
    from transformers import LlamaForCausalLM, Qwen2ForCausalLM, Qwen3ForCausalLM
    common = dict(hidden_size=m.hidden, intermediate_size=m.intermediate,
                  num_hidden_layers=m.num_layers, num_attention_heads=m.n_q_heads,
                  num_key_value_heads=m.n_kv_heads, head_dim=m.head_dim, vocab_size=m.vocab,
                  rms_norm_eps=m.rms_eps, rope_theta=m.rope_theta, tie_word_embeddings=False,
                  max_position_embeddings=4096)
    if m.qk_norm:
        cfg, cls = Qwen3Config(**common, attention_bias=False), Qwen3ForCausalLM
    elif m.qkv_bias:
        cfg, cls = Qwen2Config(**common), Qwen2ForCausalLM
    else:
        cfg, cls = LlamaConfig(**common, attention_bias=False, mlp_bias=False), LlamaForCausalLM
    cfg._attn_implementation = "sdpa"   # eager softmax runs in float32
    hf = cls(cfg).double().eval()
    sd = {"model.embed_tokens.weight": embed, "model.norm.weight": head["g_final"],
          "lm_head.weight": head["wlm"]}
    for l, p in enumerate(layers):
        pre = f"model.layers.{l}."
        sd.update({pre + "self_attn.q_proj.weight": p["wq"], pre + "self_attn.k_proj.weight": p["wk"],
                   pre + "self_attn.v_proj.weight": p["wv"], pre + "self_attn.o_proj.weight": p["wo"],
                   pre + "mlp.gate_proj.weight": p["wgate"], pre + "mlp.up_proj.weight": p["wup"],
                   pre + "mlp.down_proj.weight": p["wdown"], pre + "input_layernorm.weight": p["g_attn"],
                   pre + "post_attention_layernorm.weight": p["g_mlp"]})
        if m.qk_norm:
            sd[pre + "self_attn.q_norm.weight"] = p["g_q"]
            sd[pre + "self_attn.k_norm.weight"] = p["g_k"]
        if m.qkv_bias:
            sd[pre + "self_attn.q_proj.bias"] = p["bq"]
            sd[pre + "self_attn.k_proj.bias"] = p["bk"]
            sd[pre + "self_attn.v_proj.bias"] = p["bv"]
    missing, unexpected = hf.load_state_dict({k: torch.from_numpy(np.asarray(v)) for k, v in sd.items()},
                                             strict=False)
    assert not unexpected and all("rotary" in k for k in missing), (missing, unexpected)
    # HF builds inv_freq in float32; rebuild it in float64 so the comparison is fp64 end to end
    rot = hf.model.rotary_emb
    inv = 1.0 / (m.rope_theta ** (torch.arange(0, m.head_dim, 2, dtype=torch.float64) / m.head_dim))
    # and its forward casts angles to float32; replace it by the same formula in float64
    def fwd64(x, position_ids):
        freqs = position_ids[..., None].double() * inv[None, None, :]
        emb = torch.cat([freqs, freqs], dim=-1)
        return emb.cos().to(x.dtype), emb.sin().to(x.dtype)
    rot.forward = fwd64
    # HF RMSNorm upcasts to float32 internally; use the float64 library routine instead
    for mod in hf.modules():
        if type(mod).__name__.endswith("RMSNorm"):
            mod.forward = (lambda mm: (lambda x: torch.nn.functional.rms_norm(
                x, (x.shape[-1],), mm.weight, eps=mm.variance_epsilon)))(mod)
    return hf


@pytest.mark.parametrize("name", ["tiny", "tiny-qwen3", "tiny-qwen25"])
def test_decode_step_matches_hf(name):
    """One decode step of the oracle, fed the KV cache HF builds from a prompt, equals HF's
    full forward at the last position: per-layer inputs, logits (rel 1e-10)."""
    m = MODELS[name]
    layers, head = _model_params(m)
    embed = gen.embed_rows(SEED, np.arange(m.vocab), m.hidden)
    hf = _hf_model(m, layers, head, embed)
    rng = np.random.default_rng(0)
    for P in (0, 1, 7, 33):
        seq = rng.integers(0, m.vocab, size=P + 1)
        with torch.no_grad():
            full = hf(torch.from_numpy(seq)[None], output_hidden_states=True)
            caches = []
            if P > 0:
                pre = hf(torch.from_numpy(seq[:P])[None], use_cache=True)
                for l in range(m.num_layers):
                    lay = pre.past_key_values.layers[l]
                    k = lay.keys[0].permute(1, 0, 2).numpy()     # [P, n_kv, hd]
                    v = lay.values[0].permute(1, 0, 2).numpy()
                    Kc = np.zeros((1, P + 1, m.n_kv_heads, m.head_dim)); Kc[0, :P] = k
                    Vc = np.zeros((1, P + 1, m.n_kv_heads, m.head_dim)); Vc[0, :P] = v
                    caches.append((Kc, Vc))
            else:
                caches = [(np.zeros((1, 1, m.n_kv_heads, m.head_dim)),
                           np.zeros((1, 1, m.n_kv_heads, m.head_dim))) for _ in range(m.num_layers)]
        coll = []
        nxt, logits, _ = M.decode_step(m, layers, head, lambda t: embed[t], seq[P:], np.array([P]),
                                       caches, collect=coll)
        ref_logits = full.logits[0, -1].numpy()
        np.testing.assert_allclose(logits[0], ref_logits, rtol=1e-10, atol=1e-10 * np.abs(ref_logits).max())
        for l in range(m.num_layers):
            ref = full.hidden_states[l][0, -1].numpy()
            np.testing.assert_allclose(coll[l][0], ref, rtol=1e-10, atol=1e-12)
        assert int(nxt[0]) == int(np.argmax(ref_logits))


def test_library_ops():
    """RMSNorm, SiLU, RoPE-free attention vs torch float64 functional routines."""
    rng = np.random.default_rng(1)
    x = rng.standard_normal((5, 64)); g = rng.standard_normal(64)
    ref = torch.nn.functional.rms_norm(torch.from_numpy(x), (64,), torch.from_numpy(g), eps=1e-5)
    np.testing.assert_allclose(M.rmsnorm(x, g, 1e-5), ref.numpy(), rtol=1e-12)
    np.testing.assert_allclose(M.silu(x), torch.nn.functional.silu(torch.from_numpy(x)).numpy(), rtol=1e-12)
    m = MODELS["tiny"]
    B, T = 3, 9
    q = rng.standard_normal((B, m.n_q_heads, m.head_dim))
    Kc = rng.standard_normal((B, T, m.n_kv_heads, m.head_dim))
    Vc = rng.standard_normal((B, T, m.n_kv_heads, m.head_dim))
    pos = np.array([0, 4, 8])
    o = M.attend(m, q, Kc, Vc, pos).reshape(B, m.n_q_heads, m.head_dim)
    for b in range(B):
        n = pos[b] + 1
        qq = torch.from_numpy(q[b])[None, :, None, :]                      # [1, H, 1, hd]
        kk = torch.from_numpy(Kc[b, :n]).permute(1, 0, 2)[None]            # [1, Hkv, n, hd]
        vv = torch.from_numpy(Vc[b, :n]).permute(1, 0, 2)[None]
        ref = torch.nn.functional.scaled_dot_product_attention(qq, kk, vv, enable_gqa=True)
        np.testing.assert_allclose(o[b], ref[0, :, 0].numpy(), rtol=1e-12, atol=1e-12)


# --------------------------------------------------------------------- closed forms
def _layer_inputs(m, B=4, T=12):
    rng = np.random.default_rng(2)
    x = rng.standard_normal((B, m.hidden))
    pos = np.array([0, 3, 7, 11])[:B]
    Kc = rng.standard_normal((B, T, m.n_kv_heads, m.head_dim))
    Vc = rng.standard_normal((B, T, m.n_kv_heads, m.head_dim))
    return x, pos, Kc, Vc


def test_closed_form_zero_output_projections():
    m = MODELS["tiny"]
    p = gen.layer_params(SEED, m, 0)
    p["wo"] = np.zeros_like(p["wo"]); p["wdown"] = np.zeros_like(p["wdown"])
    x, pos, Kc, Vc = _layer_inputs(m)
    assert np.array_equal(M.decoder_layer(m, p, x, pos, Kc, Vc), x)


def test_closed_form_pos0_attention_is_v():
    m = MODELS["tiny"]
    p = gen.layer_params(SEED, m, 1)
    x, _, Kc, Vc = _layer_inputs(m)
    pos = np.zeros(4, dtype=np.int64)
    u = M.attn_norm(m, p, x)
    q, k, v = M.qkv_post(m, p, M.qkv_proj(m, p, u), pos)
    np.testing.assert_allclose(q, (u @ p["wq"].T).reshape(q.shape), rtol=1e-13)  # RoPE(pos 0) = id
    M.append_kv(Kc, Vc, k, v, pos)
    o = M.attend(m, q, Kc, Vc, pos).reshape(4, m.n_q_heads, m.head_dim)
    grp = m.n_q_heads // m.n_kv_heads
    for j in range(m.n_q_heads):
        np.testing.assert_allclose(o[:, j], v[:, j // grp], rtol=1e-13)


def test_closed_form_uniform_attention_mean_v():
    m = MODELS["tiny"]
    x, pos, Kc, Vc = _layer_inputs(m)
    q = np.zeros((4, m.n_q_heads, m.head_dim))
    o = M.attend(m, q, Kc, Vc, pos).reshape(4, m.n_q_heads, m.head_dim)
    grp = m.n_q_heads // m.n_kv_heads
    for b in range(4):
        for j in range(m.n_q_heads):
            np.testing.assert_allclose(o[b, j], Vc[b, :pos[b] + 1, j // grp].mean(0), rtol=1e-12)


def test_closed_form_rmsnorm_constant_and_rope_rotation():
    g = np.linspace(0.5, 2, 16)
    np.testing.assert_allclose(M.rmsnorm(np.full((1, 16), -3.0), g, 0.0), -g[None], rtol=1e-15)
    # RoPE preserves the norm of each (i, i+hd/2) pair and composes additively in position
    rng = np.random.default_rng(3)
    x = rng.standard_normal((1, 2, 8))
    y = M.rope(x, np.array([5]), 1e4)
    np.testing.assert_allclose(x[..., :4] ** 2 + x[..., 4:] ** 2, y[..., :4] ** 2 + y[..., 4:] ** 2, rtol=1e-12)
    np.testing.assert_allclose(M.rope(M.rope(x, np.array([2]), 1e4), np.array([3]), 1e4), y, rtol=1e-12)


def test_argmax_lowest_index_ties():
    assert list(M.argmax_lowest(np.array([[1.0, 3.0, 3.0, 0.0], [2.0, 2.0, 2.0, 2.0]]))) == [1, 0]


# --------------------------------------------------------------------- SiDP invariants
def _ranks(m, batches, seed=SEED, T=80, ctx_span=20):
    ranks = []
    base = 0
    for r, B in enumerate(batches):
        bg = np.arange(base, base + B); base += B
        pos = gen.positions(seed, bg, 0, ctx_span)
        toks = gen.tokens(seed, bg, m.vocab)
        caches = []
        for l in range(m.num_layers):
            Kc = np.zeros((B, T, m.n_kv_heads, m.head_dim)); Vc = np.zeros_like(Kc)
            if B:
                Kc[:, :T] = gen.kv(seed, gen.KCACHE, l, bg, range(T), m.n_kv_heads, m.head_dim)
                Vc[:, :T] = gen.kv(seed, gen.VCACHE, l, bg, range(T), m.n_kv_heads, m.head_dim)
            caches.append((Kc, Vc))
        ranks.append(SD.RankState(r, toks, pos, caches))
    return ranks


def _embed(m):
    E = gen.embed_rows(SEED, np.arange(m.vocab), m.hidden)
    return lambda t: E[np.asarray(t)]


@pytest.mark.parametrize("name,d,slots,order,pool", [
    ("tiny", 2, 1, "exec", "layer"), ("tiny", 2, 2, "exec", "layer"),
    ("tiny", 4, 3, "paper", "layer"), ("tiny-qwen3", 4, 2, "exec", "ffn"),
    ("tiny-qwen25", 2, 2, "exec", "ffn")])
def test_was_equals_replicated_bitwise(name, d, slots, order, pool):
    m = MODELS[name]
    layers, head = _model_params(m)
    emb = _embed(m)
    batches = [3, 2, 4, 1][:d]
    rep = SD.run_replicated(m, layers, head, emb, _ranks(m, batches), steps=3)
    log = []
    was = SD.run_was(m, layers, head, emb, _ranks(m, batches), 3, d, S.owner_map(m.num_layers, d),
                     slots, order, pool, log=log)
    for a, b in zip(rep, was):
        for ha, hb in zip(a.history, b.history):
            assert np.array_equal(ha["logits"], hb["logits"])
            assert np.array_equal(ha["next"], hb["next"])
    # every remote layer fetched exactly once per pass, into the FIFO-assigned slot
    own = S.owner_map(m.num_layers, d)
    for r in range(d):
        mine = [(t, l, s) for (rr, t, l, s) in log if rr == r]
        assert mine == S.slot_schedule(S.plan(own, d, r, order), slots, 3)


@pytest.mark.parametrize("pool", ["layer", "ffn"])
@pytest.mark.parametrize("batches", [[3, 2, 4, 1], [0, 2, 0, 5], [4, 0, 0, 0]])
def test_cas_equals_replicated_and_dummy_neutral(pool, batches):
    m = MODELS["tiny"]
    layers, head = _model_params(m)
    emb = _embed(m)
    d = len(batches)
    rep = SD.run_replicated(m, layers, head, emb, _ranks(m, batches), steps=2)
    traffic = []
    cas = SD.run_cas(m, layers, head, emb, _ranks(m, batches), 2, d, S.owner_map(m.num_layers, d),
                     pool, traffic=traffic)
    for a, b in zip(rep, cas):
        for ha, hb in zip(a.history, b.history):
            if ha is None:
                assert hb is None
                continue
            np.testing.assert_allclose(hb["logits"], ha["logits"], rtol=1e-12,
                                       atol=1e-12 * np.abs(ha["logits"]).max())
    live = [r for r, B in enumerate(batches) if B > 0]
    for (_, _, _, senders) in traffic:            # dummy ranks never move data
        assert senders == live


def test_dummy_neutrality_outputs_unchanged():
    """Live ranks' outputs do not depend on whether other ranks are dummy."""
    m = MODELS["tiny"]
    layers, head = _model_params(m)
    emb = _embed(m)
    own = S.owner_map(m.num_layers, 4)
    a = SD.run_cas(m, layers, head, emb, _ranks(m, [3, 2, 4, 1]), 1, 4, own)
    b = SD.run_cas(m, layers, head, emb, _ranks(m, [3, 2, 4, 1]), 1, 4, own)
    b2 = _ranks(m, [3, 2, 4, 1])
    b2[1] = SD.RankState(1, b2[1].tokens[:0], b2[1].pos[:0], [(K[:0], V[:0]) for K, V in b2[1].caches])
    c = SD.run_cas(m, layers, head, emb, b2, 1, 4, own)
    for r in (0, 2, 3):
        ref = a[r].history[0]["logits"]
        np.testing.assert_allclose(c[r].history[0]["logits"], ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())
    assert c[1].history[0] is None
