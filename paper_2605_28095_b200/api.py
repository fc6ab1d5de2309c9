"""Thin Python binding over libsidp.so: same names as the C ABI, marshalling only.

torch is used for device memory (caller-owned activations, KV caches, tokens) and
streams; every step of the hot path runs in the library's CUDA kernels.
"""
from __future__ import annotations

import ctypes as C

from . import _abi as A


def _stream_ptr(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def model_desc(m) -> A.ModelDesc:
    return A.ModelDesc(m.num_layers, m.hidden, m.n_q_heads, m.n_kv_heads, m.head_dim,
                       m.intermediate, m.vocab, int(m.qkv_bias), int(m.qk_norm),
                       float(m.rms_eps), float(m.rope_theta))


class KVCache:
    """Caller-owned KV cache of one rank: bf16 [L][max_batch][n_kv][max_ctx][head_dim] x 2."""

    def __init__(self, m, max_batch: int, max_ctx: int, device="cuda"):
        import torch
        shape = (m.num_layers, max_batch, m.n_kv_heads, max_ctx, m.head_dim)
        self.k = torch.empty(shape, dtype=torch.bfloat16, device=device)
        self.v = torch.empty(shape, dtype=torch.bfloat16, device=device)
        self.pos = torch.zeros(max_batch, dtype=torch.int32, device=device)
        self.max_pos = 0
        self.max_batch, self.max_ctx = max_batch, max_ctx

    def set_pos(self, pos):
        import torch
        p = torch.as_tensor(pos, dtype=torch.int32)
        self.pos[:p.numel()].copy_(p)
        self.max_pos = int(p.max()) if p.numel() else 0

    def advance(self, n: int = 1, batch: int | None = None):
        b = self.max_batch if batch is None else batch
        self.pos[:b] += n
        self.max_pos += n

    def c(self) -> A.KV:
        return A.KV(self.k.data_ptr(), self.v.data_ptr(), self.pos.data_ptr(), self.max_pos)

    def fill_synthetic(self, seed: int, b0: int, batch: int, T: int, stream=None):
        """K12 fill of positions [0, T) for rows [0, batch) (logical rows b0 + b)."""
        L = self.k.shape[0]
        nkv, smax, hd = self.k.shape[2], self.k.shape[3], self.k.shape[4]
        for l in range(L):
            for t_id, buf in ((18, self.k), (19, self.v)):   # gen.KCACHE / gen.VCACHE
                A.check(A.lib().sidp_test_gen_kv(_ptr(buf[l]), batch, nkv, smax, hd, T, b0, seed,
                                                 t_id, l, _stream_ptr(stream)), "gen_kv")


class PagedKVCache:
    """Caller-owned PAGED KV cache (sidp_kv.block_table): per layer a pool of 16-token blocks,
    bf16 [L][num_blocks][n_kv][16][head_dim] x 2, and a device block table int32
    [max_batch][max_blocks] (token t of row b in block table[b][t // 16], slot t % 16)."""
    BLOCK = 16

    def __init__(self, m, max_batch: int, max_ctx: int, num_blocks: int, device="cuda"):
        import torch
        self.max_blocks = (max_ctx + self.BLOCK - 1) // self.BLOCK
        self.num_blocks = num_blocks
        shape = (m.num_layers, num_blocks, m.n_kv_heads, self.BLOCK, m.head_dim)
        self.k = torch.zeros(shape, dtype=torch.bfloat16, device=device)
        self.v = torch.zeros(shape, dtype=torch.bfloat16, device=device)
        self.table = torch.zeros(max_batch, self.max_blocks, dtype=torch.int32, device=device)
        self.pos = torch.zeros(max_batch, dtype=torch.int32, device=device)
        self.max_pos = 0
        self.max_batch, self.max_ctx = max_batch, max_ctx

    @classmethod
    def from_contiguous(cls, kv: "KVCache", m, seed: int = 0, spare: int = 0):
        """The same cache contents in shuffled blocks: row b's c-th block goes to pool block
        perm[b * max_blocks + c] (a seeded permutation of num_blocks = B * max_blocks + spare)."""
        import torch
        B, T = kv.max_batch, kv.max_ctx
        pk = cls(m, B, T, B * ((T + cls.BLOCK - 1) // cls.BLOCK) + spare, device=kv.k.device)
        nb = pk.max_blocks
        g = torch.Generator().manual_seed(seed)
        perm = torch.randperm(pk.num_blocks, generator=g)[:B * nb]
        pk.table.copy_(perm.view(B, nb).to(torch.int32))
        for src, dst in ((kv.k, pk.k), (kv.v, pk.v)):
            L, _, nkv, _, hd = src.shape
            pad = torch.zeros(L, B, nkv, nb * cls.BLOCK, hd, dtype=src.dtype, device=src.device)
            pad[:, :, :, :T] = src
            blocks = pad.view(L, B, nkv, nb, cls.BLOCK, hd).permute(0, 1, 3, 2, 4, 5)
            dst[:, perm.to(src.device)] = blocks.reshape(L, B * nb, nkv, cls.BLOCK, hd)
        pk.pos.copy_(kv.pos)
        pk.max_pos = kv.max_pos
        return pk

    def fill_synthetic(self, seed: int, b0: int, batch: int, T: int, stream=None, perm_seed: int = 0):
        """K12 fill of positions [0, T) of rows [0, batch) (logical rows b0 + b), one layer at a
        time through a contiguous staging buffer, into a seeded shuffle of the pool's blocks."""
        import torch
        L, nb, B = self.k.shape[0], self.max_blocks, self.max_batch
        nkv, hd = self.k.shape[2], self.k.shape[4]
        g = torch.Generator().manual_seed(perm_seed)
        perm = torch.randperm(self.num_blocks, generator=g)[:B * nb]
        self.table.copy_(perm.view(B, nb).to(torch.int32))
        perm = perm.to(self.k.device)
        stage = torch.zeros(B, nkv, nb * self.BLOCK, hd, dtype=torch.bfloat16, device=self.k.device)
        for l in range(L):
            for t_id, pool in ((18, self.k), (19, self.v)):   # gen.KCACHE / gen.VCACHE
                A.check(A.lib().sidp_test_gen_kv(_ptr(stage), batch, nkv, nb * self.BLOCK, hd, T, b0,
                                                 seed, t_id, l, _stream_ptr(stream)), "gen_kv")
                blocks = stage.view(B, nkv, nb, self.BLOCK, hd).permute(0, 2, 1, 3, 4)
                pool[l][perm] = blocks.reshape(B * nb, nkv, self.BLOCK, hd)

    def to_contiguous(self, layer, which="k"):
        """Layer `layer`'s cache gathered back into [max_batch][n_kv][max_blocks*16][hd]."""
        pool = (self.k if which == "k" else self.v)[layer]
        x = pool[self.table.long()]                      # [B][nb][nkv][16][hd]
        B, nb, nkv, bt, hd = x.shape
        return x.permute(0, 2, 1, 3, 4).reshape(B, nkv, nb * bt, hd)

    set_pos = KVCache.set_pos
    advance = KVCache.advance

    def c(self) -> A.KV:
        return A.KV(self.k.data_ptr(), self.v.data_ptr(), self.pos.data_ptr(), self.max_pos,
                    self.table.data_ptr(), self.BLOCK, self.max_blocks, self.num_blocks)


class _RowsKV:
    """A paged cache seen through one block-table row per query row (prefill rows of one
    sequence share that sequence's blocks)."""

    def __init__(self, kv: "PagedKVCache", table, pos):
        self.k, self.v, self.table, self.pos = kv.k, kv.v, table, pos
        self.max_pos = int(pos.max().item()) if pos.numel() else 0
        self.max_blocks, self.num_blocks = kv.max_blocks, kv.num_blocks

    def c(self) -> A.KV:
        return A.KV(self.k.data_ptr(), self.v.data_ptr(), self.pos.data_ptr(), self.max_pos,
                    self.table.data_ptr(), PagedKVCache.BLOCK, self.max_blocks, self.num_blocks)


def prefill_rows(pos0, prompts):
    """Host side of prefill: one row per prompt token — (sequence of the row, its position
    pos0[seq] + i, its token) — and the row of each sequence's last prompt token."""
    import numpy as np
    lens = [len(p) for p in prompts]
    seq = np.concatenate([np.full(n, b) for b, n in enumerate(lens)]).astype(np.int64)
    pos = np.concatenate([int(pos0[b]) + np.arange(n) for b, n in enumerate(lens)]).astype(np.int32)
    toks = np.concatenate([np.asarray(p, dtype=np.int32) for p in prompts])
    return seq, pos, toks, np.cumsum(lens) - 1


def prefill(ctx: "Context", kv: "PagedKVCache", prompts, stream=None, logits=None,
            layer_inputs=None):
    """Prefill as ONE ragged decode step: every prompt token of every
    sequence is a row whose position is its place in the sequence, whose block-table row is its
    sequence's, so the step's KV append writes all prompt tokens into the sequence's blocks and
    each row's attention reads exactly the causal prefix [0, pos] — the library's decode kernels
    unchanged (attention re-reads the prefix per row: O(T^2) KV bytes, no flash-prefill kernel).
    prompts: per sequence b (rows 0.. of kv) an int sequence of tokens appended at kv.pos[b].
    Returns (next token per sequence, the row index of each sequence's last prompt token);
    kv.pos advances by each prompt's length.  logits / layer_inputs: optional per-row outputs."""
    import numpy as np
    import torch
    dev = kv.k.device
    lens = [len(p) for p in prompts]
    seq, pos, toks_np, last = prefill_rows(kv.pos[:len(prompts)].cpu().numpy(), prompts)
    toks = torch.from_numpy(toks_np).to(dev)
    rows = len(seq)
    view = _RowsKV(kv, kv.table[torch.from_numpy(seq).to(dev)].contiguous(),
                   torch.from_numpy(pos).to(dev))
    nxt = torch.zeros(rows, dtype=torch.int32, device=dev)
    ctx.step(toks, nxt, view, batch=rows, logits=logits, layer_inputs=layer_inputs, stream=stream)
    kv.pos[:len(prompts)] += torch.as_tensor(lens, dtype=torch.int32, device=dev)
    kv.max_pos = int(kv.pos[:len(prompts)].max().item())
    return nxt[torch.from_numpy(last).to(dev)], last


class Context:
    def __init__(self, m, *, rank=0, world=1, slots=2, cas_slots=2, order="exec", pool="layer",
                 max_batch=8, max_ctx=128, fetch_sms=24, fetch_engine="sm", stagger=True,
                 device=0, seed=20261017, layer_owner=None, alloc=True, fetch_pace_gbps=0.0,
                 compute_sms=0, slot_parts=0, fetch_ce_share=0.0):
        self.m = m
        self.rank, self.world = rank, world
        self._owner_arr = None
        own_ptr = None
        if layer_owner is not None:
            self._owner_arr = (C.c_int32 * m.num_layers)(*layer_owner)
            own_ptr = C.cast(self._owner_arr, C.POINTER(C.c_int32))
        self.cfg = A.Config(rank, world, own_ptr, slots, cas_slots,
                            A.ORDER_EXEC if order == "exec" else A.ORDER_PAPER,
                            A.POOL_LAYER if pool == "layer" else A.POOL_FFN,
                            max_batch, max_ctx, fetch_sms,
                            A.FETCH_SM if fetch_engine == "sm" else A.FETCH_CE,
                            int(bool(stagger)), device, seed, float(fetch_pace_gbps), int(compute_sms),
                            int(slot_parts), float(fetch_ce_share))
        self.desc = model_desc(m)
        h = C.c_void_p()
        A.check(A.lib().sidp_init(C.byref(self.desc), C.byref(self.cfg), C.byref(h)), "sidp_init")
        self.h = h
        self.max_batch, self.max_ctx = max_batch, max_ctx
        if alloc:
            self.alloc()

    # ---- lifecycle
    def alloc(self, arena=None):
        """arena: optional caller-owned device buffer (e.g. a torch uint8 tensor of at least
        owned_bytes()) that holds this rank's owned layers (sidp_alloc_owned); kept referenced."""
        if arena is None:
            A.check(A.lib().sidp_alloc(self.h), "sidp_alloc")
            return
        self._arena = arena
        A.check(A.lib().sidp_alloc_owned(self.h, _ptr(arena), arena.numel() * arena.element_size()),
                "sidp_alloc_owned")

    def owned_bytes(self) -> int:
        n = C.c_uint64()
        A.check(A.lib().sidp_owned_bytes(self.h, C.byref(n)), "sidp_owned_bytes")
        return n.value

    def alloc_serve_only(self, alias_of=None):
        """Owner-only rank: allocates and exports its arena, never computes (sidp.h).  alias_of
        (timing emulation only): share that serve-only context's arena instead of allocating."""
        if alias_of is None:
            A.check(A.lib().sidp_alloc_serve_only(self.h), "sidp_alloc_serve_only")
        else:
            A.check(A.lib().sidp_alloc_serve_only_alias(self.h, alias_of.h),
                    "sidp_alloc_serve_only_alias")

    def init_weights_synthetic(self, stream=None):
        A.check(A.lib().sidp_init_weights_synthetic(self.h, _stream_ptr(stream)),
                "sidp_init_weights_synthetic")

    def export_handles(self) -> bytes:
        n = C.c_size_t(0)
        A.check(A.lib().sidp_export_handles(self.h, None, C.byref(n)), "export(size)")
        buf = (C.c_char * n.value)()
        A.check(A.lib().sidp_export_handles(self.h, C.cast(buf, C.c_void_p), C.byref(n)), "export")
        return bytes(buf[:n.value])

    def import_handles(self, blobs):
        bufs = [C.create_string_buffer(b, len(b)) for b in blobs]
        ptrs = (C.c_void_p * len(bufs))(*[C.cast(b, C.c_void_p) for b in bufs])
        lens = (C.c_size_t * len(bufs))(*[len(b) for b in blobs])
        A.check(A.lib().sidp_import_handles(self.h, ptrs, lens), "sidp_import_handles")

    def destroy(self):
        if self.h:
            A.lib().sidp_destroy(self.h)
            self.h = None

    close = destroy

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    # ---- hot path
    def decode_layer(self, x, layer, mode, kv: KVCache, batch=None, stream=None):
        b = x.shape[0] if batch is None else batch
        kvc = kv.c()
        A.check(A.lib().sidp_decode_layer(self.h, _ptr(x), b, layer, mode, C.byref(kvc),
                                          _stream_ptr(stream)), "sidp_decode_layer")

    def step(self, tokens, nxt, kv: KVCache, batch=None, logits=None, layer_inputs=None,
             stream=None, advance_pos=False):
        """One decode step.  advance_pos=True lets the library write pos+1 back into kv.pos
        (and the host hint kv.max_pos is bumped here), so a decode loop launches nothing else."""
        b = tokens.shape[0] if batch is None else batch
        bt = A.Batch(tokens.data_ptr() if b else None, nxt.data_ptr() if b else None, b, kv.c(),
                     logits.data_ptr() if logits is not None else None,
                     layer_inputs.data_ptr() if layer_inputs is not None else None,
                     kv.pos.data_ptr() if advance_pos else None)
        A.check(A.lib().sidp_step(self.h, C.byref(bt), _stream_ptr(stream)), "sidp_step")
        if advance_pos:
            kv.max_pos += 1

    def set_mode(self, mode, effective_step):
        A.check(A.lib().sidp_set_mode(self.h, mode, effective_step), "sidp_set_mode")

    def set_batches(self, batches):
        arr = (C.c_int32 * len(batches))(*batches)
        A.check(A.lib().sidp_set_batches(self.h, arr), "sidp_set_batches")

    # ---- introspection
    def owner_of(self, layer) -> int:
        o = C.c_int32()
        A.check(A.lib().sidp_owner_of(self.h, layer, C.byref(o)), "sidp_owner_of")
        return o.value

    def plan(self) -> list[int]:
        n = C.c_int32()
        A.check(A.lib().sidp_get_plan(self.h, None, 0, C.byref(n)), "plan")
        arr = (C.c_int32 * max(1, n.value))()
        A.check(A.lib().sidp_get_plan(self.h, arr, n.value, C.byref(n)), "plan")
        return list(arr[:n.value])

    def schedule(self, steps: int) -> list[tuple[int, int, int]]:
        n = C.c_int32()
        A.check(A.lib().sidp_get_schedule(self.h, steps, None, None, None, 0, C.byref(n)), "sched")
        k = max(1, n.value)
        t, l, s = (C.c_int32 * k)(), (C.c_int32 * k)(), (C.c_int32 * k)()
        A.check(A.lib().sidp_get_schedule(self.h, steps, t, l, s, k, C.byref(n)), "sched")
        return list(zip(t[:n.value], l[:n.value], s[:n.value]))

    def fetch_log(self) -> list[tuple[int, int, int]]:
        n = C.c_int32()
        A.check(A.lib().sidp_get_fetch_log(self.h, None, None, None, 0, C.byref(n)), "log")
        k = max(1, n.value)
        t, l, s = (C.c_int32 * k)(), (C.c_int32 * k)(), (C.c_int32 * k)()
        A.check(A.lib().sidp_get_fetch_log(self.h, t, l, s, k, C.byref(n)), "log")
        return list(zip(t[:n.value], l[:n.value], s[:n.value]))

    def fetch_trace(self) -> list[tuple]:
        """SM fetch: device log rows (j, layer, slot, owner, epoch, t_start_ns, t_end_ns)."""
        return self._rows(A.lib().sidp_get_fetch_trace, 7)

    def consume_log(self) -> list[tuple]:
        """SM fetch: compute-side consumptions (layer, slot, tag, epoch, t_ready_ns)."""
        return self._rows(A.lib().sidp_get_consume_log, 5)

    def _rows(self, fn, w):
        n = C.c_int32()
        A.check(fn(self.h, None, 0, C.byref(n)), fn.__name__)
        k = max(1, n.value)
        buf = (C.c_int64 * (k * w))()
        A.check(fn(self.h, buf, k, C.byref(n)), fn.__name__)
        return [tuple(buf[i * w:(i + 1) * w]) for i in range(n.value)]

    def stagger_ticks(self) -> int:
        v = C.c_int32()
        A.check(A.lib().sidp_stagger_ticks(self.h, C.byref(v)), "stagger")
        return v.value

    def stats(self) -> dict:
        s = A.Stats()
        A.check(A.lib().sidp_stats(self.h, C.byref(s)), "sidp_stats")
        d = {f: getattr(s, f) for f, _ in A.Stats._fields_}
        d["timed_ms"] = list(s.timed_ms)
        d["timed_launches"] = list(s.timed_launches)
        return d

    # kernel classes for set_timing (bit positions)
    K_GATEUP, K_ATTN, K_FETCH, K_DOWN, K_QKV, K_O, K_LMHEAD = 1, 2, 3, 4, 5, 6, 7

    def set_timing(self, class_mask: int):
        A.check(A.lib().sidp_set_timing(self.h, class_mask), "sidp_set_timing")

    def layer_ptr(self, layer):
        p, q = C.c_void_p(), C.c_void_p()
        A.check(A.lib().sidp_layer_ptr(self.h, layer, C.byref(p), C.byref(q)), "layer_ptr")
        return p.value, q.value


# ---- single-kernel test hooks (same kernels as the hot path) ----
def test_gemm(x, w, out, M, N, K, epi, resid=None, bias=None, k_splits=0, ldo=None, stream=None):
    A.check(A.lib().sidp_test_gemm(_ptr(x), x.stride(0), _ptr(w), w.stride(0), M, N, K, epi,
                                   _ptr(out), out.stride(0) if ldo is None else ldo, _ptr(resid),
                                   resid.stride(0) if resid is not None else 0, _ptr(bias),
                                   k_splits, _stream_ptr(stream)), "sidp_test_gemm")


def test_gemm_qkv(x, w, bias, nq, nkv, hd, gq, gk, eps, rope, pos, q, kc, vc, smax, k_splits=0,
                  stream=None):
    M, K = x.shape
    A.check(A.lib().sidp_test_gemm_qkv(_ptr(x), x.stride(0), _ptr(w), M, K, _ptr(bias), nq, nkv, hd,
                                       _ptr(gq), _ptr(gk), eps, _ptr(rope), _ptr(pos), _ptr(q),
                                       _ptr(kc), _ptr(vc), smax, k_splits, _stream_ptr(stream)),
            "sidp_test_gemm_qkv")


def test_gemm_resid_norm(x, w, resid, g, eps, xout, u, stream=None):
    M, K = x.shape
    N = w.shape[0]
    A.check(A.lib().sidp_test_gemm_resid_norm(_ptr(x), x.stride(0), _ptr(w), M, N, K, _ptr(resid),
                                              resid.stride(0), _ptr(g), eps, _ptr(xout), _ptr(u),
                                              _stream_ptr(stream)), "sidp_test_gemm_resid_norm")


def test_mlp_fused(u, wgu, wd, resid, g, eps, act, xout, unorm, stream=None):
    M, h = u.shape
    I = wd.shape[1]
    A.check(A.lib().sidp_test_mlp_fused(_ptr(u), _ptr(wgu), _ptr(wd), _ptr(resid), M, h, I, _ptr(g),
                                        eps, _ptr(act), _ptr(xout), _ptr(unorm), _stream_ptr(stream)),
            "sidp_test_mlp_fused")


def test_gen(dst, seed, tensor, layer, kind, scale_k=0, row0=0, lcols=None, row_map=0, stream=None):
    rows, cols = dst.shape
    A.check(A.lib().sidp_test_gen(_ptr(dst), dst.stride(0), rows, cols, seed, tensor, layer, kind,
                                  scale_k, row0, cols if lcols is None else lcols, row_map,
                                  _stream_ptr(stream)), "sidp_test_gen")
