"""End-to-end parity of the CUDA path (through the C ABI) against the fp64 oracle.

Tolerance (north_star): max|gpu - oracle| <= 1e-2 * max|oracle| per layer output, bf16
weights with fp32 accumulation; the integer schedule is compared bit-exactly.
Teacher forcing: the GPU dumps every layer's bf16 input; the oracle
recomputes each layer from that dump and the same KV state.
"""
import numpy as np
import pytest
import torch

from oracle import model as OM
from oracle import schedule as OS
from sidp_inputs import MODELS, gen

from .helpers import OracleModel, oracle_layer, rank_inputs, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-2
SEED = 20261018


@pytest.fixture(scope="module")
def P():
    from paper_2605_28095_b200 import build as B
    B.build()
    import paper_2605_28095_b200 as P
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return P


class Rank:
    def __init__(self, P, m, *, rank=0, world=1, B=8, ctx=0, span=63, max_ctx=80, b0=0,
                 seed=SEED, max_batch=None, **kw):
        self.m, self.B, self.b0 = m, B, b0
        mb = max(B, 1) if max_batch is None else max_batch
        self.ctx = P.Context(m, rank=rank, world=world, max_batch=mb, max_ctx=max_ctx,
                             seed=seed, **kw)
        self.ctx.init_weights_synthetic()
        self.kv = P.KVCache(m, mb, max_ctx)          # layout uses the context's max_batch
        self.kv.fill_synthetic(seed, b0, mb, max_ctx)
        bg = np.arange(b0, b0 + B)
        self.pos = gen.positions(seed, bg, ctx, span)
        self.kv.set_pos(self.pos if B else [0])
        self.toks = torch.from_numpy(gen.tokens(seed, bg, m.vocab)).to(torch.int32).cuda()
        self.next = torch.zeros(max(B, 1), dtype=torch.int32, device="cuda")
        self.logits = torch.zeros(max(B, 1), m.vocab, dtype=torch.float32, device="cuda")
        self.dump = torch.zeros(m.num_layers, max(B, 1), m.hidden, dtype=torch.bfloat16, device="cuda")
        self.stream = torch.cuda.Stream()
        self.history = []

    def step(self):
        with torch.cuda.stream(self.stream):
            self.ctx.step(self.toks, self.next, self.kv, batch=self.B, logits=self.logits,
                          layer_inputs=self.dump, stream=self.stream)

    def finish_step(self):
        self.stream.synchronize()
        self.history.append((self.next[:self.B].clone().cpu(), self.logits[:self.B].clone().cpu(),
                             self.dump[:, :self.B].clone().cpu()))
        if self.B:
            self.toks = self.next[:self.B].clone()
            self.kv.advance(1, self.B)


@pytest.mark.parametrize("name", ["tiny", "tiny-qwen3", "tiny-qwen25"])
def test_tiny_step_teacher_forced(P, name):
    m = MODELS[name]
    R = Rank(P, m, B=8, span=63, max_ctx=80)
    R.step(); R.finish_step()
    nxt, logits, dump = R.history[0]
    om = OracleModel(m, SEED)
    _, toks, pos, caches = rank_inputs(m, SEED, 0, 8, 0, 63, 80)
    xs = dump.double().numpy()
    np.testing.assert_array_equal(xs[0], om.embed(toks))         # exact gather
    out = None
    for l in range(m.num_layers):
        out, kn, vn = oracle_layer(om, l, xs[l], pos, *caches[l])
        if l + 1 < m.num_layers:
            assert rel_err(xs[l + 1], out) <= TOL, (l, rel_err(xs[l + 1], out))
        kg = R.kv.k[l, torch.arange(8), :, torch.from_numpy(pos).long().cuda()].cpu().double().numpy()
        vg = R.kv.v[l, torch.arange(8), :, torch.from_numpy(pos).long().cuda()].cpu().double().numpy()
        assert rel_err(kg, kn) <= TOL and rel_err(vg, vn) <= TOL
    ref_logits = OM.lm_head(m, om.head, out)
    assert rel_err(logits.double().numpy(), ref_logits) <= TOL
    # the fused argmax decides in the kernel's fp32: equal to argmax of the fp32 logits
    assert (nxt.numpy() == np.argmax(logits.numpy(), axis=1)).all()


def test_tiny_multi_step_end_to_end(P):
    """Three un-forced steps (tokens fed back; the oracle follows the GPU's tokens)."""
    m = MODELS["tiny"]
    R = Rank(P, m, B=8, span=63, max_ctx=80)
    om = OracleModel(m, SEED)
    _, toks, pos, caches = rank_inputs(m, SEED, 0, 8, 0, 63, 80)
    cs = [(K.copy(), V.copy()) for K, V in caches]
    t = toks
    for s in range(3):
        R.step(); R.finish_step()
        nxt, logits, _ = R.history[-1]
        o_next, o_logits, _ = OM.decode_step(m, [om.layer(l) for l in range(m.num_layers)], om.head,
                                             om.embed, t, pos + s, cs)
        err = rel_err(logits.double().numpy(), o_logits)
        assert err <= TOL, (s, err)
        top2 = np.sort(o_logits, axis=1)[:, -2:]
        sure = (top2[:, 1] - top2[:, 0]) > 2 * err * np.abs(o_logits).max()
        assert (nxt.numpy()[sure] == o_next[sure]).all()
        t = nxt.numpy().astype(np.int64)


def _group(P, m, d, B, **kw):
    ranks = [Rank(P, m, rank=r, world=d, B=B[r], b0=sum(B[:r]), max_batch=max(B), **kw)
             for r in range(d)]
    blobs = [R.ctx.export_handles() for R in ranks]
    for R in ranks:
        R.ctx.import_handles(blobs)
    return ranks


@pytest.mark.parametrize("d,slots", [(4, 2), (8, 1)])
def test_was_serve_only_peers(P, d, slots):
    """One computing rank beside d-1 serve-only owners (sidp_alloc_serve_only: arena only, as
    bench.py --emulate-world uses them): fetch log == oracle FIFO schedule and logits BITWISE
    equal to the replicated run; the serve-only ranks refuse to compute."""
    m = MODELS["tiny"].with_layers(8)
    R = Rank(P, m, rank=0, world=d, B=5, slots=slots)
    peers = []
    for r in range(1, d):
        c = P.Context(m, rank=r, world=d, max_batch=5, max_ctx=80, seed=SEED, alloc=False)
        c.alloc_serve_only()
        c.init_weights_synthetic()
        peers.append(c)
    torch.cuda.synchronize()
    R.ctx.import_handles([R.ctx.export_handles()] + [c.export_handles() for c in peers])
    steps = 3
    for s in range(steps):
        R.step(); R.finish_step()
    pl = OS.plan(OS.owner_map(m.num_layers, d), d, 0, "exec")
    log = R.ctx.fetch_log()
    assert log == OS.slot_schedule(pl, slots, steps + 1)[:len(log)]
    assert len(log) >= steps * len(pl)
    rep = _replicated(P, m, 5, 0)
    for s in range(steps):
        rep.step(); rep.finish_step()
        assert torch.equal(rep.history[s][1], R.history[s][1]), s
    rep.ctx.destroy()
    with pytest.raises(RuntimeError):
        peers[0].step(R.toks, R.next, R.kv, batch=5)
    for c in peers:
        c.destroy()
    R.ctx.destroy()


def _replicated(P, m, B, b0, **kw):
    kw = {k: v for k, v in kw.items() if k in ("pool",)}
    return Rank(P, m, B=B, b0=b0, **kw)


@pytest.mark.parametrize("name,d,slots,order,pool", [
    ("tiny", 2, 1, "exec", "layer"), ("tiny", 2, 2, "exec", "layer"),
    ("tiny", 4, 3, "paper", "layer"), ("tiny", 4, 2, "exec", "layer"),
    ("tiny-qwen3", 4, 2, "exec", "ffn"), ("tiny-qwen25", 2, 2, "exec", "layer")])
def test_was_virtual_ranks(P, name, d, slots, order, pool):
    """WaS on d virtual ranks (one GPU): fetch log == oracle FIFO schedule bit-exactly, and
    every rank's logits are BITWISE equal to a replicated single-GPU run (fetch is verbatim)."""
    m = MODELS[name].with_layers(8)
    B = [3, 5, 2, 4][:d]
    steps = 3
    ranks = _group(P, m, d, B, slots=slots, order=order, pool=pool)
    for s in range(steps):
        for R in ranks:
            R.step()
        for R in ranks:
            R.finish_step()
    own = OS.owner_map(m.num_layers, d)
    for r, R in enumerate(ranks):
        pl = OS.plan(own, d, r, order)
        assert R.ctx.plan() == pl
        log = R.ctx.fetch_log()
        ref = OS.slot_schedule(pl, slots, steps + 1)
        assert log[:steps * len(pl)] == ref[:steps * len(pl)]
        assert log == ref[:len(log)]
        st = R.ctx.stats()
        assert st["slot_bytes"] == slots * st["layer_bytes"]
        rep = _replicated(P, m, B[r], sum(B[:r]), pool=pool)
        for s in range(steps):
            rep.step(); rep.finish_step()
            assert torch.equal(rep.history[s][1], R.history[s][1]), (r, s)
            assert torch.equal(rep.history[s][0], R.history[s][0])
        rep.ctx.destroy()
    # and against the oracle (teacher-forced last layer -> logits, step 0)
    om = OracleModel(m, SEED)
    for r, R in enumerate(ranks):
        _, toks, pos, caches = rank_inputs(m, SEED, sum(B[:r]), B[r], 0, 63, 80)
        xs = R.history[0][2].double().numpy()
        out, _, _ = oracle_layer(om, m.num_layers - 1, xs[-1], pos, *caches[-1])
        assert rel_err(R.history[0][1].double().numpy(), OM.lm_head(m, om.head, out)) <= TOL
    for R in ranks:
        R.ctx.destroy()


@pytest.mark.parametrize("pool", ["layer", "ffn"])
@pytest.mark.parametrize("B", [[3, 5], [4, 0, 2, 0], [0, 0, 0, 6], [2, 2, 2, 2]])
def test_cas_virtual_ranks(P, pool, B):
    """CaS on virtual ranks: fused owner GEMMs over the concatenated rows; dummy ranks
    (B=0) move nothing.  Per-rank results equal the replicated run within tolerance."""
    name = "tiny"
    m = MODELS[name].with_layers(4)
    d = len(B)
    ranks = _group(P, m, d, B, pool=pool)
    for R in ranks:
        R.ctx.set_batches(B)
        R.ctx.set_mode(1, 0)                      # SIDP_CAS from step 0 on every rank
    for s in range(2):
        for R in ranks:
            R.step()
        for R in ranks:
            R.finish_step()
    for R in ranks:
        st = R.ctx.stats()
        assert st["timeouts"] == 0
        assert st["mode"] == 1
    for r, R in enumerate(ranks):
        if B[r] == 0:
            continue
        rep = _replicated(P, m, B[r], sum(B[:r]), pool=pool)
        for s in range(2):
            rep.toks = R.history[s - 1][0].cuda() if s else rep.toks
            rep.step(); rep.finish_step()
            err = rel_err(R.history[s][1].double().numpy(), rep.history[s][1].double().numpy())
            assert err <= TOL, (r, s, err)
        rep.ctx.destroy()
    for R in ranks:
        R.ctx.destroy()


def test_was_layer_order_enforced(P):
    m = MODELS["tiny"]
    ranks = _group(P, m, 2, [2, 2])
    R = ranks[0]
    x = torch.zeros(2, m.hidden, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(P.SidpError) as e:
        R.ctx.decode_layer(x, 2, 0, R.kv)          # layer 0 expected first
    assert e.value.status == -4
    with pytest.raises(P.SidpError) as e:
        R.ctx.decode_layer(x, 9, 0, R.kv)
    assert e.value.status == -1
    for R in ranks:
        R.ctx.destroy()


@pytest.mark.parametrize("name,B,ctx", [("qwen3-32b", 256, 1024), ("llama-3.1-70b", 64, 512)])
def test_big_shapes_sampled_rows(P, name, B, ctx):
    """Full-size per-layer shapes (the bench's launch configuration) on 2 layers; the oracle
    recomputes sampled rows of every layer (teacher-forced) and the new k/v entries."""
    m = MODELS[name].with_layers(2)
    max_ctx = ctx + 8
    R = Rank(P, m, B=B, ctx=ctx, span=0, max_ctx=max_ctx)
    R.step(); R.finish_step()
    _, logits, dump = R.history[0]
    om = OracleModel(m, SEED)
    rows = np.array([0, 1, B // 3, B // 2, B - 2, B - 1])
    pos = np.full(len(rows), ctx)
    xs = dump[:, rows].double().numpy()
    out = None
    for l in range(m.num_layers):
        K = gen.kv(SEED, gen.KCACHE, l, rows, range(max_ctx), m.n_kv_heads, m.head_dim)
        V = gen.kv(SEED, gen.VCACHE, l, rows, range(max_ctx), m.n_kv_heads, m.head_dim)
        out, kn, _ = oracle_layer(om, l, xs[l], pos, K, V)
        if l + 1 < m.num_layers:
            assert rel_err(xs[l + 1], out) <= TOL, (l, rel_err(xs[l + 1], out))
        kg = R.kv.k[l, torch.from_numpy(rows).cuda(), :, ctx].cpu().double().numpy()
        assert rel_err(kg, kn) <= TOL
    ref = OM.lm_head(m, om.head, out)
    assert rel_err(logits[rows].double().numpy(), ref) <= TOL
    R.ctx.destroy()


def test_was_full_width_d8_serve_only_bitwise(P):
    """WaS at the bench's full per-layer shapes and launch configuration (Qwen3-32B width,
    B = 256, S_ctx = 1024; 16 layers to fit beside a replicated run): rank 0 of a d = 8 group
    whose 7 owners are serve-only contexts (as bench.py --emulate-world) fetches 14 full
    0.975 GB layers per step into 2 slots.  Logits of 2 steps are BITWISE equal to the
    replicated run (verbatim fetch, same kernels) and the fetch log equals the oracle's FIFO
    schedule."""
    m = MODELS["qwen3-32b"].with_layers(16)
    B, ctx, d, steps = 256, 1024, 8, 2
    R = Rank(P, m, rank=0, world=d, B=B, ctx=ctx, span=0, max_ctx=ctx + 8, slots=2, fetch_sms=16)
    peers = []
    for r in range(1, d):
        c = P.Context(m, rank=r, world=d, max_batch=B, max_ctx=ctx + 8, seed=SEED, alloc=False)
        c.alloc_serve_only()
        c.init_weights_synthetic()
        peers.append(c)
    torch.cuda.synchronize()
    R.ctx.import_handles([R.ctx.export_handles()] + [c.export_handles() for c in peers])
    for s in range(steps):
        R.step(); R.finish_step()
    pl = OS.plan(OS.owner_map(m.num_layers, d), d, 0, "exec")
    log = R.ctx.fetch_log()
    assert len(log) >= steps * len(pl) == steps * 14
    assert log == OS.slot_schedule(pl, 2, steps + 1)[:len(log)]
    for c in peers:
        c.destroy()
    rep = Rank(P, m, B=B, ctx=ctx, span=0, max_ctx=ctx + 8)
    for s in range(steps):
        rep.step(); rep.finish_step()
        assert torch.equal(rep.history[s][1], R.history[s][1]), s
        assert torch.equal(rep.history[s][0], R.history[s][0]), s
    rep.ctx.destroy()
    R.ctx.destroy()


def test_cuda_graph_replay_matches_eager(P):
    """An all-local step is captured once and replayed as a CUDA graph; the decoded tokens of
    several replays equal an eager run (logits requested => no graph) bit for bit."""
    m = MODELS["tiny"]
    A = Rank(P, m, B=8, span=63, max_ctx=80)
    Bq = Rank(P, m, B=8, span=63, max_ctx=80)
    for s in range(4):
        with torch.cuda.stream(A.stream):          # graph path: no logits / dumps
            A.ctx.step(A.toks, A.toks, A.kv, batch=8, stream=A.stream, advance_pos=True)
        A.stream.synchronize()
        A.history.append(A.toks.clone().cpu())
        Bq.step(); Bq.finish_step()                # eager path (logits requested)
        assert torch.equal(A.history[-1], Bq.history[-1][0]), s
    st = A.ctx.stats()
    assert st["steps"] == 4 and st["launches"] > 4 * (1 + m.num_layers * 6)
    # per-class kernel timing survives graph capture (external event-record nodes)
    A.ctx.set_timing(1 << 2)
    for s in range(3):
        with torch.cuda.stream(A.stream):
            A.ctx.step(A.toks, A.toks, A.kv, batch=8, stream=A.stream, advance_pos=True)
    A.stream.synchronize()
    st = A.ctx.stats()
    assert st["timed_launches"][2] == 3 * m.num_layers
    assert st["timed_ms"][2] > 0.0
    A.ctx.destroy()
    Bq.ctx.destroy()


@pytest.mark.parametrize("name,B,ctx,span", [("tiny", 1, 1500, 0), ("tiny", 3, 700, 900),
                                              ("tiny-qwen3", 2, 2000, 100),
                                              ("tiny", 40, 0, 1500), ("tiny-qwen3", 12, 0, 3000),
                                              ("tiny", 240, 0, 300),
                                              ("tiny", 200, 0, 60), ("tiny-qwen3", 160, 20, 40),
                                              ("tiny", 300, 0, 400), ("tiny-qwen3", 320, 100, 300)])
def test_long_context_split_kv(P, name, B, ctx, span):
    """Attention work balancing: the batch's 16-token chunks are split evenly over the CTAs, so
    small batches with long contexts split (b, kv head) pairs into pieces merged by the last
    arriving piece (split-KV), and ragged context lengths (uniform 0..span) put piece
    boundaries anywhere, including pairs of one chunk and pairs split over many CTAs.  The last
    cases have many short pairs (>= one wave of pairs, < 32 chunks each at the context bound):
    the warp-per-pair kernel, each warp finishing whole pairs of ragged lengths."""
    m = MODELS[name]
    max_ctx = ctx + span + 8
    R = Rank(P, m, B=B, ctx=ctx, span=span, max_ctx=max_ctx)
    R.step(); R.finish_step()
    _, logits, dump = R.history[0]
    om = OracleModel(m, SEED)
    bg = np.arange(B)
    pos = gen.positions(SEED, bg, ctx, span)
    xs = dump.double().numpy()
    out = None
    for l in range(m.num_layers):
        K = gen.kv(SEED, gen.KCACHE, l, bg, range(max_ctx), m.n_kv_heads, m.head_dim)
        V = gen.kv(SEED, gen.VCACHE, l, bg, range(max_ctx), m.n_kv_heads, m.head_dim)
        out, _, _ = oracle_layer(om, l, xs[l], pos, K, V)
        if l + 1 < m.num_layers:
            assert rel_err(xs[l + 1], out) <= TOL, (l, rel_err(xs[l + 1], out))
    assert rel_err(logits.double().numpy(), OM.lm_head(m, om.head, out)) <= TOL
    R.ctx.destroy()


def test_batch_one_and_max_batch(P):
    """Degenerate batch sizes: B=1 and B = max_batch with a ragged tail (M not a tile multiple)."""
    m = MODELS["tiny"]
    for B in (1, 37):
        R = Rank(P, m, B=B, span=63, max_ctx=80)
        R.step(); R.finish_step()
        _, logits, dump = R.history[0]
        om = OracleModel(m, SEED)
        _, toks, pos, caches = rank_inputs(m, SEED, 0, B, 0, 63, 80)
        xs = dump.double().numpy()
        out = None
        for l in range(m.num_layers):
            out, _, _ = oracle_layer(om, l, xs[l], pos, *caches[l])
        assert rel_err(logits.double().numpy(), OM.lm_head(m, om.head, out)) <= TOL
        R.ctx.destroy()


def test_dummy_step_was_keeps_schedule(P):
    """A WaS rank with batch 0 (dummy) still walks its ring; the fetch log stays equal to the
    oracle's FIFO schedule and the next real step is correct."""
    m = MODELS["tiny"].with_layers(8)
    ranks = _group(P, m, 2, [3, 4])
    R = ranks[0]
    with torch.cuda.stream(R.stream):
        R.ctx.step(R.toks, R.next, R.kv, batch=0, stream=R.stream)      # dummy step
    R.stream.synchronize()
    R.step(); R.finish_step()
    own = OS.owner_map(8, 2)
    log = R.ctx.fetch_log()
    ref = OS.slot_schedule(OS.plan_exec(own, 0), 2, 3)
    assert log == ref[:len(log)] and len(log) >= 2 * 4
    rep = _replicated(P, m, 3, 0)
    rep.step(); rep.finish_step()
    assert torch.equal(rep.history[0][1], R.history[0][1])
    for Rk in ranks + [rep]:
        Rk.ctx.destroy()
