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

from .helpers import OracleModel, cas_oracle_check, oracle_layer, rank_inputs, rel_err

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
    rep = _replicated(P, m, 5, 0, compute_sms=_budget(R))
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
    """Replicated (d = 1) run of the same rows; compute_sms = the WaS rank's compute-grid SM
    budget (the SM fetch holds the rest), so both run the same kernel configurations and the
    comparison can be bitwise."""
    kw = {k: v for k, v in kw.items() if k in ("pool", "compute_sms")}
    return Rank(P, m, B=B, b0=b0, **kw)


def _budget(R):
    return R.ctx.stats()["compute_sms"]


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
        rep = _replicated(P, m, B[r], sum(B[:r]), pool=pool, compute_sms=_budget(R))
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


_OM_CACHE = {}


def _oracle_model(m):
    """fp64 parameters of the 2-layer full-width models, kept for the next case of the same
    model only (a Llama-width layer is 6.8 GB in fp64)."""
    key = (m.name, m.num_layers)
    if key not in _OM_CACHE:
        _OM_CACHE.clear()
        _OM_CACHE[key] = OracleModel(m, SEED)
    return _OM_CACHE[key]


# (model, B, S_ctx, compute_sms): the M2 point in the d = 1 launch configuration (all SMs) and in
# the WaS one (132 SMs: 16 held by the SM fetch); the B_e-regime points the WaS emulation reports
# (Qwen3 B = 512-1536, Llama B = 1024 / 1536 at their max-KV contexts) in the
# WaS configuration; Qwen2.5-72B (QKV bias at h = 8192) at its M4 point
@pytest.mark.parametrize("name,B,ctx,sms", [
    ("qwen3-32b", 256, 1024, 0), ("qwen3-32b", 256, 1024, 124), ("qwen3-32b", 512, 768, 124),
    ("qwen3-32b", 1024, 384, 124), ("qwen3-32b", 1536, 256, 124),
    ("llama-3.1-70b", 64, 512, 0), ("llama-3.1-70b", 1024, 432, 124),
    ("llama-3.1-70b", 1536, 288, 124), ("qwen2.5-72b", 256, 1024, 124),
    # the CaS tail's shapes: split-KV attention in k pieces per pair (k = 128 / pairs)
    ("qwen3-32b", 16, 1024, 0), ("llama-3.1-70b", 4, 4096, 0), ("llama-3.1-70b", 1, 4096, 0)])
def test_big_shapes_sampled_rows(P, name, B, ctx, sms):
    """Full-size per-layer shapes in the launch configurations the bench times, on 2 layers;
    the oracle recomputes sampled rows of every layer (teacher-forced) and the new k/v entries."""
    m = MODELS[name].with_layers(2)
    max_ctx = ctx + 8
    R = Rank(P, m, B=B, ctx=ctx, span=0, max_ctx=max_ctx, compute_sms=sms)
    R.step(); R.finish_step()
    _, logits, dump = R.history[0]
    om = _oracle_model(m)
    rows = np.unique(np.clip([0, 1, B // 3, B // 2, B - 2, B - 1], 0, B - 1))
    pos = np.full(len(rows), ctx)
    xs = dump[:, rows].double().numpy()
    out = None
    for l in range(m.num_layers):
        K = gen.kv(SEED, gen.KCACHE, l, rows, range(max_ctx), m.n_kv_heads, m.head_dim)
        V = gen.kv(SEED, gen.VCACHE, l, rows, range(max_ctx), m.n_kv_heads, m.head_dim)
        out, kn, vn = oracle_layer(om, l, xs[l], pos, K, V)
        if l + 1 < m.num_layers:
            assert rel_err(xs[l + 1], out) <= TOL, (l, rel_err(xs[l + 1], out))
        kg = R.kv.k[l, torch.from_numpy(rows).cuda(), :, ctx].cpu().double().numpy()
        vg = R.kv.v[l, torch.from_numpy(rows).cuda(), :, ctx].cpu().double().numpy()
        assert rel_err(kg, kn) <= TOL and rel_err(vg, vn) <= TOL
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
    rep = Rank(P, m, B=B, ctx=ctx, span=0, max_ctx=ctx + 8, compute_sms=_budget(R))
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
    rep = _replicated(P, m, 3, 0, compute_sms=_budget(R))
    rep.step(); rep.finish_step()
    assert torch.equal(rep.history[0][1], R.history[0][1])
    for Rk in ranks + [rep]:
        Rk.ctx.destroy()


def _gpu_caches(R, B):
    """The rank's KV state in the oracle's layout: (K, V) [L, B, T, n_kv, hd] float64."""
    K = R.kv.k[:, :B].permute(0, 1, 3, 2, 4).double().cpu().numpy()
    V = R.kv.v[:, :B].permute(0, 1, 3, 2, 4).double().cpu().numpy()
    return K, V


@pytest.mark.parametrize("pool", ["layer", "ffn"])
@pytest.mark.parametrize("B", [[3, 5], [4, 0, 2, 0], [0, 0, 0, 6], [2, 2, 2, 2]])
def test_cas_vs_oracle(P, pool, B):
    """CaS on virtual ranks against the ORACLE's CaS (oracle/sidp.py cas_layer / run_cas), not
    against another GPU run: teacher-forced per layer and, untethered, the
    oracle's whole CaS step from the same tokens (run_cas) — logits within the north_star
    tolerance, tokens where the oracle's top-2 margin is clear.  Dummy ranks (B = 0) move
    nothing and the owner serves even when it is dummy itself."""
    from oracle import sidp as OSD
    m = MODELS["tiny"].with_layers(4)
    d = len(B)
    ranks = _group(P, m, d, B, pool=pool)
    for R in ranks:
        R.ctx.set_batches(B)
        R.ctx.set_mode(1, 0)
    for R in ranks:
        R.step()
    for R in ranks:
        R.finish_step()
    for R in ranks:
        assert R.ctx.stats()["timeouts"] == 0
    hist = {r: R.history[0] for r, R in enumerate(ranks)}
    live = [r for r in range(d) if B[r]]
    om = OracleModel(m, SEED)
    owner = OS.owner_map(m.num_layers, d)
    cas_oracle_check(m, om, d, pool, {r: hist[r][2].double().numpy() for r in live},
                     {r: hist[r][1].double().numpy() for r in live},
                     {r: _gpu_caches(ranks[r], B[r]) for r in live},
                     {r: gen.positions(SEED, np.arange(sum(B[:r]), sum(B[:r]) + B[r]), 0, 63)
                      for r in live}, TOL)
    # untethered: the oracle's CaS step from the same tokens and caches
    states = []
    for r in range(d):
        _, toks, pos, caches = rank_inputs(m, SEED, sum(B[:r]), B[r], 0, 63, 80)
        states.append(OSD.RankState(r, toks, pos, caches))
    OSD.run_cas(m, [om.layer(l) for l in range(m.num_layers)], om.head, om.embed, states, 1, d,
                owner, pool)
    for r, st in enumerate(states):
        if B[r] == 0:
            assert st.history[0] is None
            continue
        ref = st.history[0]["logits"]
        got = hist[r][1].double().numpy()
        err = rel_err(got, ref)
        assert err <= TOL, (r, err)
        top2 = np.sort(ref, axis=1)[:, -2:]
        sure = (top2[:, 1] - top2[:, 0]) > 2 * err * np.abs(ref).max()
        assert (hist[r][0].numpy()[sure] == st.history[0]["next"][sure]).all()
    for R in ranks:
        R.ctx.destroy()


@pytest.mark.parametrize("case", ["tiny-qwen3-160-20-40", "tiny-200-0-60", "tiny-300-0-400"])
def test_attention_range_walk_mode(P, case):
    """The one-wave range-walking attention partition (many short pairs split into contiguous
    chunk ranges, pieces merged by the last arriver) is only reached when the warp-per-pair
    kernel is disabled (SIDP_ATTN_WARP_CH=1, read once per process): re-run the ragged short-pair
    parity cases in a subprocess with it off, against the oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SIDP_ATTN_WARP_CH="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        f"tests/test_gpu_parity.py::test_long_context_split_kv[{case}]"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "1 passed" in r.stdout


@pytest.mark.parametrize("d,slots", [(4, 2), (8, 1)])
def test_was_cuda_graph_replay(P, d, slots):
    """WaS steps replay as a CUDA graph (device epoch flags: the ready waits and releases name
    only the slot; the fetch stream is enqueued by the host around each replay): decoded tokens
    of 5 replayed steps equal an eager WaS run's bit for bit, the device fetch log equals the
    oracle's FIFO schedule, and every consumption found the layer it expected in its slot."""
    m = MODELS["tiny"].with_layers(8)
    B = 5

    def group():
        R = Rank(P, m, rank=0, world=d, B=B, slots=slots)
        peers = []
        for r in range(1, d):
            c = P.Context(m, rank=r, world=d, max_batch=B, max_ctx=80, seed=SEED, alloc=False)
            c.alloc_serve_only()
            c.init_weights_synthetic()
            peers.append(c)
        torch.cuda.synchronize()
        R.ctx.import_handles([R.ctx.export_handles()] + [c.export_handles() for c in peers])
        return R, peers

    G, gp = group()     # graph path: no logits / dumps requested
    E, ep = group()     # eager path (logits requested)
    steps = 5
    for s in range(steps):
        with torch.cuda.stream(G.stream):
            G.ctx.step(G.toks, G.toks, G.kv, batch=B, stream=G.stream, advance_pos=True)
        G.stream.synchronize()
        G.history.append(G.toks.clone().cpu())
        E.step(); E.finish_step()
        assert torch.equal(G.history[-1], E.history[-1][0]), s
    st = G.ctx.stats()
    assert st["timeouts"] == 0 and st["fetch_sms_held"] > 0
    pl = OS.plan(OS.owner_map(m.num_layers, d), d, 0, "exec")
    log = G.ctx.fetch_log()
    assert len(log) >= steps * len(pl)
    assert log == OS.slot_schedule(pl, slots, steps + 2)[:len(log)]
    cons = G.ctx.consume_log()
    assert len(cons) == steps * len(pl)
    assert all(c[0] == c[2] for c in cons)                  # slot held the expected layer
    sched = OS.slot_schedule(pl, slots, steps)
    assert [(c[0], c[1]) for c in cons] == [(l, s) for (_, l, s) in sorted(sched, key=lambda e: (e[0], e[1]))]
    for c in gp + ep:
        c.destroy()
    G.ctx.destroy()
    E.ctx.destroy()


def test_was_windowed_graph_with_timing(P, monkeypatch):
    """The bench's WaS emulation path: ONE computing context (so the fetch of a whole step is one
    windowed launch gated on device release flags) replaying CUDA graphs while per-class kernel
    timing is on.  Regression: a blocking harvest of the fetch stream's timing events before a
    capture waited on a window whose gates need compute not yet enqueued (deadlock until the
    flag-wait timeout).  Tokens equal a replicated run's bit for bit; no timeouts."""
    monkeypatch.setenv("SIDP_CAS_TIMEOUT_MS", "4000")
    m = MODELS["tiny"].with_layers(8)
    B, d = 5, 4
    G = Rank(P, m, rank=0, world=d, B=B, slots=2)
    peers = []
    for r in range(1, d):
        c = P.Context(m, rank=r, world=d, max_batch=B, max_ctx=80, seed=SEED, alloc=False)
        c.alloc_serve_only()
        c.init_weights_synthetic()
        peers.append(c)
    torch.cuda.synchronize()
    G.ctx.import_handles([G.ctx.export_handles()] + [c.export_handles() for c in peers])
    toks = []
    for s in range(6):
        if s == 2:
            G.ctx.set_timing(sum(1 << c for c in range(1, 8)))   # every class, as the bench
        if s == 4:
            G.ctx.set_timing(1 << 3)                             # the fetch class only
        with torch.cuda.stream(G.stream):
            G.ctx.step(G.toks, G.toks, G.kv, batch=B, stream=G.stream, advance_pos=True)
        if s % 2:
            G.stream.synchronize()
            toks.append(G.toks.clone().cpu())
    G.stream.synchronize()
    st = G.ctx.stats()
    assert st["timeouts"] == 0 and st["fetch_sms_held"] > 0
    assert st["timed_launches"][3] > 0 and st["timed_ms"][3] > 0
    budget = st["compute_sms"]
    for c in peers:
        c.destroy()
    G.ctx.destroy()
    rep = Rank(P, m, B=B, compute_sms=budget)
    for s in range(6):
        with torch.cuda.stream(rep.stream):
            rep.ctx.step(rep.toks, rep.toks, rep.kv, batch=B, stream=rep.stream, advance_pos=True)
        if s % 2:
            rep.stream.synchronize()
            assert torch.equal(rep.toks.cpu(), toks[s // 2]), s
    rep.ctx.destroy()


@pytest.mark.parametrize("env,case", [
    ({"SIDP_CAS_PROLOGUE_WAIT": "1"}, "B0-layer"), ({"SIDP_CAS_PROLOGUE_WAIT": "1"}, "B1-ffn"),
    ({"SIDP_CAS_PROLOGUE_WAIT": "1"}, "B2-layer"),
    ({"SIDP_CAS_FUSED": "1"}, "B1-layer"), ({"SIDP_CAS_FUSED": "0"}, "B0-ffn")])
def test_cas_variants_vs_oracle(P, env, case):
    """The CaS ladder rungs and the flag waits folded into the consumer kernels' prologues (the
    multi-GPU default; on one shared GPU the library gates consumers with standalone wait kernels
    instead) re-run the oracle CaS test in a subprocess (the switches are read once per
    process): V3 with prologue waits forced on, V2 (fused transfer launches), V1."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        f"tests/test_gpu_parity.py::test_cas_vs_oracle[{case}]"],
                       cwd=root, env=dict(os.environ, SIDP_CAS_TIMEOUT_MS="20000", **env),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "1 passed" in r.stdout


@pytest.mark.parametrize("name,d,slots,pool", [("tiny", 4, 1, "layer"), ("tiny", 4, 2, "layer"),
                                               ("tiny-qwen3", 2, 1, "ffn"), ("tiny-qwen25", 8, 1, "layer")])
def test_was_tile_slots(P, name, d, slots, pool):
    """Tile-granular slots (sidp_config.slot_parts = 2): every pooled component
    of a slot is filled, made ready and released on its own flags, so one slot pipelines.  One
    computing rank beside d-1 serve-only owners; CUDA-graph steps and an eager step with logits
    are BITWISE equal to the replicated run; the device fetch log (one entry per layer, when its
    last part landed) equals the oracle FIFO schedule; every consumption is per part and found
    the layer it expected in that part."""
    m = MODELS[name].with_layers(8)
    B = 5
    G = Rank(P, m, rank=0, world=d, B=B, slots=slots, pool=pool, slot_parts=2)
    peers = []
    for r in range(1, d):
        c = P.Context(m, rank=r, world=d, max_batch=B, max_ctx=80, seed=SEED, alloc=False, pool=pool)
        c.alloc_serve_only()
        c.init_weights_synthetic()
        peers.append(c)
    torch.cuda.synchronize()
    G.ctx.import_handles([G.ctx.export_handles()] + [c.export_handles() for c in peers])
    steps = 4
    toks = []
    for s in range(steps):       # graph replays (no logits requested)
        with torch.cuda.stream(G.stream):
            G.ctx.step(G.toks, G.toks, G.kv, batch=B, stream=G.stream, advance_pos=True)
        G.stream.synchronize()
        toks.append(G.toks.clone().cpu())
    G.step(); G.finish_step()    # eager, logits
    st = G.ctx.stats()
    assert st["timeouts"] == 0
    pl = OS.plan(OS.owner_map(m.num_layers, d), d, 0, "exec")
    log = G.ctx.fetch_log()
    assert len(log) >= (steps + 1) * len(pl)
    assert log == OS.slot_schedule(pl, slots, steps + 3)[:len(log)]
    parts = 4 if pool == "layer" else 2
    cons = G.ctx.consume_log()
    assert len(cons) == (steps + 1) * len(pl) * parts
    assert all(c[0] == c[2] for c in cons)
    budget = st["compute_sms"]
    for c in peers:
        c.destroy()
    G.ctx.destroy()
    rep = Rank(P, m, B=B, pool=pool, compute_sms=budget)
    for s in range(steps):
        with torch.cuda.stream(rep.stream):
            rep.ctx.step(rep.toks, rep.toks, rep.kv, batch=B, stream=rep.stream, advance_pos=True)
        rep.stream.synchronize()
        assert torch.equal(rep.toks.cpu(), toks[s]), s
    rep.step(); rep.finish_step()
    assert torch.equal(rep.history[0][1], G.history[0][1])
    rep.ctx.destroy()


def test_was_tile_slots_full_width_one_slot(P):
    """One tile-granular slot at the bench's full Qwen3-32B width (B = 256, S_ctx = 1024, 12
    layers; d = 8 with serve-only owners): about one layer of cache memory, logits bitwise equal
    to the replicated run, fetch log == oracle schedule."""
    m = MODELS["qwen3-32b"].with_layers(12)
    B, ctx, d, steps = 256, 1024, 8, 2
    R = Rank(P, m, rank=0, world=d, B=B, ctx=ctx, span=0, max_ctx=ctx + 8, slots=1, slot_parts=2)
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
    st = R.ctx.stats()
    assert st["timeouts"] == 0 and st["slot_bytes"] == st["layer_bytes"]
    pl = OS.plan(OS.owner_map(m.num_layers, d), d, 0, "exec")
    log = R.ctx.fetch_log()
    assert log == OS.slot_schedule(pl, 1, steps + 1)[:len(log)] and len(log) >= steps * len(pl)
    for c in peers:
        c.destroy()
    rep = Rank(P, m, B=B, ctx=ctx, span=0, max_ctx=ctx + 8, compute_sms=st["compute_sms"])
    for s in range(steps):
        rep.step(); rep.finish_step()
        assert torch.equal(rep.history[s][1], R.history[s][1]), s
    rep.ctx.destroy()
    R.ctx.destroy()


@pytest.mark.parametrize("d,slots,share", [(4, 2, 0.5), (8, 1, 0.25), (2, 2, 0.9)])
def test_was_hybrid_fetch(P, d, slots, share):
    """Hybrid fetch (sidp_config.fetch_ce_share): the copy engine writes a prefix of every layer,
    the SM kernel the rest, both counted into the same fill epoch.  One computing rank beside
    serve-only owners, CUDA-graph steps and an eager step with logits: BITWISE equal to the
    replicated run; the device fetch log equals the oracle FIFO schedule."""
    m = MODELS["tiny"].with_layers(8)
    B = 5
    G = Rank(P, m, rank=0, world=d, B=B, slots=slots, fetch_ce_share=share)
    peers = []
    for r in range(1, d):
        c = P.Context(m, rank=r, world=d, max_batch=B, max_ctx=80, seed=SEED, alloc=False)
        c.alloc_serve_only()
        c.init_weights_synthetic()
        peers.append(c)
    torch.cuda.synchronize()
    G.ctx.import_handles([G.ctx.export_handles()] + [c.export_handles() for c in peers])
    toks = []
    for s in range(4):
        with torch.cuda.stream(G.stream):
            G.ctx.step(G.toks, G.toks, G.kv, batch=B, stream=G.stream, advance_pos=True)
        G.stream.synchronize()
        toks.append(G.toks.clone().cpu())
    G.step(); G.finish_step()
    st = G.ctx.stats()
    assert st["timeouts"] == 0
    pl = OS.plan(OS.owner_map(m.num_layers, d), d, 0, "exec")
    log = G.ctx.fetch_log()
    assert len(log) >= 5 * len(pl)
    assert log == OS.slot_schedule(pl, slots, 8)[:len(log)]
    budget = st["compute_sms"]
    for c in peers:
        c.destroy()
    G.ctx.destroy()
    rep = Rank(P, m, B=B, compute_sms=budget)
    for s in range(4):
        with torch.cuda.stream(rep.stream):
            rep.ctx.step(rep.toks, rep.toks, rep.kv, batch=B, stream=rep.stream, advance_pos=True)
        rep.stream.synchronize()
        assert torch.equal(rep.toks.cpu(), toks[s]), s
    rep.step(); rep.finish_step()
    assert torch.equal(rep.history[0][1], G.history[0][1])
    rep.ctx.destroy()


@pytest.mark.parametrize("pool,B", [("layer", [3, 5]), ("layer", [4, 0, 2, 0]), ("ffn", [2, 2, 2, 2])])
def test_cas_graph_replay(P, pool, B):
    """CaS steps replay as CUDA graphs (flag values relative to a device round-trip counter that
    each step's first kernel advances): the tokens of 5 graph-replayed CaS steps on virtual ranks
    equal an eager CaS run's bit for bit (eager = logits requested, so never captured), and the
    live ranks replayed graphs."""
    m = MODELS["tiny"].with_layers(4)
    d = len(B)
    steps = 5

    def group():
        ranks = _group(P, m, d, B, pool=pool)
        for R in ranks:
            R.ctx.set_batches(B)
            R.ctx.set_mode(1, 0)
        return ranks

    G = group()
    E = group()
    for s in range(steps):
        for R in G:
            with torch.cuda.stream(R.stream):
                R.ctx.step(R.toks, R.toks, R.kv, batch=R.B, stream=R.stream, advance_pos=R.B > 0)
        for R in E:
            R.step()
        for R in G:
            R.stream.synchronize()
        for R in E:
            R.finish_step()
        for r in range(d):
            if B[r]:
                assert torch.equal(G[r].toks[:B[r]].cpu(), E[r].history[-1][0]), (s, r)
    for r, R in enumerate(G):
        st = R.ctx.stats()
        assert st["timeouts"] == 0
        if B[r]:
            assert st["graph_replays"] >= steps - 1, st["graph_replays"]
    for R in G + E:
        R.ctx.destroy()


def test_alloc_owned_torch_arena(P):
    """sidp_alloc_owned: the owned layers in a caller-owned torch buffer give
    bit-identical WaS results to the library-allocated arena (virtual ranks, d = 2), and bad
    arenas are rejected with SIDP_EINVAL before anything is allocated."""
    m = MODELS["tiny"].with_layers(4)
    B = [3, 5]

    outs = []
    for torch_arena in (False, True):
        ranks = []
        for r in range(2):
            ctx = P.Context(m, rank=r, world=2, max_batch=max(B), max_ctx=80, seed=SEED, alloc=False)
            nb = ctx.owned_bytes()
            assert nb > 0
            if torch_arena:
                seg = torch.empty(nb + 8192, dtype=torch.uint8, device="cuda")
                with pytest.raises(P.SidpError):            # too small
                    ctx.alloc(seg[:nb - 256])
                with pytest.raises(P.SidpError):            # misaligned
                    ctx.alloc(seg[8:8 + nb])
                ctx.alloc(seg[2048:2048 + nb])
            else:
                ctx.alloc()
            ranks.append(ctx)
        for ctx in ranks:
            ctx.init_weights_synthetic()
        blobs = [c.export_handles() for c in ranks]
        for c in ranks:
            c.import_handles(blobs)
        res = []
        for r, ctx in enumerate(ranks):
            mb = max(B)
            kv = P.KVCache(m, mb, 80)
            kv.fill_synthetic(SEED, sum(B[:r]), mb, 80)
            bg = np.arange(sum(B[:r]), sum(B[:r]) + B[r])
            kv.set_pos(gen.positions(SEED, bg, 0, 63))
            toks = torch.from_numpy(gen.tokens(SEED, bg, m.vocab)).to(torch.int32).cuda()
            nxt = torch.zeros(mb, dtype=torch.int32, device="cuda")
            logits = torch.zeros(mb, m.vocab, dtype=torch.float32, device="cuda")
            ctx.step(toks, nxt, kv, batch=B[r], logits=logits)
            torch.cuda.synchronize()
            res.append(logits[:B[r]].cpu().clone())
        outs.append(res)
        for c in ranks:
            c.destroy()
    for r in range(2):
        assert torch.equal(outs[0][r], outs[1][r]), r


@pytest.mark.parametrize("parts,fetch", [(1, "sm"), (2, "sm"), (1, "ce")])
def test_was_slot_verify(P, monkeypatch, parts, fetch):
    """Debug slot check (SIDP_SLOT_VERIFY=1, SURVEY.md §5 slot-checksum mode): every landed slot
    (whole, or each tile part) is compared word for word with the owner's blob right after its
    ready wait, before the layer's first reader; over graph-replayed and eager WaS steps every
    consumption is checked and no word differs (the fetch is verbatim), and the
    check itself leaves the logits bit-identical."""
    monkeypatch.setenv("SIDP_SLOT_VERIFY", "1")
    m = MODELS["tiny"].with_layers(8)
    d, B, pool = 4, 5, "layer"
    G = Rank(P, m, rank=0, world=d, B=B, slots=2, pool=pool, slot_parts=parts, fetch_engine=fetch)
    peers = []
    for r in range(1, d):
        c = P.Context(m, rank=r, world=d, max_batch=B, max_ctx=80, seed=SEED, alloc=False, pool=pool)
        c.alloc_serve_only()
        c.init_weights_synthetic()
        peers.append(c)
    torch.cuda.synchronize()
    G.ctx.import_handles([G.ctx.export_handles()] + [c.export_handles() for c in peers])
    steps = 3
    for s in range(steps):
        with torch.cuda.stream(G.stream):
            G.ctx.step(G.toks, G.toks, G.kv, batch=B, stream=G.stream, advance_pos=True)
        G.stream.synchronize()
    G.step(); G.finish_step()
    st = G.ctx.stats()
    remote = sum(1 for l in range(m.num_layers) if OS.owner_map(m.num_layers, d)[l] != 0)
    assert st["timeouts"] == 0
    assert st["slot_checks"] == (steps + 1) * remote * (4 if parts > 1 else 1), st["slot_checks"]
    assert st["slot_mismatches"] == 0
    for c in peers:
        c.destroy()
    G.ctx.destroy()
    monkeypatch.delenv("SIDP_SLOT_VERIFY")
    rep = Rank(P, m, B=B, pool=pool, compute_sms=st["compute_sms"])
    for s in range(steps):
        with torch.cuda.stream(rep.stream):
            rep.ctx.step(rep.toks, rep.toks, rep.kv, batch=B, stream=rep.stream, advance_pos=True)
        rep.stream.synchronize()
    rep.step(); rep.finish_step()
    assert torch.equal(rep.history[0][1], G.history[0][1])
    rep.ctx.destroy()


@pytest.mark.parametrize("name,B,ctx,span,layers", [
    ("tiny", 8, 0, 63, 4), ("tiny-qwen3", 6, 20, 40, 4),
    ("qwen3-32b", 256, 1000, 24, 2),          # pair-mode / warp-per-pair attention
    ("llama-3.1-70b", 4, 4000, 90, 2),        # few pairs: split-KV pieces
    ("qwen3-32b", 1024, 200, 56, 2)])         # many short pairs
def test_paged_kv_bitwise(P, name, B, ctx, span, layers):
    """Paged KV (sidp_kv.block_table, 16-token blocks): the same cache contents
    scattered over a shuffled block pool give BIT-IDENTICAL logits to the contiguous layout over
    several decode steps (CUDA-graph replays and eager steps; appends crossing block boundaries),
    and every appended k/v lands in the right block."""
    m = MODELS[name].with_layers(layers)
    max_ctx = ctx + span + 8
    ctxt = P.Context(m, max_batch=B, max_ctx=max_ctx, seed=SEED)
    ctxt.init_weights_synthetic()
    kv = P.KVCache(m, B, max_ctx)
    kv.fill_synthetic(SEED, 0, B, max_ctx)
    bg = np.arange(B)
    kv.set_pos(gen.positions(SEED, bg, ctx, span))
    torch.cuda.synchronize()
    pk = P.PagedKVCache.from_contiguous(kv, m, seed=7, spare=5)
    toks = torch.from_numpy(gen.tokens(SEED, bg, m.vocab)).to(torch.int32).cuda()
    outs = []
    for cache in (kv, pk):
        t = toks.clone()
        nxt = torch.zeros(B, dtype=torch.int32, device="cuda")
        logits = torch.zeros(B, m.vocab, dtype=torch.float32, device="cuda")
        res = []
        for s in range(4):
            if s < 2:      # graph-replayed steps (no logits), tokens fed back
                ctxt.step(t, t, cache, batch=B, advance_pos=True)
                torch.cuda.synchronize()
                res.append(t.cpu().clone())
            else:
                ctxt.step(t, nxt, cache, batch=B, logits=logits, advance_pos=True)
                torch.cuda.synchronize()
                res.append(logits.cpu().clone())
                t = nxt.clone()
        outs.append(res)
    for s in range(4):
        assert torch.equal(outs[0][s], outs[1][s]), s
    # the appended entries of every layer, gathered back through the block table
    p0 = torch.from_numpy(gen.positions(SEED, bg, ctx, span)).long()
    ar = torch.arange(B)
    for l in range(layers):
        for which, ref in (("k", kv.k[l]), ("v", kv.v[l])):
            got = pk.to_contiguous(l, which)
            for s in range(4):
                assert torch.equal(got[ar, :, p0 + s].cpu(), ref[ar, :, p0 + s].cpu()), (l, which, s)
    ctxt.destroy()


def test_paged_kv_fused_qkv_epilogue():
    """The paged KV append also from the fused token-major QKV epilogue (SIDP_FUSED_QKV=1, read
    once per process): the paged tests re-run in a subprocess with it on."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, SIDP_FUSED_QKV="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        __file__, "-k", "paged_kv_bitwise"], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("name,layers", [("tiny", 4), ("tiny-qwen3", 4), ("tiny-qwen25", 4),
                                         ("qwen3-32b", 2)])   # 8-head groups: transposed attention
def test_prefill_vs_oracle(P, name, layers):
    """Prefill as one ragged step over a paged cache: prompts of 5, 17 and 33
    tokens (crossing 16-token blocks) appended to three sequences with existing contexts.  Per
    layer, teacher-forced (C-N8): every prompt row's layer output and new k/v against the fp64
    oracle from the GPU's layer input and the sequence's KV state (the oracle attends over the
    row's causal prefix, the earlier prompt rows' entries included), and the logits."""
    m = MODELS[name].with_layers(layers)
    S, lens, pos0 = 3, [5, 17, 33], [10, 0, 20]
    rows, max_ctx = sum(lens), 80
    ctxt = P.Context(m, max_batch=rows, max_ctx=max_ctx, seed=SEED)
    ctxt.init_weights_synthetic()
    pk = P.PagedKVCache(m, S, max_ctx, S * (max_ctx // 16) + 3)
    pk.fill_synthetic(SEED, 0, S, max_ctx, perm_seed=3)
    pk.set_pos(pos0)
    g = np.random.default_rng(5)
    prompts = [g.integers(0, m.vocab, n) for n in lens]
    logits = torch.zeros(rows, m.vocab, dtype=torch.float32, device="cuda")
    dump = torch.zeros(m.num_layers, rows, m.hidden, dtype=torch.bfloat16, device="cuda")
    nxt, last = P.prefill(ctxt, pk, prompts, logits=logits, layer_inputs=dump)
    torch.cuda.synchronize()
    assert pk.pos[:S].cpu().tolist() == [p + n for p, n in zip(pos0, lens)]
    om = OracleModel(m, SEED)
    seq = np.concatenate([np.full(n, b) for b, n in enumerate(lens)])
    pos = np.concatenate([pos0[b] + np.arange(n) for b, n in enumerate(lens)])
    xs = dump.double().cpu().numpy()
    lg = logits.double().cpu().numpy()
    for l in range(m.num_layers):
        K = pk.to_contiguous(l, "k").permute(0, 2, 1, 3).double().cpu().numpy()[seq]   # [rows][T][nkv][hd]
        V = pk.to_contiguous(l, "v").permute(0, 2, 1, 3).double().cpu().numpy()[seq]
        out, kn, vn = oracle_layer(om, l, xs[l], pos, K, V)
        b = np.arange(rows)
        errs = [rel_err(K[b, pos], kn), rel_err(V[b, pos], vn)]
        if l + 1 < m.num_layers:
            errs.append(rel_err(xs[l + 1], out))
        elif m.vocab <= 10000:   # full-width heads (6 GB in fp64) are checked by the step tests
            errs.append(rel_err(lg, OM.lm_head(m, om.head, out)))
        assert max(errs) <= TOL, (l, errs)
    assert (nxt.cpu().numpy() == np.argmax(lg[last], axis=1)).all()
    ctxt.destroy()


def test_paged_kv_cas_bitwise(P):
    """Paged KV under CaS (the requester's qkv_post appends and attention reads through the block
    table while the owners compute the linears): bit-identical to the contiguous layout."""
    m = MODELS["tiny"].with_layers(4)
    B = [3, 5]
    outs = []
    for paged in (False, True):
        ranks = _group(P, m, 2, B)
        for r, R in enumerate(ranks):
            if paged:
                R.kv = P.PagedKVCache.from_contiguous(R.kv, m, seed=11 + r, spare=2)
            R.ctx.set_batches(B)
            R.ctx.set_mode(1, 0)
        for s in range(2):
            for R in ranks:
                R.step()
            for R in ranks:
                R.finish_step()
        outs.append([[h[1] for h in R.history] for R in ranks])
        for R in ranks:
            assert R.ctx.stats()["timeouts"] == 0
            R.ctx.destroy()
    assert all(torch.equal(a, b) for ra, rb in zip(outs[0], outs[1]) for a, b in zip(ra, rb))


def test_paged_kv_rejects_bad_geometry(P):
    """sidp_kv validation (sidp.h): a block size other than 16 or a table shorter than max_ctx
    is SIDP_EINVAL before anything is enqueued."""
    m = MODELS["tiny"].with_layers(2)
    ctxt = P.Context(m, max_batch=2, max_ctx=64, seed=SEED)
    ctxt.init_weights_synthetic()
    pk = P.PagedKVCache(m, 2, 64, 8)
    pk.set_pos([3, 5])
    toks = torch.zeros(2, dtype=torch.int32, device="cuda")
    import paper_2605_28095_b200._abi as A

    class Bad:
        def __init__(self, **over):
            self.pos, self.max_pos, self.over = pk.pos, pk.max_pos, over

        def c(self):
            f = dict(block_tokens=16, max_blocks=pk.max_blocks, num_blocks=pk.num_blocks)
            f.update(self.over)
            return A.KV(pk.k.data_ptr(), pk.v.data_ptr(), pk.pos.data_ptr(), pk.max_pos,
                        pk.table.data_ptr(), f["block_tokens"], f["max_blocks"], f["num_blocks"])

    for over in (dict(block_tokens=32), dict(max_blocks=2), dict(num_blocks=0)):
        with pytest.raises(P.SidpError) as e:
            ctxt.step(toks, toks, Bad(**over), batch=2)
        assert e.value.status == -1, over
    ctxt.step(toks, toks, pk, batch=2)     # the valid geometry runs
    torch.cuda.synchronize()
    ctxt.destroy()
