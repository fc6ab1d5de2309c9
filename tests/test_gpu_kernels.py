"""Single-kernel parity on the GPU (through the C-ABI test hooks, same kernels as the hot path).

* K12 generator: bit-exact vs sidp_inputs.gen (the shared seeded generator).
* tcgen05 GEMM: vs the fp64 product of the same bf16 operands, over tile-spanning shapes with
  ragged tails, forced split-K counts and every fused epilogue.
"""
import numpy as np
import pytest
import torch

from sidp_inputs import gen

pytestmark = pytest.mark.gpu
SEED = 20261017


@pytest.fixture(scope="module")
def P():
    from paper_2605_28095_b200 import build as B
    B.build()
    import paper_2605_28095_b200 as P
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return P


def _lvl(shape, gen_, scale=1.0):
    return (torch.randint(-128, 128, shape, generator=gen_).to(torch.float32) / 128 * scale).to(torch.bfloat16)


# ------------------------------------------------------------------ K12
def test_gen_weights_bit_exact(P):
    dst = torch.empty(96, 5120, dtype=torch.bfloat16, device="cuda")
    P.test_gen(dst, SEED, gen.WQ, 3, 0, scale_k=5120, row0=40)
    ref = gen.weight(SEED, gen.WQ, 3, 136, 5120)[40:]
    assert torch.equal(dst.cpu().double(), torch.from_numpy(ref))


def test_gen_gate_up_interleave_bit_exact(P):
    I, K = 192, 256
    dst = torch.empty(2 * I, K, dtype=torch.bfloat16, device="cuda")
    P.test_gen(dst, SEED, gen.WGATE, 1, 0, scale_k=K, row_map=1)
    g = gen.weight(SEED, gen.WGATE, 1, I, K)
    u = gen.weight(SEED, gen.WUP, 1, I, K)
    ref = np.concatenate([np.concatenate([g[8 * t:8 * t + 8], u[8 * t:8 * t + 8]])
                          for t in range(I // 8)])
    assert torch.equal(dst.cpu().double(), torch.from_numpy(ref))


def test_gen_gain_bias_unit_kv_bit_exact(P):
    for kind, tid, fn in ((1, gen.G_ATTN, lambda: gen.gain(SEED, gen.G_ATTN, 2, 512)),
                          (2, gen.BQ, lambda: gen.bias(SEED, gen.BQ, 2, 512))):
        dst = torch.empty(1, 512, dtype=torch.bfloat16, device="cuda")
        P.test_gen(dst, SEED, tid, 2, kind)
        assert torch.equal(dst.cpu().double()[0], torch.from_numpy(fn()))
    E = torch.empty(64, 256, dtype=torch.bfloat16, device="cuda")
    P.test_gen(E, SEED, gen.EMBED, 0, 3)
    assert torch.equal(E.cpu().double(), torch.from_numpy(gen.embed_rows(SEED, np.arange(64), 256)))
    import ctypes
    B, nkv, smax, hd, T = 3, 2, 40, 64, 33
    cache = torch.zeros(B, nkv, smax, hd, dtype=torch.bfloat16, device="cuda")
    P._abi.check(P._abi.lib().sidp_test_gen_kv(ctypes.c_void_p(cache.data_ptr()), B, nkv, smax, hd, T,
                                               5, SEED, gen.KCACHE, 1,
                                               ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)), "kv")
    ref = gen.kv(SEED, gen.KCACHE, 1, np.arange(5, 5 + B), range(T), nkv, hd)     # [B, T, g, d]
    got = cache.cpu().double().permute(0, 2, 1, 3)[:, :T]
    assert torch.equal(got, torch.from_numpy(ref))


# ------------------------------------------------------------------ tcgen05 GEMM
SHAPES = [(1, 128, 64), (8, 256, 256), (16, 384, 512), (37, 1000, 320), (100, 640, 1024),
          (256, 512, 5120), (300, 256, 512), (513, 128, 128), (64, 10240, 5120),
          (256, 10240, 5120), (200, 3440, 512)]   # token-major feature tiles of 144 / odd 16s


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("splits", [1, 3, 0, -1])
def test_gemm_f32(P, M, N, K, splits):
    g = torch.Generator().manual_seed(M * 7 + N + K)
    x = _lvl((M, K), g).cuda()
    w = _lvl((N, K), g, 2.0 ** -5).cuda()
    out = torch.full((M, N), float("nan"), dtype=torch.float32, device="cuda")
    P.test_gemm(x, w, out, M, N, K, 0, k_splits=splits)
    torch.cuda.synchronize()
    ref = x.cpu().double() @ w.cpu().double().T
    err = (out.cpu().double() - ref).abs().max().item()
    assert err <= 1e-5 * ref.abs().max().item() + 1e-6, err


@pytest.mark.parametrize("M,N,K", [(8, 256, 256), (37, 1000, 320), (256, 512, 2048)])
@pytest.mark.parametrize("orient", [0, -1])
def test_gemm_bf16_bias_and_residual(P, M, N, K, orient):
    g = torch.Generator().manual_seed(1)
    x = _lvl((M, K), g).cuda()
    w = _lvl((N, K), g, 2.0 ** -5).cuda()
    bias = _lvl((N,), g, 0.125).cuda()
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    P.test_gemm(x, w, out, M, N, K, 1, bias=bias, k_splits=2 if orient == 0 else -1)
    ref = x.cpu().double() @ w.cpu().double().T + bias.cpu().double()
    torch.cuda.synchronize()
    d = (out.cpu().double() - ref).abs()
    assert (d <= ref.abs() * 2.0 ** -8 + 1e-6 * ref.abs().max()).all()
    # residual, in place (out aliases resid)
    r = _lvl((M, N), g).cuda()
    ref2 = x.cpu().double() @ w.cpu().double().T + r.cpu().double()
    P.test_gemm(x, w, r, M, N, K, 2, resid=r, k_splits=orient)
    torch.cuda.synchronize()
    d2 = (r.cpu().double() - ref2).abs()
    assert (d2 <= ref2.abs() * 2.0 ** -8 + 1e-6 * ref2.abs().max()).all()


@pytest.mark.parametrize("M,N,K", [(8, 256, 256), (100, 640, 1024), (256, 5120, 8192),
                                   (200, 1000, 2048), (300, 512, 512), (128, 2048, 25600)])
def test_gemm_deferred_fixup_resid_norm(P, M, N, K):
    """EPI_PARTIAL stream-K slices summed by resid_norm: x2 = x W^T + resid, u = RMSNorm(x2) g
    (SURVEY.md a8+a9 / a11+a5), vs the fp64 product of the same bf16 operands."""
    g = torch.Generator().manual_seed(M + N + K)
    x = _lvl((M, K), g).cuda()
    w = _lvl((N, K), g, 2.0 ** -6).cuda()
    r = _lvl((M, N), g).cuda()
    gain = (1 + _lvl((N,), g, 2.0 ** -3).float()).to(torch.bfloat16).cuda()
    xout = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device="cuda")
    u = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device="cuda")
    eps = 1e-6
    P.test_gemm_resid_norm(x, w, r, gain, eps, xout, u)
    torch.cuda.synchronize()
    ref = x.cpu().double() @ w.cpu().double().T + r.cpu().double()
    got = xout.cpu().double()
    assert ((got - ref).abs() <= ref.abs() * 2.0 ** -8 + 1e-6 * ref.abs().max()).all()
    ur = got * torch.rsqrt((got * got).mean(-1, keepdim=True) + eps) * gain.cpu().double()
    assert ((u.cpu().double() - ur).abs() <= ur.abs() * 2.0 ** -7 + 1e-6 * ur.abs().max()).all()
    # in place (resid aliases xout), as the hot path runs it
    r2 = r.clone()
    P.test_gemm_resid_norm(x, w, r2, gain, eps, r2, u)
    torch.cuda.synchronize()
    assert torch.equal(r2, xout)


@pytest.mark.parametrize("M,N,K", [(1024, 5120, 2048), (600, 9728, 4096), (1024, 5120, 8192)])
def test_gemm_hybrid_streamk_tail(P, M, N, K):
    """Tile counts just over one wave of the 74 CTA pairs (80, 76 tiles): a whole-tile wave +
    a stream-K tail whose partials live in per-cluster buffers (gemm_reduce_kernel), for the
    fp32 (+bias), residual and SiLU*mul epilogues, vs fp64 of the same operands."""
    g = torch.Generator().manual_seed(M + N)
    x = _lvl((M, K), g).cuda()
    w = _lvl((N, K), g, 2.0 ** -6).cuda()
    bias = _lvl((N,), g, 0.125).cuda()
    xd, wd = x.cpu().double(), w.cpu().double()
    out = torch.full((M, N), float("nan"), dtype=torch.float32, device="cuda")
    P.test_gemm(x, w, out, M, N, K, 0, bias=bias)
    r = _lvl((M, N), g).cuda()
    ref2 = xd @ wd.T + r.cpu().double()
    P.test_gemm(x, w, r, M, N, K, 2, resid=r)
    act = torch.full((M, N // 2), float("nan"), dtype=torch.bfloat16, device="cuda")
    P.test_gemm(x, w, act, M, N, K, 3)   # rows read as interleaved [gate 8 | up 8] groups
    torch.cuda.synchronize()
    ref = xd @ wd.T + bias.cpu().double()
    assert (out.cpu().double() - ref).abs().max().item() <= 1e-5 * ref.abs().max().item() + 1e-6
    d2 = (r.cpu().double() - ref2).abs()
    assert (d2 <= ref2.abs() * 2.0 ** -8 + 1e-6 * ref2.abs().max()).all()
    y = (xd @ wd.T).view(M, N // 16, 2, 8)
    gate, up = y[:, :, 0, :].reshape(M, N // 2), y[:, :, 1, :].reshape(M, N // 2)
    refs = gate / (1 + torch.exp(-gate)) * up
    d3 = (act.cpu().double() - refs).abs()
    assert (d3 <= refs.abs() * 2.0 ** -7 + 1e-4 * refs.abs().max()).all()


@pytest.mark.parametrize("M,h,I", [(8, 256, 768), (256, 1024, 3072), (200, 5120, 25600),
                                   (256, 5120, 25600), (64, 2048, 9472), (300, 1024, 3072),
                                   (512, 5120, 25600), (448, 2048, 5120)])
def test_mlp_fused(P, M, h, I):
    """Fused gate/up -> down launch (SURVEY.md a10 + a11) + resid_norm, vs fp64 of the same bf16
    operands: act within bf16 rounding, xout = resid + act Wd^T and u = RMSNorm(xout) g."""
    g = torch.Generator().manual_seed(M + h + I)
    u = _lvl((M, h), g).cuda()
    wg = _lvl((I, h), g, 2.0 ** -5)
    wu = _lvl((I, h), g, 2.0 ** -5)
    wgu = torch.cat([torch.cat([wg[8 * t:8 * t + 8], wu[8 * t:8 * t + 8]]) for t in range(I // 8)]).cuda()
    wd = _lvl((h, I), g, 2.0 ** -7).cuda()
    r = _lvl((M, h), g).cuda()
    gain = (1 + _lvl((h,), g, 2.0 ** -3).float()).to(torch.bfloat16).cuda()
    act = torch.full((M, I), float("nan"), dtype=torch.bfloat16, device="cuda")
    xout = torch.full((M, h), float("nan"), dtype=torch.bfloat16, device="cuda")
    un = torch.full((M, h), float("nan"), dtype=torch.bfloat16, device="cuda")
    for _ in range(2):   # twice: the tile counters must be reset by the previous launch
        P.test_mlp_fused(u, wgu, wd, r, gain, 1e-6, act, xout, un)
        torch.cuda.synchronize()
    ud = u.cpu().double()
    a_, b_ = ud @ wg.double().T, ud @ wu.double().T
    aref = a_ / (1 + torch.exp(-a_)) * b_
    d = (act.cpu().double() - aref).abs()
    assert (d <= aref.abs() * 2.0 ** -7 + 1e-4 * aref.abs().max()).all()
    xref = r.cpu().double() + act.cpu().double() @ wd.cpu().double().T   # from the GPU's act
    got = xout.cpu().double()
    assert ((got - xref).abs() <= xref.abs() * 2.0 ** -8 + 1e-5 * xref.abs().max()).all()
    uref = got * torch.rsqrt((got * got).mean(-1, keepdim=True) + 1e-6) * gain.cpu().double()
    assert ((un.cpu().double() - uref).abs() <= uref.abs() * 2.0 ** -7 + 1e-6 * uref.abs().max()).all()


@pytest.mark.parametrize("M,F,K,splits", [(8, 64, 256, 1), (33, 192, 512, 0), (256, 640, 1024, 4),
                                          (200, 328, 512, -1), (300, 1040, 256, -1), (40, 200, 256, -1)])
def test_gemm_silu_mul(P, M, F, K, splits):
    g = torch.Generator().manual_seed(2)
    x = _lvl((M, K), g).cuda()
    wg = _lvl((F, K), g, 2.0 ** -4)
    wu = _lvl((F, K), g, 2.0 ** -4)
    packed = torch.cat([torch.cat([wg[8 * t:8 * t + 8], wu[8 * t:8 * t + 8]]) for t in range(F // 8)]).cuda()
    out = torch.empty(M, F, dtype=torch.bfloat16, device="cuda")
    P.test_gemm(x, packed, out, M, 2 * F, K, 3, k_splits=splits)
    torch.cuda.synchronize()
    xd = x.cpu().double()
    a, b = xd @ wg.double().T, xd @ wu.double().T
    ref = a / (1 + torch.exp(-a)) * b
    d = (out.cpu().double() - ref).abs()
    assert (d <= ref.abs() * 2.0 ** -7 + 1e-4 * ref.abs().max()).all()


@pytest.mark.parametrize("M,N,K", [(1, 1024, 256), (8, 151936 // 8, 512), (200, 2000, 256)])
@pytest.mark.parametrize("orient", [0, -1])
def test_gemm_fused_argmax(P, M, N, K, orient):
    g = torch.Generator().manual_seed(3)
    x = _lvl((M, K), g).cuda()
    w = _lvl((N, K), g, 2.0 ** -4).cuda()
    packed = torch.zeros(M, dtype=torch.int64, device="cuda")
    P.test_gemm(x, w, packed, M, N, K, 4, ldo=0, k_splits=orient)
    logits = torch.empty(M, N, dtype=torch.float32, device="cuda")
    P.test_gemm(x, w, logits, M, N, K, 0)
    torch.cuda.synchronize()
    idx = (0xFFFFFFFF - (packed.cpu() & 0xFFFFFFFF)).numpy()
    ref = (x.cpu().double() @ w.cpu().double().T).numpy()
    lg = logits.cpu().numpy()
    # the decision is taken in the kernel's fp32: must equal argmax (lowest index) of fp32 logits
    assert (idx == np.argmax(lg, axis=1)).all()
    top2 = np.sort(ref, axis=1)[:, -2:]
    sure = (top2[:, 1] - top2[:, 0]) > 1e-4
    assert (idx[sure] == np.argmax(ref, axis=1)[sure]).all()


# fused QKV GEMM (a6): GEMM + bias + per-head RMSNorm + RoPE + q / KV-cache stores in one launch
def _qkv_reference(x, w, bias, nq, nkv, hd, gq, gk, eps, rope, pos):
    """fp64 torch reference of the fused epilogue on the same bf16 operands."""
    y = x.double() @ w.double().T
    if bias is not None:
        y = y + bias.double()
    M = x.shape[0]
    y = y.view(M, nq + 2 * nkv, hd)
    q, k, v = y[:, :nq], y[:, nq:nq + nkv], y[:, nq + nkv:]

    def norm(t, g):
        if g is None:
            return t
        return t * torch.rsqrt(t.pow(2).mean(-1, keepdim=True) + eps) * g.double()

    cs = rope.double()[pos.long()]                      # [M, hd/2, 2]
    c, s = cs[..., 0][:, None, :], cs[..., 1][:, None, :]

    def rot(t):
        a, b = t[..., :hd // 2], t[..., hd // 2:]
        return torch.cat([a * c - b * s, b * c + a * s], -1)

    return rot(norm(q, gq)), rot(norm(k, gk)), v


@pytest.mark.parametrize("M,K,nq,nkv,hd,qk_norm,bias,splits", [
    (256, 5120, 64, 8, 128, True, False, 0),      # Qwen3-32B shape, token-major head tiles
    (300, 1024, 16, 4, 128, True, True, 0),       # ragged token tail, QKV bias (Qwen2.5)
    (1024, 2048, 32, 8, 128, False, False, 0),    # Llama-like, several token pairs
    (200, 512, 8, 2, 64, True, True, 0),          # hd 64
    (64, 1024, 16, 4, 128, True, True, 0),        # below the token-major threshold (W-major)
    (256, 1024, 16, 4, 128, True, False, 1),      # W-major whole tiles forced
])
def test_gemm_qkv_fused(P, M, K, nq, nkv, hd, qk_norm, bias, splits):
    g = torch.Generator().manual_seed(M + K + nq)
    N = (nq + 2 * nkv) * hd
    x = _lvl((M, K), g).cuda()
    w = _lvl((N, K), g, 2.0 ** -5).cuda()
    b = _lvl((N,), g, 0.125).cuda() if bias else None
    gq = (1 + _lvl((hd,), g, 0.25).float()).to(torch.bfloat16).cuda() if qk_norm else None
    gk = (1 + _lvl((hd,), g, 0.25).float()).to(torch.bfloat16).cuda() if qk_norm else None
    smax = 64
    pos = torch.randint(0, smax, (M,), generator=g, dtype=torch.int32).cuda()
    ang = torch.arange(smax, dtype=torch.float64)[:, None] * 10000.0 ** (
        -torch.arange(0, hd, 2, dtype=torch.float64) / hd)[None, :]
    rope = torch.stack([ang.cos(), ang.sin()], -1).float().cuda()      # [smax, hd/2, 2]
    q = torch.full((M, nq, hd), float("nan"), dtype=torch.bfloat16, device="cuda")
    kc = torch.zeros(M, nkv, smax, hd, dtype=torch.bfloat16, device="cuda")
    vc = torch.zeros_like(kc)
    eps = 1e-6
    for _ in range(2):   # twice: the split-tile arrival counters must be back at zero
        P.test_gemm_qkv(x, w, b, nq, nkv, hd, gq, gk, eps, rope, pos, q, kc, vc, smax, k_splits=splits)
    torch.cuda.synchronize()
    rq, rk, rv = _qkv_reference(x.cpu(), w.cpu(), None if b is None else b.cpu(), nq, nkv, hd,
                                None if gq is None else gq.cpu(), None if gk is None else gk.cpu(),
                                eps, rope.cpu(), pos.cpu())
    ar = torch.arange(M)
    pk = kc.cpu()[ar, :, pos.cpu().long()].double()                     # [M, nkv, hd]
    pv = vc.cpu()[ar, :, pos.cpu().long()].double()
    for got, ref in ((q.cpu().double(), rq), (pk, rk), (pv, rv)):
        err = (got - ref).abs().max().item()
        assert err <= 2.0 ** -7 * ref.abs().max().item(), err
    # nothing written outside the new tokens' cache rows
    mask = torch.ones(M, smax, dtype=torch.bool)
    mask[ar, pos.cpu().long()] = False
    assert kc.cpu().permute(0, 2, 1, 3)[mask].abs().max().item() == 0
