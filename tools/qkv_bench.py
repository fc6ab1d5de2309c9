"""Fused QKV GEMM (EPI_QKV, token-major head tiles) vs the plain fp32 GEMM (EPI_F32) + qkv_post
cost, at the Qwen3-32B QKV shape.  CUDA events, weight copies rotated past L2.
Usage: python tools/qkv_bench.py [M,...]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_28095_b200 as P

Ms = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else [256, 1024]
K, nq, nkv, hd = 5120, 64, 8, 128
N = (nq + 2 * nkv) * hd
copies = 8
ws = [(torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(copies)]
gq = torch.ones(hd, dtype=torch.bfloat16, device="cuda")
smax = 1100
ang = torch.arange(smax, dtype=torch.float64)[:, None] * 1e6 ** (-torch.arange(0, hd, 2, dtype=torch.float64) / hd)
rope = torch.stack([ang.cos(), ang.sin()], -1).float().cuda()


def timeit(fn, reps=20):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(reps):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for M in Ms:
    x = (torch.randn(M, K, device="cuda")).to(torch.bfloat16)
    pos = torch.full((M,), 1024, dtype=torch.int32, device="cuda")
    q = torch.empty(M, nq, hd, dtype=torch.bfloat16, device="cuda")
    kc = torch.empty(M, nkv, smax, hd, dtype=torch.bfloat16, device="cuda")
    vc = torch.empty_like(kc)
    out = torch.empty(M, N, dtype=torch.float32, device="cuda")
    t_f32 = timeit(lambda i: P.test_gemm(x, ws[i % copies], out, M, N, K, 0))
    res = {"M": M, "f32_gemm_us": round(t_f32, 1)}
    for ks in [int(v) for v in os.environ.get("KS", "0,1").split(",")]:
        try:
            res[f"qkv_fused_k{ks}_us"] = round(timeit(lambda i: P.test_gemm_qkv(
                x, ws[i % copies], None, nq, nkv, hd, gq, gq, 1e-6, rope, pos, q, kc, vc, smax,
                k_splits=ks)), 1)
        except Exception as e:   # noqa: BLE001
            res[f"qkv_fused_k{ks}_us"] = str(e)[:80]
    print(res, flush=True)
