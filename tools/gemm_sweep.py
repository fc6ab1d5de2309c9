"""Per-k-block vs fixed cost of the GEMM kernel (debug modes via SIDP_GEMM_DEBUG)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_28095_b200 as P
M = 256
tag = os.environ.get("TAG", "")
for N, epi in [(51200, 3), (51200, 0), (5120, 0)]:
    for K in [64, 512, 2048, 5120]:
        w = torch.randn(N, K, device="cuda").to(torch.bfloat16)
        x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        out = torch.empty(M, N // 2 if epi == 3 else N, device="cuda",
                          dtype=torch.bfloat16 if epi == 3 else torch.float32)
        for _ in range(3):
            P.test_gemm(x, w, out, M, N, K, epi, k_splits=1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            P.test_gemm(x, w, out, M, N, K, epi, k_splits=1)
        e1.record(); torch.cuda.synchronize()
        print(f"{tag} N={N} K={K} epi={epi}: {e0.elapsed_time(e1)/10*1e3:8.1f} us", flush=True)
