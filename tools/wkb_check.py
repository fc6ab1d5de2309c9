"""k-block-major W (SIDP_TEST_GEMM_WKB=1): GEMM results vs fp64 for both orientations."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_28095_b200 as P
for (M, N, K) in [(16, 1024, 512), (256, 512, 5120), (100, 640, 128), (256, 10240, 1024), (8, 256, 64)]:
    for orient in (0, 1, -1, 3):
        g = torch.Generator().manual_seed(5)
        x = (torch.randint(-8, 8, (M, K), generator=g).float() / 8).bfloat16().cuda()
        w = (torch.randint(-8, 8, (N, K), generator=g).float() / 256).bfloat16().cuda()
        wkb = w.view(N, K // 64, 64).transpose(0, 1).contiguous().view(N, K)
        out = torch.full((M, N), float("nan"), device="cuda")
        P.test_gemm(x, wkb, out, M, N, K, 0, k_splits=orient)
        torch.cuda.synchronize()
        ref = (x.double() @ w.double().T).float()
        bad = int((~((out - ref).abs() <= 1e-3 * ref.abs().max() + 1e-6)).sum())
        print(f"M={M} N={N} K={K} splits={orient}: bad={bad}", flush=True)
