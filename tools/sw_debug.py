"""Token-major GEMM debug: error pattern per BNF for one shape."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch
    import paper_2605_28095_b200 as P
    M, N, K = map(int, sys.argv[2:5])
    g = torch.Generator().manual_seed(5)
    x = (torch.randint(-8, 8, (M, K), generator=g).float() / 8).bfloat16().cuda()
    w = (torch.randint(-8, 8, (N, K), generator=g).float() / 256).bfloat16().cuda()
    out = torch.full((M, N), float("nan"), device="cuda")
    P.test_gemm(x, w, out, M, N, K, 0, k_splits=1)
    torch.cuda.synchronize()
    ref = (x.double() @ w.double().T).float()
    bad = ~((out - ref).abs() <= 1e-3 * ref.abs().max() + 1e-6)
    rows = bad.any(1).nonzero().flatten().tolist()
    cols = bad.any(0).nonzero().flatten().tolist()
    print(f"BNF={os.environ.get('SIDP_GEMM_SW_BNF')} M={M} N={N} K={K}: bad={int(bad.sum())} "
          f"rows[{len(rows)}]={rows[:6]}..{rows[-3:]} cols[{len(cols)}]={cols[:6]}..{cols[-3:]} nan={int(out.isnan().sum())}")
    sys.exit(0)
for shape in [(256, 512, 5120), (256, 512, 256), (128, 1024, 512)]:
    for bnf in [16, 32, 64, 80, 128, 256]:
        env = dict(os.environ, SIDP_GEMM_SW_BNF=str(bnf))
        subprocess.run([sys.executable, __file__, "child", *map(str, shape)], env=env)
