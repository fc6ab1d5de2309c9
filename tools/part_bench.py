"""Time the runtime's partial GEMM + resid_norm (O / down shapes) at a given M, CUDA events,
rotated weight copies.  Usage: python tools/part_bench.py M [o|down]..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_28095_b200 as P

M = int(sys.argv[1])
shapes = {"o": (5120, 8192), "down": (5120, 25600), "o70": (8192, 8192), "down70": (8192, 28672)}
for name in sys.argv[2:] or ["o", "down"]:
    N, K = shapes[name]
    copies = max(2, int(600e6 // (N * K * 2)) + 1)
    ws = [torch.randn(N, K, device="cuda").to(torch.bfloat16) * 0.02 for _ in range(copies)]
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    r = torch.randn(M, N, device="cuda").to(torch.bfloat16)
    g = torch.ones(N, device="cuda", dtype=torch.bfloat16)
    xo = torch.empty_like(r); u = torch.empty_like(r)
    f = lambda i: P.test_gemm_resid_norm(x, ws[i % copies], r, g, 1e-6, xo, u)
    for i in range(3): f(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(20): f(i)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    print(f"{os.environ.get('TAG','')} part {name:6s} M={M} N={N} K={K}: {us:7.1f} us (GEMM + resid_norm)  {2*M*N*K/us/1e6:7.1f} TFLOP/s", flush=True)
