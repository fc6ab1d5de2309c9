"""Microbenchmark of the tcgen05 decode GEMM at the hot-path shapes (CUDA events; several
weight copies rotated so no launch hits L2), beside cuBLAS (torch.matmul) on the same shape.
Usage: python tools/gemm_bench.py [M] [shape,...] [splits,...]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_28095_b200 as P

M = int(sys.argv[1]) if len(sys.argv) > 1 else 256
shapes = {"qkv": (10240, 5120, 0), "o": (5120, 8192, 2), "gate_up": (51200, 5120, 3),
          "down": (5120, 25600, 2), "lm": (151936, 5120, 0),
          # Llama-3.1-70B
          "l_qkv": (10240, 8192, 0), "l_o": (8192, 8192, 2), "l_gate_up": (57344, 8192, 3),
          "l_down": (8192, 28672, 2)}
only = sys.argv[2].split(",") if len(sys.argv) > 2 and sys.argv[2] != "all" else list(shapes)
splits_list = [int(s) for s in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0, 1]
tag = os.environ.get("TAG", "")


SERIAL = os.environ.get("SERIAL", "0") != "0"   # an event between launches: no PDL overlap
gap = torch.cuda.Event()


def timeit(fn, copies, reps=20):
    for i in range(2):
        fn(i % copies)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(reps):
        if SERIAL:
            gap.record()
        fn(i % copies)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for name in only:
    N, K, epi = shapes[name]
    copies = max(2, int(600e6 // (N * K * 2)) + 1)
    ws = [torch.randn(N, K, device="cuda").to(torch.bfloat16) * 0.02 for _ in range(copies)]
    if os.environ.get("SIDP_TEST_GEMM_WKB", "0") != "0":   # k-block-major copies [K/64][N][64]
        ws = [w.view(N, K // 64, 64).transpose(0, 1).contiguous().view(N, K) for w in ws]
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    if os.environ.get("SIDP_TEST_GEMM_XKB", "0") != "0":   # k-block-major X [K/64][M][64]
        x = x.view(M, K // 64, 64).transpose(0, 1).contiguous().view(M, K)
    if epi == 3:
        out = torch.empty(M, N // 2, device="cuda", dtype=torch.bfloat16)
    elif epi == 2:
        out = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    else:
        out = torch.empty(M, N, device="cuda", dtype=torch.float32)
    fl, by = 2.0 * M * N * K, 2.0 * N * K
    for splits in splits_list:
        us = timeit(lambda i: P.test_gemm(x, ws[i], out, M, N, K, epi,
                                          resid=out if epi == 2 else None, k_splits=splits), copies)
        print(f"{tag} {name:8s} M={M} N={N} K={K} splits={splits}: {us:8.1f} us  {fl/us/1e6:7.1f} TFLOP/s  {by/us/1e3:7.1f} GB/s", flush=True)
    if os.environ.get("NO_CUBLAS"):
        continue
    us = timeit(lambda i: torch.matmul(x, ws[i].t()), copies)
    print(f"{tag} {name:8s} M={M} N={N} K={K} cuBLAS : {us:8.1f} us  {fl/us/1e6:7.1f} TFLOP/s  {by/us/1e3:7.1f} GB/s", flush=True)
