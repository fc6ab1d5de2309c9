"""Compute-kernel slowdown beside a resident SM fetch CTA: times the gate/up
GEMM (M = 1024) and prints its per-CTA milestones (SIDP_GEMM_TRACE=1) alone and while a long
unpaced 1-CTA fetch runs on another stream.  Usage: SIDP_GEMM_TRACE=1 python tools/corun_probe.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_28095_b200 as P

sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
nbytes = 6 << 30
src = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
dst = torch.empty_like(src)
M, N, K = 1024, 51200, 5120
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
w = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
out = torch.empty(M, N // 2, device="cuda", dtype=torch.bfloat16)


def run(tag, n=3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(sb):
        e0.record(sb)
        for _ in range(n):
            P.test_gemm(x, w, out, M, N, K, 3, stream=sb)
        e1.record(sb)
    sb.synchronize()
    print(f"{tag}: gate/up M={M} {e0.elapsed_time(e1) / n * 1e3:.1f} us", flush=True)


run("alone")
lib = P._abi.lib()
P._abi.check(lib.sidp_test_fetch(dst.data_ptr(), src.data_ptr(), nbytes, 1, 0, sa.cuda_stream), "fetch")
run("beside a 1-CTA fetch")
sa.synchronize()
run("alone again")
