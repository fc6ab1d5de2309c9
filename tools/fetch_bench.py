"""K1 fetch-kernel bandwidth on one GPU (local HBM -> HBM copy of one pooled layer) for several
CTA counts, beside the copy engine (cudaMemcpyAsync).  NVLink peer bandwidth cannot be measured
on the 1-GPU pool; this bounds the kernel's own issue capability.  engine 3 = the kernel exactly as
the WaS ring runs it (claimed chunk groups, completion published).  Prints one JSON line."""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_28095_b200 as P

nbytes = int(float(os.environ.get("BYTES", 975e6)))
src = torch.empty(nbytes // 2, dtype=torch.bfloat16, device="cuda").fill_(1.0)
dst = torch.empty_like(src)
res = {"bytes": nbytes}
L = P._abi.lib()
L.sidp_test_fetch.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int32, C.c_int32, C.c_void_p]
runs = [(c, 0) for c in [8, 16, 32, 64]] + [(c, 3) for c in [16, 24, 32, 48]] + [(0, 1)]
if os.environ.get("ONLY_LDG"):
    runs = [(int(c), 2) for c in os.environ.get("ONLY_LDG").split(",")]
elif os.environ.get("ONLY_RING"):
    runs = [(int(c), 3) for c in os.environ.get("ONLY_RING").split(",")]
for ctas, engine in runs:
    for _ in range(2):
        P._abi.check(L.sidp_test_fetch(dst.data_ptr(), src.data_ptr(), nbytes, ctas, engine, None), "fetch")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        P._abi.check(L.sidp_test_fetch(dst.data_ptr(), src.data_ptr(), nbytes, ctas, engine, None), "fetch")
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    key = {1: "copy_engine", 2: f"ldg_fetch_{ctas}ctas", 3: f"ring_fetch_{ctas}ctas"}.get(engine, f"sm_fetch_{ctas}ctas")
    res[key] = {"ms": ms, "GBps_read": nbytes / ms / 1e6}
assert torch.equal(dst, src)
print(json.dumps(res))
