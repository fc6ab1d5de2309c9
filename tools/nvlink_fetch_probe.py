"""NVLink evidence for the WaS fetch (needs >= 2 GPUs; prints {"skipped": ...} otherwise): one
pooled layer copied from GPU `--src` (the owner) into GPU `--dst` (the reader) by the fetch
kernel exactly as the ring runs it (sidp_test_fetch engine 3: TMA bulk copies from the peer VA,
claimed chunk groups), by the round-1 LDG/STG kernel (engine 2) and by the copy engine (engine 1),
CUDA-event timed; the kernel result is checked bit for bit.  Under ncu (one process, the reader's
launches), tools/profile.sh reads nvlrx__bytes.sum / nvltx__bytes.sum beside dram__bytes.
    python tools/nvlink_fetch_probe.py [--bytes 975e6] [--src 1] [--dst 0] [--ctas 16,24,32]"""
import argparse, ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

ap = argparse.ArgumentParser()
ap.add_argument("--bytes", type=float, default=975e6)
ap.add_argument("--src", type=int, default=1)
ap.add_argument("--dst", type=int, default=0)
ap.add_argument("--ctas", default="16,24,32")
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
if torch.cuda.device_count() < 2:
    print(json.dumps({"skipped": f"{torch.cuda.device_count()} GPU(s) visible, the probe needs 2"}))
    sys.exit(0)
import paper_2605_28095_b200 as P
L = P._abi.lib()
L.sidp_test_fetch.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int32, C.c_int32, C.c_void_p]
n = int(a.bytes) // 16 * 16
src = torch.randint(-30000, 30000, (n // 2,), dtype=torch.int16, device=f"cuda:{a.src}")
torch.cuda.set_device(a.dst)
dst = torch.empty(n // 2, dtype=torch.int16, device=f"cuda:{a.dst}")
torch.cuda.synchronize(a.src)
res = {"bytes": n, "src_gpu": a.src, "dst_gpu": a.dst,
       "peer_access": torch.cuda.can_device_access_peer(a.dst, a.src)}
runs = [(int(c), 3) for c in a.ctas.split(",")] + [(24, 2), (0, 1)]
for ctas, engine in runs:
    try:
        dst.zero_()
        for _ in range(2):
            P._abi.check(L.sidp_test_fetch(dst.data_ptr(), src.data_ptr(), n, ctas, engine, None), "fetch")
        torch.cuda.synchronize(a.dst)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            P._abi.check(L.sidp_test_fetch(dst.data_ptr(), src.data_ptr(), n, ctas, engine, None), "fetch")
        e1.record()
        torch.cuda.synchronize(a.dst)
        ms = e0.elapsed_time(e1) / a.reps
        ok = bool(torch.equal(dst.cpu(), src.cpu()))
        key = {1: "copy_engine", 2: f"ldg_{ctas}ctas", 3: f"ring_fetch_{ctas}ctas"}[engine]
        res[key] = {"ms": ms, "GBps": n / ms / 1e6, "bitwise": ok}
    except Exception as e:   # e.g. a bulk copy from a peer VA refused by this driver
        res[f"engine{engine}_{ctas}"] = {"error": str(e)[:200]}
print(json.dumps(res))
