"""HBM read-only bandwidth probe (torch ops): sum-reduce of a 4 GiB bf16 tensor vs a copy.
Answers whether the attention kernel (read-only, 6.21 TB/s under ncu) has headroom above the
copy-based MEASURED_PEAKS figure."""
import torch
x = torch.empty(2 * 1024**3, dtype=torch.bfloat16, device="cuda").uniform_()
y = torch.empty_like(x)
def t(fn, n=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n / 1e3
b = x.numel() * 2
s = t(lambda: x.sum(dtype=torch.float32))
c = t(lambda: y.copy_(x))
print(f"read-only sum: {b / s / 1e9:.0f} GB/s   copy: {2 * b / c / 1e9:.0f} GB/s (read+write)")
