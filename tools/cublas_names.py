import torch
from torch.profiler import profile, ProfilerActivity
for (M,N,K) in [(256,10240,5120),(256,5120,8192),(256,51200,5120),(256,5120,25600)]:
    x=torch.randn(M,K,device="cuda",dtype=torch.bfloat16); w=torch.randn(N,K,device="cuda",dtype=torch.bfloat16)
    for _ in range(3): torch.matmul(x,w.t())
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(5): torch.matmul(x,w.t())
        torch.cuda.synchronize()
    for e in prof.key_averages():
        if e.device_type.name=="CUDA" or "gemm" in e.key.lower() or "xmma" in e.key.lower():
            print(M,N,K, e.key[:200], round(e.device_time_total/e.count,1) if e.count else None)
