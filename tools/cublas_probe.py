import torch
for (M,N,K) in [(256,5120,8192),(256,5120,25600),(256,10240,5120),(256,51200,5120),(16,5120,8192)]:
    x=torch.randn(M,K,device='cuda',dtype=torch.bfloat16); w=torch.randn(N,K,device='cuda',dtype=torch.bfloat16)
    for _ in range(3): y=x@w.t()
    torch.cuda.synchronize()
