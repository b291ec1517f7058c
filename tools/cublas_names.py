import torch
from torch.profiler import profile, ProfilerActivity
for M, N, K in [(320, 12288, 4096), (320, 4096, 4096), (320, 16384, 4096), (320, 4096, 16384), (8, 12288, 4096), (128, 12288, 4096)]:
    x = torch.randn(M, K, device="cuda").bfloat16(); w = torch.randn(N, K, device="cuda").bfloat16()
    torch.matmul(x, w.T); torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as p:
        torch.matmul(x, w.T); torch.cuda.synchronize()
    names = [e.name for e in p.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    print(M, N, K, names)
