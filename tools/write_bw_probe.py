import torch, time
x = torch.empty(8 * 1024**3 // 8, dtype=torch.float64, device='cuda')
h = torch.empty(8 * 1024**3 // 8, dtype=torch.float16, device='cuda')
for name, f, nbytes in [("memset zero (write only)", lambda: x.zero_(), x.numel()*8),
                        ("torch h->d copy_", lambda: x.copy_(h), x.numel()*10)]:
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): f()
    e1.record(); torch.cuda.synchronize()
    ms=e0.elapsed_time(e1)/5
    print(f"{name}: {nbytes/ms/1e6:.0f} GB/s")
