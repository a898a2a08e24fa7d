import torch
x=torch.empty(1<<28,dtype=torch.float32,device='cuda')  # 1 GiB
y=torch.empty_like(x)
for name,f in [("fill",lambda: x.fill_(1.0)),("copy",lambda: y.copy_(x)),("sum",lambda: x.sum())]:
    for _ in range(3): f()
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10): f()
    e.record(); torch.cuda.synchronize()
    ms=s.elapsed_time(e)/10
    by = (1<<30)*(2 if name=="copy" else 1)
    print(name, ms, by/ms/1e6, "GB/s")
