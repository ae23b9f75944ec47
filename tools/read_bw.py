import torch
x = torch.empty(4 * 1024**3, dtype=torch.bfloat16, device="cuda").fill_(1)   # 8 GiB
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for f, name in ((lambda: x.amax(), "amax"), (lambda: x.sum(), "sum")):
    f(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        a.record(); f(); b.record(); torch.cuda.synchronize(); best = min(best, a.elapsed_time(b))
    print(f"torch {name} read-only over 8 GiB: {x.numel()*2/best/1e6:.1f} GB/s")
