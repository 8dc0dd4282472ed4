"""Write / copy bandwidth reference points on this GPU (context for kernel (e))."""
import torch
x = torch.empty(8192 * 8192, dtype=torch.int32, device="cuda")
y = torch.empty_like(x)
fl = torch.ones(1 << 28, dtype=torch.int32, device="cuda")
def t(fn, n=10):
    for _ in range(3): fn()
    ts = []
    for _ in range(n):
        fl.sum(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]
ms = t(lambda: x.fill_(7)); print(f"fill 256MB: {ms*1e3:.1f} us  {268435456/ms/1e6:.0f} GB/s")
ms = t(lambda: y.copy_(x)); print(f"copy 256MB: {ms*1e3:.1f} us  {2*268435456/ms/1e6:.0f} GB/s (r+w)")
