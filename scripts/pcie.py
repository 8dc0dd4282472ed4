"""PCIe reference points on this box: pinned H2D / D2H copy bandwidth (256 MiB), one direction and both at once."""
import torch
n = 256 << 20
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, k=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(k):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return min(ts)
ms = t(lambda: h.copy_(d, non_blocking=True)); print(f"D2H {n/ms/1e6:.1f} GB/s")
ms = t(lambda: d.copy_(h, non_blocking=True)); print(f"H2D {n/ms/1e6:.1f} GB/s")
def both():
    with torch.cuda.stream(s1): h.copy_(d, non_blocking=True)
    with torch.cuda.stream(s2): d2.copy_(h2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
ms = t(both); print(f"D2H+H2D concurrent: {2*n/ms/1e6:.1f} GB/s total, {n/ms/1e6:.1f} each")
