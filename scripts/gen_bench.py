"""GPU random_image generator: throughput and parity with the host generator (debug aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1712_09789_b200 as ccl
for (w, h) in [(8192, 8192), (32768, 32768)]:
    out = torch.empty((h, w), dtype=torch.uint8, device="cuda")
    ccl.random_image_device(w, h, 0.5, 0, out)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); ccl.random_image_device(w, h, 0.5, 0, out); torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    t1 = time.perf_counter(); ref = ccl.random_image(w, h, 0.5, 0); ht = time.perf_counter() - t1
    print(f"{w}x{h}: gpu {dt*1e3:.2f} ms (incl. host jump tables), host {ht*1e3:.0f} ms, equal={np.array_equal(out.cpu().numpy(), ref)}")
