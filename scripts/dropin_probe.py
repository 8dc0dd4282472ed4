import time, ctypes, numpy as np, sys, os
sys.path.insert(0, '/root/repo')
import paper_1712_09789_b200 as ccl
from paper_1712_09789_b200 import _lib, _ctx, _u8p, _u32p, _check
img = ccl.random_image(8192, 8192, 0.5, 0)
h, w = img.shape
ctx = _ctx(0)
ms = ctypes.c_float()
def call(out):
    _check(_lib.ccl_label_host(ctx.handle, img.ctypes.data_as(_u8p), w, h, out.ctypes.data_as(_u32p), 0, ctypes.byref(ms)))
out = np.empty((h, w), np.uint32); call(out)
for name, fn in [("np.empty", lambda: np.empty((h, w), np.uint32)),
                 ("np.empty + fill", lambda: np.full((h, w), 7, np.uint32)),
                 ("label_host into a touched buffer", lambda: call(out)),
                 ("label_image (new output)", lambda: ccl.label_image(img))]:
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
    print(f"{name:36s} {sorted(ts)[2]*1e3:8.2f} ms")
print("cpus", os.cpu_count())
