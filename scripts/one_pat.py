"""Label one pattern image a few times (profiling driver): one_pat.py <pattern|dD|zeros> [n]."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1712_09789_b200 as ccl  # noqa: E402
name = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
if name == "zeros":
    import numpy as np
    img_np = np.zeros((n, n), np.uint8)
else:
    img_np = ccl.random_image(n, n, float(name[1:]), 0) if name.startswith("d") else ccl.pattern_image(name, n, n)
img = torch.from_numpy(img_np).cuda()
for _ in range(3):
    out, t = ccl.label_device(img, sync=True)
print(name, {k: round(v * 1e3, 1) for k, v in t.items()})
