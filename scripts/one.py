"""Label one image a few times (profiling driver)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1712_09789_b200 as ccl
w = int(sys.argv[1]) if len(sys.argv) > 1 else 512
h = int(sys.argv[2]) if len(sys.argv) > 2 else w
img = torch.from_numpy(ccl.random_image(w, h, 0.5, 0)).cuda()
for _ in range(3):
    out, t = ccl.label_device(img, sync=True)
print(t)
