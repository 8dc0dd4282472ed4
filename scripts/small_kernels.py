"""Per-kernel device durations for small images (run under ncu --metrics
gpu__time_duration.sum): 512^2 and 2048^2 d=0.5, a few warm calls each."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1712_09789_b200 as ccl  # noqa: E402

for w in (512, 2048):
    img = torch.from_numpy(ccl.random_image(w, w, 0.5, 0)).cuda()
    out = torch.empty((w, w), dtype=torch.uint32, device="cuda")
    for _ in range(4):
        ccl.label_device(img, out)
    torch.cuda.synchronize()
