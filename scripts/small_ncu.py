import sys; sys.path.insert(0,'.')
import torch, paper_1712_09789_b200 as ccl
for w in (512, 2048):
    img = torch.from_numpy(ccl.random_image(w, w, 0.5, 0)).cuda()
    out = torch.empty((w, w), dtype=torch.uint32, device="cuda")
    for _ in range(3): ccl.label_device(img, out)
    torch.cuda.synchronize()
