"""Small-image latency vs throughput of the device path (SURVEY configs 1-2):
single-call device time (CUDA events around one un-split call, median) and
back-to-back throughput (events around 200 calls), L2 not flushed."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1712_09789_b200 as ccl  # noqa: E402

for (w, d) in [(512, 0.5), (2048, 0.1), (2048, 0.5), (2048, 0.9), (8192, 0.5)]:
    img = torch.from_numpy(ccl.random_image(w, w, d, 0)).cuda()
    out = torch.empty((w, w), dtype=torch.uint32, device="cuda")
    s = torch.cuda.current_stream()
    for _ in range(5):
        ccl.label_device(img, out)
    torch.cuda.synchronize()
    lat = []
    for _ in range(50):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        ccl.label_device(img, out)
        e1.record(s)
        torch.cuda.synchronize()
        lat.append(e0.elapsed_time(e1) * 1e3)
    lat.sort()
    n = 200
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(n):
        ccl.label_device(img, out)
    e1.record(s)
    torch.cuda.synchronize()
    thr = e0.elapsed_time(e1) * 1e3 / n
    print(f"{w}^2 d={d}: single call {lat[len(lat) // 2]:7.1f} us ({w * w / lat[len(lat) // 2] / 1e3:6.1f} Gpx/s)  "
          f"back-to-back {thr:7.1f} us/call ({w * w / thr / 1e3:6.1f} Gpx/s)")
