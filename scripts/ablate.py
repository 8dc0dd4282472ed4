"""Timing ablations of the device path (graph-replayed, PDL-chained): the
exposed cost of each kernel = full step minus the step without it
(CCL_DEBUG_SKIP bits, set per subprocess; labels are wrong when skipping)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def child(name, n):
    import torch
    import paper_1712_09789_b200 as ccl
    if name == "zeros":
        import numpy as np
        img_np = np.zeros((n, n), np.uint8)
    elif name.startswith("d"):
        img_np = ccl.random_image(n, n, float(name[1:]), 0)
    else:
        img_np = ccl.pattern_image(name, n, n)
    img = torch.from_numpy(img_np).cuda()
    out = torch.empty(img.shape, dtype=torch.uint32, device="cuda")
    fl = torch.ones(1 << 28, dtype=torch.int32, device="cuda")
    for _ in range(5):
        ccl.label_device(img, out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(15):
        fl.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ccl.label_device(img, out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    print(f"{ts[len(ts) // 2]:.1f}")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child(sys.argv[2], int(sys.argv[3]))
        raise SystemExit
    n = int(os.environ.get("ABL_N", "8192"))
    for name in os.environ.get("ABL_IMGS", "d0.5,zeros,d0.7,spiral").split(","):
        res = {}
        for tag, mask in [("full", 0), ("-d", 2), ("-d2", 4), ("-e", 8), ("-d2-e", 12), ("a only", 14), ("-a", 1)]:
            env = dict(os.environ, CCL_DEBUG_SKIP=str(mask))
            r = subprocess.run([sys.executable, __file__, "--child", name, str(n)], env=env, capture_output=True,
                               text=True)
            res[tag] = r.stdout.strip() or r.stderr.strip()[-200:]
        print(f"{name:8s} {n}: " + "  ".join(f"{k}={v}" for k, v in res.items()), flush=True)
