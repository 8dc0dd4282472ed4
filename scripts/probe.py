"""Quick GPU probe: per-kernel device times on the headline workload and a few
stress patterns (not the bench contract; see bench.py)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1712_09789_b200 as ccl  # noqa: E402


CHECK = os.environ.get("PROBE_CHECK", "1") == "1"


def flush(buf):
    buf.sum()  # read 1 GiB of clean data: evicts (and writes back) everything in L2


def run(name, img_np, variant="c2fl", iters=10):
    img = torch.from_numpy(img_np).cuda()
    out = torch.empty(img.shape, dtype=torch.uint32, device="cuda")
    fl = torch.ones(1 << 28, dtype=torch.int32, device="cuda")
    for _ in range(3):
        ccl.label_device(img, out, variant=variant, sync=True)
    ts = []
    for _ in range(iters):
        flush(fl)
        torch.cuda.synchronize()
        _, t = ccl.label_device(img, out, variant=variant, sync=True)
        ts.append(t)
    med = lambda k: sorted(x[k] for x in ts)[len(ts) // 2]
    ok = ""
    if CHECK:
        import numpy as np
        import oracle
        ok = " OK" if np.array_equal(out.cpu().numpy(), oracle.sequential_ccl(img_np)) else " MISMATCH"

    px = img.numel()
    tot = med("total_ms")
    gbs = px * 5 / (tot * 1e-3) / 1e9
    print(f"{name:28s} {variant:6s} local {med('local_ms')*1e3:7.1f}us merge {med('merge_ms')*1e3:7.1f}us "
          f"final {med('final_ms')*1e3:7.1f}us total {tot*1e3:7.1f}us  {px/tot/1e6:8.1f} Gpx/s  {gbs:7.0f} GB/s{ok}")


def run_batch(n=128):
    import numpy as np
    frames = torch.from_numpy(np.stack([ccl.random_image(1920, 1080, 0.5, s) for s in range(n)])).cuda()
    out = torch.empty(frames.shape, dtype=torch.uint32, device="cuda")
    fl = torch.ones(1 << 28, dtype=torch.int32, device="cuda")
    for _ in range(3):
        ccl.label_batch_device(frames, out)
    ts = []
    for _ in range(5):
        flush(fl)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ccl.label_batch_device(frames, out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    print(f"batch {n} x 1920x1080 d0.5        total {ms*1e3:9.1f}us  {frames.numel()/ms/1e6:8.1f} Gpx/s")


def run_big():
    img_np = ccl.random_image(32768, 32768, 0.5, 0)
    run("random 32768 d0.5", img_np, iters=3)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--all", action="store_true")
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--shapes", action="store_true")
    ap.add_argument("--modes", action="store_true")
    a = ap.parse_args()
    print(torch.cuda.get_device_name(), "tile", ccl.tile_shape())
    if a.modes:
        run_batch()
        run_big()
        raise SystemExit
    run("random 8192 d0.5", ccl.random_image(8192, 8192, 0.5, 0))
    if a.shapes:
        import numpy as np
        run("zeros 8192", np.zeros((8192, 8192), np.uint8))
        run("ones 8192", np.ones((8192, 8192), np.uint8))
        for d in (0.1, 0.3, 0.9):
            run(f"random 8192 d{d}", ccl.random_image(8192, 8192, d, 0))
        run("random 8192 d0.5", ccl.random_image(8192, 8192, 0.5, 0), "rc2fl")
    if a.quick:
        run("spiral 8192", ccl.pattern_image("spiral", 8192, 8192))
        run("random 8192 d0.7", ccl.random_image(8192, 8192, 0.7, 0))
    if a.all:
        for v in ["rc2fl", "cc2fl", "nc2fl"]:
            run("random 8192 d0.5", ccl.random_image(8192, 8192, 0.5, 0), v)
        for d in (0.1, 0.3, 0.7, 0.9):
            run(f"random 8192 d{d}", ccl.random_image(8192, 8192, d, 0))
        for k in ("blobs", "spiral", "stripes", "checkerboard"):
            run(f"{k} 8192", ccl.pattern_image(k, 8192, 8192))
        run("random 2048 d0.5", ccl.random_image(2048, 2048, 0.5, 0))
        for d in (0.1, 0.3, 0.7, 0.9):
            run(f"random 2048 d{d}", ccl.random_image(2048, 2048, d, 0))
        run("random 512 d0.5", ccl.random_image(512, 512, 0.5, 0))
