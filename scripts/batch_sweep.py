"""Config 4 (1024 x 1080p frames) on one GPU: batch pipelining knobs
(CCL_PIPE, CCL_PIPE_TILES, CCL_PIPE_A, CCL_PIPE_E) -- device time per batch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1712_09789_b200 as ccl  # noqa: E402

w, h, n = 1920, 1080, 1024
frames = torch.empty((n, h, w), dtype=torch.uint8, device="cuda")
for j in range(n):
    ccl.random_image_device(w, h, 0.5, j, out=frames[j])
out = torch.empty((n, h, w), dtype=torch.uint32, device="cuda")
fl = torch.ones(1 << 28, dtype=torch.int32, device="cuda")
ref = None


def run(tag, **env):
    global ref
    for k in ("CCL_PIPE", "CCL_PIPE_TILES", "CCL_PIPE_A", "CCL_PIPE_E"):
        os.environ.pop(k, None)
    for k, v in env.items():
        os.environ[k] = str(v)
    for _ in range(2):
        ccl.label_batch_device(frames, out)
    ts = []
    for _ in range(5):
        fl.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ccl.label_batch_device(frames, out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[2]
    h_ = int(out[::97].sum().item())
    if ref is None:
        ref = h_
    print(f"{tag:34s} {ms:7.3f} ms  {n * w * h / ms / 1e6:7.1f} Gpx/s  {'OK' if h_ == ref else 'MISMATCH'}", flush=True)


run("no pipeline", CCL_PIPE=0)
import itertools
for tiles in [int(x) for x in os.environ.get("SWEEP_TILES", "12288,16384,24576").split(",")]:
    pairs = os.environ.get("SWEEP_PAIRS", "8:2,8:3,7:3,9:2,10:2,6:4,4:4,5:3,9:1,10:1,7:2,6:2")
    for a, e in [tuple(int(v) for v in p.split(":")) for p in pairs.split(",")]:
        run(f"tiles {tiles} a{a} e{e}", CCL_PIPE_TILES=tiles, CCL_PIPE_A=a, CCL_PIPE_E=e)
