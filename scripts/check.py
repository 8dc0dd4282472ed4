"""Quick GPU parity sweep (debug aid, not a test): label a handful of images
with every variant and compare against the oracle; print the first mismatch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1712_09789_b200 as ccl  # noqa: E402


def check(name, img, variants=("c2fl", "rc2fl", "cc2fl", "nc2fl")):
    want = oracle.sequential_ccl(img)
    ok = True
    for v in variants:
        d = torch.from_numpy(np.ascontiguousarray(img)).cuda()
        got, _ = ccl.label_device(d, variant=v, sync=True)
        got = got.cpu().numpy()
        if not np.array_equal(got, want):
            ok = False
            bad = np.argwhere(got != want)
            y, x = bad[0]
            print(f"FAIL {name} {v}: {len(bad)} px differ; first ({y},{x}) got {got[y, x]:#x} want {want[y, x]:#x}")
    if ok:
        print(f"ok   {name}")
    return ok


if __name__ == "__main__":
    allok = True
    for (w, h) in [(1, 1), (33, 7), (64, 64), (256, 32), (257, 33), (300, 1), (1, 300), (517, 391), (1920, 1080),
                   (2048, 2048)]:
        for d in (0.1, 0.5, 0.7, 0.95):
            allok &= check(f"random {w}x{h} d{d}", ccl.random_image(w, h, d, 7))
    for k in ("blobs", "spiral", "stripes", "checkerboard"):
        allok &= check(f"{k} 1024", ccl.pattern_image(k, 1024, 1024))
    allok &= check("ones 777x333", np.ones((333, 777), np.uint8))
    allok &= check("zeros 777x333", np.zeros((333, 777), np.uint8))
    rng = np.random.default_rng(1)
    allok &= check("bytes{0,1,2,255}", rng.choice(np.array([0, 1, 2, 255], np.uint8), size=(300, 500)))
    print("ALL OK" if allok else "SOME FAILED")
