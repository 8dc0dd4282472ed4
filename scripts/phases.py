"""Per-phase cycle breakdown of kernel (a) (needs a -DCCL_PHASES=1 build; debug aid).
usage: CCL_LIB_PATH=..._phases1.so python scripts/phases.py [w] [kind]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1712_09789_b200 as ccl  # noqa: E402

NAMES = ["records+top", "masks", "prefix+coarse", "jumps", "unions", "flatten+marks", "tagging", "table",
         "B:wait prev", "B:mask wait+build", "B:bands+coarse+ulist", "B:jumps+unions", "B:marks", "B:table+store",
         "B:records"]
lib = ccl._lib
f = lib.ccl_debug_phases
f.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
w = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
kinds = sys.argv[2:] or ["random0.5"]
for kind in kinds:
    if kind.startswith("random"):
        img = ccl.random_image(w, w, float(kind[6:]), 0)
    elif kind == "zeros":
        img = np.zeros((w, w), np.uint8)
    else:
        img = ccl.pattern_image(kind, w, w)
    d = torch.from_numpy(img).cuda()
    for _ in range(2):
        ccl.label_device(d, sync=True)
    buf = (ctypes.c_ulonglong * 16)()
    f(buf, 1)
    n = 5
    for _ in range(n):
        ccl.label_device(d, sync=True)
    f(buf, 1)
    vals = [buf[i] / n for i in range(16)]
    tot = sum(vals) or 1
    print(f"{kind}: total {tot / 1e6:.1f} Mcycles (thread-0 sum over CTAs per run)")
    for i, nm in enumerate(NAMES):
        if not vals[i]:
            continue
        print(f"  {nm:16s} {vals[i] / 1e6:8.2f} M  {100 * vals[i] / tot:5.1f}%")
