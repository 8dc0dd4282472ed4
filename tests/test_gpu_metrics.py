"""Instrumented metrics mode: the CCL_METRICS=1 build of
the library counts, per 128x64 tile of kernel (a), the parent-link steps of
root finding and the CAS attempts of unions (reference BlockMetrics,
forest.hpp:12-29), plus border-merge and resolve totals -- and labels exactly
like the product build.  Runs in a subprocess (one library per process)."""
import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(REPO, "paper_1712_09789_b200", "_lib", "libccl_b200_metrics1.so")

SCRIPT = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
import numpy as np
import torch
import oracle
import paper_1712_09789_b200 as ccl
assert ccl.metrics_build()
out = {}
for d in (0.1, 0.5, 0.9):
    img = ccl.random_image(2048, 2048, d, 0)
    rep = ccl.label_image(img)
    assert np.array_equal(rep.label_map.labels, oracle.sequential_ccl(img)), d
    m = ccl.read_metrics()
    s = ccl.aggregate_metrics(rep)
    out[str(d)] = {"shape": list(m["find"].shape), "find": int(m["find"].sum()), "cas": int(m["cas"].sum()),
                   "border_find": m["border_find"], "border_cas": m["border_cas"],
                   "resolve_find": m["resolve_find"], "blocks": [rep.blocks_x, rep.blocks_y],
                   "n_block": len(rep.per_block), "mean_atomics": s.mean_atomics,
                   "border_phase": [rep.border_phase.findroot_iterations, rep.border_phase.atomic_ops]}
z = ccl.label_image(np.zeros((640, 512), np.uint8))
m = ccl.read_metrics()
out["zeros"] = {"find": int(m["find"].sum()), "cas": int(m["cas"].sum()), "border": m["border_find"] + m["border_cas"],
                "shape": list(m["find"].shape)}
frames = torch.from_numpy(np.stack([ccl.random_image(256, 192, 0.5, i) for i in range(3)])).cuda()
lab = ccl.label_batch_device(frames)
torch.cuda.synchronize()
m = ccl.read_metrics(ccl._ctx(0))
out["batch"] = {"shape": list(m["find"].shape)}
print(json.dumps(out))
"""


@pytest.mark.gpu
def test_metrics_build_counts_and_labels_exactly():
    assert os.path.exists(LIB), "build() builds the instrumented library"
    env = dict(os.environ, CCL_LIB_PATH=LIB)
    r = subprocess.run([sys.executable, "-c", SCRIPT, REPO], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    tw, th = 128, 64
    for d in ("0.1", "0.5", "0.9"):
        o = out[d]
        assert o["shape"] == [1, 2048 // th, 2048 // tw]
        assert o["blocks"] == [2048 // tw, 2048 // th] and o["n_block"] == (2048 // tw) * (2048 // th)
        assert o["find"] > 0 and o["cas"] > 0
        assert o["border_find"] + o["border_cas"] > 0 and o["border_cas"] > 0
        assert o["border_phase"] == [o["border_find"], o["border_cas"]]
        assert abs(o["mean_atomics"] - o["cas"] / o["n_block"]) < 1e-6
    # more foreground adjacencies -> more unions than at d=0.1
    assert out["0.5"]["cas"] > out["0.1"]["cas"]
    assert out["zeros"] == {"find": 0, "cas": 0, "border": 0, "shape": [1, 10, 4]}
    assert out["batch"]["shape"] == [3, 3, 2]
