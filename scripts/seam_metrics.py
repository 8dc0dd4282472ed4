"""Kernel (d) union work (find steps, CAS attempts) of one 8192^2 image with an
instrumented library (CCL_LIB_PATH=...metrics build): seam_metrics.py <image>"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_1712_09789_b200 as ccl  # noqa: E402
name = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
img = ccl.random_image(n, n, float(name[1:]), 0) if name.startswith("d") else ccl.pattern_image(name, n, n)
assert ccl.metrics_build()
for _ in range(3):
    ccl.label_image(img)
    m = ccl.read_metrics()
    print(name, os.path.basename(os.environ.get("CCL_LIB_PATH", "")), "border_find", m["border_find"], "border_cas", m["border_cas"],
          "resolve_find", m["resolve_find"], "local find", int(m["find"].sum()), "cas", int(m["cas"].sum()))
