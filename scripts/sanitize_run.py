"""Workload for compute-sanitizer (scripts/sanitize.sh): every kernel of the
labeler on small inputs, through the C-ABI host paths, checked bit-exact
against the oracle (test infrastructure) so a sanitizer run is also a parity run."""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import oracle  # noqa: E402
import paper_1712_09789_b200 as ccl  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1] == "small":  # full hazard listing (racecheck)
    for name, img in [("random512", ccl.random_image(512, 512, 0.5, 0)),
                      ("spiral256", ccl.pattern_image("spiral", 256, 256))]:
        assert np.array_equal(ccl.label_image(img).label_map.labels, oracle.sequential_ccl(img)), name
        print("ok", name, flush=True)
    print("SANITIZE_RUN_DONE")
    sys.exit(0)
cases = [("random2048", ccl.random_image(2048, 2048, 0.5, 0)),
         ("spiral1024", ccl.pattern_image("spiral", 1024, 1024)),
         ("checker512", ccl.pattern_image("checkerboard", 512, 512)),
         ("random1000x777_unaligned", ccl.random_image(1000, 777, 0.6, 3))]
for name, img in cases:
    got = ccl.label_image(img).label_map.labels
    assert np.array_equal(got, oracle.sequential_ccl(img)), name
    print("ok", name, flush=True)
img = ccl.random_image(1003, 777, 0.58, 5)
rep = ccl.label_strips(img, [0, 0, 0])
assert np.array_equal(rep.label_map.labels, oracle.sequential_ccl(img)), "strips"
print("ok strips3", flush=True)
for v in ("rc2fl", "cc2fl", "nc2fl"):
    img = ccl.random_image(700, 300, 0.55, 9)
    assert np.array_equal(ccl.label_image(img, variant=v).label_map.labels, oracle.sequential_ccl(img)), v
    print("ok", v, flush=True)
print("SANITIZE_RUN_DONE")
