"""Instrumented-build counters vs density (the paper's Figs. 7-10 quantities on
the GPU's tiles): mean find steps and CAS attempts per 128x64 tile of kernel
(a), border-merge and resolve totals.  Run with the metrics library:
  CCL_LIB_PATH=paper_1712_09789_b200/_lib/libccl_b200_metrics1.so python scripts/metrics_sweep.py [w]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_09789_b200 as ccl  # noqa: E402

assert ccl.metrics_build(), "needs the CCL_METRICS=1 library (CCL_LIB_PATH)"
w = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
print(f"{w}x{w} random, seed 0; per 128x64 tile of kernel (a): mean / max find steps and CAS attempts")
print(f"{'density':>7} {'find mean':>10} {'find max':>9} {'cas mean':>9} {'cas max':>8} {'border find':>12} "
      f"{'border cas':>11} {'resolve find':>13}")
for i in range(1, 10):
    d = i / 10
    rep = ccl.label_image(ccl.random_image(w, w, d, 0))
    m = ccl.read_metrics()
    f, c = m["find"], m["cas"]
    print(f"{d:7.1f} {f.mean():10.1f} {f.max():9d} {c.mean():9.1f} {c.max():8d} {m['border_find']:12d} "
          f"{m['border_cas']:11d} {m['resolve_find']:13d}")
for kind in ("blobs", "spiral", "stripes", "checkerboard"):
    ccl.label_image(ccl.pattern_image(kind, w, w))
    m = ccl.read_metrics()
    f, c = m["find"], m["cas"]
    print(f"{kind:>12} find mean {f.mean():.1f} cas mean {c.mean():.1f} border find {m['border_find']} "
          f"border cas {m['border_cas']} resolve find {m['resolve_find']}")
