"""A/B timing of experiment libraries (graph-replayed device path, L2 flushed
between steps, trimmed mean of 15), each library in its own process, with a
bit-exactness check against the oracle.
usage: CMP_IMGS=d0.5,zeros,... python scripts/cmp_libs.py lib1.so lib2.so ..."""
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def make(name, n):
    import numpy as np
    import paper_1712_09789_b200 as ccl
    if name == "zeros":
        return np.zeros((n, n), np.uint8)
    if name.startswith("d"):
        return ccl.random_image(n, n, float(name[1:]), 0)
    return ccl.pattern_image(name, n, n)


def child(names, n, check):
    import numpy as np
    import torch
    import oracle
    out_lines = []
    for name in names:
        img_np = make(name, n)
        img = torch.from_numpy(img_np).cuda()
        out = torch.empty(img.shape, dtype=torch.uint32, device="cuda")
        fl = torch.ones(1 << 28, dtype=torch.int32, device="cuda")
        import paper_1712_09789_b200 as ccl
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
        ts = ts[3:-3]
        _, t = ccl.label_device(img, out, sync=True)
        ok = ""
        if check:
            ok = " OK" if np.array_equal(out.cpu().numpy(), oracle.sequential_ccl(img_np)) else " MISMATCH"
        out_lines.append(f"{name}:{sum(ts) / len(ts):.1f}(a{t['local_ms'] * 1e3:.0f}){ok}")
    print("  ".join(out_lines))


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(sys.argv[2].split(","), int(sys.argv[3]), sys.argv[4] == "1")
        raise SystemExit
    names = os.environ.get("CMP_IMGS", "d0.5,zeros,d0.3,d0.7,spiral,blobs").split(",")
    n = int(os.environ.get("CMP_N", "8192"))
    check = os.environ.get("CMP_CHECK", "1")
    reps = int(os.environ.get("CMP_REPS", "1"))
    for r in range(reps):
        for lib in sys.argv[1:]:
            env = dict(os.environ, CCL_LIB_PATH=lib)
            try:
                p = subprocess.run([sys.executable, __file__, "--child", ",".join(names), str(n), check], env=env,
                                   capture_output=True, text=True, timeout=int(os.environ.get("CMP_TIMEOUT", "240")))
            except subprocess.TimeoutExpired:
                print(f"{os.path.basename(lib):36s} TIMEOUT", flush=True)
                continue
            print(f"{os.path.basename(lib):36s} " + (p.stdout.strip() or p.stderr.strip()[-300:]), flush=True)
