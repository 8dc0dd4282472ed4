"""(a)+(d) only timing per library (CCL_DEBUG_SKIP=12), mean of 30 graph replays."""
import os, subprocess, sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
def child(names, n):
    import torch, numpy as np
    import paper_1712_09789_b200 as ccl
    res = []
    for name in names:
        img_np = np.zeros((n, n), np.uint8) if name == "zeros" else (ccl.random_image(n, n, float(name[1:]), 0) if name.startswith("d") else ccl.pattern_image(name, n, n))
        img = torch.from_numpy(img_np).cuda(); out = torch.empty(img.shape, dtype=torch.uint32, device="cuda")
        fl = torch.ones(1 << 28, dtype=torch.int32, device="cuda")
        for _ in range(5): ccl.label_device(img, out)
        torch.cuda.synchronize(); ts = []
        for _ in range(30):
            fl.sum(); e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); ccl.label_device(img, out); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort(); ts = ts[3:-3]
        res.append(f"{name}:{sum(ts)/len(ts):.1f}")
    print("  ".join(res))
if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(sys.argv[2].split(","), int(sys.argv[3])); raise SystemExit
    names = os.environ.get("CMP_IMGS", "d0.5,zeros,d0.7,spiral").split(",")
    for lib in sys.argv[1:]:
        for skip in os.environ.get("SKIPS", "0,12,14").split(","):
            env = dict(os.environ, CCL_LIB_PATH=lib, CCL_DEBUG_SKIP=skip)
            p = subprocess.run([sys.executable, __file__, "--child", ",".join(names), os.environ.get("CMP_N", "8192")], env=env, capture_output=True, text=True)
            print(f"{os.path.basename(lib):34s} skip={skip:3s} " + (p.stdout.strip() or p.stderr.strip()[-300:]), flush=True)
