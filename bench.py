"""Benchmark: Gpixels/s labeled on 8192^2 random binary d=0.5 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one labeling pass (kernels a-e) over one 8192x8192 u8 image
resident in HBM; `value` = pixels / device time (CUDA events on the launching
stream, L2 flushed by a 1 GiB read between steps).  N>1 (torchrun, one rank
per GPU): weak-scaling strip mode, rank k labels rows [8192k, 8192(k+1)) of
random_image(8192, 8192N, 0.5, 0), generated on each GPU (global raster labels), with the NCCL seam exchange
inside the timed step; value = total pixels / max-over-ranks step time.

`e2e` = same metric through the public host API (ccl_label_host via
paper_1712_09789_b200.label_image path) with pinned host buffers, H2D + D2H
inside the timed region.  `--impl reference` times the reference CPU labeler
(oracle/_ref, compiled from /root/reference) on the host cores instead.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

W = H = 8192
DENSITY, SEED = 0.5, 0
BYTES_PER_PX = 5  # algorithmic: 1 B u8 image in + 4 B u32 label out
METRIC = "Gpixels/s labeled (8192^2 random binary, d=0.5)"


def dist_env():
    r = int(os.environ.get("RANK", "0"))
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    lr = int(os.environ.get("LOCAL_RANK", str(r)))
    return r, ws, lr


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(img_np, max_seconds=20.0):
    """Reference CPU labeler on the host cores (oracle/_ref) — reported baseline only."""
    import numpy as np
    import oracle
    n = os.cpu_count() or 1
    try:
        if not oracle.ref_available():
            oracle.build()
        if oracle.ref_available():
            oracle.ref_label_image(img_np, 32, 32, "c2fl", n)  # warm
            times = []
            t_end = time.time() + max_seconds
            while len(times) < 3 and (time.time() < t_end or not times):
                _, ms = oracle.ref_label_image(img_np, 32, 32, "c2fl", n)
                times.append(ms)
            ms = statistics.median(times)
            out = {"value": img_np.size / (ms * 1e-3) / 1e9, "unit": "Gpixels/s", "cores": n, "kind": "reference",
                   "sample": f"full {img_np.shape[1]}x{img_np.shape[0]} image, ccl_ref::label_image C2FL 32x32 "
                             f"workers={n}, median of {len(times)} (RunReport.wall_time)",
                   "cpu_model": _cpu_model(), "hardware_concurrency": n}
            # SURVEY §8d also asks for one worker: a bounded 2048-row sample of the same image
            sub = np.ascontiguousarray(img_np[:2048])
            _, ms1 = oracle.ref_label_image(sub, 32, 32, "c2fl", 1)
            out["workers1"] = {"value": sub.size / (ms1 * 1e-3) / 1e9, "unit": "Gpixels/s",
                               "sample": f"first 2048 rows ({sub.shape[1]}x{sub.shape[0]}), workers=1, 1 run"}
            return out
    except Exception as e:  # pragma: no cover
        print(f"[bench] reference baseline failed: {e}", file=sys.stderr)
    t0 = time.perf_counter()
    oracle.sequential_ccl(img_np)
    s = time.perf_counter() - t0
    return {"value": img_np.size / s / 1e9, "unit": "Gpixels/s", "cores": 1, "kind": "port",
            "sample": "full image, oracle sequential_ccl (C port), 1 run"}


def run_reference_impl(args):
    """--impl reference: the reference CPU implementation, rank 0 only."""
    rank, ws, _ = dist_env()
    if rank != 0:
        return
    import oracle
    import numpy as np
    if not oracle.ref_available():
        try:
            oracle.build()
        except Exception:
            pass
    n = os.cpu_count() or 1
    use_ref = oracle.ref_available()
    img = (oracle.ref_random_image if use_ref else oracle.random_image)(W, H, DENSITY, SEED)
    rows = H
    # bound the run to a few minutes: shrink the per-step sample if needed
    t0 = time.perf_counter()
    if use_ref:
        oracle.ref_label_image(img, 32, 32, "c2fl", n)
    else:
        oracle.sequential_ccl(img)
    per = time.perf_counter() - t0
    budget = 150.0
    if per * (args.steps + args.warmup) > budget:
        rows = max(256, int(H * budget / (per * (args.steps + args.warmup))) // 32 * 32)
    sample = np.ascontiguousarray(img[:rows])
    for _ in range(args.warmup):
        (oracle.ref_label_image(sample, 32, 32, "c2fl", n) if use_ref else oracle.sequential_ccl(sample))
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        if use_ref:
            _, ms = oracle.ref_label_image(sample, 32, 32, "c2fl", n)
            times.append(ms * 1e-3)
        else:
            oracle.sequential_ccl(sample)
            times.append(time.perf_counter() - t0)
    mean_s = statistics.mean(times)
    val = sample.size / mean_s / 1e9
    desc = (f"{W}x{rows} rows of the 8192^2 d=0.5 seed-0 image per step, "
            + (f"ccl_ref::label_image C2FL 32x32 workers={n} (RunReport.wall_time)" if use_ref
               else "oracle sequential_ccl port, 1 thread"))
    line = {"metric": METRIC, "value": val, "unit": "Gpixels/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean_s * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": "random8192", "width": W, "height": rows, "density": DENSITY, "seed": SEED},
            "cpu_baseline": {"value": val, "unit": "Gpixels/s", "cores": n if use_ref else 1,
                             "kind": "reference" if use_ref else "port", "sample": desc},
            "e2e": {"value": val, "unit": "Gpixels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--variant", default="c2fl")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        run_reference_impl(args)
        return

    import numpy as np
    import torch
    import paper_1712_09789_b200 as ccl

    rank, ws, lrank = dist_env()
    torch.cuda.set_device(lrank)
    dev = torch.device("cuda", lrank)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.Stream(device=dev)
    flush = torch.empty(1 << 28, dtype=torch.int32, device=dev).fill_(1)  # 1 GiB, read between steps

    if ws == 1:
        img_np = ccl.random_image(W, H, DENSITY, SEED)
        img = torch.from_numpy(img_np).to(dev)
    else:  # rows [8192k, 8192(k+1)) of random_image(8192, 8192N, 0.5, 0), generated on this GPU
        img = ccl.random_image_device(W, H, DENSITY, SEED, row0=rank * H, device=lrank)
    out = torch.empty((H, W), dtype=torch.uint32, device=dev)
    ctx = ccl.Context(lrank)

    if ws == 1:
        def step():
            return ccl.label_device(img, out, variant=args.variant, stream=stream, ctx=ctx)
    else:
        from paper_1712_09789_b200 import strips
        strip = strips.StripLabeler(ctx, W, H, row0=rank * H, full_h=H * ws, rank=rank, world=ws, device=dev)

        def step():
            return strip.label(img, out, variant=args.variant, stream=stream)

    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    clk = ClockSampler(lrank)
    clk.start()  # sampling spans the (>= 1 s) warm-up soak and the timed region
    t_soak = time.perf_counter()
    with torch.cuda.stream(stream):
        i = 0
        while i < args.warmup or time.perf_counter() - t_soak < 1.0:
            step()
            i += 1
            if i % 50 == 0:
                torch.cuda.synchronize(dev)
    torch.cuda.synchronize(dev)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    with torch.cuda.stream(stream):
        for i in range(args.steps):
            flush.sum()  # evicts the previous step's labels from L2 (outside the timed interval)
            ev0[i].record(stream)
            step()
            ev1[i].record(stream)
    torch.cuda.synchronize(dev)
    clocks = clk.stop()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    step_ms = [a.elapsed_time(b) for a, b in zip(ev0, ev1)]
    mean_ms = statistics.mean(step_ms)
    if ws > 1:
        t = torch.tensor([mean_ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        mean_ms = float(t.item())
    px_total = W * H * ws
    value = px_total / (mean_ms * 1e-3) / 1e9

    # per-kernel split of one step (same stream, events between launches)
    if ws == 1:
        kms = []
        for _ in range(5):
            flush.sum()
            torch.cuda.synchronize(dev)
            _, t = ccl.label_device(img, out, variant=args.variant, stream=stream, sync=True, ctx=ctx)
            kms.append(t)
        kern = {k: statistics.median(x[k] for x in kms) for k in ("local_ms", "merge_ms", "final_ms", "total_ms")}
    else:
        kern = None

    line = None
    if rank == 0:
        peak, peak_src = peaks()
        if kern:
            dom = max(("local_ms", "merge_ms", "final_ms"), key=lambda k: kern[k])
            dom_bytes = {"local_ms": W * H * 1, "merge_ms": 0, "final_ms": W * H * BYTES_PER_PX}[dom]
            achieved = dom_bytes / (kern[dom] * 1e-3) / 1e9
            roof = {"bound": "hbm", "kernel": {"local_ms": "k_local (a-c)", "merge_ms": "k_seams (d)",
                                                "final_ms": "k_final (e)"}[dom],
                    "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": traffic_from_profiles(dom), "peak_source": peak_src,
                    "algorithmic_bytes_per_launch": dom_bytes}
        else:
            roof = None
        path_achieved = px_total / ws * BYTES_PER_PX / (mean_ms * 1e-3) / 1e9
        line = {
            "metric": METRIC, "value": value, "unit": "Gpixels/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": mean_ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic (reference xoshiro256** generator, seed 0)",
            "config": {"workload": "random8192" if ws == 1 else
                       f"strips of random_image(8192, {8192 * ws}, 0.5, 0) (8192 rows/GPU)",
                       "width": W, "height": H * ws, "density": DENSITY, "seed": SEED, "variant": args.variant,
                       "tile": list(ccl.tile_shape()), "l2_flush": "1 GiB read between timed steps",
                       "parallelism": "single GPU" if ws == 1 else f"{ws} strips, NCCL seam all-gather"},
            "roofline": roof,
            "roofline_path": {"bound": "hbm", "achieved": path_achieved, "peak": peak, "unit": "GB/s",
                              "frac": path_achieved / peak, "bytes_per_px": BYTES_PER_PX},
            "kernels_ms": kern,
            "gpu_launches": ccl.launches_per_label() * args.steps + (0 if ws == 1 else 9 * args.steps),
            "clocks": clocks,
        }
        if ws == 1:
            line["e2e"] = e2e_host_api(ccl, img_np, args)
        if ws == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(img_np)
    if ws > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    if line:
        print(json.dumps(line), flush=True)


def traffic_from_profiles(kernel_key):
    """dram bytes per launch of the dominant kernel from the committed ncu summary, if any."""
    try:
        with open(os.path.join(REPO, "profiles", "traffic.json")) as f:
            t = json.load(f)
        return t.get(kernel_key)
    except Exception:
        return None


def e2e_host_api(ccl, img_np, args):
    """Public host API end to end: pinned host image -> H2D -> kernels -> D2H labels, every step.

    A stream of images through ccl_label_host_async on two alternating contexts
    (one image's upload overlaps the previous image's label download: PCIe is
    full duplex); the synchronous ccl_label_host time of one call is reported
    beside it."""
    import numpy as np
    import torch
    h_img = torch.empty(img_np.shape, dtype=torch.uint8, pin_memory=True)
    h_img.numpy()[:] = img_np
    outs = [torch.empty(img_np.shape, dtype=torch.int32, pin_memory=True) for _ in range(2)]
    a = h_img.numpy()
    o = [t.numpy().view(np.uint32) for t in outs]
    dev = torch.cuda.current_device()
    v = int(ccl.Variant.parse(args.variant))
    ctxs = [ccl.Context(dev), ccl.Context(dev)]
    ms = ctypes.c_float()

    def sync_call():
        ccl._check(ccl._lib.ccl_label_host(ctxs[0].handle, a.ctypes.data_as(ccl._u8p), W, H,
                                           o[0].ctypes.data_as(ccl._u32p), v, ctypes.byref(ms)))

    def stream(n):
        for k in range(n):
            c = ctxs[k & 1]
            if k >= 2:  # this context's previous image must be home before its buffers are reused
                ccl._check(ccl._lib.ccl_ctx_sync(c.handle))
            ccl._check(ccl._lib.ccl_label_host_async(c.handle, a.ctypes.data_as(ccl._u8p), W, H,
                                                     o[k & 1].ctypes.data_as(ccl._u32p), v))
        for c in ctxs:
            ccl._check(ccl._lib.ccl_ctx_sync(c.handle))

    for _ in range(max(1, args.warmup)):
        sync_call()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        sync_call()
        ts.append(time.perf_counter() - t0)
    s_sync = statistics.mean(ts)
    stream(max(2, args.warmup))
    n = max(6, min(args.steps, 20))
    t0 = time.perf_counter()
    stream(n)
    s = (time.perf_counter() - t0) / n
    return {"value": W * H / s / 1e9, "unit": "Gpixels/s", "h2d_bytes_per_step": W * H,
            "d2h_bytes_per_step": W * H * 4,
            "api": "ccl_label_host_async on two alternating contexts (C-ABI of ccl::label_image's host path): "
                   "every step uploads its image and downloads its labels; consecutive steps overlap",
            "ms_per_step": s * 1e3,
            "sync_call": {"value": W * H / s_sync / 1e9, "unit": "Gpixels/s", "ms_per_step": s_sync * 1e3,
                          "api": "ccl_label_host, one blocking call"}}


if __name__ == "__main__":
    main()
