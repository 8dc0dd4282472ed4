"""Benchmark: Gpixels/s labeled (BASELINE.json: 8192^2 random binary d=0.5).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload random8192|strips32768|batch1080|sweep2048|patterns8192|parity512]

One step = one labeling pass (kernels (a)-(e), plus the seam exchange in strip
mode) over one synthetic input already resident in HBM; `value` = pixels /
device time (CUDA events on the launching stream, L2 flushed by a 1 GiB read
between steps; max over ranks).  Workloads (BASELINE.json configs):

  random8192   (default at N=1) config 3 headline: random_image(8192, 8192, 0.5, 0).
               The line also carries "configs": every other north_star config
               measured on this GPU in the same run (configs 1, 2, 3, 4 and the
               N=1 point of 5), and the CPU baselines.
  strips32768  (default at N>1) config 5: random_image(32768, 32768, 0.5, 0) in N
               strips of 32768/N rows, one per rank (STRONG scaling); the seam
               exchange runs inside the library (NVLink peer stores + device
               flags, strip groups).  Rank 0 also labels the whole image alone
               (`n1_value`) so the efficiency is self-contained.
  batch1080    config 4: 1024 frames random_image(1920, 1080, 0.5, s), 1024/N
               frames per rank in one batched launch per kernel, no communication.
  sweep2048 / patterns8192 / parity512: configs 2, 3 (blobs, spiral, stripes,
               checkerboard) and 1 on their own line.

`e2e` = the same metric through the public host API with host buffers (H2D and
D2H inside the timed region).  `--impl reference` times the reference CPU
labeler (oracle/_ref, compiled from /root/reference) on this host's cores.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
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

BYTES_PER_PX = 5  # algorithmic: 1 B u8 image in + 4 B u32 label out
METRIC = "Gpixels/s labeled (8192^2 random binary, d=0.5)"
METRICS = {"random8192": METRIC,
           "strips32768": "Gpixels/s labeled (32768^2 random d=0.5, strip-partitioned)",
           "batch1080": "Gpixels/s labeled (1024 x 1920x1080 random d=0.5 frames)"}
DATA = "synthetic (reference xoshiro256** generator / reference patterns)"
SWEEP = [0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9]
PATTERNS = ["blobs", "spiral", "stripes", "checkerboard"]


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


# ------------------------------------------------------------ CPU baselines
def _median_ms(fn, reps):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        r = fn()
        ts.append(r if r is not None else (time.perf_counter() - t0) * 1e3)
    return statistics.median(ts)


def cpu_baseline(img_np):
    """The reference CPU labeler on this host's cores -- reported
    baseline only: all cores (median of 3 on the full image), one worker and the
    single-thread sequential_ccl oracle (medians of 3 on a 2048-row sample)."""
    import numpy as np
    import oracle
    n = os.cpu_count() or 1
    if not oracle.ref_available():
        try:
            oracle.build()
        except Exception:
            pass
    if not oracle.ref_available():  # pragma: no cover - the box always has oracle/_ref
        s = _median_ms(lambda: (oracle.sequential_ccl(img_np), None)[1], 1)
        return {"value": img_np.size / (s * 1e-3) / 1e9, "unit": "Gpixels/s", "cores": 1, "kind": "port",
                "sample": "full image, oracle sequential_ccl (C port), 1 run"}
    oracle.ref_label_image(img_np, 32, 32, "c2fl", n)  # warm
    ms = _median_ms(lambda: oracle.ref_label_image(img_np, 32, 32, "c2fl", n)[1], 3)
    out = {"value": img_np.size / (ms * 1e-3) / 1e9, "unit": "Gpixels/s", "cores": n, "kind": "reference",
           "sample": f"full {img_np.shape[1]}x{img_np.shape[0]} image, ccl_ref::label_image C2FL 32x32 "
                     f"workers={n}, median of 3 (RunReport.wall_time)",
           "cpu_model": _cpu_model(), "hardware_concurrency": n}
    sub = np.ascontiguousarray(img_np[:2048])
    ms1 = _median_ms(lambda: oracle.ref_label_image(sub, 32, 32, "c2fl", 1)[1], 3)
    out["workers1"] = {"value": sub.size / (ms1 * 1e-3) / 1e9, "unit": "Gpixels/s", "cores": 1,
                       "sample": f"first 2048 rows ({sub.shape[1]}x2048), ccl_ref::label_image workers=1, median of 3"}
    mss = _median_ms(lambda: (oracle.ref_sequential_ccl(sub), None)[1], 3)
    out["sequential_ccl"] = {"value": sub.size / (mss * 1e-3) / 1e9, "unit": "Gpixels/s", "cores": 1,
                             "sample": "first 2048 rows, ccl_ref::sequential_ccl (proj/src/oracle.cpp:34-50), "
                                       "median of 3 (wall clock)"}
    return out


def cpu_baseline_batch(w=1920, h=1080, frames=64):
    """Config 4 on the CPU: hardware_concurrency concurrent label_image(workers=1)
    calls, one frame each, over a bounded sample of frames."""
    import oracle
    n = os.cpu_count() or 1
    imgs = [oracle.ref_random_image(w, h, 0.5, s) for s in range(frames)]
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(n) as ex:  # ctypes releases the GIL
        list(ex.map(lambda im: oracle.ref_label_image(im, 32, 32, "c2fl", 1), imgs))
    s = time.perf_counter() - t0
    return {"value": frames * w * h / s / 1e9, "unit": "Gpixels/s", "cores": n, "kind": "reference",
            "sample": f"frames 0..{frames - 1} of the 1024-frame batch, {n} concurrent ccl_ref::label_image "
                      "workers=1 calls (wall clock)"}


# ------------------------------------------------------------ reference arm
def run_reference_impl(args):
    """--impl reference: the reference CPU implementation on this host, rank 0 only."""
    rank, ws, _ = dist_env()
    if rank != 0:
        return
    import numpy as np
    import oracle
    if not oracle.ref_available():
        try:
            oracle.build()
        except Exception:
            pass
    use_ref = oracle.ref_available()
    n = os.cpu_count() or 1
    workload = args.workload or ("random8192" if ws == 1 else "strips32768")
    gen = oracle.ref_random_image if use_ref else oracle.random_image
    if workload == "batch1080":
        W_, H_ = 1920, 1080
        per_frame = []
        frames = [gen(W_, H_, 0.5, s) for s in range(2 * n)]
        for _ in range(args.warmup):
            with cf.ThreadPoolExecutor(n) as ex:
                list(ex.map(lambda im: oracle.ref_label_image(im, 32, 32, "c2fl", 1), frames[:n]))
        for _ in range(args.steps):
            t0 = time.perf_counter()
            with cf.ThreadPoolExecutor(n) as ex:
                list(ex.map(lambda im: oracle.ref_label_image(im, 32, 32, "c2fl", 1), frames))
            per_frame.append(time.perf_counter() - t0)
        mean_s = statistics.mean(per_frame)
        px = len(frames) * W_ * H_
        desc = f"{len(frames)} of the 1024 frames per step, {n} concurrent ccl_ref::label_image workers=1 calls"
        cfg = {"workload": workload, "width": W_, "height": H_, "frames": 1024, "density": 0.5}
    else:
        W_ = H_ = 32768 if workload == "strips32768" else 8192
        img = gen(W_, 2048 if W_ == 32768 else H_, 0.5, 0)  # 32768: the first rows of the image
        t0 = time.perf_counter()
        oracle.ref_label_image(img, 32, 32, "c2fl", n) if use_ref else oracle.sequential_ccl(img)
        per = time.perf_counter() - t0
        rows = img.shape[0]
        budget = 150.0
        if per * (args.steps + args.warmup) > budget:
            rows = max(256, int(rows * budget / (per * (args.steps + args.warmup))) // 32 * 32)
        sample = np.ascontiguousarray(img[:rows])
        for _ in range(args.warmup):
            oracle.ref_label_image(sample, 32, 32, "c2fl", n) if use_ref else oracle.sequential_ccl(sample)
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            if use_ref:
                times.append(oracle.ref_label_image(sample, 32, 32, "c2fl", n)[1] * 1e-3)
            else:
                oracle.sequential_ccl(sample)
                times.append(time.perf_counter() - t0)
        mean_s = statistics.mean(times)
        px = sample.size
        desc = (f"{W_}x{rows} rows of random_image({W_}, {H_}, 0.5, 0) per step, "
                + (f"ccl_ref::label_image C2FL 32x32 workers={n} (RunReport.wall_time)" if use_ref
                   else "oracle sequential_ccl port, 1 thread"))
        cfg = {"workload": workload, "width": W_, "height": H_, "density": 0.5, "seed": 0}
    val = px / mean_s / 1e9
    line = {"metric": METRICS.get(workload, f"Gpixels/s labeled ({workload})"), "value": val,
            "unit": "Gpixels/s", "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": mean_s * 1e3, "higher_is_better": True,
            "scaling": "weak" if workload == "random8192" else "strong", "vs_baseline": None, "dtype": "u32",
            "data": DATA, "config": cfg,
            "cpu_baseline": {"value": val, "unit": "Gpixels/s", "cores": n if use_ref else 1,
                             "kind": "reference" if use_ref else "port", "sample": desc},
            "e2e": {"value": val, "unit": "Gpixels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ device timing
class Timer:
    """K timed steps on `stream`, L2 flushed between them, events on the stream."""

    def __init__(self, dev, stream):
        import torch
        self.torch, self.dev, self.stream = torch, dev, stream
        self.flush = torch.empty(1 << 28, dtype=torch.int32, device=dev).fill_(1)  # 1 GiB

    def run(self, step, steps, warmup, soak_s=0.0):
        torch = self.torch
        with torch.cuda.stream(self.stream):
            t0 = time.perf_counter()
            i = 0
            while i < warmup or time.perf_counter() - t0 < soak_s:
                step()
                i += 1
                if i % 50 == 0:
                    torch.cuda.synchronize(self.dev)
        torch.cuda.synchronize(self.dev)
        ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        with torch.cuda.stream(self.stream):
            for i in range(steps):
                self.flush.sum()  # evicts the previous step's data from L2 (outside the timed interval)
                ev0[i].record(self.stream)
                step()
                ev1[i].record(self.stream)
        torch.cuda.synchronize(self.dev)
        return statistics.mean(a.elapsed_time(b) for a, b in zip(ev0, ev1))


def cpu_ref_gpx(img_np, reps=3):
    """Reference CPU labeler (oracle/_ref, all host cores) on one image: Gpx/s, median of `reps`."""
    import oracle
    if not oracle.ref_available():
        return None
    n = os.cpu_count() or 1
    ms = _median_ms(lambda: oracle.ref_label_image(img_np, 32, 32, "c2fl", n)[1], reps)
    return img_np.size / (ms * 1e-3) / 1e9


def measure_configs(ccl, timer, ctx, dev, stream, steps=5, warmup=3, cpu=True):
    """Every other north_star config on this GPU, device-resident, L2 flushed
    between steps (per-config throughput visible in the driver's bench line),
    each with the reference CPU labeler's throughput on the same image beside
    it (`cpu_gpx_s`, all host cores; 32768^2: its first 2048 rows)."""
    import numpy as np
    import torch
    out = {}

    def one(img, w, h):
        lab = torch.empty((h, w), dtype=torch.uint32, device=dev)
        ms = timer.run(lambda: ccl.label_device(img, lab, stream=stream, ctx=ctx), steps, warmup)
        r = {"ms": ms, "gpx_s": w * h / (ms * 1e-3) / 1e9}
        if cpu:
            host = img.cpu().numpy() if h <= 8192 else np.ascontiguousarray(img[:2048].cpu().numpy())
            r["cpu_gpx_s"] = cpu_ref_gpx(host)
        return r

    img = ccl.random_image_device(512, 512, 0.5, 0, device=dev.index)
    out["1_parity512"] = one(img, 512, 512)
    out["2_sweep2048"] = {f"d{d:.1f}": one(ccl.random_image_device(2048, 2048, d, 0, device=dev.index), 2048, 2048)
                          for d in SWEEP}
    pats = {}
    for kind in PATTERNS:
        a = torch.from_numpy(ccl.pattern_image(kind, 8192, 8192)).to(dev)
        pats[kind] = one(a, 8192, 8192)
        del a
    for d in (0.1, 0.3, 0.7, 0.9):
        pats[f"random_d{d}"] = one(ccl.random_image_device(8192, 8192, d, 0, device=dev.index), 8192, 8192)
    out["3_8192"] = pats
    out["4_batch1080"] = batch_point(ccl, timer, ctx, dev, stream, 1024, steps=3, warmup=2)
    torch.cuda.empty_cache()
    big = ccl.random_image_device(32768, 32768, 0.5, 0, device=dev.index)
    out["5_single32768"] = one(big, 32768, 32768)
    out["5_strip_rank_model"] = strip_rank_model(ccl, big, dev, stream, ctx)
    del big
    torch.cuda.empty_cache()
    return out


def strip_rank_model(ccl, img, dev, stream, ctx, ns=(2, 4, 8), reps=4):
    """Config 5 on ONE GPU as a per-rank cost model: for N strips, the kernels
    rank N/2 runs in a multi-GPU step -- (a)+(d) on its 32768/N rows, the seam
    export, the seam union-find over all N exports, (d2)+(e) -- timed back to
    back with CUDA events (every other strip's export prepared first).  The
    NVLink exchange of N x 16 W bytes is not included (one GPU here).
    `projected_gpx_s` = 32768^2 / rank step: the strong-scaling curve the
    multi-GPU run should approach (scripts/strip_model.py prints the phases)."""
    import torch
    from paper_1712_09789_b200 import _lib, _check
    from paper_1712_09789_b200.strips import split_rows
    H, W = img.shape
    s = stream.cuda_stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    out = torch.empty((H, W), dtype=torch.uint32, device=dev)
    res = {}
    for n in ns:
        parts = split_rows(H, n)
        seams = torch.empty((n, 4 * W), dtype=torch.int32, device=dev)
        scratch = torch.empty(int(_lib.ccl_strip_scratch_words(n, W)), dtype=torch.int32, device=dev)
        works = [torch.zeros(int(_lib.ccl_work_bytes(W, h, 1)), dtype=torch.uint8, device=dev) for _, h in parts]
        k = n // 2

        def phase1(j):
            r0, h = parts[j]
            im, lo = img[r0:r0 + h], out[r0:r0 + h]
            _check(_lib.ccl_strip_local(ctx.handle, im.data_ptr(), im.stride(0), W, h, r0, H, lo.data_ptr(),
                                        works[j].data_ptr(), 0, s))
            _check(_lib.ccl_strip_seam_export(ctx.handle, W, h, r0, H, j, lo.data_ptr(), works[j].data_ptr(),
                                              seams[j].data_ptr(), s))

        for j in range(n):
            phase1(j)
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(torch.cuda.ExternalStream(s) if stream is None else stream)
            phase1(k)
            r0, h = parts[k]
            lo = out[r0:r0 + h]
            _check(_lib.ccl_strip_seam_resolve(ctx.handle, seams.data_ptr(), n, k, W, h, r0, H, lo.data_ptr(),
                                               works[k].data_ptr(), scratch.data_ptr(), s))
            _check(_lib.ccl_strip_final(ctx.handle, W, h, r0, H, lo.data_ptr(), works[k].data_ptr(), 0, s))
            e1.record(torch.cuda.ExternalStream(s) if stream is None else stream)
            torch.cuda.synchronize(dev)
            ts.append(e0.elapsed_time(e1))
        ms = sorted(ts)[len(ts) // 2]
        res[f"N{n}"] = {"rank_ms": ms, "projected_gpx_s": H * W / (ms * 1e-3) / 1e9, "rows_per_rank": parts[k][1]}
        del seams, scratch, works
    res["note"] = ("per-rank kernels of the N-GPU step measured on one GPU (L2 warm between phases, no flush); "
                   "the NVLink seam exchange (N x 16 W bytes) is not included")
    torch.cuda.empty_cache()
    return res


def batch_point(ccl, timer, ctx, dev, stream, nframes, first=0, steps=3, warmup=2):
    import torch
    w, h = 1920, 1080
    frames = torch.empty((nframes, h, w), dtype=torch.uint8, device=dev)
    for j in range(nframes):
        ccl.random_image_device(w, h, 0.5, first + j, out=frames[j], device=dev.index)
    lab = torch.empty((nframes, h, w), dtype=torch.uint32, device=dev)
    ms = timer.run(lambda: ccl.label_batch_device(frames, lab, stream=stream, ctx=ctx), steps, warmup)
    del frames, lab
    return {"ms": ms, "gpx_s": nframes * w * h / (ms * 1e-3) / 1e9, "frames": nframes}


# ------------------------------------------------------------ end to end
def e2e_host_api(ccl, img_np, args):
    """Public host API end to end: host image -> H2D -> kernels -> D2H labels, every step.

    Headline: a stream of images through ccl_label_host_async on two
    alternating contexts with page-locked buffers (one image's upload overlaps
    the previous image's label download: PCIe is full duplex).  Beside it: one
    blocking ccl_label_host call, and the drop-in ccl::label_image semantics on
    PAGEABLE memory (numpy in, a fresh numpy label map out: the C++
    ccl::label_image on std::vectors does the same work)."""
    import numpy as np
    import torch
    H_, W_ = img_np.shape
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
        ccl._check(ccl._lib.ccl_label_host(ctxs[0].handle, a.ctypes.data_as(ccl._u8p), W_, H_,
                                           o[0].ctypes.data_as(ccl._u32p), v, ctypes.byref(ms)))

    def stream(n):
        for k in range(n):
            c = ctxs[k & 1]
            if k >= 2:  # this context's previous image must be home before its buffers are reused
                ccl._check(ccl._lib.ccl_ctx_sync(c.handle))
            ccl._check(ccl._lib.ccl_label_host_async(c.handle, a.ctypes.data_as(ccl._u8p), W_, H_,
                                                     o[k & 1].ctypes.data_as(ccl._u32p), v))
        for c in ctxs:
            ccl._check(ccl._lib.ccl_ctx_sync(c.handle))

    for _ in range(max(1, args.warmup)):
        sync_call()
    s_sync = statistics.mean(_timed(sync_call) for _ in range(5))
    stream(max(2, args.warmup))
    n = max(6, min(args.steps, 20))
    t0 = time.perf_counter()
    stream(n)
    s = (time.perf_counter() - t0) / n
    for _ in range(2):
        ccl.label_image(img_np)
    s_page = statistics.mean(_timed(lambda: ccl.label_image(img_np)) for _ in range(3))
    px = W_ * H_
    return {"value": px / s / 1e9, "unit": "Gpixels/s", "h2d_bytes_per_step": px, "d2h_bytes_per_step": px * 4,
            "api": "ccl_label_host_async on two alternating contexts (C-ABI of ccl::label_image's host path), "
                   "page-locked buffers: every step uploads its image and downloads its labels; consecutive "
                   "steps overlap",
            "ms_per_step": s * 1e3,
            "sync_call": {"value": px / s_sync / 1e9, "unit": "Gpixels/s", "ms_per_step": s_sync * 1e3,
                          "api": "ccl_label_host, one blocking call, page-locked buffers"},
            "dropin_pageable": {"value": px / s_page / 1e9, "unit": "Gpixels/s", "ms_per_step": s_page * 1e3,
                                "api": "label_image(numpy image) -> RunReport with a new numpy label map: "
                                       "pageable H2D + kernels + pageable D2H, one blocking call"}}


def _timed(fn):
    t0 = time.perf_counter()
    fn()
    return time.perf_counter() - t0


def traffic_from_profiles(kernel_key):
    """dram bytes per launch of the dominant kernel from the committed ncu summary, if any."""
    try:
        with open(os.path.join(REPO, "profiles", "traffic.json")) as f:
            return json.load(f).get(kernel_key)
    except Exception:
        return None


def _max_over_ranks(x, ws, dev):
    if ws == 1:
        return x
    import torch
    gloo = torch.distributed.get_backend() == "gloo"
    t = torch.tensor([x], device="cpu" if gloo else dev, dtype=torch.float64)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None,
                    choices=["random8192", "strips32768", "batch1080", "sweep2048", "patterns8192", "parity512"])
    ap.add_argument("--variant", default="c2fl")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config table of the N=1 line")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        run_reference_impl(args)
        return

    import numpy as np
    import torch
    import paper_1712_09789_b200 as ccl

    rank, ws, lrank = dist_env()
    workload = args.workload or ("random8192" if ws == 1 else "strips32768")
    # CCL_BENCH_ONE_GPU=1: every rank on GPU 0 with gloo (a functional check of
    # the N>1 paths on a one-GPU box; ranks then time-slice one GPU, so the
    # numbers are not scaling numbers)
    one_gpu = os.environ.get("CCL_BENCH_ONE_GPU") == "1"
    if one_gpu:
        lrank = 0
    torch.cuda.set_device(lrank)
    dev = torch.device("cuda", lrank)
    if ws > 1:
        import torch.distributed as dist
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.Stream(device=dev)
    timer = Timer(dev, stream)
    ctx = ccl.Context(lrank)
    peak, peak_src = peaks()
    clk = ClockSampler(lrank)
    extra = {}
    kern = None
    launches_per_step = ccl.launches_per_label()

    if workload in ("random8192", "patterns8192", "parity512", "sweep2048") and ws > 1:
        raise SystemExit(f"--workload {workload} is a single-GPU config (use strips32768 / batch1080 for N>1)")
    if workload == "random8192":
        W_ = H_ = 8192
        img_np = ccl.random_image(W_, H_, 0.5, 0)
        img = torch.from_numpy(img_np).to(dev)
        out = torch.empty((H_, W_), dtype=torch.uint32, device=dev)
        step = lambda: ccl.label_device(img, out, variant=args.variant, stream=stream, ctx=ctx)  # noqa: E731
        px_step, scaling = W_ * H_, "weak"
        cfg = {"workload": "random8192", "width": W_, "height": H_, "density": 0.5, "seed": 0,
               "variant": args.variant, "tile": list(ccl.tile_shape())}
        metric = METRIC
    elif workload == "strips32768":
        from paper_1712_09789_b200.strips import StripLabeler
        W_ = H_ = 32768
        lab = StripLabeler(ctx, W_, H_, rank, ws)
        img = ccl.random_image_device(W_, lab.h, 0.5, 0, row0=lab.row0, device=lrank)  # this rank's rows
        out = torch.empty((lab.h, W_), dtype=torch.uint32, device=dev)
        step = lambda: lab.label(img, out, variant=args.variant, stream=stream)  # noqa: E731
        px_step, scaling = W_ * H_, "strong"
        launches_per_step = lab.launches
        cfg = {"workload": "strips32768", "width": W_, "height": H_, "density": 0.5, "seed": 0,
               "strips": ws, "rows_per_gpu": lab.h, "variant": args.variant,
               "exchange": "in-library: 16*W-byte seam export stored into every rank's exchange area "
                           "(CUDA IPC, NVLink peer stores) + device epoch flags; no host round trip"}
        metric = METRICS["strips32768"]
    elif workload == "batch1080":
        w, h, total = 1920, 1080, 1024
        per = total // ws + (1 if rank < total % ws else 0)
        first = rank * (total // ws) + min(rank, total % ws)
        frames = torch.empty((per, h, w), dtype=torch.uint8, device=dev)
        for j in range(per):
            ccl.random_image_device(w, h, 0.5, first + j, out=frames[j], device=lrank)
        out = torch.empty((per, h, w), dtype=torch.uint32, device=dev)
        step = lambda: ccl.label_batch_device(frames, out, variant=args.variant, stream=stream, ctx=ctx)  # noqa
        px_step, scaling = total * w * h, "strong"
        cfg = {"workload": "batch1080", "width": w, "height": h, "frames": total, "frames_per_gpu": per,
               "density": 0.5, "seeds": "0..1023", "variant": args.variant}
        metric = METRICS["batch1080"]
    else:  # single-GPU config lines
        key = {"sweep2048": "2_sweep2048", "patterns8192": "3_8192", "parity512": "1_parity512"}[workload]
        table = measure_single(ccl, timer, ctx, dev, stream, workload, args)
        vals = [v["gpx_s"] for v in table.values()] if "gpx_s" not in table else [table["gpx_s"]]
        line = {"metric": f"Gpixels/s labeled ({workload})", "value": statistics.mean(vals), "unit": "Gpixels/s",
                "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": DATA,
                "config": {"workload": workload, "value": "mean over the cases"}, key: table}
        print(json.dumps(line), flush=True)
        return

    clk.start()
    mean_ms = timer.run(step, args.steps, args.warmup, soak_s=1.0)
    clocks = clk.stop()
    if ws > 1:
        torch.distributed.barrier()
    mean_ms = _max_over_ranks(mean_ms, ws, dev)
    value = px_step / (mean_ms * 1e-3) / 1e9

    if workload == "random8192":  # per-kernel split of one step (events between the launches)
        kms = []
        for _ in range(5):
            timer.flush.sum()
            torch.cuda.synchronize(dev)
            _, t = ccl.label_device(img, out, variant=args.variant, stream=stream, sync=True, ctx=ctx)
            kms.append(t)
        kern = {k: statistics.median(x[k] for x in kms) for k in ("local_ms", "merge_ms", "final_ms", "total_ms")}
    if workload == "strips32768" and rank == 0:
        # the N=1 point of the same image on this GPU (self-contained efficiency)
        del img, out
        torch.cuda.empty_cache()
        big = ccl.random_image_device(32768, 32768, 0.5, 0, device=lrank)
        lab1 = torch.empty((32768, 32768), dtype=torch.uint32, device=dev)
        ms1 = timer.run(lambda: ccl.label_device(big, lab1, stream=stream, ctx=ctx), 5, 3)
        extra["n1_value"] = 32768 * 32768 / (ms1 * 1e-3) / 1e9
        extra["n1_ms_per_step"] = ms1
        del big, lab1
        torch.cuda.empty_cache()

    line = None
    if rank == 0:
        if kern:
            achieved = 1 * px_step / (kern["local_ms"] * 1e-3) / 1e9
            roof = {"bound": "hbm", "kernel": "k_local_band (a)-(c)", "achieved": achieved, "peak": peak,
                    "unit": "GB/s", "frac": achieved / peak, "traffic": traffic_from_profiles("local_ms"),
                    "peak_source": peak_src, "algorithmic_bytes_per_launch": px_step,
                    "bytes_per_px": 1}
        else:
            roof = None
        per_gpu_px = px_step / (ws if scaling == "strong" else 1)
        path_achieved = per_gpu_px * BYTES_PER_PX / (mean_ms * 1e-3) / 1e9
        line = {"metric": metric, "value": value, "unit": "Gpixels/s", "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": mean_ms, "higher_is_better": True, "scaling": scaling,
                "vs_baseline": None, "dtype": "u32", "data": DATA,
                "config": dict(cfg, l2_flush="1 GiB read between timed steps",
                               parallelism="single GPU" if ws == 1 else f"{ws} GPUs, one process each"),
                "roofline": roof,
                "roofline_path": {"bound": "hbm", "achieved": path_achieved, "peak": peak, "unit": "GB/s",
                                  "frac": path_achieved / peak, "bytes_per_px": BYTES_PER_PX,
                                  "note": "per GPU: 5 B/px x pixels per GPU / step time"},
                "kernels_ms": kern, "gpu_launches": launches_per_step * args.steps, "clocks": clocks}
        line.update(extra)
        if workload == "random8192":
            line["e2e"] = e2e_host_api(ccl, img_np, args)
            if not args.no_cpu_baseline:
                line["cpu_baseline"] = cpu_baseline(img_np)
            if not args.no_configs:
                line["configs"] = measure_configs(ccl, timer, ctx, dev, stream, cpu=not args.no_cpu_baseline)
                if not args.no_cpu_baseline:
                    line["configs"]["4_batch1080"]["cpu_baseline"] = cpu_baseline_batch()
    if workload != "random8192":  # e2e through the host API on every rank, max over ranks
        e2e = e2e_distributed(ccl, workload, args, ctx, dev, rank, ws, lab if workload == "strips32768" else None,
                              frames if workload == "batch1080" else None, stream)
        if line:
            line["e2e"] = e2e
    if ws > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    if line:
        print(json.dumps(line), flush=True)


def measure_single(ccl, timer, ctx, dev, stream, workload, args):
    import torch
    steps, warmup = args.steps, args.warmup

    def one(img, w, h):
        lab = torch.empty((h, w), dtype=torch.uint32, device=dev)
        ms = timer.run(lambda: ccl.label_device(img, lab, stream=stream, ctx=ctx), steps, warmup)
        return {"ms": ms, "gpx_s": w * h / (ms * 1e-3) / 1e9}

    if workload == "parity512":
        return one(ccl.random_image_device(512, 512, 0.5, 0, device=dev.index), 512, 512)
    if workload == "sweep2048":
        return {f"d{d:.1f}": one(ccl.random_image_device(2048, 2048, d, 0, device=dev.index), 2048, 2048)
                for d in SWEEP}
    return {k: one(torch.from_numpy(ccl.pattern_image(k, 8192, 8192)).to(dev), 8192, 8192) for k in PATTERNS}


def e2e_distributed(ccl, workload, args, ctx, dev, rank, ws, lab, frames, stream):
    """Strips / batch end to end: every rank uploads its share from page-locked
    host memory, labels it and downloads its labels each step (wall clock on
    each rank, max over ranks)."""
    import torch
    if workload == "strips32768":
        h_img = torch.empty((lab.h, 32768), dtype=torch.uint8, pin_memory=True)
        h_img.copy_(ccl.random_image_device(32768, lab.h, 0.5, 0, row0=lab.row0, device=dev.index).cpu())
        h_out = torch.empty((lab.h, 32768), dtype=torch.int32, pin_memory=True)
        d_img = torch.empty((lab.h, 32768), dtype=torch.uint8, device=dev)
        d_out = torch.empty((lab.h, 32768), dtype=torch.int32, device=dev)
        px_total = 32768 * 32768
        bi, bo = h_img.numel(), h_out.numel() * 4

        def step():
            with torch.cuda.stream(stream):
                d_img.copy_(h_img, non_blocking=True)
                lab.label(d_img, d_out, stream=stream)
                h_out.copy_(d_out, non_blocking=True)
            stream.synchronize()
        api = "StripLabeler.label (ccl_strip_group_label) with the rank's rows H2D before and labels D2H after"
    else:
        per = frames.shape[0]
        h_img = frames.cpu().pin_memory()
        h_out = torch.empty(tuple(frames.shape), dtype=torch.int32, pin_memory=True)
        d_out = torch.empty(tuple(frames.shape), dtype=torch.int32, device=dev)
        d_img = torch.empty_like(frames)
        px_total = 1024 * 1920 * 1080
        bi, bo = h_img.numel(), h_out.numel() * 4

        def step():
            with torch.cuda.stream(stream):
                d_img.copy_(h_img, non_blocking=True)
                ccl.label_batch_device(d_img, d_out.view(torch.uint32), stream=stream, ctx=ctx)
                h_out.copy_(d_out, non_blocking=True)
            stream.synchronize()
        api = f"label_batch_device on the rank's {per} frames, H2D before and D2H after (page-locked)"
    for _ in range(2):
        step()
    if ws > 1:
        torch.distributed.barrier()
    n = 3
    t0 = time.perf_counter()
    for _ in range(n):
        step()
    s = _max_over_ranks((time.perf_counter() - t0) / n, ws, dev)
    return {"value": px_total / s / 1e9, "unit": "Gpixels/s", "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo,
            "ms_per_step": s * 1e3, "api": api, "note": "bytes per rank per step; value over all ranks"}


if __name__ == "__main__":
    main()
