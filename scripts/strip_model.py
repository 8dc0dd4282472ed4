"""Per-rank cost of config 5's strip protocol, measured on ONE GPU: for N = 1, 2,
4, 8 strips of random_image(32768, 32768, 0.5, 0), rank k's own kernels --
ccl_strip_local ((a)+(d) on its 32768/N rows), ccl_strip_seam_export,
ccl_strip_seam_resolve (the union-find over all N exports, done redundantly by
every rank) and ccl_strip_final ((d2)+(e)) -- timed with CUDA events (L2
flushed before each), for the middle strip.  The NVLink exchange of the
N x 16 W bytes is not included (a multi-GPU box only).  Prints the projected
whole-image Gpx/s = 32768^2 / max-rank time and the strong-scaling efficiency
against the N = 1 step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1712_09789_b200 as ccl  # noqa: E402
from paper_1712_09789_b200 import _lib, _check, _ctx  # noqa: E402
from paper_1712_09789_b200.strips import split_rows  # noqa: E402

W = H = 32768
img = torch.empty((H, W), dtype=torch.uint8, device="cuda")
ccl.random_image_device(W, H, 0.5, 0, out=img)
out = torch.empty((H, W), dtype=torch.uint32, device="cuda")
fl = torch.ones(1 << 28, dtype=torch.int32, device="cuda")
ctx = _ctx(0)
s = torch.cuda.current_stream().cuda_stream


def ev():
    return torch.cuda.Event(enable_timing=True)


def median(xs):
    xs = sorted(xs)
    return xs[len(xs) // 2]


base = None
for n in (1, 2, 4, 8):
    parts = split_rows(H, n)
    seams = torch.empty((n, 4 * W), dtype=torch.int32, device="cuda")
    scratch = torch.empty(int(_lib.ccl_strip_scratch_words(n, W)), dtype=torch.int32, device="cuda")
    works = [torch.zeros(int(_lib.ccl_work_bytes(W, h, 1)), dtype=torch.uint8, device="cuda") for _, h in parts]
    k = n // 2
    r0k, hk = parts[k]
    times = {"local": [], "export": [], "resolve": [], "final": []}
    for rep in range(6):
        # every strip's phase 1 (the exports rank k needs), then rank k's phases timed
        for j, (r0, h) in enumerate(parts):
            im, lo = img[r0:r0 + h], out[r0:r0 + h]
            if j == k:
                fl.sum()
                e = [ev() for _ in range(3)]
                e[0].record()
            _check(_lib.ccl_strip_local(ctx.handle, im.data_ptr(), im.stride(0), W, h, r0, H, lo.data_ptr(),
                                        works[j].data_ptr(), 0, s))
            if j == k:
                e[1].record()
            _check(_lib.ccl_strip_seam_export(ctx.handle, W, h, r0, H, j, lo.data_ptr(), works[j].data_ptr(),
                                              seams[j].data_ptr(), s))
            if j == k:
                e[2].record()
                torch.cuda.synchronize()
                if rep:
                    times["local"].append(e[0].elapsed_time(e[1]))
                    times["export"].append(e[1].elapsed_time(e[2]))
        lo = out[r0k:r0k + hk]
        fl.sum()
        e = [ev() for _ in range(3)]
        e[0].record()
        _check(_lib.ccl_strip_seam_resolve(ctx.handle, seams.data_ptr(), n, k, W, hk, r0k, H, lo.data_ptr(),
                                           works[k].data_ptr(), scratch.data_ptr(), s))
        e[1].record()
        _check(_lib.ccl_strip_final(ctx.handle, W, hk, r0k, H, lo.data_ptr(), works[k].data_ptr(), 0, s))
        e[2].record()
        torch.cuda.synchronize()
        if rep:
            times["resolve"].append(e[0].elapsed_time(e[1]))
            times["final"].append(e[1].elapsed_time(e[2]))
    t = {key: median(v) for key, v in times.items()}
    tot = sum(t.values())
    if base is None:
        base = tot
    gpx = W * H / (tot * 1e-3) / 1e9
    eff = base / (n * tot)
    print(f"N={n}: strip {hk} rows  local {t['local']*1e3:7.1f}  export {t['export']*1e3:5.1f}  "
          f"resolve {t['resolve']*1e3:6.1f}  final {t['final']*1e3:7.1f} us  -> rank step {tot*1e3:7.1f} us, "
          f"projected {gpx:7.1f} Gpx/s, efficiency {eff*100:5.1f} % (exchange of {n * 16 * W / 2**20:.1f} MiB not included)",
          flush=True)
