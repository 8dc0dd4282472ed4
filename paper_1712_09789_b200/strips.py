"""Strip mode: one image split into horizontal strips, one strip per GPU/rank.

Protocol (include/ccl_cuda.h, csrc/ccl_aux.cu):
  1. ccl_strip_local         kernels (a)(b)(c)(d) on the strip, labels in
                             GLOBAL raster space (x + (row0 + y) * W)
  2. ccl_strip_seam_export   4*W u32: strip roots of the top/bottom rows and
                             the first seam node carrying each root
  3. all-gather              NCCL all_gather_into_tensor of every strip's 4*W
                             words (the only cross-GPU traffic: 16*W bytes/GPU)
  4. ccl_strip_seam_resolve  identical union-find over all seam nodes on every
                             rank, then each rank writes its seam roots' final
                             labels into its own forest
  5. ccl_strip_final         kernel (e)

Every strip except the last must have a height that is a multiple of the tile
height (``split_rows`` produces such a split).
"""
from __future__ import annotations

import ctypes

from . import _check, _lib, _stream_ptr, Context, Variant, tile_shape


def split_rows(full_h: int, n: int) -> list[tuple[int, int]]:
    """(row0, h) per strip: near-equal heights, all but the last a multiple of the tile height."""
    th = tile_shape()[1]
    tiles = -(-full_h // th)
    out, r0 = [], 0
    for k in range(n):
        t = tiles // n + (1 if k < tiles % n else 0)
        h = min(t * th, full_h - r0) if k < n - 1 else full_h - r0
        out.append((r0, h))
        r0 += h
    if any(h <= 0 for _, h in out):
        raise ValueError(f"image of {full_h} rows too small for {n} strips")
    return out


def exchange_seams(seam_local, world: int, group=None):
    """All-gather every strip's 4*W seam words (works for NCCL and gloo tensors)."""
    import torch
    import torch.distributed as dist
    flat = seam_local.reshape(-1)
    out = torch.empty(world * flat.numel(), dtype=seam_local.dtype, device=seam_local.device)
    dist.all_gather_into_tensor(out, flat, group=group)
    return out.view((world,) + tuple(seam_local.shape))


class StripLabeler:
    """Labels this rank's strip; the seam exchange runs over torch.distributed."""

    def __init__(self, ctx: Context, w: int, h: int, row0: int, full_h: int, rank: int, world: int, device,
                 group=None):
        import torch
        self.ctx, self.w, self.h, self.row0, self.full_h = ctx, w, h, row0, full_h
        self.rank, self.world, self.group = rank, world, group
        self.seam = torch.empty(4 * w, dtype=torch.int32, device=device)
        self.scratch = torch.empty(int(_lib.ccl_strip_scratch_words(world, w)), dtype=torch.int32, device=device)
        self.work = torch.zeros(int(_lib.ccl_work_bytes(w, h, 1)), dtype=torch.uint8, device=device)

    def label(self, img, out, variant="c2fl", stream=None):
        import torch
        v = int(Variant.parse(variant))
        s = _stream_ptr(stream)
        c = self.ctx.handle
        _check(_lib.ccl_strip_local(c, img.data_ptr(), img.stride(0), self.w, self.h, self.row0, self.full_h,
                                    out.data_ptr(), self.work.data_ptr(), v, s))
        _check(_lib.ccl_strip_seam_export(c, self.w, self.h, self.row0, self.full_h, self.rank, out.data_ptr(),
                                          self.work.data_ptr(), self.seam.data_ptr(), s))
        if stream is not None and not isinstance(stream, int):
            with torch.cuda.stream(stream):
                allseams = exchange_seams(self.seam, self.world, self.group)
        else:
            allseams = exchange_seams(self.seam, self.world, self.group)
            if stream is not None:  # raw stream handle: keep the gather alive until it has run
                torch.cuda.current_stream().synchronize()
        _check(_lib.ccl_strip_seam_resolve(c, allseams.data_ptr(), self.world, self.rank, self.w, self.h, self.row0,
                                           self.full_h, out.data_ptr(), self.work.data_ptr(), self.scratch.data_ptr(),
                                           s))
        _check(_lib.ccl_strip_final(c, self.w, self.h, self.row0, self.full_h, out.data_ptr(), self.work.data_ptr(),
                                    v, s))
        return out


def label_strips_single_gpu(img, n_strips: int, variant="c2fl", stream=None, ctx: Context | None = None):
    """Run the strip protocol with ``n_strips`` virtual strips on one device.

    Same kernels as the multi-GPU path; the all-gather is a device-local
    concatenation.  Returns the (H, W) uint32 global label map."""
    import torch
    from . import _ctx
    if stream is not None and not isinstance(stream, int):
        # temporaries are allocated on (and freed back to) the stream the
        # kernels run on, so the caching allocator cannot hand them out early
        with torch.cuda.stream(stream):
            return label_strips_single_gpu(img, n_strips, variant, None, ctx)
    h_full, w = img.shape
    ctx = ctx or _ctx(img.device.index or 0)
    v = int(Variant.parse(variant))
    s = _stream_ptr(stream)
    out = torch.empty((h_full, w), dtype=torch.uint32, device=img.device)
    parts = split_rows(h_full, n_strips)
    seams = torch.empty((n_strips, 4 * w), dtype=torch.int32, device=img.device)
    scratch = torch.empty(int(_lib.ccl_strip_scratch_words(n_strips, w)), dtype=torch.int32, device=img.device)
    views = []
    for k, (r0, h) in enumerate(parts):
        im, lo = img[r0:r0 + h], out[r0:r0 + h]
        wk = torch.zeros(int(_lib.ccl_work_bytes(w, h, 1)), dtype=torch.uint8, device=img.device)
        views.append((im, lo, r0, h, wk))
        _check(_lib.ccl_strip_local(ctx.handle, im.data_ptr(), im.stride(0), w, h, r0, h_full, lo.data_ptr(),
                                    wk.data_ptr(), v, s))
        _check(_lib.ccl_strip_seam_export(ctx.handle, w, h, r0, h_full, k, lo.data_ptr(), wk.data_ptr(),
                                          seams[k].data_ptr(), s))
    for k, (im, lo, r0, h, wk) in enumerate(views):
        _check(_lib.ccl_strip_seam_resolve(ctx.handle, seams.data_ptr(), n_strips, k, w, h, r0, h_full, lo.data_ptr(),
                                           wk.data_ptr(), scratch.data_ptr(), s))
    for k, (im, lo, r0, h, wk) in enumerate(views):
        _check(_lib.ccl_strip_final(ctx.handle, w, h, r0, h_full, lo.data_ptr(), wk.data_ptr(), v, s))
    return out
