"""Strip mode: one image split into horizontal strips, one strip per GPU/rank.

Protocol (include/ccl_cuda.h, csrc/ccl_aux.cu):
  1. ccl_strip_local         kernels (a)(b)(c)(d) on the strip, labels in
                             GLOBAL raster space (x + (row0 + y) * W)
  2. ccl_strip_seam_export   4*W u32: strip roots of the top/bottom rows and
                             the first seam node carrying each root
  3. exchange               every strip's 4*W words stored into every rank's
                             exchange area over NVLink + device epoch flags
                             (library strip groups, StripLabeler); a device-
                             local concatenation for virtual strips
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


def gather_handles(mine: bytes, world: int, group=None) -> bytes:
    """All ranks' exchange-area handles concatenated in rank order (setup only;
    any torch.distributed backend)."""
    if world == 1:
        return mine
    import torch.distributed as dist
    allh = [None] * world
    dist.all_gather_object(allh, mine, group=group)
    if any(len(h) != len(mine) for h in allh):
        raise RuntimeError("strip group handles differ in size across ranks")
    return b"".join(allh)


class StripLabeler:
    """This rank's strip of an N-GPU strip labeling (one process per GPU).

    The seam exchange runs INSIDE the library (include/ccl_cuda.h strip
    groups): each step stores this rank's 16*W-byte seam export into every
    rank's exchange area over NVLink (areas shared with CUDA IPC handles) and
    waits on device flags -- no host round trip, no torch collective in the
    step.  torch.distributed is used once, at construction, to all-gather the
    IPC handles (any backend; ``group`` selects the process group)."""

    def __init__(self, ctx: Context, w: int, full_h: int, rank: int, world: int, group=None):
        self.ctx, self.w, self.full_h, self.rank, self.world = ctx, w, full_h, rank, world
        hb = int(_lib.ccl_strip_group_handle_bytes())
        handle = ctypes.create_string_buffer(hb)
        g = ctypes.c_void_p()
        _check(_lib.ccl_strip_group_create(ctx.handle, rank, world, w, full_h, ctypes.byref(g), handle))
        self._g = g
        blob = ctypes.create_string_buffer(gather_handles(bytes(handle.raw), world, group), hb * world)
        _check(_lib.ccl_strip_group_connect(g, blob))
        r0, h = ctypes.c_uint32(), ctypes.c_uint32()
        _check(_lib.ccl_strip_group_rows(g, ctypes.byref(r0), ctypes.byref(h)))
        self.row0, self.h = int(r0.value), int(h.value)

    @property
    def launches(self) -> int:
        return int(_lib.ccl_strip_group_launches(self._g))

    def label(self, img, out, variant="c2fl", stream=None):
        """img: (h, W) uint8 CUDA tensor holding rows [row0, row0+h); out: (h, W)
        32-bit tensor, receives GLOBAL raster labels.  Asynchronous on stream."""
        _check(_lib.ccl_strip_group_label(self._g, img.data_ptr(), img.stride(0), out.data_ptr(),
                                          int(Variant.parse(variant)), _stream_ptr(stream)))
        return out

    def close(self):
        if getattr(self, "_g", None):
            _lib.ccl_strip_group_destroy(self._g)
            self._g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


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
