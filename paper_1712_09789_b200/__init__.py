"""B200-native block-based coarse-to-fine connected-components labeler.

Python mirror of the reference's C++ API (``/root/reference/proj/include/ccl``)
over the C-ABI of ``include/ccl_cuda.h`` (library ``_lib/libccl_b200.so``,
sm_100a).  Same names, argument meaning and error behaviour as the reference:

    label_image(img, cfg=BlockConfig(), variant=Variant.C2FL, workers=1) -> RunReport
        pipeline.hpp:33-34 / pipeline.cpp:11-52; ValueError (the reference's
        std::invalid_argument) for an invalid cfg, workers == 0 or a 0x0 image.
    compact_labels(label_map) -> LabelMap          (pipeline.cpp:54-70)
    random_image / pattern_image                   (generate.cpp:9-106)

plus device-resident entry points for torch tensors already in HBM
(``label_device``, ``label_batch_device``, ``compact_device``) and the
multi-GPU strip mode (``strips.label_strip_distributed``).

There is no CPU fallback: importing this package without the built CUDA
library raises ImportError, and every call without an sm_100 device raises
DeviceError.
"""
from __future__ import annotations

import ctypes
import enum
import os
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "BG", "BlockConfig", "Variant", "LabelMap", "RunReport", "DeviceError", "label_image", "compact_labels",
    "random_image", "pattern_image", "label_device", "label_batch_device", "compact_device", "Context",
    "tile_shape", "lib_path", "write_label_map", "read_label_map", "label_to_cclm", "random_image_device",
]

BG = 0xFFFFFFFF
_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("CCL_LIB_PATH") or os.path.join(_HERE, "_lib", "libccl_b200.so")


def lib_path() -> str:
    return _LIB_PATH


if not os.path.exists(_LIB_PATH):
    raise ImportError(
        f"{_LIB_PATH} is missing: build the CUDA library first (python __graft_entry__.py build "
        "or python paper_1712_09789_b200/_build.py). There is no CPU fallback.")

_lib = ctypes.CDLL(_LIB_PATH)
_vp = ctypes.c_void_p
_u8p = ctypes.POINTER(ctypes.c_uint8)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_sz = ctypes.c_size_t
_u32 = ctypes.c_uint32


class _Timing(ctypes.Structure):
    _fields_ = [("local_ms", ctypes.c_float), ("merge_ms", ctypes.c_float), ("final_ms", ctypes.c_float),
                ("total_ms", ctypes.c_float)]


def _sig(name, res, *args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_c = ctypes.c_int
_sig("ccl_ctx_create", _c, _c, ctypes.POINTER(_vp))
_sig("ccl_ctx_destroy", None, _vp)
_sig("ccl_ctx_stream", _vp, _vp)
_sig("ccl_label_device", _c, _vp, _vp, _sz, _u32, _u32, _vp, _c, _vp, _c, ctypes.POINTER(_Timing))
_sig("ccl_label_host", _c, _vp, _u8p, _u32, _u32, _u32p, _c, ctypes.POINTER(ctypes.c_float))
_sig("ccl_label_host_async", _c, _vp, _u8p, _u32, _u32, _u32p, _c)
_sig("ccl_ctx_sync", _c, _vp)
_sig("ccl_label_batch", _c, _vp, _vp, _sz, _sz, _u32, _u32, _u32, _vp, _c, _vp)
_sig("ccl_strip_local", _c, _vp, _vp, _sz, _u32, _u32, _u32, _u32, _vp, _vp, _c, _vp)
_sig("ccl_strip_seam_export", _c, _vp, _u32, _u32, _u32, _u32, _u32, _vp, _vp, _vp, _vp)
_sig("ccl_strip_seam_resolve", _c, _vp, _vp, _u32, _u32, _u32, _u32, _u32, _u32, _vp, _vp, _vp, _vp)
_sig("ccl_strip_final", _c, _vp, _u32, _u32, _u32, _u32, _vp, _vp, _c, _vp)
_sig("ccl_strip_scratch_words", _sz, _u32, _u32)
_sig("ccl_gen_random_device", _c, _vp, _vp, _u32, _u32, _u32, ctypes.c_double, ctypes.c_uint64, _vp)
_sig("ccl_label_to_cclm", _c, _vp, _u8p, _u32, _u32, _c, ctypes.c_char_p, ctypes.POINTER(ctypes.c_uint64))
_sig("ccl_write_label_map", _c, _u32p, _u32, _u32, _c, _c, ctypes.c_char_p)
_sig("ccl_read_label_map", _c, ctypes.c_char_p, _u32p, _sz, _u32p, _u32p)
_sig("ccl_io_last_error", ctypes.c_char_p)
_sig("ccl_work_bytes", _sz, _u32, _u32, _u32)
_sig("ccl_compact_device", _c, _vp, _vp, _u32, _u32, _vp, _vp, ctypes.POINTER(ctypes.c_uint64), _vp)
_sig("ccl_compact_scratch_words", _sz, _u32, _u32)
_sig("ccl_tile_shape", None, _u32p, _u32p)
_sig("ccl_launches_per_label", _c)
_sig("ccl_metrics_build", _c)
_sig("ccl_strip_group_handle_bytes", _sz)
_sig("ccl_strip_group_create", _c, _vp, _u32, _u32, _u32, _u32, ctypes.POINTER(_vp), ctypes.c_char_p)
_sig("ccl_strip_group_connect", _c, _vp, ctypes.c_char_p)
_sig("ccl_strip_group_rows", _c, _vp, _u32p, _u32p)
_sig("ccl_strip_group_label", _c, _vp, _vp, _sz, _vp, _c, _vp)
_sig("ccl_strip_group_launches", _c, _vp)
_sig("ccl_strip_group_destroy", None, _vp)
_sig("ccl_release_caches", None)
_sig("ccl_label_strips", _c, ctypes.POINTER(_c), _c, _u8p, _u32, _u32, _u32p, _c, ctypes.POINTER(ctypes.c_float))
_sig("ccl_read_metrics", _c, _vp, _u32p, _u32p, _sz, ctypes.POINTER(ctypes.c_uint64), _u32p, _u32p, _u32p)
_sig("ccl_gen_random", _c, _u8p, _u32, _u32, ctypes.c_double, ctypes.c_uint64)
_sig("ccl_gen_pattern", _c, _u8p, _c, _u32, _u32, _u32, ctypes.c_double, ctypes.c_uint64)
_sig("ccl_last_error", ctypes.c_char_p)
_sig("ccl_version", ctypes.c_char_p)

C_ABI_SYMBOLS = [
    "ccl_ctx_create", "ccl_ctx_destroy", "ccl_ctx_stream", "ccl_label_device", "ccl_label_host", "ccl_label_batch",
    "ccl_label_host_async", "ccl_ctx_sync",
    "ccl_gen_random_device", "ccl_label_to_cclm", "ccl_write_label_map", "ccl_read_label_map", "ccl_io_last_error",
    "ccl_strip_local", "ccl_strip_seam_export", "ccl_strip_seam_resolve", "ccl_strip_final",
    "ccl_strip_scratch_words", "ccl_work_bytes", "ccl_compact_device", "ccl_compact_scratch_words", "ccl_tile_shape",
    "ccl_launches_per_label", "ccl_label_strips", "ccl_strip_group_handle_bytes", "ccl_strip_group_create",
    "ccl_strip_group_connect", "ccl_strip_group_rows", "ccl_strip_group_label", "ccl_strip_group_launches",
    "ccl_strip_group_destroy", "ccl_release_caches", "ccl_metrics_build", "ccl_read_metrics", "ccl_gen_random", "ccl_gen_pattern", "ccl_last_error", "ccl_version",
]

_EINVAL, _ENOMEM, _ECUDA, _ENODEV = 1, 2, 3, 4


class DeviceError(RuntimeError):
    """A CUDA failure below the C-ABI (the C++ API's ccl::DeviceError)."""

    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


def _check(status: int) -> None:
    if status == 0:
        return
    msg = (_lib.ccl_last_error() or b"").decode()
    if status == _EINVAL:
        raise ValueError(msg)
    raise DeviceError(status, msg)


def tile_shape() -> tuple[int, int]:
    w, h = _u32(), _u32()
    _lib.ccl_tile_shape(ctypes.byref(w), ctypes.byref(h))
    return int(w.value), int(h.value)


def launches_per_label() -> int:
    return int(_lib.ccl_launches_per_label())


# --------------------------------------------------------------------- types
class Variant(enum.IntEnum):
    """image.hpp:68-73; output-invariant, selects the kernel's local strategy."""
    C2FL = 0
    RC2FL = 1
    CC2FL = 2
    NC2FL = 3

    @staticmethod
    def parse(s: "str | Variant | int") -> "Variant":
        if isinstance(s, Variant):
            return s
        if isinstance(s, int):
            return Variant(s)
        try:
            return Variant[s.upper()]
        except KeyError:
            raise ValueError(f"unknown variant: {s}") from None


@dataclass
class BlockConfig:
    """image.hpp:55-66 (validated; the GPU tile is internal)."""
    block_w: int = 32
    block_h: int = 32
    slot_ceiling: int = 4096

    def slots(self) -> int:
        return self.block_w * self.block_h

    def valid(self) -> bool:
        return self.block_w >= 1 and self.block_h >= 1 and self.slots() <= self.slot_ceiling


@dataclass
class LabelMap:
    width: int
    height: int
    labels: np.ndarray  # (H, W) uint32
    compacted: bool = False


@dataclass
class BlockMetrics:
    block_id: int = 0
    findroot_iterations: int = 0
    atomic_ops: int = 0


@dataclass
class RunReport:
    """pipeline.hpp:15-26.  wall_time_ms = CUDA-event device time of the kernels."""
    label_map: LabelMap
    blocks_x: int
    blocks_y: int
    wall_time_ms: float
    variant: Variant
    cfg: BlockConfig
    worker_count: int
    per_block: list = field(default_factory=list)
    border_phase: BlockMetrics = field(default_factory=BlockMetrics)
    resolve_phase: BlockMetrics = field(default_factory=BlockMetrics)


# ------------------------------------------------------------------- context
class Context:
    """One ccl_ctx (device, stream, workspace).  Not shared across threads."""

    def __init__(self, device: int = 0):
        h = _vp()
        _check(_lib.ccl_ctx_create(device, ctypes.byref(h)))
        self._h = h
        self.device = device

    @property
    def handle(self):
        return self._h

    @property
    def stream(self) -> int:
        return int(_lib.ccl_ctx_stream(self._h) or 0)

    def close(self):
        if getattr(self, "_h", None):
            _lib.ccl_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


import atexit as _atexit
import threading as _threading

_tls = _threading.local()
_all_ctxs: list = []  # every implicit context, released at interpreter exit


def _ctx(device: int = 0) -> Context:
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
        _all_ctxs.append(ctxs[device])
    return ctxs[device]


@_atexit.register
def _release_contexts():
    _lib.ccl_release_caches()
    for c in _all_ctxs:
        c.close()
    _all_ctxs.clear()


# ------------------------------------------------------------- the drop-in
def _as_image(img) -> np.ndarray:
    a = np.ascontiguousarray(img, dtype=np.uint8)
    if a.ndim != 2:
        raise ValueError("image must be a 2-D (H, W) uint8 array")
    if a.shape[0] == 0 or a.shape[1] == 0:
        raise ValueError("image dimensions must be at least 1x1")
    return a


def label_image(img, cfg: BlockConfig | None = None, variant="c2fl", workers: int = 1,
                device: int = 0) -> RunReport:
    """The reference's ``ccl::label_image`` (pipeline.cpp:11-52) on the GPU."""
    cfg = cfg or BlockConfig()
    if not cfg.valid():
        raise ValueError("block configuration invalid or over the scratch ceiling")
    if workers == 0:
        raise ValueError("workers must be >= 1")
    v = Variant.parse(variant)
    a = _as_image(img)
    h, w = a.shape
    out = np.empty((h, w), dtype=np.uint32)
    ms = ctypes.c_float()
    _check(_lib.ccl_label_host(_ctx(device).handle, a.ctypes.data_as(_u8p), w, h, out.ctypes.data_as(_u32p), int(v),
                               ctypes.byref(ms)))
    bx, by = -(-w // cfg.block_w), -(-h // cfg.block_h)
    rep = RunReport(label_map=LabelMap(w, h, out), blocks_x=bx, blocks_y=by, wall_time_ms=float(ms.value),
                    variant=v, cfg=cfg, worker_count=workers,
                    per_block=[BlockMetrics(block_id=i) for i in range(bx * by)] if bx * by <= 1 << 16 else [])
    if metrics_build():  # instrumented library: counters per GPU tile (see read_metrics)
        m = read_metrics(_ctx(device))
        rep.blocks_x, rep.blocks_y = m["tiles_x"], m["tiles_y"]
        rep.per_block = [BlockMetrics(i, int(f), int(c))
                         for i, (f, c) in enumerate(zip(m["find"].ravel(), m["cas"].ravel()))]
        rep.border_phase = BlockMetrics(0, m["border_find"], m["border_cas"])
        rep.resolve_phase = BlockMetrics(0, m["resolve_find"], 0)
    return rep


def label_strips(img, devices=(0,), variant="c2fl") -> RunReport:
    """``ccl::label_image_strips``: one host image over the listed GPUs of this
    process (horizontal strips, seams exchanged by peer copies; a device may
    repeat), the same label map as ``label_image``."""
    if len(devices) == 0:
        raise ValueError("no devices")
    v = Variant.parse(variant)
    a = _as_image(img)
    h, w = a.shape
    out = np.empty((h, w), dtype=np.uint32)
    ms = ctypes.c_float()
    devs = (_c * len(devices))(*devices)
    _check(_lib.ccl_label_strips(devs, len(devices), a.ctypes.data_as(_u8p), w, h, out.ctypes.data_as(_u32p), int(v),
                                 ctypes.byref(ms)))
    cfg = BlockConfig()
    bx, by = -(-w // cfg.block_w), -(-h // cfg.block_h)
    return RunReport(label_map=LabelMap(w, h, out), blocks_x=bx, blocks_y=by, wall_time_ms=float(ms.value),
                     variant=v, cfg=cfg, worker_count=len(devices))


def metrics_build() -> bool:
    """True when the loaded library is the instrumented build (CCL_METRICS=1)."""
    return bool(_lib.ccl_metrics_build())


def read_metrics(ctx: "Context | None" = None, device: int = 0) -> dict:
    """Counters of the last labeling call on ``ctx`` (instrumented build only;
    reference BlockMetrics, forest.hpp:12-29): per 128x64 tile of kernel (a)
    the parent-link steps of root finding and the CAS attempts of unions
    (arrays shaped (frames, tiles_y, tiles_x)), plus the border-merge and
    resolve totals."""
    c = (ctx or _ctx(device)).handle
    tx, ty, nf = _u32(), _u32(), _u32()
    _check(_lib.ccl_read_metrics(c, None, None, 0, None, ctypes.byref(tx), ctypes.byref(ty), ctypes.byref(nf)))
    n = tx.value * ty.value * nf.value
    f = np.zeros(n, np.uint32)
    a = np.zeros(n, np.uint32)
    ph = (ctypes.c_uint64 * 4)()
    _check(_lib.ccl_read_metrics(c, f.ctypes.data_as(_u32p), a.ctypes.data_as(_u32p), n, ph, ctypes.byref(tx),
                                 ctypes.byref(ty), ctypes.byref(nf)))
    shape = (nf.value, ty.value, tx.value)
    return {"tiles_x": tx.value, "tiles_y": ty.value, "frames": nf.value, "find": f.reshape(shape),
            "cas": a.reshape(shape), "border_find": int(ph[0]), "border_cas": int(ph[1]), "resolve_find": int(ph[2])}


@dataclass
class MetricsSummary:
    """pipeline.hpp MetricsSummary: per-block grids and means."""
    grid_w: int = 0
    grid_h: int = 0
    iterations_grid: list = field(default_factory=list)
    atomics_grid: list = field(default_factory=list)
    mean_iterations: float = 0.0
    mean_atomics: float = 0.0


def aggregate_metrics(report: RunReport) -> MetricsSummary:
    """pipeline.cpp:72-91: grids of the per-block counters and their means."""
    s = MetricsSummary(report.blocks_x, report.blocks_y)
    s.iterations_grid = [m.findroot_iterations for m in report.per_block]
    s.atomics_grid = [m.atomic_ops for m in report.per_block]
    if report.per_block:
        s.mean_iterations = sum(s.iterations_grid) / len(report.per_block)
        s.mean_atomics = sum(s.atomics_grid) / len(report.per_block)
    return s


def compact_labels(lm: LabelMap) -> LabelMap:
    """pipeline.cpp:54-70 for a host label map (GPU version: compact_device)."""
    if lm.compacted:
        return lm
    raw = lm.labels.ravel()
    fg = raw != BG
    roots = np.unique(raw[fg])  # roots are component minima: first appearance == ascending order
    out = np.zeros(raw.shape, dtype=np.uint32)
    out[fg] = np.searchsorted(roots, raw[fg]).astype(np.uint32) + 1
    return LabelMap(lm.width, lm.height, out.reshape(lm.labels.shape), True)


# ---------------------------------------------------------------- label-map files
_FORMATS = {"raw": 0, "csv": 1, "pgm16": 2}


def write_label_map(lm: LabelMap, path: str, fmt: str = "raw") -> None:
    """label_io.cpp:66-76: compact, then write raw CCLM / csv / pgm16 (host only).
    ValueError for an unknown format or an I/O / overflow failure."""
    if fmt not in _FORMATS:
        raise ValueError(f"unknown label map format: {fmt}")
    lab = np.ascontiguousarray(lm.labels, dtype=np.uint32)
    rc = _lib.ccl_write_label_map(lab.ctypes.data_as(_u32p), lm.width, lm.height, int(lm.compacted),
                                  _FORMATS[fmt], os.fsencode(path))
    if rc != 0:
        raise ValueError(_lib.ccl_io_last_error().decode())


def read_label_map(path: str) -> LabelMap:
    """label_io.cpp:78-94: a compacted map from a CCLM file."""
    w, h = _u32(), _u32()
    if _lib.ccl_read_label_map(os.fsencode(path), None, 0, ctypes.byref(w), ctypes.byref(h)) != 0:
        raise ValueError(_lib.ccl_io_last_error().decode())
    out = np.empty((h.value, w.value), dtype=np.uint32)
    if _lib.ccl_read_label_map(os.fsencode(path), out.ctypes.data_as(_u32p), out.size, None, None) != 0:
        raise ValueError(_lib.ccl_io_last_error().decode())
    return LabelMap(w.value, h.value, out, True)


def label_to_cclm(img, path: str, variant="c2fl", device: int = 0) -> int:
    """Label on the GPU, compact on the GPU, stream the CCLM file (device->host
    copies overlap the file writes).  Returns the number of components K."""
    a = _as_image(img)
    k = ctypes.c_uint64()
    _check(_lib.ccl_label_to_cclm(_ctx(device).handle, a.ctypes.data_as(_u8p), a.shape[1], a.shape[0],
                                  int(Variant.parse(variant)), os.fsencode(path), ctypes.byref(k)))
    return int(k.value)


# ---------------------------------------------------------------- generators
_PATTERNS = {"stripes": 0, "spiral": 1, "blobs": 2, "checkerboard": 3}


def random_image(w: int, h: int, density: float, seed: int) -> np.ndarray:
    out = np.empty((h, w), dtype=np.uint8)
    _check(_lib.ccl_gen_random(out.ctypes.data_as(_u8p), w, h, density, seed))
    return out


def random_image_device(w: int, h: int, density: float, seed: int, out=None, stream=None, device: int = 0,
                        row0: int = 0):
    """random_image generated on the GPU (xoshiro256** jump-ahead), byte-identical
    with random_image; rows [row0, row0+h) of a taller image when row0 > 0.
    Returns an (h, w) uint8 torch tensor on the device."""
    torch = _torch()
    if out is None:
        out = torch.empty((h, w), dtype=torch.uint8, device=f"cuda:{device}")
    _check(_lib.ccl_gen_random_device(_ctx(device).handle, out.data_ptr(), w, h, int(row0), float(density), int(seed),
                                      _stream_ptr(stream)))
    return out


def pattern_image(kind: str, w: int, h: int, period: int = 2, density: float = 0.5, seed: int = 0) -> np.ndarray:
    if kind not in _PATTERNS:
        raise ValueError(f"unknown pattern kind: {kind}")
    out = np.empty((h, w), dtype=np.uint8)
    _check(_lib.ccl_gen_pattern(out.ctypes.data_as(_u8p), _PATTERNS[kind], w, h, period, density, seed))
    return out


# ------------------------------------------------------- device (torch) path
def _torch():
    import torch
    return torch


def _stream_ptr(stream) -> int:
    torch = _torch()
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def label_device(img, out=None, variant="c2fl", stream=None, sync: bool = False, ctx: Context | None = None):
    """Label a (H, W) or (H, pitch) uint8 CUDA tensor already in HBM.

    Returns a (H, W) uint32 CUDA tensor (raw-root labels).  Asynchronous on
    ``stream`` (default: torch's current stream) unless ``sync``; with
    ``sync`` returns ``(labels, timing_dict)``.
    """
    torch = _torch()
    if img.dtype != torch.uint8 or img.dim() != 2 or not img.is_cuda:
        raise ValueError("img must be a 2-D uint8 CUDA tensor")
    if img.stride(1) != 1:
        raise ValueError("img rows must be contiguous")
    h, w = img.shape
    pitch = img.stride(0)
    dev = img.device.index or 0
    ctx = ctx or _ctx(dev)
    if out is None:
        out = torch.empty((h, w), dtype=torch.uint32, device=img.device)
    elif out.shape != (h, w) or not out.is_contiguous() or out.element_size() != 4:
        raise ValueError("out must be a contiguous (H, W) 32-bit tensor")
    t = _Timing()
    _check(_lib.ccl_label_device(ctx.handle, img.data_ptr(), pitch, w, h, out.data_ptr(), int(Variant.parse(variant)),
                                 _stream_ptr(stream), 1 if sync else 0, ctypes.byref(t)))
    if sync:
        return out, {"local_ms": t.local_ms, "merge_ms": t.merge_ms, "final_ms": t.final_ms, "total_ms": t.total_ms}
    return out


def label_batch_device(frames, out=None, variant="c2fl", stream=None, ctx: Context | None = None):
    """Label a (F, H, W) uint8 CUDA tensor of frames in one launch per kernel.

    Labels are per-frame raster indices; returns (F, H, W) uint32."""
    torch = _torch()
    if frames.dtype != torch.uint8 or frames.dim() != 3 or not frames.is_cuda or frames.stride(2) != 1:
        raise ValueError("frames must be a (F, H, W) uint8 CUDA tensor with contiguous rows")
    f, h, w = frames.shape
    ctx = ctx or _ctx(frames.device.index or 0)
    if out is None:
        out = torch.empty((f, h, w), dtype=torch.uint32, device=frames.device)
    step = 65535
    for f0 in range(0, f, step):
        n = min(step, f - f0)
        _check(_lib.ccl_label_batch(ctx.handle, frames[f0].data_ptr(), frames.stride(1), frames.stride(0), n, w, h,
                                    out[f0].data_ptr(), int(Variant.parse(variant)), _stream_ptr(stream)))
    return out


def compact_device(raw, out=None, stream=None, ctx: Context | None = None):
    """GPU compaction (pipeline.cpp:54-70): returns (compacted uint32 tensor, K)."""
    torch = _torch()
    h, w = raw.shape
    ctx = ctx or _ctx(raw.device.index or 0)
    if out is None:
        out = torch.empty((h, w), dtype=torch.uint32, device=raw.device)
    scratch = torch.empty(int(_lib.ccl_compact_scratch_words(w, h)), dtype=torch.uint32, device=raw.device)
    k = ctypes.c_uint64()
    _check(_lib.ccl_compact_device(ctx.handle, raw.data_ptr(), w, h, out.data_ptr(), scratch.data_ptr(),
                                   ctypes.byref(k), _stream_ptr(stream)))
    return out, int(k.value)
