"""TEST INFRASTRUCTURE ONLY — the parity checker, never the product.

ctypes bindings for
  * ``_build/libccl_oracle.so`` — the plain-C restatement in ``ccl_oracle.c``
  * ``_ref/libccl_ref.so``      — the unmodified reference CPU labeler compiled
                                   from /root/reference (see ``Makefile``)

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  The product
(``paper_1712_09789_b200``) never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(_HERE, "_build", "libccl_oracle.so")
REF_SO = os.path.join(_HERE, "_ref", "libccl_ref.so")
BG = 0xFFFFFFFF

PATTERNS = {"stripes": 0, "spiral": 1, "blobs": 2, "checkerboard": 3}
VARIANTS = {"c2fl": 0, "rc2fl": 1, "cc2fl": 2, "nc2fl": 3}

_u8p = ctypes.POINTER(ctypes.c_uint8)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_u64p = ctypes.POINTER(ctypes.c_uint64)


def build() -> None:
    """Compile the oracle (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def _p8(a):
    return a.ctypes.data_as(_u8p)


def _p32(a):
    return a.ctypes.data_as(_u32p)


_orc = None
_ref = None


def _load_oracle():
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            build()
        lib = ctypes.CDLL(ORACLE_SO)
        lib.orc_random_image.argtypes = [_u8p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_double, ctypes.c_uint64]
        lib.orc_random_image.restype = ctypes.c_int
        lib.orc_pattern_image.argtypes = [_u8p, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                          ctypes.c_double, ctypes.c_uint64]
        lib.orc_pattern_image.restype = ctypes.c_int
        lib.orc_sequential_ccl.argtypes = [_u8p, ctypes.c_uint32, ctypes.c_uint32, _u32p]
        lib.orc_sequential_ccl.restype = None
        lib.orc_label_blocks.argtypes = [_u8p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                         ctypes.c_int, _u32p]
        lib.orc_label_blocks.restype = ctypes.c_int
        lib.orc_compact.argtypes = [_u32p, ctypes.c_uint64, _u32p]
        lib.orc_compact.restype = ctypes.c_uint32
        lib.orc_count.argtypes = [_u32p, ctypes.c_uint64, _u64p, _u64p]
        lib.orc_count.restype = None
        lib.orc_fnv1a64_u32.argtypes = [_u32p, ctypes.c_uint64]
        lib.orc_fnv1a64_u32.restype = ctypes.c_uint64
        _orc = lib
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _load_ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} missing (build oracle/ in a container with /root/reference)")
        lib = ctypes.CDLL(REF_SO)
        lib.ref_random_image.argtypes = [_u8p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_double, ctypes.c_uint64]
        lib.ref_random_image.restype = ctypes.c_int
        lib.ref_pattern_image.argtypes = [_u8p, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                          ctypes.c_double, ctypes.c_uint64]
        lib.ref_pattern_image.restype = ctypes.c_int
        lib.ref_label_image.argtypes = [_u8p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                        ctypes.c_int, ctypes.c_uint, _u32p, ctypes.POINTER(ctypes.c_double)]
        lib.ref_label_image.restype = ctypes.c_int
        lib.ref_sequential_ccl.argtypes = [_u8p, ctypes.c_uint32, ctypes.c_uint32, _u32p]
        lib.ref_sequential_ccl.restype = ctypes.c_int
        lib.ref_write_label_map.argtypes = [_u32p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_char_p]
        lib.ref_write_label_map.restype = ctypes.c_int
        lib.ref_hardware_concurrency.argtypes = []
        lib.ref_hardware_concurrency.restype = ctypes.c_uint
        _ref = lib
    return _ref


# ---------------------------------------------------------------- oracle port
def random_image(w: int, h: int, density: float, seed: int) -> np.ndarray:
    out = np.empty((h, w), dtype=np.uint8)
    if _load_oracle().orc_random_image(_p8(out), w, h, density, seed) != 0:
        raise ValueError("density must be in [0, 1]")
    return out


def pattern_image(kind: str, w: int, h: int, period: int = 2, density: float = 0.5, seed: int = 0) -> np.ndarray:
    out = np.empty((h, w), dtype=np.uint8)
    if _load_oracle().orc_pattern_image(_p8(out), PATTERNS[kind], w, h, period, density, seed) != 0:
        raise ValueError(f"bad pattern parameters for {kind}")
    return out


def sequential_ccl(img: np.ndarray) -> np.ndarray:
    img = np.ascontiguousarray(img, dtype=np.uint8)
    h, w = img.shape
    out = np.empty((h, w), dtype=np.uint32)
    _load_oracle().orc_sequential_ccl(_p8(img), w, h, _p32(out))
    return out


def label_blocks(img: np.ndarray, bw: int = 32, bh: int = 32, variant: str = "c2fl") -> np.ndarray:
    img = np.ascontiguousarray(img, dtype=np.uint8)
    h, w = img.shape
    out = np.empty((h, w), dtype=np.uint32)
    rc = _load_oracle().orc_label_blocks(_p8(img), w, h, bw, bh, VARIANTS[variant], _p32(out))
    if rc != 0:
        raise ValueError("invalid block config / variant")
    return out


def compact(raw: np.ndarray) -> tuple[np.ndarray, int]:
    raw = np.ascontiguousarray(raw, dtype=np.uint32)
    out = np.empty_like(raw)
    k = _load_oracle().orc_compact(_p32(raw), raw.size, _p32(out))
    return out, int(k)


def count(raw: np.ndarray) -> tuple[int, int]:
    """(K, foreground count) of a raw-root map: K = #{p : labels[p] == p}."""
    raw = np.ascontiguousarray(raw, dtype=np.uint32)
    k = ctypes.c_uint64()
    fg = ctypes.c_uint64()
    _load_oracle().orc_count(_p32(raw), raw.size, ctypes.byref(k), ctypes.byref(fg))
    return int(k.value), int(fg.value)


def fnv1a64(raw: np.ndarray) -> int:
    raw = np.ascontiguousarray(raw, dtype=np.uint32)
    return int(_load_oracle().orc_fnv1a64_u32(_p32(raw), raw.size))


# ------------------------------------------------------------- the reference
def ref_random_image(w: int, h: int, density: float, seed: int) -> np.ndarray:
    out = np.empty((h, w), dtype=np.uint8)
    if _load_ref().ref_random_image(_p8(out), w, h, density, seed) != 0:
        raise ValueError("density must be in [0, 1]")
    return out


def ref_pattern_image(kind: str, w: int, h: int, period: int = 2, density: float = 0.5, seed: int = 0) -> np.ndarray:
    out = np.empty((h, w), dtype=np.uint8)
    if _load_ref().ref_pattern_image(_p8(out), PATTERNS[kind], w, h, period, density, seed) != 0:
        raise ValueError(f"bad pattern parameters for {kind}")
    return out


def ref_label_image(img: np.ndarray, bw: int = 32, bh: int = 32, variant: str = "c2fl",
                    workers: int = 1) -> tuple[np.ndarray, float]:
    """The reference ``ccl::label_image`` (pipeline.cpp:11-52); returns (raw map, wall_ms)."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    h, w = img.shape
    out = np.empty((h, w), dtype=np.uint32)
    ms = ctypes.c_double()
    rc = _load_ref().ref_label_image(_p8(img), w, h, bw, bh, VARIANTS[variant], workers, _p32(out), ctypes.byref(ms))
    if rc == -1:
        raise ValueError("invalid argument (reference label_image)")
    if rc != 0:
        raise RuntimeError("reference label_image failed")
    return out, float(ms.value)


def ref_sequential_ccl(img: np.ndarray) -> np.ndarray:
    img = np.ascontiguousarray(img, dtype=np.uint8)
    h, w = img.shape
    out = np.empty((h, w), dtype=np.uint32)
    if _load_ref().ref_sequential_ccl(_p8(img), w, h, _p32(out)) != 0:
        raise RuntimeError("reference sequential_ccl failed")
    return out


def ref_write_label_map(labels: np.ndarray, path: str, fmt: str = "raw", compacted: bool = False) -> None:
    """The reference's write_label_map (label_io.cpp:66-76) on a raw or compacted map.
    Only "raw" is safe to call in-process (csv/pgm16 format through iostreams,
    which crash with the libstdc++ state of a Python process)."""
    lab = np.ascontiguousarray(labels, dtype=np.uint32)
    h, w = lab.shape
    rc = _load_ref().ref_write_label_map(_p32(lab), w, h, int(compacted), {"raw": 0, "csv": 1, "pgm16": 2}[fmt],
                                         path.encode())
    if rc != 0:
        raise ValueError("reference write_label_map failed")


def ref_hardware_concurrency() -> int:
    return int(_load_ref().ref_hardware_concurrency())
