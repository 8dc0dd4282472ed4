"""In-tree build of the native library ``_lib/libccl_b200.so`` (sm_100a only).

Every CUDA and host C++ source under ``csrc/`` is compiled with nvcc
(``-gencode arch=compute_100a,code=sm_100a -lineinfo``) and linked into one
shared library exporting the C-ABI of ``include/ccl_cuda.h`` and the C++ API
of ``include/ccl/*.hpp``.  The .so is git-ignored but lives in the tree, so it
travels to the GPU box with ``gpurun``.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(OUT_DIR, "libccl_b200.so")


def _exp_defs() -> list[str]:
    """Experiment knobs: CCL_TILE=WXxWY and CCL_DEFS="NAME=V,NAME=V" (e.g.
    CCL_DEFS=CCL_JUMP=1,CCL_WAVE=1).  A non-default build gets its own library
    name, so the in-tree default library is never clobbered by an experiment."""
    fl = []
    tile = os.environ.get("CCL_TILE")
    if tile:
        wx, wy = tile.lower().split("x")
        fl += [f"-DCCL_TILE_WX={int(wx)}", f"-DCCL_TILE_WY={int(wy)}"]
    for d in filter(None, os.environ.get("CCL_DEFS", "").split(",")):
        fl.append("-D" + d.strip())
    return fl


def _exp_xflags() -> list[str]:
    """Experiment compiler flags (CCL_XFLAGS="-Xptxas,--allow-expensive-optimizations=true"); tagged as x<hash>."""
    return [f for f in os.environ.get("CCL_XFLAGS", "").split(",") if f]


def exp_tag() -> str:
    t = "_".join(f.replace("-DCCL_", "").replace("=", "").lower() for f in _exp_defs())
    if _exp_xflags():
        import hashlib
        t += ("_" if t else "") + "x" + hashlib.sha1(",".join(_exp_xflags()).encode()).hexdigest()[:6]
    return t


def lib_for_tag(tag: str | None) -> str:
    return LIB if not tag else os.path.join(OUT_DIR, f"libccl_b200_{tag}.so")


OBJ_DIR = os.path.join(REPO, "build", "obj")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[str]:
    out = []
    for root, _, files in os.walk(CSRC):
        for f in sorted(files):
            if f.endswith((".cu", ".cpp")):
                out.append(os.path.join(root, f))
    return sorted(out)


def _flags(extra: list[str] | None = None) -> list[str]:
    fl = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
                 "-I", os.path.join(REPO, "include"), "-I", CSRC]
    fl += _exp_defs() + _exp_xflags()
    return fl + (extra or [])


def _needs(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [src] + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    deps += [os.path.join(REPO, "include", d, f) for d in ("", "ccl")
             for f in os.listdir(os.path.join(REPO, "include", d)) if f.endswith((".h", ".hpp"))]
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    nvcc = _nvcc()
    os.makedirs(OBJ_DIR, exist_ok=True)
    os.makedirs(OUT_DIR, exist_ok=True)
    srcs = sources()
    tag = exp_tag() or "default"
    objs = [os.path.join(OBJ_DIR, os.path.relpath(s, CSRC).replace(os.sep, "__") + f".{tag}.o") for s in srcs]
    jobs = []
    for s, o in zip(srcs, objs):
        if force or _needs(o, s):
            cmd = [nvcc] + _flags(["-Xptxas", "-v"] if verbose else []) + ["-c", s, "-o", o]
            if s.endswith(".cpp"):
                cmd = [nvcc] + _flags() + ["-x", "cu", "-c", s, "-o", o]
            jobs.append(cmd)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for r in ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), jobs):
            if verbose and (r.stdout or r.stderr):
                print(r.stdout + r.stderr, file=sys.stderr)
            if r.returncode != 0:
                raise RuntimeError("nvcc failed:\n" + " ".join(r.args) + "\n" + r.stdout + r.stderr)
    lib = lib_for_tag(exp_tag() or None)
    if force or jobs or not os.path.exists(lib) or any(os.path.getmtime(o) > os.path.getmtime(lib) for o in objs):
        tmp = lib + ".tmp"
        link = [nvcc] + ARCH + ["-shared", "-o", tmp] + objs + ["-lcudart_static", "-lrt", "-lpthread", "-ldl"]
        r = subprocess.run(link, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n" + r.stdout + r.stderr)
        os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
