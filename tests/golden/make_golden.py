"""Generate the committed golden fixtures from the REFERENCE ITSELF.

Run in a container that has /root/reference (oracle/_ref is built from it):

    python tests/golden/make_golden.py            # small fixtures + known answers
    python tests/golden/make_golden.py --big      # also 32768^2 and the 1024-frame batch

Outputs (committed):
  tests/golden/small_cases.npz   — small images (incl. SPEC.md examples, odd
                                    shapes, non-binary bytes) with the raw-root
                                    map produced by the reference
                                    ccl_ref::label_image (pipeline.cpp:11-52)
  tests/golden/known_answers.json — K, foreground count and FNV-1a-64 of the
                                    raw-root map (u32 LE bytes) of the
                                    reference ccl_ref::sequential_ccl
                                    (oracle.cpp:34-50) on the SURVEY.md
                                    Appendix A inputs (reference generators).

The GPU box never runs this script (no /root/reference there); tests read the
committed files only.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import oracle as o  # noqa: E402


def spec_cases():
    """SPEC.md worked examples (as image arrays)."""
    cases = {}
    cases["spec_lshape_4x4"] = np.array([[1, 0, 0, 0], [1, 0, 0, 0], [1, 1, 1, 0], [0, 0, 0, 0]], np.uint8)
    cases["spec_refine_4x4"] = np.array([[1, 1, 0, 0], [0, 1, 0, 1], [0, 1, 1, 1], [0, 0, 0, 1]], np.uint8)
    cases["spec_two_bars_3x2"] = np.array([[1, 0, 1], [1, 0, 1]], np.uint8)
    cases["spec_1x1_fg"] = np.array([[1]], np.uint8)
    cases["spec_1x1_bg"] = np.array([[0]], np.uint8)
    cases["spec_checker_4x4"] = o.ref_pattern_image("checkerboard", 4, 4)
    cases["spec_stripes_p2_h8"] = o.ref_pattern_image("stripes", 8, 8, period=2)
    cases["spec_spiral_64"] = o.ref_pattern_image("spiral", 64, 64)
    cases["spec_allfg_32"] = np.ones((32, 32), np.uint8)
    return cases


def random_cases():
    cases = {}
    rng = np.random.default_rng(1712)
    shapes = [(1, 1), (1, 37), (37, 1), (5, 7), (7, 5), (31, 33), (33, 31), (64, 64), (97, 131), (130, 257),
              (255, 513), (16, 1000), (1000, 16)]
    for i, (h, w) in enumerate(shapes):
        for d in (0.1, 0.5, 0.62, 0.9):
            cases[f"rand_{h}x{w}_d{d}"] = o.ref_random_image(w, h, d, 1000 + i)
    # non-binary bytes: only byte==1 is foreground
    for i, (h, w) in enumerate([(40, 72), (129, 65)]):
        cases[f"bytes_{h}x{w}"] = rng.choice(np.array([0, 1, 2, 255], np.uint8), size=(h, w), p=[.3, .4, .15, .15])
    for kind in ("stripes", "spiral", "blobs", "checkerboard"):
        cases[f"pattern_{kind}_200x300"] = o.ref_pattern_image(kind, 300, 200, period=6 if kind == "stripes" else 2)
    return cases


def known_answers(big: bool):
    items = []
    def add(name, img):
        t = time.time()
        lab = o.ref_sequential_ccl(img)
        k, fg = o.count(lab)
        items.append({"name": name, "h": int(img.shape[0]), "w": int(img.shape[1]), "fg": fg, "K": k,
                      "fnv1a64_raw": f"{o.fnv1a64(lab):016x}"})
        print(name, k, fg, items[-1]["fnv1a64_raw"], f"{time.time() - t:.1f}s", flush=True)

    add("random_512_d0.5_s0", o.ref_random_image(512, 512, 0.5, 0))
    for d10 in range(1, 10):
        d = d10 / 10
        add(f"random_2048_d{d}_s0", o.ref_random_image(2048, 2048, d, 0))
    add("random_8192_d0.5_s0", o.ref_random_image(8192, 8192, 0.5, 0))
    add("blobs_8192_d0.5_s0", o.ref_pattern_image("blobs", 8192, 8192, density=0.5, seed=0))
    add("spiral_8192", o.ref_pattern_image("spiral", 8192, 8192))
    add("stripes_8192_p2", o.ref_pattern_image("stripes", 8192, 8192, period=2))
    add("checkerboard_8192", o.ref_pattern_image("checkerboard", 8192, 8192))
    add("frame_1920x1080_d0.5_s0", o.ref_random_image(1920, 1080, 0.5, 0))
    add("frame_1920x1080_d0.5_s1023", o.ref_random_image(1920, 1080, 0.5, 1023))
    if big:
        xor, sk, sfg = 0, 0, 0
        t = time.time()
        for s in range(1024):
            lab = o.ref_sequential_ccl(o.ref_random_image(1920, 1080, 0.5, s))
            k, fg = o.count(lab)
            xor ^= o.fnv1a64(lab)
            sk += k
            sfg += fg
        items.append({"name": "batch_1920x1080x1024_d0.5_seeds0-1023", "h": 1080, "w": 1920, "frames": 1024,
                      "fg": sfg, "K": sk, "fnv1a64_raw_xor": f"{xor:016x}"})
        print("batch", sk, sfg, f"{xor:016x}", f"{time.time() - t:.1f}s", flush=True)
        add("random_32768_d0.5_s0", o.ref_random_image(32768, 32768, 0.5, 0))
    return items


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    args = ap.parse_args()
    o.build()
    cases = {**spec_cases(), **random_cases()}
    arrays = {}
    for name, img in cases.items():
        img = np.ascontiguousarray(img, np.uint8)
        lab, _ = o.ref_label_image(img, 32, 32, "c2fl", 1)
        seq = o.ref_sequential_ccl(img)
        assert (lab == seq).all(), name
        arrays[f"img__{name}"] = img
        arrays[f"lab__{name}"] = lab
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **arrays)
    print(f"wrote {len(cases)} small cases")
    path = os.path.join(HERE, "known_answers.json")
    old = {}
    if os.path.exists(path):
        old = {d["name"]: d for d in json.load(open(path))["answers"]}
    for it in known_answers(args.big):
        old[it["name"]] = it
    json.dump({"source": "reference ccl_ref::sequential_ccl via oracle/_ref (tests/golden/make_golden.py)",
               "hash": "FNV-1a-64 over raw-root u32 little-endian bytes, offset 0xcbf29ce484222325, prime 0x100000001b3",
               "answers": list(old.values())}, open(path, "w"), indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
