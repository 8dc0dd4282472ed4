"""GPU tests of the batch, strip (virtual multi-GPU), compaction and C++
drop-in paths; bit-exact against the oracle / the reference."""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ccl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1712_09789_b200 as ccl
    return ccl


def test_batch_frames(ccl, oracle_mod):
    import torch
    frames = np.stack([ccl.random_image(500, 300, 0.5, s) for s in range(9)])
    frames[3] = ccl.pattern_image("spiral", 500, 300)
    frames[4] = 1
    frames[5] = 0
    got = ccl.label_batch_device(torch.from_numpy(frames).cuda()).cpu().numpy()
    for f in range(len(frames)):
        assert np.array_equal(got[f], oracle_mod.sequential_ccl(frames[f])), f


def test_batch_1080p_known_answers(ccl, oracle_mod, known_answers):
    import torch
    frames = torch.from_numpy(np.stack([ccl.random_image(1920, 1080, 0.5, s) for s in (0, 1023)])).cuda()
    got = ccl.label_batch_device(frames).cpu().numpy()
    for f, name in enumerate(["frame_1920x1080_d0.5_s0", "frame_1920x1080_d0.5_s1023"]):
        k, fg = oracle_mod.count(got[f])
        assert (k, fg) == (known_answers[name]["K"], known_answers[name]["fg"])
        assert f"{oracle_mod.fnv1a64(got[f]):016x}" == known_answers[name]["fnv1a64_raw"]


@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("kind", ["random", "spiral", "stripes", "blobs", "checkerboard"])
def test_virtual_strips(ccl, oracle_mod, kind, n):
    import torch
    from paper_1712_09789_b200.strips import label_strips_single_gpu
    w, h = 1024, 1024 + 96
    img = ccl.random_image(w, h, 0.55, 3) if kind == "random" else ccl.pattern_image(kind, w, h, period=6)
    got = label_strips_single_gpu(torch.from_numpy(img).cuda(), n).cpu().numpy()
    want = oracle_mod.sequential_ccl(img)
    assert np.array_equal(got, want), (kind, n, int((got != want).sum()))


def test_virtual_strips_odd_width(ccl, oracle_mod):
    import torch
    from paper_1712_09789_b200.strips import label_strips_single_gpu
    for (w, h, n) in [(97, 200, 3), (1, 640, 5), (300, 64, 2), (1003, 300, 4)]:
        img = ccl.random_image(w, h, 0.6, w + h)
        got = label_strips_single_gpu(torch.from_numpy(img).cuda(), n).cpu().numpy()
        assert np.array_equal(got, oracle_mod.sequential_ccl(img)), (w, h, n)


def test_compact_device(ccl, oracle_mod):
    import torch
    for (w, h, d) in [(512, 512, 0.5), (97, 131, 0.3), (1, 1, 1.0), (2048, 2048, 0.7), (1000, 333, 0.05)]:
        img = ccl.random_image(w, h, d, 1)
        raw = ccl.label_device(torch.from_numpy(img).cuda())
        comp, k = ccl.compact_device(raw)
        want, kw = oracle_mod.compact(oracle_mod.sequential_ccl(img))
        assert k == kw
        assert np.array_equal(comp.cpu().numpy(), want)


def test_cpp_dropin(ccl, oracle_mod, tmp_path):
    if not oracle_mod.ref_available():
        pytest.skip("oracle/_ref not available")
    exe = str(tmp_path / "dropin_test")
    lib_dir = os.path.dirname(ccl.lib_path())
    ref_dir = os.path.dirname(oracle_mod.REF_SO)
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(REPO, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(REPO, "tests", "cpp", "dropin_test.cpp"), "-o", exe, "-L", lib_dir, "-lccl_b200",
           "-L", ref_dir, "-lccl_ref", f"-Wl,-rpath,{lib_dir}:{ref_dir}", "-pthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr
