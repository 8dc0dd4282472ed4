"""north_star configs 4 and 5 at full size, through the batch and strip paths
(SURVEY §8(e)), against the reference's own known answers
(tests/golden/known_answers.json, made by tests/golden/make_golden.py from
ccl_ref::sequential_ccl, proj/src/oracle.cpp:34-50).

* config 4: 1024 frames of random_image(1920, 1080, 0.5, s), s = 0..1023,
  labeled through label_batch_device in per-GPU shares (1024/N frames per GPU
  for N = 1, 2, 4, 8 -- the frame split bench.py uses); the XOR of the
  per-frame FNV-1a-64 hashes, sum K and sum fg must match.
* config 5: random_image(32768, 32768, 0.5, 0) split in N strips of 32768/N
  rows (N = 2, 4, 8) through the strip protocol (virtual strips on one GPU,
  the same kernels and seam exchange as the multi-GPU path) and through the
  host API ccl_label_strips; FNV, K and fg must match the single-image answer.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ccl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1712_09789_b200 as ccl
    return ccl


def _hash_frames(oracle_mod, lab_dev):
    """(sum K, sum fg, XOR of FNV) of a (F, H, W) device label tensor."""
    sk = sfg = 0
    x = 0
    host = lab_dev.cpu().numpy().view(np.uint32)
    for f in range(host.shape[0]):
        k, fg = oracle_mod.count(host[f])
        sk += k
        sfg += fg
        x ^= oracle_mod.fnv1a64(host[f])
    return sk, sfg, x


def test_config4_batch_1024_frames(ccl, oracle_mod, known_answers):
    import torch
    ka = known_answers["batch_1920x1080x1024_d0.5_seeds0-1023"]
    w, h, nf = 1920, 1080, 1024
    chunk = 128  # one per-GPU share at N = 8
    frames = torch.empty((chunk, h, w), dtype=torch.uint8, device="cuda")
    out = torch.empty((chunk, h, w), dtype=torch.uint32, device="cuda")
    sk = sfg = x = 0
    for f0 in range(0, nf, chunk):
        for j in range(chunk):
            ccl.random_image_device(w, h, 0.5, f0 + j, out=frames[j])
        ccl.label_batch_device(frames, out=out)
        k, fg, hx = _hash_frames(oracle_mod, out)
        sk, sfg, x = sk + k, sfg + fg, x ^ hx
    assert (sk, sfg) == (ka["K"], ka["fg"])
    assert f"{x:016x}" == ka["fnv1a64_raw_xor"]


@pytest.mark.parametrize("share", [1024, 512, 256])
def test_config4_batch_shares(ccl, oracle_mod, known_answers, share):
    """The first per-GPU share at N = 1, 2, 4 in ONE batched launch per
    kernel; every frame equals the per-frame answer of a 2-frame batch."""
    import torch
    w, h = 1920, 1080
    frames = torch.empty((share, h, w), dtype=torch.uint8, device="cuda")
    for j in range(share):
        ccl.random_image_device(w, h, 0.5, j, out=frames[j])
    lab = ccl.label_batch_device(frames)
    del frames
    # frame 0 known answer, and spot frames against the oracle
    k, fg = oracle_mod.count(lab[0].cpu().numpy().view(np.uint32))
    ka = known_answers["frame_1920x1080_d0.5_s0"]
    assert (k, fg) == (ka["K"], ka["fg"])
    for j in (1, share // 2, share - 1):
        want = oracle_mod.sequential_ccl(ccl.random_image(w, h, 0.5, j))
        assert np.array_equal(lab[j].cpu().numpy().view(np.uint32), want), j


@pytest.fixture(scope="module")
def img32768(ccl):
    return ccl.random_image_device(32768, 32768, 0.5, 0)


def _check_32768(oracle_mod, known_answers, lab_host):
    ka = known_answers["random_32768_d0.5_s0"]
    k, fg = oracle_mod.count(lab_host)
    assert (k, fg) == (ka["K"], ka["fg"])
    assert f"{oracle_mod.fnv1a64(lab_host):016x}" == ka["fnv1a64_raw"]


@pytest.mark.parametrize("n", [2, 4, 8])
def test_config5_strips_32768(ccl, oracle_mod, known_answers, img32768, n):
    import torch
    from paper_1712_09789_b200.strips import label_strips_single_gpu
    lab = label_strips_single_gpu(img32768, n)
    torch.cuda.synchronize()
    host = lab.cpu().numpy().view(np.uint32)
    del lab
    _check_32768(oracle_mod, known_answers, host)


def test_config5_label_strips_host_api_32768(ccl, oracle_mod, known_answers, img32768):
    """ccl_label_strips (ccl::label_image_strips) over 8 virtual strips."""
    host_img = img32768.cpu().numpy()
    rep = ccl.label_strips(host_img, [0] * 8)
    _check_32768(oracle_mod, known_answers, rep.label_map.labels)
