"""Randomised GPU parity (hypothesis): arbitrary shapes, densities, byte
values, variants and row pitches through the C-ABI, bit-exact against the
oracle (the reference's canonical raw-root map, oracle.cpp:34-50)."""
import os
import numpy as np
import pytest

hypothesis = pytest.importorskip("hypothesis")
from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

VARIANTS = ["c2fl", "rc2fl", "cc2fl", "nc2fl"]


@pytest.mark.gpu
@settings(max_examples=int(os.environ.get("CCL_FUZZ_EXAMPLES", "300")), deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(w=st.integers(1, 700), h=st.integers(1, 300), density=st.floats(0.0, 1.0), seed=st.integers(0, 2**31),
       variant=st.sampled_from(VARIANTS), junk=st.booleans(), pad=st.integers(0, 37))
def test_random_images(ccl, oracle_mod, w, h, density, seed, variant, junk, pad):
    import torch
    rng = np.random.default_rng(seed)
    img = (rng.random((h, w)) < density).astype(np.uint8)
    if junk:  # non-binary bytes are background (foreground iff byte == 1)
        img = np.where(rng.random((h, w)) < 0.2, rng.choice(np.array([0, 2, 3, 255], np.uint8), (h, w)), img)
    want = oracle_mod.sequential_ccl(img)
    buf = torch.zeros((h, w + pad), dtype=torch.uint8)  # pitch w+pad (unaligned pitches take the generic loads)
    buf[:, :w] = torch.from_numpy(img)
    got, _ = ccl.label_device(buf.cuda()[:, :w], variant=variant, sync=True)
    assert np.array_equal(got.cpu().numpy(), want)


@pytest.mark.gpu
@settings(max_examples=int(os.environ.get("CCL_FUZZ_EXAMPLES_MODES", "60")), deadline=None,
          suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(w=st.integers(1, 600), h=st.integers(1, 400), n=st.integers(1, 6), density=st.floats(0.3, 0.8),
       seed=st.integers(0, 2**31), kind=st.sampled_from(["random", "spiral", "stripes", "blobs"]))
def test_random_strips(ccl, oracle_mod, w, h, n, density, seed, kind):
    """The strip protocol (virtual strips on one GPU: kernels (a)-(d) per strip,
    seam export, the exchange layout, seam union-find, (d2)+(e)) on random
    shapes and strip counts."""
    import torch
    from paper_1712_09789_b200.strips import label_strips_single_gpu
    th = ccl.tile_shape()[1]
    n = max(1, min(n, -(-h // th)))  # every strip but the last is a whole number of tile rows
    img = ccl.random_image(w, h, density, seed) if kind == "random" else ccl.pattern_image(kind, w, h, period=3)
    got = label_strips_single_gpu(torch.from_numpy(img).cuda(), n).cpu().numpy()
    assert np.array_equal(got, oracle_mod.sequential_ccl(img))


@pytest.mark.gpu
@settings(max_examples=int(os.environ.get("CCL_FUZZ_EXAMPLES_MODES", "60")), deadline=None,
          suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(w=st.integers(1, 300), h=st.integers(1, 200), frames=st.integers(1, 40), chunk_tiles=st.integers(1, 64),
       seed=st.integers(0, 2**31))
def test_random_batches(ccl, oracle_mod, monkeypatch, w, h, frames, chunk_tiles, seed):
    """ccl_label_batch on random frame shapes and counts, pipelined in chunks
    of random size (CCL_PIPE_TILES) or as one launch when too few frames."""
    import torch
    monkeypatch.setenv("CCL_PIPE_TILES", str(chunk_tiles))
    rng = np.random.default_rng(seed)
    dens = rng.random(frames)
    batch = np.stack([(rng.random((h, w)) < d).astype(np.uint8) for d in dens])
    got = ccl.label_batch_device(torch.from_numpy(batch).cuda()).cpu().numpy()
    for f in range(frames):
        assert np.array_equal(got[f], oracle_mod.sequential_ccl(batch[f])), f
