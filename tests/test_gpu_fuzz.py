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
