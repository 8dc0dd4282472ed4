"""GPU parity: the CUDA path (through the C-ABI) against the oracle and the
reference's own golden outputs.  Bar: bit-exact raw-root label maps."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

VARIANTS = ["c2fl", "rc2fl", "cc2fl", "nc2fl"]


@pytest.fixture(scope="module")
def ccl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1712_09789_b200 as ccl
    return ccl


def _gpu_label(ccl, img, variant="c2fl"):
    return ccl.label_image(img, variant=variant).label_map.labels


def _first_diff(a, b):
    d = np.argwhere(a != b)
    if len(d) == 0:
        return "identical"
    y, x = d[0]
    return f"{len(d)} px differ; first at (x={x}, y={y}): got {a[y, x]:#x} want {b[y, x]:#x}"


@pytest.mark.parametrize("variant", VARIANTS)
def test_golden_small_cases(ccl, small_cases, variant):
    for name, (img, want) in small_cases.items():
        got = _gpu_label(ccl, img, variant)
        assert np.array_equal(got, want), f"{name} [{variant}]: {_first_diff(got, want)}"


def test_known_answers_512_and_sweep(ccl, known_answers, oracle_mod):
    cases = [("random_512_d0.5_s0", 512, 512, 0.5, 0)] + [
        (f"random_2048_d{d / 10}_s0", 2048, 2048, d / 10, 0) for d in range(1, 10)]
    for name, w, h, d, s in cases:
        img = ccl.random_image(w, h, d, s)
        lab = _gpu_label(ccl, img)
        k, fg = oracle_mod.count(lab)
        ka = known_answers[name]
        assert (k, fg) == (ka["K"], ka["fg"]), name
        assert f"{oracle_mod.fnv1a64(lab):016x}" == ka["fnv1a64_raw"], name


@pytest.mark.parametrize("density", [0.05, 0.3, 0.5, 0.593, 0.7, 0.95])
@pytest.mark.parametrize("shape", [(1, 1), (1, 257), (300, 1), (31, 33), (97, 131), (255, 513), (1080, 1920),
                                   (64, 4096), (4096, 48)])
def test_random_vs_oracle(ccl, oracle_mod, density, shape):
    h, w = shape
    img = ccl.random_image(w, h, density, 7 + h * 31 + w)
    want = oracle_mod.sequential_ccl(img)
    for v in VARIANTS:
        got = _gpu_label(ccl, img, v)
        assert np.array_equal(got, want), f"{shape} d={density} {v}: {_first_diff(got, want)}"


def test_non_binary_bytes(ccl, oracle_mod):
    rng = np.random.default_rng(5)
    for shape in [(64, 64), (257, 300), (1000, 1000)]:
        img = rng.choice(np.array([0, 1, 2, 3, 255], np.uint8), size=shape, p=[.3, .4, .1, .1, .1])
        want = oracle_mod.sequential_ccl(img)
        got = _gpu_label(ccl, img)
        assert np.array_equal(got, want), _first_diff(got, want)


@pytest.mark.parametrize("kind", ["stripes", "spiral", "blobs", "checkerboard"])
def test_patterns(ccl, oracle_mod, kind):
    for (w, h) in [(1000, 777), (2048, 2048), (333, 4000)]:
        img = ccl.pattern_image(kind, w, h, period=2 if kind != "stripes" else 6)
        want = oracle_mod.sequential_ccl(img)
        for v in VARIANTS:
            got = _gpu_label(ccl, img, v)
            assert np.array_equal(got, want), f"{kind} {w}x{h} {v}: {_first_diff(got, want)}"


def test_edge_images(ccl, oracle_mod):
    for shape in [(1, 1), (5, 1), (1, 5), (33, 257), (64, 512), (1024, 1024)]:
        for fill in (0, 1):
            img = np.full(shape, fill, np.uint8)
            want = oracle_mod.sequential_ccl(img)
            got = _gpu_label(ccl, img)
            assert np.array_equal(got, want), f"{shape} fill={fill}"


@pytest.mark.slow
@pytest.mark.parametrize("name,kind", [("random_8192_d0.5_s0", "random"), ("blobs_8192_d0.5_s0", "blobs"),
                                       ("spiral_8192", "spiral"), ("stripes_8192_p2", "stripes"),
                                       ("checkerboard_8192", "checkerboard")])
def test_known_answers_8192(ccl, known_answers, oracle_mod, name, kind):
    import torch
    if kind == "random":
        img = ccl.random_image(8192, 8192, 0.5, 0)
    else:
        img = ccl.pattern_image(kind, 8192, 8192, period=2, density=0.5, seed=0)
    d_img = torch.from_numpy(img).cuda()
    lab = ccl.label_device(d_img).cpu().numpy()
    k, fg = oracle_mod.count(lab)
    ka = known_answers[name]
    assert (k, fg) == (ka["K"], ka["fg"]), name
    assert f"{oracle_mod.fnv1a64(lab):016x}" == ka["fnv1a64_raw"], name


def test_device_path_pitched(ccl, oracle_mod):
    import torch
    img = ccl.random_image(1000, 700, 0.55, 3)
    want = oracle_mod.sequential_ccl(img)
    buf = torch.zeros((700, 1024), dtype=torch.uint8, device="cuda")
    buf[:, :1000] = torch.from_numpy(img).cuda()
    got = ccl.label_device(buf[:, :1000]).cpu().numpy()
    assert np.array_equal(got, want), _first_diff(got, want)
    # unaligned pitch -> generic (non-TMA) load path
    buf2 = torch.zeros((700, 1003), dtype=torch.uint8, device="cuda")
    buf2[:, :1000] = torch.from_numpy(img).cuda()
    got2 = ccl.label_device(buf2[:, :1000]).cpu().numpy()
    assert np.array_equal(got2, want), _first_diff(got2, want)


def test_repeat_determinism(ccl):
    import torch
    img = torch.from_numpy(ccl.random_image(4096, 4096, 0.6, 11)).cuda()
    first = ccl.label_device(img).clone()
    for _ in range(5):
        assert torch.equal(ccl.label_device(img), first)


def test_errors(ccl):
    img = np.zeros((4, 4), np.uint8)
    with pytest.raises(ValueError):
        ccl.label_image(img, cfg=ccl.BlockConfig(0, 32))
    with pytest.raises(ValueError):
        ccl.label_image(img, cfg=ccl.BlockConfig(128, 64))
    with pytest.raises(ValueError):
        ccl.label_image(img, workers=0)
    with pytest.raises(ValueError):
        ccl.label_image(np.zeros((0, 5), np.uint8))
    with pytest.raises(ValueError):
        ccl.label_image(img, variant="bogus")


def test_mixed_structures(ccl, oracle_mod):
    """Tiles mixing vertically repeated run starts (vertical stripes, checkerboard
    blocks: kernel (e)'s rotated run-start scatter, and tables staged in parts)
    with random noise, so warps of one tile take different (e) paths; a dense
    band exercises the union-list capacity of kernel (a)."""
    rng = np.random.default_rng(11)
    h, w = 1111, 1537
    img = (rng.random((h, w)) < 0.5).astype(np.uint8)
    img[:, 100:400] = (np.arange(300) % 2 == 0)[None, :]           # vertical stripes, period 2
    yy, xx = np.mgrid[0:400, 0:300]
    img[300:700, 500:800] = ((yy + xx) % 2 == 0)                      # checkerboard block
    img[800:1000, :] = (rng.random((200, w)) < 0.85)                  # dense band
    img[:, 1200:1203] = 1                                             # long vertical bars across tiles
    want = oracle_mod.sequential_ccl(img)
    for v in VARIANTS:
        got = _gpu_label(ccl, img, v)
        assert np.array_equal(got, want), f"{v}: {_first_diff(got, want)}"
