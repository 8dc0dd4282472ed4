"""CPU tests pinning the oracle (test infrastructure) against the reference's
own outputs: SPEC.md examples, SURVEY.md Appendix A known answers, the
committed golden fixtures (made by the reference itself) and, when
oracle/_ref is built, the live reference labeler."""
import numpy as np
import pytest

BG = 0xFFFFFFFF


def test_spec_examples(oracle_mod):
    o = oracle_mod
    # SPEC.md:401 L-shape -> all fg labeled 0
    lab = o.sequential_ccl(np.array([[1, 0, 0, 0], [1, 0, 0, 0], [1, 1, 1, 0], [0, 0, 0, 0]], np.uint8))
    assert set(lab[lab != BG].tolist()) == {0}
    # SPEC.md:222 -> all 8 fg share root 0
    lab = o.sequential_ccl(np.array([[1, 1, 0, 0], [0, 1, 0, 1], [0, 1, 1, 1], [0, 0, 0, 1]], np.uint8))
    assert (lab[lab != BG] == 0).all() and (lab != BG).sum() == 8
    # SPEC.md:306 two bars -> {0,3}->0, {2,5}->2
    lab = o.sequential_ccl(np.array([[1, 0, 1], [1, 0, 1]], np.uint8)).ravel().tolist()
    assert lab == [0, BG, 2, 0, BG, 2]
    # SPEC.md:348 1x1 fg -> 0
    assert o.sequential_ccl(np.ones((1, 1), np.uint8)).tolist() == [[0]]
    # SPEC.md:421-423 stripes p2 h8 -> 4 comps; checkerboard 4x4 -> 8 singletons; spiral -> 1
    assert o.count(o.sequential_ccl(o.pattern_image("stripes", 8, 8, period=2)))[0] == 4
    k, fg = o.count(o.sequential_ccl(o.pattern_image("checkerboard", 4, 4)))
    assert (k, fg) == (8, 8)
    assert o.count(o.sequential_ccl(o.pattern_image("spiral", 64, 64)))[0] == 1


def test_byte_predicate_is_eq1(oracle_mod):
    img = np.array([[1, 2, 1], [255, 1, 0]], np.uint8)
    lab = oracle_mod.sequential_ccl(img).ravel().tolist()
    assert lab == [0, BG, 2, BG, 4, BG]


def test_golden_fixtures(oracle_mod, small_cases):
    for name, (img, want) in small_cases.items():
        got = oracle_mod.sequential_ccl(img)
        assert np.array_equal(got, want), name


@pytest.mark.parametrize("variant", ["c2fl", "rc2fl", "cc2fl", "nc2fl"])
@pytest.mark.parametrize("block", [(32, 32), (8, 8), (16, 16), (5, 7), (1, 1), (64, 64)])
def test_block_restatement_matches_golden(oracle_mod, small_cases, variant, block):
    for name, (img, want) in list(small_cases.items())[::3]:
        got = oracle_mod.label_blocks(img, block[0], block[1], variant)
        assert np.array_equal(got, want), (name, variant, block)


def test_known_answers(oracle_mod, known_answers):
    o = oracle_mod
    cases = [("random_512_d0.5_s0", lambda: o.random_image(512, 512, 0.5, 0))]
    cases += [(f"random_2048_d{d / 10}_s0", (lambda d=d: o.random_image(2048, 2048, d / 10, 0))) for d in range(1, 10)]
    cases += [("frame_1920x1080_d0.5_s0", lambda: o.random_image(1920, 1080, 0.5, 0)),
              ("frame_1920x1080_d0.5_s1023", lambda: o.random_image(1920, 1080, 0.5, 1023))]
    for name, mk in cases:
        lab = o.sequential_ccl(mk())
        k, fg = o.count(lab)
        ka = known_answers[name]
        assert (k, fg) == (ka["K"], ka["fg"]), name
        assert f"{o.fnv1a64(lab):016x}" == ka["fnv1a64_raw"], name


def test_appendix_a_counts(known_answers):
    """K / fg of SURVEY.md Appendix A, reproduced by the reference here."""
    exp = {"random_512_d0.5_s0": (17469, 131508), "random_8192_d0.5_s0": (4415243, 33557554),
           "blobs_8192_d0.5_s0": (12, 26254800), "spiral_8192": (1, 33564671), "stripes_8192_p2": (4096, 33554432),
           "checkerboard_8192": (33554432, 33554432), "frame_1920x1080_d0.5_s0": (136855, 1037365),
           "random_32768_d0.5_s0": (70618584, 536888580)}
    for name, (k, fg) in exp.items():
        if name in known_answers:
            assert (known_answers[name]["K"], known_answers[name]["fg"]) == (k, fg), name


def test_generators_match_reference(oracle_mod):
    o = oracle_mod
    if not o.ref_available():
        pytest.skip("oracle/_ref not built (no /root/reference)")
    for (w, h, d, s) in [(97, 131, 0.3, 5), (512, 512, 0.5, 0), (1, 1000, 0.9, 2)]:
        assert np.array_equal(o.random_image(w, h, d, s), o.ref_random_image(w, h, d, s))
    for kind in ("stripes", "spiral", "blobs", "checkerboard"):
        assert np.array_equal(o.pattern_image(kind, 257, 190, period=4), o.ref_pattern_image(kind, 257, 190, period=4))


def test_oracle_vs_live_reference(oracle_mod):
    o = oracle_mod
    if not o.ref_available():
        pytest.skip("oracle/_ref not built (no /root/reference)")
    rng = np.random.default_rng(3)
    for i in range(20):
        h, w = int(rng.integers(1, 200)), int(rng.integers(1, 200))
        img = o.ref_random_image(w, h, float(rng.uniform(0.05, 0.95)), i)
        want = o.ref_sequential_ccl(img)
        assert np.array_equal(o.sequential_ccl(img), want)
        ref_blocks, _ = o.ref_label_image(img, 16, 8, "nc2fl", 3)
        assert np.array_equal(ref_blocks, want)
        assert np.array_equal(o.label_blocks(img, 16, 8, "cc2fl"), want)


def test_scipy_second_oracle(oracle_mod):
    ndimage = pytest.importorskip("scipy.ndimage")
    img = oracle_mod.random_image(300, 200, 0.55, 9)
    raw = oracle_mod.sequential_ccl(img)
    comp, k = oracle_mod.compact(raw)
    lab, n = ndimage.label(img == 1)
    assert k == n
    assert np.array_equal(comp, lab.astype(np.uint32))


def test_compact(oracle_mod):
    raw = np.array([[BG, 1, 1], [3, BG, 1]], np.uint32)
    out, k = oracle_mod.compact(raw)
    assert k == 2 and out.tolist() == [[0, 1, 1], [2, 0, 1]]
