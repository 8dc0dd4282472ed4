"""CPU tests of the product boundary: the sm_100a library loads, exports every
symbol declared in include/*.h, its host-side logic (validation, generators,
host compaction) behaves like the reference — no GPU compute calls here."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ccl():
    import paper_1712_09789_b200 as ccl
    return ccl


def _declared_c_functions():
    src = open(os.path.join(REPO, "include", "ccl_cuda.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ccl_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_c_abi_symbol(ccl):
    lib = ctypes.CDLL(ccl.lib_path())
    decl = _declared_c_functions()
    assert len(decl) >= 15
    missing = [s for s in decl if not hasattr(lib, s)]
    assert not missing, missing
    assert set(decl) == set(ccl.C_ABI_SYMBOLS)


def test_library_exports_cpp_api(ccl):
    out = subprocess.run(["nm", "-D", "--defined-only", "-C", ccl.lib_path()], capture_output=True, text=True).stdout
    for sym in ["ccl::label_image(ccl::BinaryImage const&, ccl::BlockConfig const&, ccl::Variant, unsigned int)",
                "ccl::compact_labels(ccl::LabelMap const&)", "ccl::aggregate_metrics(ccl::RunReport const&)",
                "ccl::random_image(unsigned int, unsigned int, double, unsigned long)",
                "ccl::pattern_image(ccl::PatternKind, unsigned int, unsigned int, ccl::PatternParams const&)",
                "ccl::label_batch("]:
        assert sym in out, sym


def test_library_is_sm100a_only(ccl):
    out = subprocess.run(["cuobjdump", "--list-elf", ccl.lib_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_generators_match_oracle(ccl, oracle_mod):
    for (w, h, d, s) in [(97, 131, 0.3, 5), (512, 512, 0.5, 0), (1, 1000, 0.9, 2), (2048, 64, 0.1, 7)]:
        assert np.array_equal(ccl.random_image(w, h, d, s), oracle_mod.random_image(w, h, d, s))
    for kind in ("stripes", "spiral", "blobs", "checkerboard"):
        assert np.array_equal(ccl.pattern_image(kind, 257, 190, period=4, seed=3),
                              oracle_mod.pattern_image(kind, 257, 190, period=4, seed=3))
    with pytest.raises(ValueError):
        ccl.random_image(4, 4, 1.5, 0)
    with pytest.raises(ValueError):
        ccl.pattern_image("stripes", 4, 4, period=1)
    with pytest.raises(ValueError):
        ccl.pattern_image("bogus", 4, 4)


def test_validation_before_device(ccl):
    """invalid cfg / workers / size raise ValueError (std::invalid_argument) first."""
    img = np.zeros((4, 4), np.uint8)
    with pytest.raises(ValueError):
        ccl.label_image(img, cfg=ccl.BlockConfig(0, 32))
    with pytest.raises(ValueError):
        ccl.label_image(img, cfg=ccl.BlockConfig(65, 64))
    with pytest.raises(ValueError):
        ccl.label_image(img, workers=0)
    with pytest.raises(ValueError):
        ccl.label_image(np.zeros((0, 3), np.uint8))
    with pytest.raises(ValueError):
        ccl.Variant.parse("x2fl")


def test_no_device_fails_loudly(ccl):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(ccl.DeviceError):
        ccl.label_image(np.ones((8, 8), np.uint8))


def test_host_compact_matches_oracle(ccl, oracle_mod, small_cases):
    for name, (img, raw) in list(small_cases.items())[:20]:
        want, k = oracle_mod.compact(raw)
        got = ccl.compact_labels(ccl.LabelMap(raw.shape[1], raw.shape[0], raw))
        assert np.array_equal(got.labels, want), name
        assert got.compacted


def test_strip_split(ccl):
    from paper_1712_09789_b200.strips import split_rows
    th = ccl.tile_shape()[1]
    for full_h, n in [(8192 * 8, 8), (1080, 3), (1000, 4), (33, 1), (2 * th, 2)]:
        parts = split_rows(full_h, n)
        assert sum(h for _, h in parts) == full_h and len(parts) == n
        assert all(h % th == 0 for _, h in parts[:-1])
        assert parts[0][0] == 0 and all(parts[i][0] + parts[i][1] == parts[i + 1][0] for i in range(n - 1))


def test_tile_shape(ccl):
    tw, th = ccl.tile_shape()
    assert tw % 32 == 0 and th % 32 == 0 and th <= 256


def test_metrics_build_exports_and_product_refuses(ccl):
    """The instrumented library (CCL_METRICS=1) exports the same C-ABI; the
    product library reports it is not instrumented (no GPU calls)."""
    path = os.path.join(os.path.dirname(ccl.lib_path()), "libccl_b200_metrics1.so")
    assert os.path.exists(path), "build() also builds the metrics library"
    inst = ctypes.CDLL(path)
    prod = ctypes.CDLL(ccl.lib_path())
    assert [s for s in _declared_c_functions() if not hasattr(inst, s)] == []
    assert inst.ccl_metrics_build() == 1 and prod.ccl_metrics_build() == 0
    assert not ccl.metrics_build()
    f = prod.ccl_read_metrics
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_size_t] + [ctypes.c_void_p] * 4
    assert f(None, None, None, 0, None, None, None, None) == 1  # CCL_EINVAL


def test_aggregate_metrics_mirror(ccl):
    """pipeline.cpp:72-91 restated: grids in block order and their means."""
    lm = ccl.LabelMap(4, 4, np.zeros((4, 4), np.uint32))
    rep = ccl.RunReport(lm, 2, 1, 0.0, ccl.Variant.C2FL, ccl.BlockConfig(), 1,
                        per_block=[ccl.BlockMetrics(0, 3, 1), ccl.BlockMetrics(1, 5, 0)])
    s = ccl.aggregate_metrics(rep)
    assert (s.grid_w, s.grid_h) == (2, 1)
    assert s.iterations_grid == [3, 5] and s.atomics_grid == [1, 0]
    assert s.mean_iterations == 4.0 and s.mean_atomics == 0.5
