"""Label-map files (reference proj/src/label_io.cpp:27-94,
SPEC.md:455-466): host writers byte-identical with the reference's, CCLM
round trips, and the GPU label -> compact -> CCLM stream path."""
import os

import numpy as np
import pytest


def _ref_or_skip(oracle_mod):
    if not oracle_mod.ref_available():
        pytest.skip("oracle/_ref not built")


def test_spec_examples(ccl, tmp_path):
    # 1x1 background, raw -> 13 header bytes + 4 payload bytes
    p = str(tmp_path / "bg.cclm")
    ccl.write_label_map(ccl.LabelMap(1, 1, np.full((1, 1), ccl.BG, np.uint32)), p, "raw")
    data = open(p, "rb").read()
    assert len(data) == 17 and data[:5] == b"CCLM\x01" and data[13:] == b"\x00\x00\x00\x00"
    # 2x1 map [1, 2] csv -> "1,2"
    p = str(tmp_path / "m.csv")
    ccl.write_label_map(ccl.LabelMap(2, 1, np.array([[1, 2]], np.uint32), True), p, "csv")
    assert open(p).read() == "1,2\n"


def _expected(raw, fmt):
    """csv / pgm16 bytes per SPEC.md:458 (LF rows, no trailing comma; P5 header, 16-bit BE)."""
    import oracle
    c, k = oracle.compact(raw)
    if fmt == "csv":
        return "".join(",".join(str(v) for v in row) + "\n" for row in c).encode()
    h, w = c.shape
    return f"P5\n{w} {h}\n{max(k, 1)}\n".encode() + c.astype(">u2").tobytes()


@pytest.mark.parametrize("fmt", ["raw", "csv", "pgm16"])
def test_writer_matches_reference(ccl, oracle_mod, tmp_path, fmt):
    # raw: byte-identical with the reference's own writer (label_io.cpp:27-33);
    # csv / pgm16: the reference writer formats numbers through iostreams, which
    # crash inside this Python process (its libccl_ref.so carries its own
    # libstdc++), so those bytes are checked against the SPEC.md:458 layout
    if fmt == "raw":
        _ref_or_skip(oracle_mod)
    for (w, h, d, s) in [(1, 1, 1.0, 0), (37, 11, 0.5, 1), (128, 64, 0.3, 2), (300, 7, 0.7, 3)]:
        img = oracle_mod.random_image(w, h, d, s)
        raw = oracle_mod.sequential_ccl(img)
        mine = str(tmp_path / f"m.{fmt}")
        ccl.write_label_map(ccl.LabelMap(w, h, raw), mine, fmt)
        if fmt == "raw":
            ref = str(tmp_path / f"r.{fmt}")
            oracle_mod.ref_write_label_map(raw, ref, fmt)
            want = open(ref, "rb").read()
        else:
            want = _expected(raw, fmt)
        assert open(mine, "rb").read() == want, (fmt, w, h)


def test_round_trip_100_maps(ccl, oracle_mod, tmp_path):
    # acceptance criterion 10: CCLM write -> read is lossless
    rng = np.random.default_rng(5)
    p = str(tmp_path / "rt.cclm")
    for i in range(100):
        w, h = int(rng.integers(1, 60)), int(rng.integers(1, 60))
        img = oracle_mod.random_image(w, h, float(rng.uniform(0.05, 0.95)), i)
        raw = oracle_mod.sequential_ccl(img)
        ccl.write_label_map(ccl.LabelMap(w, h, raw), p, "raw")
        back = ccl.read_label_map(p)
        want, _ = oracle_mod.compact(raw)
        assert back.compacted and (back.width, back.height) == (w, h)
        assert np.array_equal(back.labels, want)


def test_errors(ccl, tmp_path):
    bad = tmp_path / "bad.cclm"
    bad.write_bytes(b"NOPE\x01")
    with pytest.raises(ValueError, match="not a CCLM"):
        ccl.read_label_map(str(bad))
    bad.write_bytes(b"CCLM\x02" + b"\x01\x00\x00\x00" * 2)
    with pytest.raises(ValueError, match="version"):
        ccl.read_label_map(str(bad))
    bad.write_bytes(b"CCLM\x01" + b"\x02\x00\x00\x00" * 2 + b"\x00" * 5)
    with pytest.raises(ValueError, match="truncated"):
        ccl.read_label_map(str(bad))
    with pytest.raises(ValueError, match="cannot open"):
        ccl.read_label_map(str(tmp_path / "missing.cclm"))
    many = np.arange(70000, dtype=np.uint32).reshape(1, 70000)  # 70000 singleton components
    with pytest.raises(ValueError, match="65535"):
        ccl.write_label_map(ccl.LabelMap(70000, 1, many), str(tmp_path / "x.pgm"), "pgm16")
    with pytest.raises(ValueError, match="unknown"):
        ccl.write_label_map(ccl.LabelMap(1, 1, np.zeros((1, 1), np.uint32)), str(tmp_path / "x"), "png")


@pytest.mark.gpu
def test_label_to_cclm_stream(ccl, oracle_mod, tmp_path):
    # chunked device->file copies: sizes below, at and above one 16 MiB chunk
    for (w, h, d) in [(1, 1, 1.0), (517, 391, 0.5), (2048, 2048, 0.6), (4096, 1100, 0.5)]:
        img = ccl.random_image(w, h, d, 9)
        p = str(tmp_path / "gpu.cclm")
        k = ccl.label_to_cclm(img, p)
        want, kw = oracle_mod.compact(oracle_mod.sequential_ccl(img))
        assert k == kw
        assert os.path.getsize(p) == 13 + 4 * w * h
        back = ccl.read_label_map(p)
        assert np.array_equal(back.labels, want)
