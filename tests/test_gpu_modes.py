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
    th = ccl.tile_shape()[1]
    for (w, h, n) in [(97, 3 * th + 8, 3), (1, 10 * th, 5), (300, 2 * th, 2), (1003, 300, 4)]:
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


def _strip_rank(rank, world, port, w, full_h, q):
    """One rank of the strip protocol on the real kernels (shared GPU, gloo exchange)."""
    import os
    import sys
    import numpy as np
    import torch
    import torch.distributed as dist
    sys.path.insert(0, REPO)
    import paper_1712_09789_b200 as ccl
    from paper_1712_09789_b200.strips import StripLabeler, split_rows
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        img = ccl.random_image(w, full_h, 0.58, 21)
        dev = torch.device("cuda", 0)
        lab = StripLabeler(ccl.Context(0), w, full_h, rank, world)
        row0, h = lab.row0, lab.h
        assert (row0, h) == split_rows(full_h, world)[rank]
        d_img = torch.from_numpy(np.ascontiguousarray(img[row0:row0 + h])).to(dev)
        out = torch.empty((h, w), dtype=torch.uint32, device=dev)
        for _ in range(2):  # repeated steps: both export parities, epochs advance
            out.fill_(7)
            lab.label(d_img, out)
            torch.cuda.synchronize()
        for _ in range(6):  # back to back, no host sync: ranks drift apart by a step
            lab.label(d_img, out)
        torch.cuda.synchronize()
        mine = out.cpu().view(torch.int32)
        hmax = max(hh for _, hh in split_rows(full_h, world))
        pad = torch.zeros((hmax, w), dtype=torch.int32)
        pad[:h] = mine
        parts = [torch.zeros((hmax, w), dtype=torch.int32) for _ in range(world)]
        dist.all_gather(parts, pad)
        if rank == 0:
            got = torch.cat([parts[k][:split_rows(full_h, world)[k][1]] for k in range(world)]).numpy().view(np.uint32)
            import oracle
            q.put(bool(np.array_equal(got, oracle.sequential_ccl(img))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_strip_labeler_multiprocess(ccl, world):
    """StripLabeler (the bench's N>1 path) in `world` processes sharing one GPU:
    library strip groups with CUDA IPC exchange areas and device flags (the
    handles are all-gathered over gloo once)."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_strip_rank, args=(r, world, port, 1500, 256 * world + 77, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=5) is True


@pytest.mark.slow
def test_known_answer_32768(ccl, oracle_mod, known_answers):
    """Config 5 image on one B200 (5.4 GB working set): K / fg / FNV vs the reference."""
    import torch
    ka = known_answers.get("random_32768_d0.5_s0")
    if ka is None:
        pytest.skip("known answer not generated")
    img = torch.from_numpy(ccl.random_image(32768, 32768, 0.5, 0)).cuda()
    lab = ccl.label_device(img)
    del img
    lab = lab.cpu().numpy()
    k, fg = oracle_mod.count(lab)
    assert (k, fg) == (ka["K"], ka["fg"])
    assert f"{oracle_mod.fnv1a64(lab):016x}" == ka["fnv1a64_raw"]


@pytest.mark.gpu
def test_random_image_device_matches_host(ccl):
    # xoshiro256** jump-ahead per chunk, byte-identical with
    # the host generator (reference generate.cpp:9-18)
    for (w, h, d, s) in [(1, 1, 0.5, 0), (17, 3, 0.3, 7), (1920, 1080, 0.5, 1023), (2048, 2048, 0.1, 0),
                         (4096, 1000, 0.9, 12345), (8192, 8192, 0.5, 0)]:
        got = ccl.random_image_device(w, h, d, s).cpu().numpy()
        full = ccl.random_image(w, h, d, s)
        assert np.array_equal(got, full), (w, h, d, s)
        if h >= 3:  # one strip of the same image
            r0 = h // 3
            strip = ccl.random_image_device(w, h - r0, d, s, row0=r0).cpu().numpy()
            assert np.array_equal(strip, full[r0:]), (w, h, d, s, r0)


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["c2fl", "rc2fl", "cc2fl", "nc2fl"])
def test_virtual_strips_variants(ccl, oracle_mod, variant):
    # every variant through the strip protocol (ccl_strip_final must expand the
    # node layout the strip's kernel (a) used), aligned and unaligned pitches
    import torch
    from paper_1712_09789_b200.strips import label_strips_single_gpu
    th = ccl.tile_shape()[1]
    for (w, h, n) in [(256, 4 * th, 3), (97, 3 * th + 5, 2)]:
        img = ccl.random_image(w, h, 0.55, 11 + w)
        got = label_strips_single_gpu(torch.from_numpy(img).cuda(), n, variant=variant).cpu().numpy()
        assert np.array_equal(got, oracle_mod.sequential_ccl(img)), (variant, w, h, n)


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0, 0]])
@pytest.mark.parametrize("kind", ["random", "spiral", "checkerboard"])
def test_label_strips_multi_device_api(ccl, oracle_mod, kind, devices):
    """ccl_label_strips / label_strips: one host image over a device list (one
    GPU listed n times = n strips with peer-copy seam exchange on one device)."""
    w, h = 1003, 777
    img = ccl.random_image(w, h, 0.58, 5) if kind == "random" else ccl.pattern_image(kind, w, h, period=5)
    rep = ccl.label_strips(img, devices)
    assert np.array_equal(rep.label_map.labels, oracle_mod.sequential_ccl(img)), (kind, devices)
    assert rep.worker_count == len(devices) and rep.wall_time_ms > 0


def test_label_strips_errors(ccl):
    img = np.ones((100, 50), np.uint8)
    with pytest.raises(ValueError):
        ccl.label_strips(img, [])
    th = ccl.tile_shape()[1]
    with pytest.raises(ValueError):  # more strips than tile rows
        ccl.label_strips(np.ones((th, 50), np.uint8), [0, 0])


def test_device_path_graph_replay(ccl, oracle_mod):
    """Repeated ccl_label_device calls on the same buffers replay a cached CUDA
    graph: new image content in the same buffer, then other buffers / shapes."""
    import torch
    w, h = 700, 500
    img = torch.empty((h, w), dtype=torch.uint8, device="cuda")
    out = torch.empty((h, w), dtype=torch.uint32, device="cuda")
    for seed in range(4):  # same pointers every call: capture once, then replays
        a = ccl.random_image(w, h, 0.45 + 0.05 * seed, seed)
        img.copy_(torch.from_numpy(a))
        ccl.label_device(img, out)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint32), oracle_mod.sequential_ccl(a)), seed
    for (ww, hh) in [(300, 200), (w, h)]:  # other buffers / shape, then the first graph again
        a = ccl.random_image(ww, hh, 0.6, ww)
        got = ccl.label_device(torch.from_numpy(a).cuda())
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy().view(np.uint32), oracle_mod.sequential_ccl(a))
    a = ccl.pattern_image("spiral", w, h)
    img.copy_(torch.from_numpy(a))
    ccl.label_device(img, out)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().view(np.uint32), oracle_mod.sequential_ccl(a))


def test_label_host_async_two_contexts(ccl, oracle_mod):
    """ccl_label_host_async + ccl_ctx_sync: a stream of host images on two
    alternating contexts (pinned buffers), every result bit-exact."""
    import ctypes
    import torch
    w, h = 640, 480
    imgs = [ccl.random_image(w, h, 0.4 + 0.05 * k, k) for k in range(5)]
    hin = [torch.from_numpy(a).pin_memory() for a in imgs]
    hout = [torch.empty((h, w), dtype=torch.int32).pin_memory() for _ in imgs]
    ctxs = [ccl.Context(0), ccl.Context(0)]
    for k in range(len(imgs)):
        c = ctxs[k & 1]
        if k >= 2:
            ccl._check(ccl._lib.ccl_ctx_sync(c.handle))
            done = hout[k - 2].numpy().view(np.uint32)
            assert np.array_equal(done, oracle_mod.sequential_ccl(imgs[k - 2])), k - 2
        ccl._check(ccl._lib.ccl_label_host_async(
            c.handle, ctypes.cast(hin[k].data_ptr(), ccl._u8p), w, h,
            ctypes.cast(hout[k].data_ptr(), ccl._u32p), 0))
    for c in ctxs:
        ccl._check(ccl._lib.ccl_ctx_sync(c.handle))
    for k in (len(imgs) - 2, len(imgs) - 1):
        assert np.array_equal(hout[k].numpy().view(np.uint32), oracle_mod.sequential_ccl(imgs[k])), k


@pytest.mark.parametrize("pipe_tiles", ["50", "8192"])
def test_batch_pipelined_chunks(ccl, oracle_mod, monkeypatch, pipe_tiles):
    """ccl_label_batch as a two-stream pipeline of frame chunks (kernels (a)+(d)
    of chunk j+1 beside (d2)+(e) of chunk j): small chunks forced through
    CCL_PIPE_TILES, mixed content, ragged last chunk; every frame bit-exact."""
    import torch
    monkeypatch.setenv("CCL_PIPE_TILES", pipe_tiles)
    w, h, n = 500, 300, 41
    frames = np.stack([ccl.random_image(w, h, 0.3 + 0.01 * s, s) for s in range(n)])
    frames[7] = ccl.pattern_image("spiral", w, h)
    frames[8] = 1
    frames[9] = 0
    frames[10] = ccl.pattern_image("checkerboard", w, h)
    got = ccl.label_batch_device(torch.from_numpy(frames).cuda()).cpu().numpy()
    for f in range(n):
        assert np.array_equal(got[f], oracle_mod.sequential_ccl(frames[f])), f
