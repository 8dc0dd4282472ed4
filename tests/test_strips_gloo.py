"""world_size-2 (and 3) gloo test of the strip-mode host protocol on CPU.

Each rank labels its strip, exports the 4*W seam words in exactly the layout
the CUDA kernels produce (csrc/ccl_aux.cu: roots of the top/bottom rows, then
the global seam-node rep of each), exchanges them with ``strips.exchange_seams``
over gloo (the all-gather the library's strip groups perform with NVLink peer
stores: every rank ends with every strip's export in rank order), checks the
product's setup step ``strips.gather_handles`` (IPC handles, rank order), runs the seam union-find and applies the
remap.  The per-strip labeling and the seam arithmetic here are a test-only
numpy restatement of the kernels; the GPU path itself is covered by
tests/test_gpu_modes.py::test_virtual_strips.  The stitched result must be
bit-exact with the oracle on the full image.
"""
import os
import socket

import numpy as np
import pytest

BG = 0xFFFFFFFF


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _strip_export(lab_strip, base, w, k, edge_below):
    """Port of k_strip_roots / k_strip_repmin / k_strip_reps (always export the top row)."""
    h = lab_strip.shape[0]
    roots = np.full(2 * w, BG, np.int64)
    roots[:w] = lab_strip[0]
    if edge_below:
        roots[w:] = lab_strip[h - 1]
    reps = np.full(2 * w, BG, np.int64)
    first_bottom = {}
    for x in range(w):
        r = roots[w + x]
        if r != BG and (r - base) >= w:
            first_bottom.setdefault(int(r), x)
    for i in range(2 * w):
        r = roots[i]
        if r == BG:
            continue
        rl = int(r) - base
        local = rl if rl < w else w + first_bottom[int(r)]
        reps[i] = k * 2 * w + local
    return np.concatenate([roots, reps]).astype(np.uint32)


def _seam_resolve(all_seams, n, w):
    """Port of k_seam_union + k_seam_apply (sequential): seam-root -> final label."""
    all_seams = all_seams.astype(np.int64)
    par = np.concatenate([all_seams[s, 2 * w:] for s in range(n)])
    key = np.concatenate([all_seams[s, :2 * w] for s in range(n)])

    def find(j):
        while par[j] != j:
            j = par[j]
        return j
    for s in range(n - 1):
        for x in range(w):
            a, b = s * 2 * w + w + x, (s + 1) * 2 * w + x
            if key[a] == BG or key[b] == BG:
                continue
            ra, rb = find(a), find(b)
            if ra == rb:
                continue
            if key[ra] > key[rb]:
                ra, rb = rb, ra
            par[rb] = ra
    remap = {}
    for j in range(n * 2 * w):
        if key[j] != BG:
            remap[int(key[j])] = int(key[find(j)])
    return remap


def _worker(rank, world, port, w, full_h, q):
    import torch
    import torch.distributed as dist
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    from paper_1712_09789_b200.strips import exchange_seams, gather_handles
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # strip-group setup: every rank's 64-byte IPC handle, rank order
        blob = gather_handles(bytes([rank + 1]) * 64, world)
        assert blob == b"".join(bytes([k + 1]) * 64 for k in range(world)), "handle all-gather"
        img = oracle.random_image(w, full_h, 0.58, 12) if w != 96 else oracle.pattern_image("spiral", w, full_h)
        th = 32
        tiles = -(-full_h // th)
        parts, r0 = [], 0
        for k in range(world):
            t = tiles // world + (1 if k < tiles % world else 0)
            h = min(t * th, full_h - r0) if k < world - 1 else full_h - r0
            parts.append((r0, h))
            r0 += h
        row0, h = parts[rank]
        base = row0 * w
        strip = img[row0:row0 + h]
        lab = oracle.sequential_ccl(strip).astype(np.int64)
        lab = np.where(lab == BG, BG, lab + base)  # global raster space
        seam = torch.from_numpy(_strip_export(lab, base, w, rank, row0 + h < full_h).view(np.int32).copy())
        allseams = exchange_seams(seam, world).numpy().view(np.uint32)
        remap = _seam_resolve(allseams, world, w)
        final = np.vectorize(lambda v: remap.get(int(v), int(v)), otypes=[np.int64])(lab) if remap else lab
        hmax = max(hh for _, hh in parts)
        mine = torch.zeros((hmax, w), dtype=torch.int64)
        mine[:h] = torch.from_numpy(final)
        full = [torch.zeros((hmax, w), dtype=torch.int64) for k in range(world)]
        dist.all_gather(full, mine)
        if rank == 0:
            got = torch.cat([full[k][:parts[k][1]] for k in range(world)]).numpy().astype(np.uint32)
            want = oracle.sequential_ccl(img)
            q.put(bool(np.array_equal(got, want)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,w,full_h", [(2, 64, 160), (2, 96, 96), (3, 50, 200)])
def test_strip_protocol_gloo(world, w, full_h):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, w, full_h, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=5) is True
