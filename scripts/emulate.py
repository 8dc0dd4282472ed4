"""Sequential Python emulation of the kernel algorithm (debug aid only).

Mirrors csrc/ccl_kernels.cu step by step (word masks, run nodes, coarse
column links, has_lower_in_run refinement, flatten, seam marking, A/D/E) so a
wrong label can be traced without a GPU."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

M32 = 0xFFFFFFFF
BG = 0xFFFFFFFF


def hi_bit_le(s, b):
    v = s & (M32 >> (31 - b))
    return v.bit_length() - 1


def has_lower_in_run(m, o):
    return (((m + o) & M32) ^ m ^ o) & m


def bits(x):
    while x:
        b = (x & -x).bit_length() - 1
        yield b
        x &= x - 1


def emulate(img, WX=8, WY=1, variant=0):
    H, W = img.shape
    TW, TH = 32 * WX, 32 * WY
    PS = TW + 1
    ntx, nty = -(-W // TW), -(-H // TH)
    fgimg = (img == 1)
    L = np.full(W * H, 0xDEADBEEF, dtype=np.uint64)

    def tile(tx, ty):
        x0, y0 = tx * TW, ty * TH
        P = {}
        masks = np.zeros((TH, WX), dtype=np.uint64)
        for r in range(TH):
            for wx in range(WX):
                m = 0
                for b in range(32):
                    y, x = y0 + r, x0 + 32 * wx + b
                    if y < H and x < W and fgimg[y, x]:
                        m |= 1 << b
                masks[r, wx] = m
        RUNS = variant in (0, 1)
        st_of = lambda m: (m & ~(m << 1) & M32) if RUNS else m
        for r in range(TH):
            for wx in range(WX):
                m = int(masks[r, wx]); um = int(masks[r - 1, wx]) if r > 0 else 0
                st, ust = st_of(m), st_of(um)
                nb = r * PS + 32 * wx
                for b in bits(st):
                    par = nb + b
                    if variant == 0:
                        mb = m >> b
                        ov = (((mb & ~(mb + 1)) << b) & M32) & um
                        if ov:
                            par = nb - PS + hi_bit_le(ust, (ov & -ov).bit_length() - 1)
                    elif variant == 2 and (um >> b) & 1:
                        par = nb + b - PS
                    P[nb + b] = par

        def find(x):
            while P[x] != x:
                x = P[x]
            return x

        def union(a, b):
            a, b = find(a), find(b)
            if a == b:
                return
            if a < b:
                a, b = b, a
            P[a] = b

        for r in range(TH):
            for wx in range(WX):
                m = int(masks[r, wx]); um = int(masks[r - 1, wx]) if r > 0 else 0
                st, ust = st_of(m), st_of(um)
                nb = r * PS + 32 * wx
                if RUNS:
                    o = m & um
                    U = o & ~(o << 1) & M32
                    if variant == 0:
                        U &= has_lower_in_run(m, o)
                    for b in bits(U):
                        union(nb + hi_bit_le(st, b), nb - PS + hi_bit_le(ust, b))
                else:
                    if variant == 3:
                        for b in bits(m & um):
                            union(nb + b, nb + b - PS)
                    hp = (m & (m << 1) & M32) & ~(um & (um << 1) & M32)
                    for b in bits(hp):
                        union(nb + b, nb + b - 1)
                if wx > 0 and (m & 1):
                    lm = int(masks[r, wx - 1])
                    if lm >> 31:
                        lst = st_of(lm)
                        union(nb, nb - 32 + (lst.bit_length() - 1))
        for k in list(P):  # (the kernel needs two passes here, see the CUDA comment)
            P[k] = find(k)
        F = set()
        has_top, has_bot = ty > 0, ty + 1 < nty
        has_left, has_right = tx > 0, tx + 1 < ntx
        for wx in range(WX):
            if has_top:
                for b in bits(st_of(int(masks[0, wx]))):
                    F.add(P[32 * wx + b])
            if has_bot:
                for b in bits(st_of(int(masks[TH - 1, wx]))):
                    F.add(P[(TH - 1) * PS + 32 * wx + b])
        for r in range(TH):
            m0 = int(masks[r, 0])
            if has_left and m0 & 1:
                F.add(P[r * PS])
            ml = int(masks[r, WX - 1])
            if has_right and ml >> 31:
                F.add(P[r * PS + 32 * (WX - 1) + hi_bit_le(st_of(ml), 31)])
        gid = lambda n: (y0 + n // PS) * W + x0 + n % PS

        def local_label(y, x):  # root node of pixel (y, x) of this tile
            r, c = y - y0, x - x0
            wx, b = c // 32, c % 32
            st = st_of(int(masks[r, wx]))
            return P[r * PS + 32 * wx + hi_bit_le(st, b)]
        return P, F, gid, local_label, masks

    tiles = {}
    # kernel A
    for ty in range(nty):
        for tx in range(ntx):
            P, F, gid, ll, masks = tile(tx, ty)
            tiles[(tx, ty)] = (P, F, gid, ll)
            for n in F:
                L[gid(n)] = gid(n)
            x0, y0 = tx * TW, ty * TH
            rows = []
            if ty > 0:
                rows.append(y0)
            if ty + 1 < nty:
                rows.append(y0 + TH - 1)
            for y in rows:
                for x in range(x0, min(x0 + TW, W)):
                    L[y * W + x] = gid(ll(y, x)) if fgimg[y, x] else BG
            for y in range(y0, min(y0 + TH, H)):
                if tx > 0:
                    L[y * W + x0] = gid(ll(y, x0)) if fgimg[y, x0] else BG
                if tx + 1 < ntx:
                    L[y * W + x0 + TW - 1] = gid(ll(y, x0 + TW - 1)) if fgimg[y, x0 + TW - 1] else BG

    def gfind(x):
        while L[x] != x:
            x = int(L[x])
            assert x < W * H, "chain reached an unregistered entry"
        return x

    def gunion(a, b):
        a, b = gfind(a), gfind(b)
        if a != b:
            if a < b:
                a, b = b, a
            L[a] = b
    # kernel D
    for k in range(1, nty):
        y = k * TH
        for x in range(W):
            a, b = int(L[y * W + x]), int(L[(y - 1) * W + x])
            if a != BG and b != BG:
                gunion(a, b)
    for k in range(1, ntx):
        x = k * TW
        for y in range(H):
            a, b = int(L[y * W + x]), int(L[y * W + x - 1])
            if a != BG and b != BG:
                gunion(a, b)
    # kernel E
    out = np.full(W * H, BG, dtype=np.uint64)
    for (tx, ty), (P, F, gid, ll) in tiles.items():
        x0, y0 = tx * TW, ty * TH
        for y in range(y0, min(y0 + TH, H)):
            for x in range(x0, min(x0 + TW, W)):
                if fgimg[y, x]:
                    R = ll(y, x)
                    out[y * W + x] = gfind(gid(R)) if R in F else gid(R)
    return out.reshape(H, W).astype(np.uint32)


if __name__ == "__main__":
    import oracle as o
    img = o.pattern_image("spiral", 300, 200)
    want = o.sequential_ccl(img)
    for v in range(4):
        got = emulate(img, variant=v)
        d = np.argwhere(got != want)
        print("variant", v, "mismatches", len(d), d[:5].tolist())
