/*
 * ccl_oracle.c — TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * A plain-C, single-threaded restatement of the reference CPU labeler's
 * algorithm for the `ccl::label_image` path (arXiv 1712.09789 as restated in
 * /root/reference/proj).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load this library.  The product path
 * (paper_1712_09789_b200 / libccl_b200.so) never links or calls it.
 *
 * Parity pinning: tests/test_oracle.py checks this file against
 *   - the SPEC.md worked examples,
 *   - SURVEY.md Appendix A known answers (K, fg count, FNV-1a-64 of the
 *     raw-root map) produced by the reference's own sequential_ccl,
 *   - the reference itself compiled from /root/reference into oracle/_ref
 *     (oracle/Makefile), on seeded random/pattern images,
 *   - the committed golden fixtures in tests/golden/ (made by
 *     tests/golden/make_golden.py from oracle/_ref).
 *
 * Conventions kept from the reference:
 *   - foreground iff byte == 1 (oracle.cpp:41-43, local_labeler.cpp:59,64)
 *   - raw-root label = minimum raster index x + y*W of the 4-connected
 *     component (image.hpp:41-43); background = 0xFFFFFFFF (image.hpp:15)
 *   - compacted labels 1..K in raster order of first appearance, bg 0
 *     (pipeline.cpp:54-70)
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define ORC_BG 0xFFFFFFFFu

/* ------------------------------------------------------------------ */
/* Generator: xoshiro256** seeded by splitmix64 (generate.hpp:15-43).  */
/* ------------------------------------------------------------------ */
typedef struct { uint64_t s[4]; } orc_rng;

static uint64_t orc_rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }

static void orc_rng_seed(orc_rng* r, uint64_t seed) {
    /* splitmix64 stream, four outputs fill the state (generate.hpp:17-26) */
    uint64_t x = seed;
    for (int i = 0; i < 4; ++i) {
        x += 0x9e3779b97f4a7c15ull;
        uint64_t z = x;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        r->s[i] = z ^ (z >> 31);
    }
}

static uint64_t orc_rng_next(orc_rng* r) {
    /* xoshiro256** step (generate.hpp:28-38) */
    uint64_t* s = r->s;
    const uint64_t out = orc_rotl(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = orc_rotl(s[3], 45);
    return out;
}

/* random_image (generate.cpp:9-18): one draw per pixel in raster order,
 * fg iff (next >> 11) < floor(density * 2^53). Returns -1 on bad density. */
int orc_random_image(uint8_t* out, uint32_t w, uint32_t h, double density, uint64_t seed) {
    if (!(density >= 0.0 && density <= 1.0)) return -1;
    orc_rng r;
    orc_rng_seed(&r, seed);
    const uint64_t thr = (uint64_t)(density * 9007199254740992.0);
    const uint64_t n = (uint64_t)w * h;
    for (uint64_t i = 0; i < n; ++i) out[i] = (orc_rng_next(&r) >> 11) < thr ? 1 : 0;
    return 0;
}

/* pattern_image (generate.cpp:30-106). kind: 0 stripes, 1 spiral, 2 blobs,
 * 3 checkerboard. Returns -1 on invalid parameters. */
int orc_pattern_image(uint8_t* out, int kind, uint32_t w, uint32_t h,
                      uint32_t period, double density, uint64_t seed) {
    const uint64_t n = (uint64_t)w * h;
    memset(out, 0, n);
    if (kind == 0) {                      /* stripes: rows y%period < period/2 */
        if (period < 2) return -1;
        const uint32_t thick = period / 2;
        for (uint32_t y = 0; y < h; ++y)
            if (y % period < thick) memset(out + (uint64_t)y * w, 1, w);
        return 0;
    }
    if (kind == 1) {                      /* spiral: rings at inset 0,2,4,... bridged inward */
        for (uint32_t in = 0; 2u * in < w && 2u * in < h; in += 2) {
            const uint32_t x1 = w - 1 - in, y1 = h - 1 - in;
            for (uint32_t x = in; x <= x1; ++x) {
                out[x + (uint64_t)in * w] = 1;
                out[x + (uint64_t)y1 * w] = 1;
            }
            for (uint32_t y = in; y <= y1; ++y) {
                out[in + (uint64_t)y * w] = 1;
                out[x1 + (uint64_t)y * w] = 1;
            }
            if (2u * (in + 2) < w && 2u * (in + 2) < h) out[(in + 2) + (uint64_t)(in + 1) * w] = 1;
        }
        return 0;
    }
    if (kind == 2) {                      /* blobs: seeded discs, radius max(2, min(w,h)/16) */
        const double mn = (double)(w < h ? w : h);
        const double radius = mn / 16.0 > 2.0 ? mn / 16.0 : 2.0;
        const double area = 3.14159265358979323846 * radius * radius;
        long long cnt = llround(density * (double)w * (double)h / area);
        uint64_t count = cnt < 1 ? 1 : (uint64_t)cnt;
        orc_rng r;
        orc_rng_seed(&r, seed);
        const int64_t r2 = (int64_t)(radius * radius);
        const int64_t ri = (int64_t)radius;
        for (uint64_t i = 0; i < count; ++i) {
            const int64_t cx = (int64_t)(orc_rng_next(&r) % w);
            const int64_t cy = (int64_t)(orc_rng_next(&r) % h);
            int64_t ylo = cy - ri < 0 ? 0 : cy - ri;
            int64_t yhi = cy + ri > (int64_t)h - 1 ? (int64_t)h - 1 : cy + ri;
            int64_t xlo = cx - ri < 0 ? 0 : cx - ri;
            int64_t xhi = cx + ri > (int64_t)w - 1 ? (int64_t)w - 1 : cx + ri;
            for (int64_t y = ylo; y <= yhi; ++y)
                for (int64_t x = xlo; x <= xhi; ++x)
                    if ((x - cx) * (x - cx) + (y - cy) * (y - cy) <= r2) out[x + y * (int64_t)w] = 1;
        }
        return 0;
    }
    if (kind == 3) {                      /* checkerboard: (x+y) even */
        for (uint32_t y = 0; y < h; ++y)
            for (uint32_t x = 0; x < w; ++x) out[x + (uint64_t)y * w] = ((x + y) % 2 == 0);
        return 0;
    }
    return -1;
}

/* ------------------------------------------------------------------ */
/* Sequential two-pass union-find (oracle.cpp:10-50).                  */
/* ------------------------------------------------------------------ */
static uint32_t orc_find(uint32_t* par, uint32_t i) {
    uint32_t root = i;
    while (par[root] != root) root = par[root];
    while (par[i] != root) {               /* full path compression */
        uint32_t nx = par[i];
        par[i] = root;
        i = nx;
    }
    return root;
}

static void orc_unite(uint32_t* par, uint32_t a, uint32_t b) {
    uint32_t ra = orc_find(par, a), rb = orc_find(par, b);
    if (ra == rb) return;
    if (ra < rb) par[rb] = ra; else par[ra] = rb;   /* min-union: roots are class minima */
}

/* labels: W*H u32 out (raw-root form). Uses labels as the parent array. */
void orc_sequential_ccl(const uint8_t* img, uint32_t w, uint32_t h, uint32_t* labels) {
    const uint64_t n = (uint64_t)w * h;
    for (uint64_t i = 0; i < n; ++i) labels[i] = (uint32_t)i;
    for (uint64_t i = 0; i < n; ++i) {
        if (img[i] != 1) continue;
        if (i % w > 0 && img[i - 1] == 1) orc_unite(labels, (uint32_t)i, (uint32_t)(i - 1));
        if (i >= w && img[i - w] == 1) orc_unite(labels, (uint32_t)i, (uint32_t)(i - w));
    }
    /* second pass: resolve in ascending order; roots precede members so a
     * single ascending sweep that reads the (already final) parent suffices
     * after compression.  Background gets the sentinel afterwards. */
    for (uint64_t i = 0; i < n; ++i)
        if (img[i] == 1) labels[i] = orc_find(labels, (uint32_t)i);
    for (uint64_t i = 0; i < n; ++i)
        if (img[i] != 1) labels[i] = ORC_BG;
}

/* ------------------------------------------------------------------ */
/* Block-based three-step restatement (pipeline.cpp:11-52) — single    */
/* threaded, used to pin the block/variant semantics on small images.  */
/* ------------------------------------------------------------------ */
static uint32_t orc_root_nocompress(const uint32_t* par, uint32_t i) {
    while (par[i] != i) i = par[i];
    return i;
}

static void orc_merge(uint32_t* par, uint32_t a, uint32_t b) {
    /* forest.hpp:98-111 with a single thread: the CAS always succeeds */
    uint32_t ra = orc_root_nocompress(par, a), rb = orc_root_nocompress(par, b);
    if (ra == rb) return;
    if (ra < rb) par[rb] = ra; else par[ra] = rb;
}

/* variant: 0 C2FL, 1 RC2FL, 2 CC2FL, 3 NC2FL (image.hpp:73) */
int orc_label_blocks(const uint8_t* img, uint32_t w, uint32_t h, uint32_t bw, uint32_t bh,
                     int variant, uint32_t* labels) {
    if (bw < 1 || bh < 1 || (uint64_t)bw * bh > 4096 || variant < 0 || variant > 3) return -1;
    const uint64_t n = (uint64_t)w * h;
    const uint32_t slots = bw * bh;
    uint32_t* par = (uint32_t*)malloc(sizeof(uint32_t) * slots);
    uint32_t* snap = (uint32_t*)malloc(sizeof(uint32_t) * slots);
    uint8_t* px = (uint8_t*)malloc(slots);
    if (!par || !snap || !px) { free(par); free(snap); free(px); return -2; }
    /* step 1: local labeling of every block, written as global parents */
    for (uint32_t y0 = 0; y0 < h; y0 += bh) {
        for (uint32_t x0 = 0; x0 < w; x0 += bw) {
            const uint32_t bwt = (w - x0) < bw ? (w - x0) : bw;    /* truncated edge blocks */
            const uint32_t bht = (h - y0) < bh ? (h - y0) : bh;
            const uint32_t ns = bwt * bht;
            for (uint32_t ly = 0; ly < bht; ++ly)
                memcpy(px + ly * bwt, img + x0 + (uint64_t)(y0 + ly) * w, bwt);
            for (uint32_t i = 0; i < ns; ++i) par[i] = i;
            const int row_scan = (variant == 0 || variant == 1);
            const int col_scan = (variant == 0 || variant == 2);
            if (row_scan) {                 /* local_labeler.cpp:30-38, snapshot semantics */
                memcpy(snap, par, sizeof(uint32_t) * ns);
                for (uint32_t i = 0; i < ns; ++i)
                    if (i % bwt != 0 && px[i] == px[i - 1]) par[i] = snap[i - 1];
            }
            if (col_scan) {                 /* local_labeler.cpp:40-48 */
                memcpy(snap, par, sizeof(uint32_t) * ns);
                for (uint32_t i = bwt; i < ns; ++i)
                    if (px[i] == px[i - bwt]) par[i] = snap[i - bwt];
            }
            for (uint32_t i = 0; i < ns; ++i) par[i] = orc_root_nocompress(par, i);   /* flatten_all */
            const int ref_rows = (variant != 1);
            const int ref_cols = (variant == 1 || variant == 3);
            if (ref_rows)                   /* refine rows, local_labeler.cpp:58-61 */
                for (uint32_t i = 0; i < ns; ++i)
                    if (i % bwt != 0 && px[i] == 1 && px[i - 1] == 1) orc_merge(par, i, i - 1);
            if (ref_cols)                   /* refine columns, local_labeler.cpp:63-66 */
                for (uint32_t i = bwt; i < ns; ++i)
                    if (px[i] == 1 && px[i - bwt] == 1) orc_merge(par, i, i - bwt);
            for (uint32_t i = 0; i < ns; ++i) par[i] = orc_root_nocompress(par, i);
            for (uint32_t i = 0; i < ns; ++i) {        /* convert_ids, local_labeler.cpp:102-112 */
                const uint32_t r = par[i];
                const uint64_t g = (uint64_t)(x0 + r % bwt) + (uint64_t)(y0 + r / bwt) * w;
                labels[(uint64_t)(x0 + i % bwt) + (uint64_t)(y0 + i / bwt) * w] = (uint32_t)g;
            }
        }
    }
    free(par); free(snap); free(px);
    /* step 2: one border-merge pass over interior block boundaries (boundary.cpp:7-35) */
    for (uint32_t x = bw; x < w; x += bw)
        for (uint32_t y = 0; y < h; ++y) {
            const uint64_t p = x + (uint64_t)y * w;
            if (img[p] == 1 && img[p - 1] == 1) orc_merge(labels, (uint32_t)p, (uint32_t)(p - 1));
        }
    for (uint32_t y = bh; y < h; y += bh)
        for (uint32_t x = 0; x < w; ++x) {
            const uint64_t p = x + (uint64_t)y * w;
            if (img[p] == 1 && img[p - w] == 1) orc_merge(labels, (uint32_t)p, (uint32_t)(p - w));
        }
    /* step 3: resolve (boundary.cpp:37-55); ascending order keeps it single-pass */
    for (uint64_t p = 0; p < n; ++p)
        if (img[p] == 1) labels[p] = orc_root_nocompress(labels, (uint32_t)p);
    for (uint64_t p = 0; p < n; ++p)
        if (img[p] != 1) labels[p] = ORC_BG;
    return 0;
}

/* compact_labels (pipeline.cpp:54-70): 1..K in order of first appearance. */
uint32_t orc_compact(const uint32_t* raw, uint64_t n, uint32_t* out) {
    uint32_t* remap = (uint32_t*)calloc(n ? n : 1, sizeof(uint32_t));
    uint32_t next = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const uint32_t v = raw[i];
        if (v == ORC_BG) { out[i] = 0; continue; }
        if (remap[v] == 0) remap[v] = ++next;
        out[i] = remap[v];
    }
    free(remap);
    return next;
}

/* K = #{p : labels[p] == p} and foreground count, for known-answer checks. */
void orc_count(const uint32_t* raw, uint64_t n, uint64_t* k_out, uint64_t* fg_out) {
    uint64_t k = 0, fg = 0;
    for (uint64_t i = 0; i < n; ++i) {
        if (raw[i] != ORC_BG) ++fg;
        if (raw[i] == (uint32_t)i) ++k;
    }
    *k_out = k;
    *fg_out = fg;
}

/* FNV-1a-64 over the u32 little-endian label bytes. */
uint64_t orc_fnv1a64_u32(const uint32_t* v, uint64_t n) {
    uint64_t hsh = 0xcbf29ce484222325ull;
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t x = v[i];
        for (int b = 0; b < 4; ++b) {
            hsh ^= (x >> (8 * b)) & 0xFFu;
            hsh *= 0x100000001b3ull;
        }
    }
    return hsh;
}
