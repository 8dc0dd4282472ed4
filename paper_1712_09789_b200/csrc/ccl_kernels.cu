// ccl_kernels.cu — the hand-written sm_100a kernels of the labeler.
//
//   (a)+(b)+(c)  k_local_band (C2FL, the default)  : persistent, one 128x64
//                           tile per CTA at a time, TMA-staged.  Lane = a 2-row
//                           band of one 32-px word: band runs from bit masks,
//                           COMPACT node ids in tile raster order (prefix
//                           counts), one coarse loop over per-run marker bits
//                           (links to the band above / root codes), a
//                           pointer-jump round where runs mostly link, shared-
//                           memory min-union refinement over node HANDLES (the
//                           entries' byte offsets), seam-touching roots registered
//                           in the compact global forest, then a node table of
//                           root codes.  Hands off, per tile: row masks, band
//                           prefixes / starts, the table, the seam-root list and
//                           the seam records (root of every border pixel).
//                k_local<VAR> : the same on row runs for the RC2FL / CC2FL / NC2FL
//                           variants (coarse scans per the reference's variant).
//   (d)          k_seams  : boundary-only pass (Algorithm 2) over the seam
//                           records: one warp per four 32-pair chunks, one union
//                           per distinct pair, min-key CAS union-find in the
//                           compact L2-resident forest.
//   (d2)         k_resolve: each tile's seam-touching roots climb to their class
//                           root once; the final labels go into the tile's list.
//   (e)          k_final  : persistent 3-stage pipeline: expands every band run
//                           to its two rows in a 128B-swizzled staging tile and
//                           writes every label exactly once (TMA stores).  It
//                           never re-reads the image.
//   (d), (d2), (e) are programmatic dependent launches of (a); the chain is
//   graph-replayed by the C-ABI.
//
// Node ids are assigned in tile raster order, so the min-id root of a class is
// its min raster position (forest.hpp:44-111 invariant parent <= self), which
// is the component's min pixel: the reference's canonical label
// (image.hpp:41-43) after convert_ids (local_labeler.cpp:102-112).
//
// The reference's block config / variant are honoured for validation and
// strategy selection; the GPU tile is an internal constant (labels are
// tile-shape invariant: SPEC.md "Variant equivalence", "Scheduler independence").
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>

#include "ccl_device.cuh"
#include "ccl_internal.h"

namespace cclk {

template <int WX_, int WY_, int WPL_ = 1, int RPL_ = 1>
struct Cfg {
    static constexpr int WX = WX_, WY = WY_;  // warps across / down the tile
    static constexpr int WPL = WPL_;          // 32-px row words per lane
    static constexpr int RPL = RPL_;          // rows per lane (2: a lane owns a 2-row band)
    static constexpr int WPR = WX * WPL;      // row words per tile row
    static constexpr int TW = 32 * WPR, TH = 32 * RPL * WY, NT = 32 * WX * WY, NWARP = WX * WY;
    static constexpr int PX = TW * TH;
    static constexpr int MAXF = 2 * TW + 2 * TH;  // bound on seam-touching roots (one per boundary run)
    // work buffer (global) per tile, in u32 words:
    //   head [nF, nodes, -, -] | row-word masks | per-word node prefix (u16) |
    //   seam-root list (global index; resolved label after k_resolve) |
    //   seam records (local root of every border pixel: top, bottom, left, right) | node table (u16)
    static constexpr int MW = TH * WPR;  // row words
    static constexpr int W_HEAD = 0;
    static constexpr int W_MASK = 4;
    static constexpr int W_PF = W_MASK + MW;
    static constexpr int BSW = (TH / 2) * WPR;  // band-start words (band kernel (a) only)
    static constexpr int W_BS = W_PF + MW / 2;
    static constexpr int W_LIST = W_BS + BSW;
    static constexpr int W_REC = W_LIST + MAXF;
    static constexpr int W_TBL = W_REC + 2 * TW + 2 * TH;
    static constexpr int TILE_WORDS = (W_TBL + PX / 2 + 31) / 32 * 32;  // table sized for pixel nodes; 128B lines
    static_assert((2 * MAXF) % 32 == 0, "per-tile forest segments are whole 128B lines");
    static constexpr int S1_BYTES = (W_BS - W_HEAD) * 4;         // head + masks + prefixes: one copy
    static constexpr int S1_BYTES_BAND = (W_LIST - W_HEAD) * 4;  // ... + band starts (band kernel (a))
    // After the tiles: the COMPACT global forest, one {parent, key} u32 pair per
    // possible seam-touching root (node n = tile * MAXF + rank, key = the root's
    // global raster index), then the strip-mode area (edge rows + their roots).
    static_assert(TW <= 256 && TH <= 256, "TMA box dims are limited to 256");
    static_assert(PX <= 0x4000, "positions are 14-bit codes (root entries are 0x8000 | code)");
    static_assert(MW % 8 == 0, "16-byte alignment of the work-buffer sections");
};

// Kernel (a)'s CTA layout; kernels (d), (d2) and the work-buffer layout only
// depend on the tile shape.  Kernel (e) has its own warp layout over the same
// tile (one 32-px word per lane): same TW, TH, MW, MAXF, hence the same work tile.
using TileCfg = Cfg<CCL_TILE_WX, CCL_TILE_WY, CCL_WPL>;
using ECfg = Cfg<CCL_TILE_WX * CCL_WPL, CCL_TILE_WY, 1>;
// 2-row band kernels: (a) lane = band with CCL_BWPL words; (e) lane = band, one word.
using BandCfg = Cfg<TileCfg::WPR / CCL_BWPL, TileCfg::TH / 64, CCL_BWPL, 2>;
using BandECfg = Cfg<TileCfg::WPR, TileCfg::TH / 64, 1, 2>;
static_assert(BandCfg::TW == TileCfg::TW && BandCfg::TH == TileCfg::TH && BandCfg::TILE_WORDS == TileCfg::TILE_WORDS,
              "band kernel (a) writes the same work tiles");
static_assert(BandECfg::TILE_WORDS == TileCfg::TILE_WORDS, "band kernel (e) reads the same work tiles");

// Kernel (a) shared memory, per node granularity (runs: <= PX/2 nodes).
template <class C, bool RUNS, bool BAND = false>
struct ALayout {
    static constexpr int MAXN = RUNS ? C::PX / 2 : C::PX;
    static constexpr int P_OFF = 0;                                        // u16 parents / root codes, then the table
    static constexpr int FB_OFF = P_OFF + MAXN * 2;                        // seam-root bitmap
    static constexpr int M_OFF = FB_OFF + ((MAXN / 32 * 4 + 127) / 128) * 128;  // row-word masks
    static constexpr int PF16_OFF = M_OFF + C::MW * 4;                     // u16 prefixes (contiguous: one bulk store)
    static constexpr int BS_OFF = PF16_OFF + C::MW * 2;                    // band starts (band kernel)
    static constexpr int PF_OFF = BS_OFF + (BAND ? C::BSW * 4 : 0);        // u32 counts / prefixes (row kernel)
    static constexpr int BT_OFF = PF_OFF + (BAND ? 0 : C::MW * 4);         // band totals (+ total)
    static constexpr int FR_OFF = BT_OFF + (BAND && C::WY == 1 ? 0 : 128);  // [count, global idx of seam roots]
    static constexpr int UL_CAP = BAND ? CCL_BULCAP : CCL_ULCAP;           // union pairs per warp
    static constexpr int UL_OFF = ((FR_OFF + (1 + C::MAXF) * 4) + 127) / 128 * 128;
    static constexpr int BN_OFF = UL_OFF + C::NWARP * UL_CAP * 4;          // border-pixel nodes (band kernel)
    static constexpr int BN_END = BN_OFF + (BAND ? (C::MAXF * 2 + 127) / 128 * 128 : 0);
    // band kernel with CCL_AIMG_OVERLAY: the TMA tile lands in the node table
    // (dead between the table's bulk store and the next coarse scan)
    static constexpr bool OVL = BAND && CCL_AIMG_OVERLAY;
    static_assert(!OVL || MAXN * 2 >= C::PX, "tile bytes fit in the node table");
    static constexpr int IMG_OFF = OVL ? P_OFF : BN_END;
    static constexpr int BAR_OFF = OVL ? BN_END : IMG_OFF + C::PX;
    // band kernel: the prefix counts live in the seam-root list (written only
    // after the last prefix read and a barrier); its TMA load is unswizzled,
    // so a 128 B base alignment is enough
    static constexpr int CNT_OFF = BAND ? FR_OFF + 16 : PF_OFF;
    static constexpr int ALIGN = BAND ? 128 : 1024;
    static constexpr int SMEM = BAR_OFF + (BAND ? 16 : 64) + ALIGN;  // + runtime base alignment slack
    static_assert(!BAND || (C::TH / 2) * C::WX * 4 + 16 <= C::MAXF * 4, "band counts fit in the seam-root list");
};

// Kernel (e) shared memory: 3 head/mask stages, 2 table/label stages, staging.
template <class C, bool RUNS, bool BAND = false>
struct ELayout {
    static constexpr int S1B = BAND ? C::S1_BYTES_BAND : C::S1_BYTES;
    static constexpr int S1 = (S1B + 127) / 128 * 128;
    // u16 node table; band tiles with more than TBLN nodes (checkerboard-like)
    // read their table from the work tile in global memory instead
    static constexpr int TBLN = BAND ? CCL_ETBL : (RUNS ? C::PX / 2 : C::PX);
    static constexpr int TBLB = TBLN * 2;
    static constexpr int S2 = (C::MAXF * 4 + TBLB + 127) / 128 * 128;     // resolved labels + table
    static constexpr int S1_OFF = 0;
    static constexpr int S2_OFF = S1_OFF + 3 * S1;
    static constexpr int STG_OFF = ((S2_OFF + 2 * S2) + 1023) / 1024 * 1024;
    static constexpr int BAR_OFF = STG_OFF + C::NWARP * C::WPL * C::RPL * 4096;
    static constexpr int SMEM = BAR_OFF + 64 + 1024;
};

// Node entries (u16): a non-root holds its parent id (< 0x8000); a root holds
// its CODE = kRoot | position-in-tile, or kRoot | kSeam | rank once it is
// known to touch a tile side (rank = index in the tile's seam-root list).
// The node table handed to kernel (e) is the array of every node's root code.
constexpr uint32_t kRoot = 0x8000u;
constexpr uint32_t kSeam = 0x4000u;
constexpr uint32_t kCode = 0x3FFFu;

// Phase timing of kernel (a) (experiment builds with -DCCL_PHASES=1 only):
// thread 0 accumulates clock64() deltas between consecutive barriers.
#if CCL_PHASES
__device__ unsigned long long g_phase_cycles[16];
#define CCL_PH_INIT() unsigned long long ph_t0 = clock64(), ph_acc[16] = {}
#define CCL_PH(k)                                         \
    do {                                                  \
        if (threadIdx.x == 0) {                           \
            const unsigned long long t1_ = clock64();     \
            ph_acc[k] += t1_ - ph_t0;                     \
            ph_t0 = t1_;                                  \
        }                                                 \
    } while (0)
#define CCL_PH_DONE()                                                              \
    do {                                                                           \
        if (threadIdx.x == 0)                                                      \
            for (int k_ = 0; k_ < 16; ++k_) atomicAdd(&g_phase_cycles[k_], ph_acc[k_]); \
    } while (0)
#else
#define CCL_PH_INIT() (void)0
#define CCL_PH(k) (void)0
#define CCL_PH_DONE() (void)0
#endif

// Node parents are u16; unions are CAS min-unions on the 16-bit entries.
using node_t = uint16_t;
__device__ __forceinline__ uint32_t nfind(node_t* P, uint32_t x, Ctr& m) {
    volatile node_t* vP = P;
    uint32_t p = vP[x];
    while (!(p & kRoot)) {
        m.step();
        const uint32_t gp = vP[p];
        if (gp & kRoot) return p;
        vP[x] = node_t(gp);  // path halving (ancestor only)
        x = gp;
        p = vP[x];
    }
    return x;
}
// nfind that also hands back the root's entry (its code): no re-read by the caller
// Band kernel node HANDLES: a node's handle is its id << kNS = the byte offset
// of its entry in the table, so a parent entry addresses its parent's entry
// directly (LDS [handle + base], no index arithmetic per hop of a walk).
// Handles stay below 0x2000 (4096 nodes), clear of the kRoot / kSeam code bits.
constexpr uint32_t kNS = 1u;
__device__ __forceinline__ volatile node_t* nslot(node_t* P, uint32_t h) {
    return reinterpret_cast<volatile node_t*>(reinterpret_cast<char*>(P) + h);
}
__device__ __forceinline__ uint32_t nfind_code(node_t* P, uint32_t x, uint32_t& code, Ctr& m) {
    uint32_t p = *nslot(P, x);
    while (!(p & kRoot)) {
        m.step();
        const uint32_t gp = *nslot(P, p);
        if (gp & kRoot) {
            code = gp;
            return p;
        }
        *nslot(P, x) = node_t(gp);  // path halving (ancestor only)
        x = gp;
        p = *nslot(P, x);
    }
    code = p;
    return x;
}
__device__ __forceinline__ void nunion(node_t* P, uint32_t a, uint32_t b, Ctr& m) {
    volatile node_t* vP = P;
    for (;;) {
        a = nfind(P, a, m);
        b = nfind(P, b, m);
        if (a == b) return;
        if (a < b) { const uint32_t t = a; a = b; b = t; }
        const uint32_t ca = vP[a];  // a's root code: link a below b unless a got linked meanwhile
        if (ca & kRoot) m.cas();
        if ((ca & kRoot) && atomicCAS(reinterpret_cast<unsigned short*>(P + a), static_cast<unsigned short>(ca),
                                      static_cast<unsigned short>(b)) == ca)
            return;
    }
}

// Instrumented builds: counters of a warp flushed to the per-tile grid / the
// per-phase totals (layout in ccl_internal.h, Geo::metrics).  Whole warps only.
__device__ __forceinline__ void metrics_tile(const Geo& g, uint32_t t, Ctr& m) {
#if CCL_METRICS
    const uint32_t f = __reduce_add_sync(0xffffffffu, m.f), c = __reduce_add_sync(0xffffffffu, m.c);
    if ((threadIdx.x & 31) == 0 && g.metrics) {
        if (f) atomicAdd(g.metrics + 8 + 2 * size_t(t), f);
        if (c) atomicAdd(g.metrics + 8 + 2 * size_t(t) + 1, c);
    }
    m.f = m.c = 0;
#endif
}
__device__ __forceinline__ void metrics_phase(const Geo& g, int k, Ctr& m) {
#if CCL_METRICS
    const uint32_t f = __reduce_add_sync(0xffffffffu, m.f), c = __reduce_add_sync(0xffffffffu, m.c);
    if ((threadIdx.x & 31) == 0 && g.metrics) {
        unsigned long long* ph = reinterpret_cast<unsigned long long*>(g.metrics);
        if (f) atomicAdd(ph + k, static_cast<unsigned long long>(f));
        if (c) atomicAdd(ph + k + 1, static_cast<unsigned long long>(c));
    }
    m.f = m.c = 0;
#endif
}

// Dynamic shared memory rounded up to ALIGN bytes (1024 B: 128B-swizzled TMA
// tiles).  The base is rounded as a 32-bit shared address, passed through an
// empty asm and converted back: the compiler still sees a shared pointer
// (LDS/STS with 32-bit addresses, not generic LD/ST) but can no longer
// re-derive the base from SR_CgaCtaId inside every loop (4 instructions per
// trip under kernel (a)'s register cap); it keeps it in a uniform register.
template <uint32_t ALIGN = 1024>
__device__ __forceinline__ uint8_t* aligned_smem() {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint32_t a = (smem_u32(smem_raw) + (ALIGN - 1)) & ~(ALIGN - 1);
    asm volatile("" : "+r"(a));
    return static_cast<uint8_t*>(__cvta_shared_to_generic(a));
}

// Work-buffer view of one tile (tile index tg over frames x tile rows x tile cols).
template <class C>
__device__ __forceinline__ uint32_t* work_tile(uint32_t* work, size_t tg) {
    return work + tg * size_t(C::TILE_WORDS);
}

template <class C>
__device__ __forceinline__ Forest forest_of(uint32_t* work, uint32_t ntiles) {
    return Forest{work + size_t(ntiles) * C::TILE_WORDS};
}
template <class C>
__device__ __forceinline__ uint32_t* strip_area(uint32_t* work, uint32_t ntiles) {
    return work + size_t(ntiles) * C::TILE_WORDS + 2 * size_t(ntiles) * C::MAXF;
}

// Linear tile index -> (tx, ty, frame).
struct TileId {
    uint32_t tx, ty, fz;
};
__device__ __forceinline__ TileId tile_of(uint32_t t, const Geo& g) {
    const uint32_t per = g.ntx * g.nty;
    const uint32_t fz = t / per, r = t - fz * per;
    const uint32_t ty = r / g.ntx;
    return TileId{r - ty * g.ntx, ty, fz};
}
// Persistent tile walk t, t + G, t + 2G, ... without a division per step:
// the stride G is decomposed once into (frames, rows, columns) of tiles.
struct TileWalk {
    TileId cur, step;
    uint32_t ntx, nty;
    __device__ __forceinline__ TileWalk(uint32_t t0, uint32_t G, const Geo& g)
        : cur(tile_of(t0, g)), step(tile_of(G, g)), ntx(g.ntx), nty(g.nty) {}
    __device__ __forceinline__ void advance() {
        cur.tx += step.tx;
        cur.ty += step.ty;
        cur.fz += step.fz;
        if (cur.tx >= ntx) { cur.tx -= ntx; ++cur.ty; }
        if (cur.ty >= nty) { cur.ty -= nty; ++cur.fz; }
    }
};

// Programmatic dependent launch: a dependent grid may be launched while its
// predecessor drains; it must wait for the predecessor before touching its output.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_store_hint(void* gdst, const void* ssrc, uint32_t bytes, uint64_t pol) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
                 "r"(smem_u32(ssrc)), "r"(bytes), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void bulk_load(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(sdst)),
                 "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// Node starts of one row word: runs (a run continuing from the word on its
// left is not restarted, so a tile-row run is ONE node) or fg pixels.
template <bool RUNS>
__device__ __forceinline__ uint32_t word_starts(uint32_t m, uint32_t lm) {
    if (!RUNS) return m;
    const uint32_t cont = (lm >> 31) & m & 1u;
    return m & ~((m << 1) | cont);
}

// Inclusive warp scan: shfl.up hands back whether the source lane exists, so
// each step is a shuffle and a predicated add (no lane compare and select).
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1)
        asm("{\n\t.reg .u32 t;\n\t.reg .pred p;\n\t"
            "shfl.sync.up.b32 t|p, %0, %1, 0, 0xffffffff;\n\t"
            "@p add.u32 %0, %0, t;\n\t}"
            : "+r"(v)
            : "r"(d));
    return v;
}

// Raster-order node prefix of every row word of the tile.  Each lane owns
// word (row, wx) with `cnt` node starts; CNT is scratch for the counts.
// Returns the number of nodes that start before this word; *total = nodes in
// the tile.  Two barriers (one when the tile is a single warp row).
template <class C>
__device__ __forceinline__ uint32_t tile_prefix(uint32_t cnt, uint32_t* CNT, uint32_t* BT, int row, int wx, int wy,
                                                int lane, uint32_t* total) {
    CNT[row * C::WX + wx] = cnt;
    __syncthreads();
    uint32_t left = 0, rowtot = 0;
#pragma unroll
    for (int w = 0; w < C::WX; ++w) {
        const uint32_t c = CNT[row * C::WX + w];
        left += (w < wx) ? c : 0u;
        rowtot += c;
    }
    const uint32_t inc = warp_incl_scan(rowtot);
    uint32_t band = 0, tot;
    if (C::WY == 1) {
        tot = __shfl_sync(0xffffffffu, inc, 31);
    } else {
        if (wx == 0 && lane == 31) BT[wy] = inc;
        __syncthreads();
        tot = 0;
#pragma unroll
        for (int b = 0; b < C::WY; ++b) {
            const uint32_t t = BT[b];
            band += (b < wy) ? t : 0u;
            tot += t;
        }
    }
    *total = tot;
    return band + inc - rowtot + left;
}

// Index of the lowest set bit of x != 0 (FLO only; __ffs costs a BREV more on the XU pipe).
__device__ __forceinline__ uint32_t lowbit(uint32_t x) { return 31u - __clz(x & (0u - x)); }

// Id of the node holding bit b of a word with starts st and prefix pfx (a bit
// before the word's first start belongs to the node continuing from the left).
__device__ __forceinline__ uint32_t node_of(uint32_t pfx, uint32_t st, uint32_t b) {
    return pfx + __popc(st << (31u - b)) - 1u;  // the starts at or below bit b
}
// Bits b of o such that some bit of o lies strictly below b inside the same
// run of m (o must be a subset of m): the carry-in vector of m + o, within m.
__device__ __forceinline__ uint32_t lower_in_run(uint32_t m, uint32_t o) {
    return ((m + o) ^ m ^ o) & m;
}

template <class C>
__device__ __forceinline__ uint32_t pos_gidx(uint32_t pos, uint32_t x0, uint32_t y0, const Geo& g) {
    constexpr int SH = __builtin_ctz(C::TW);
    return (g.row0 + y0 + (pos >> SH)) * g.W + x0 + (pos & (C::TW - 1));  // global raster index (convert_ids)
}

// ------------------------------------------------------------------ kernel (a)(b)(c)
// Persistent: CTA b labels tiles b, b + G, b + 2G, ... (G = gridDim.x).  The
// next tile's image is TMA-loaded into the staging buffer as soon as the
// current tile's masks are built, so the load overlaps a whole tile of work.
template <class C, int VAR, bool TMA>
__global__ void __launch_bounds__(C::NT, CCL_MINB)
    k_local(const __grid_constant__ CUtensorMap tm_img, const uint8_t* img, uint32_t* L, uint32_t* work, Geo g,
            uint32_t ntiles) {
    constexpr bool RUNS = (VAR == 0 || VAR == 1);
    using A = ALayout<C, RUNS>;
    uint8_t* smem = aligned_smem();
    node_t* P = reinterpret_cast<node_t*>(smem + A::P_OFF);
    uint32_t* FB = reinterpret_cast<uint32_t*>(smem + A::FB_OFF);
    uint32_t* M = reinterpret_cast<uint32_t*>(smem + A::M_OFF);
    uint16_t* PF16 = reinterpret_cast<uint16_t*>(smem + A::PF16_OFF);
    uint32_t* CNT = reinterpret_cast<uint32_t*>(smem + A::CNT_OFF);
    uint32_t* BT = reinterpret_cast<uint32_t*>(smem + A::BT_OFF);
    uint32_t* FR = reinterpret_cast<uint32_t*>(smem + A::FR_OFF);
    uint8_t* IMG = smem + A::IMG_OFF;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + A::BAR_OFF);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wx = warp % C::WX, wy = warp / C::WX;
    const int row = wy * 32 + lane;
    const int col0 = wx * 32 * C::WPL;  // first pixel column of this lane's words
    const int wc0 = wx * C::WPL;        // first word column
    const Forest fst = forest_of<C>(work, ntiles);
    uint32_t* SE = strip_area<C>(work, ntiles);  // strip mode: edge-row nodes [top W | bottom W]

    auto issue_at = [&](const TileId& q) {  // TMA 2-D tile load, OOB -> 0 == background
        mbar_expect_tx(bar, C::PX);
        if (CCL_HINTS)
            tma_load_3d_hint(IMG, &tm_img, int(q.tx * C::TW), int(q.ty * C::TH), int(q.fz), bar, policy_evict_first());
        else
            tma_load_3d(IMG, &tm_img, int(q.tx * C::TW), int(q.ty * C::TH), int(q.fz), bar);
    };
    if (TMA && tid == 0) {
        prefetch_tmap(&tm_img);
        mbar_init(bar, 1);
        if (blockIdx.x < ntiles) issue_at(tile_of(blockIdx.x, g));
    }

    CCL_PH_INIT();
    Ctr mc;  // instrumented builds: this thread's find steps / CAS attempts of the current tile
    uint32_t it = 0;
    TileWalk walk(blockIdx.x, gridDim.x, g);
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it, walk.advance()) {
        const TileId ti = walk.cur;
        const uint32_t tx = ti.tx, ty = ti.ty;
        const uint32_t x0 = tx * C::TW, y0 = ty * C::TH;
        uint32_t* wt = work_tile<C>(work, t);

        // the previous tile's bulk stores must have read P / M / PF16, and its
        // last phase must be done with every smem array
        if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncthreads();
        CCL_PH(0);
        for (int i = tid; i < A::MAXN / 32; i += C::NT) FB[i] = 0u;
        if (tid == 0) FR[0] = 0u;

        // ---- row-word foreground masks (byte == 1)
        if (TMA) {
            mbar_wait(bar, it & 1u);
            constexpr int CPR = C::TW / 16;
            uint16_t* M16 = reinterpret_cast<uint16_t*>(M);
#pragma unroll
            for (int c = tid; c < C::TH * CPR; c += C::NT) {
                const uint4 q = *reinterpret_cast<const uint4*>(IMG + c * 16);
                M16[c] = static_cast<uint16_t>(eq1_mask16(q));
            }
        } else {
            const uint32_t gy = y0 + row;
#pragma unroll
            for (int k = 0; k < C::WPL; ++k) {
                uint32_t mm = 0u;
                if (gy < g.H) {
                    const uint8_t* src = img + size_t(ti.fz) * g.frame_pitch + size_t(gy) * g.img_pitch;
                    for (int b = 0; b < 32; ++b) {
                        const uint32_t gx = x0 + col0 + 32 * k + b;
                        if (gx < g.W && src[gx] == 1) mm |= 1u << b;
                    }
                }
                M[row * C::WPR + wx * C::WPL + k] = mm;
            }
        }
        __syncthreads();
        CCL_PH(1);
        if (TMA && tid == 0 && t + gridDim.x < ntiles) {  // staging buffer is dead: prefetch the next tile
            TileWalk nx = walk;
            nx.advance();
            issue_at(nx.cur);
        }

        // this lane's WPL row words (row, wc0 + k), their left / upper neighbours
        uint32_t m[C::WPL], lm[C::WPL], um[C::WPL], lum[C::WPL], st[C::WPL], ust[C::WPL];
#pragma unroll
        for (int k = 0; k < C::WPL; ++k) {
            const int wc = wc0 + k;
            m[k] = M[row * C::WPR + wc];
            um[k] = row > 0 ? M[(row - 1) * C::WPR + wc] : 0u;
            lm[k] = k > 0 ? m[k - 1] : (wc > 0 ? M[row * C::WPR + wc - 1] : 0u);
            lum[k] = k > 0 ? um[k - 1] : ((row > 0 && wc > 0) ? M[(row - 1) * C::WPR + wc - 1] : 0u);
            st[k] = word_starts<RUNS>(m[k], lm[k]);
            ust[k] = word_starts<RUNS>(um[k], lum[k]);
        }

        // ---- coarse row scan: node ids in tile raster order
        uint32_t nodes, cnt = 0, ucnt0 = 0;
#pragma unroll
        for (int k = 0; k < C::WPL; ++k) cnt += __popc(st[k]);
        const uint32_t pfx0 = tile_prefix<C>(cnt, CNT, BT, row, wx, wy, lane, &nodes);
        uint32_t upfx0 = __shfl_up_sync(0xffffffffu, pfx0, 1);
        if (lane == 0) {  // words above belong to the warp band above: prefix from the counts
            uint32_t rest = 0, left = 0;
#pragma unroll
            for (int w = 0; w < C::WX; ++w) {
                rest += (row > 0 && w >= wx) ? CNT[(row - 1) * C::WX + w] : 0u;
                left += (w < wx) ? CNT[row * C::WX + w] : 0u;
            }
            upfx0 = pfx0 - left - rest;
        }
        (void)ucnt0;
        uint32_t pfx[C::WPL], upfx[C::WPL];
#pragma unroll
        for (int k = 0; k < C::WPL; ++k) {
            pfx[k] = k > 0 ? pfx[k - 1] + __popc(st[k - 1]) : pfx0;
            upfx[k] = k > 0 ? upfx[k - 1] + __popc(ust[k - 1]) : upfx0;
            PF16[row * C::WPR + wc0 + k] = uint16_t(pfx[k]);
        }

        // ---- init + coarse column scan (plain stores, no atomics): every node is
        // its own parent, except that C2FL links a run to the upper run holding
        // its first overlap inside its word and CC2FL links a pixel to the pixel above.
        uint32_t o[C::WPL], os[C::WPL], first[C::WPL];
#pragma unroll
        for (int k = 0; k < C::WPL; ++k) {
            o[k] = m[k] & um[k];
            const uint32_t ocont = (o[k] & 1u) & ((lm[k] & lum[k]) >> 31);  // overlap continuing from the left
            os[k] = (o[k] & ~(o[k] << 1)) & ~ocont;                       // one bit per (node, upper node) overlap
            first[k] = 0u;                                                // overlaps handled by a coarse link
            if (VAR == 0) first[k] = os[k] & ~lower_in_run(m[k], o[k]) & ~((st[k] & 1u) ? 0u : (m[k] & ~(m[k] + 1u)));
            if (VAR == 2) first[k] = o[k];
            const uint32_t rowpos = uint32_t(row * C::TW + col0 + 32 * k);
            // every node starts as a root carrying its position ...
            uint16_t* dst = P + pfx[k];
            uint32_t tt = st[k];
            while (tt) {
                const uint32_t b = __ffs(tt) - 1;
                tt &= tt - 1;
                *dst++ = node_t(kRoot | (rowpos + b));
            }
            // ... then the coarse links overwrite the linked ones: one per
            // first-overlap bit f (C2FL) / fg pixel with fg above (CC2FL)
            uint32_t ff = first[k];
            while (ff) {
                const uint32_t f = __ffs(ff) - 1;
                ff &= ff - 1;
                P[node_of(pfx[k], st[k], f)] = node_t(node_of(upfx[k], ust[k], f));
            }
        }
        // refinement pairs (run, upper run) not covered by a coarse link go to
        // this warp's union list, so the unions are spread over all 32 lanes
        // instead of serialising on the lanes that own many of them
        uint32_t U[C::WPL];
        uint32_t cu = 0;
#pragma unroll
        for (int k = 0; k < C::WPL; ++k) {
            U[k] = RUNS ? (os[k] & ~first[k]) : 0u;
            cu += __popc(U[k]);
        }
        uint32_t* UL = reinterpret_cast<uint32_t*>(smem + A::UL_OFF) + warp * A::UL_CAP;
        uint32_t nul;
        {
            uint32_t inc = cu;
#pragma unroll
            for (int j = 1; j < 32; j <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, j);
                if (lane >= j) inc += y;
            }
            const bool fits = inc <= uint32_t(A::UL_CAP);
            nul = __reduce_max_sync(0xffffffffu, fits ? inc : 0u);  // entries actually listed
            if (fits) {  // all of this lane's pairs fit: list them
                uint32_t* dst = UL + (inc - cu);
#pragma unroll
                for (int k = 0; k < C::WPL; ++k) {
                    while (U[k]) {
                        const uint32_t b = __ffs(U[k]) - 1;
                        U[k] &= U[k] - 1;
                        *dst++ = node_of(pfx[k], st[k], b) | (node_of(upfx[k], ust[k], b) << 16);
                    }
                }
            }
        }
        __syncthreads();
        CCL_PH(2);

        // ---- pointer jumping over the coarse forest (balanced over node ids):
        // coarse links form vertical chains; each round halves their length.
        if (VAR == 0 || VAR == 2) {
#pragma unroll 1
            for (int j = 0; j < CCL_JUMP; ++j) {
                volatile node_t* vP = P;
                for (uint32_t id = tid; id < nodes; id += C::NT) {
                    const uint32_t p = vP[id];
                    const uint32_t pp = (p & kRoot) ? p : vP[p];
                    if (!(p & kRoot)) mc.step();
                    if (!(pp & kRoot)) vP[id] = node_t(pp);
                }
                // no barrier after the last round: jumps and unions only ever
                // replace an entry by an ancestor, and unions CAS root entries only
                if (j + 1 < CCL_JUMP) __syncthreads();
                CCL_PH(3);
            }
        }

        // ---- refinement: min-union of the adjacencies the coarse scans did not link
        {
            for (uint32_t k = lane; k < nul; k += 32) {
                const uint32_t pr = UL[k];
                nunion(P, pr & 0xFFFFu, pr >> 16, mc);
            }
#pragma unroll
            for (int k = 0; k < C::WPL; ++k) {
                uint32_t Uk = RUNS ? U[k] : ((VAR == 3) ? o[k] : 0u);  // NC2FL: every vertical pixel pair
                while (Uk) {                                          // pairs that did not fit in the list
                    const uint32_t b = __ffs(Uk) - 1;
                    Uk &= Uk - 1;
                    nunion(P, node_of(pfx[k], st[k], b), node_of(upfx[k], ust[k], b), mc);
                }
                if (!RUNS) {  // horizontal pixel pairs (incl. the word boundary), minus closed 2x2 squares
                    const uint32_t hm = m[k] & ((m[k] << 1) | ((lm[k] >> 31) & 1u));
                    const uint32_t hu = um[k] & ((um[k] << 1) | ((lum[k] >> 31) & 1u));
                    uint32_t hp = (VAR == 2) ? (hm & ~hu) : hm;
                    while (hp) {
                        const uint32_t b = __ffs(hp) - 1;
                        hp &= hp - 1;
                        const uint32_t id = node_of(pfx[k], st[k], b);
                        nunion(P, id, id - 1, mc);  // the left neighbour is the previous fg pixel in raster order
                    }
                }
            }
        }
        __syncthreads();
        CCL_PH(4);

        // ---- seam-touching roots (components reaching a side that faces a
        // neighbour tile/strip), balanced over all threads: each is marked once
        // in the FB bitmap; the winner ranks it, registers it in the global
        // forest and replaces its code by kRoot | kSeam | rank.
        const bool has_top = ty > 0 || g.edge_above;
        const bool has_bot = ty + 1 < g.nty || g.edge_below;
        const bool has_left = tx > 0, has_right = tx + 1 < g.ntx;
        {
            const uint32_t top_n = PF16[C::WPR];               // nodes in row 0
            const uint32_t bot0 = PF16[(C::TH - 1) * C::WPR];  // first node of the last row
            const uint32_t n1 = has_top ? top_n : 0u;
            const uint32_t n2 = n1 + (has_bot ? nodes - bot0 : 0u);
            const uint32_t n3 = n2 + (has_left ? uint32_t(C::TH) : 0u);
            const uint32_t n4 = n3 + (has_right ? uint32_t(C::TH) : 0u);
            for (uint32_t i = tid; i < n4; i += C::NT) {
                uint32_t id;
                if (i < n1) {
                    id = i;
                } else if (i < n2) {
                    id = bot0 + (i - n1);
                } else if (i < n3) {
                    const uint32_t r = i - n2;
                    if (!(M[r * C::WPR] & 1u)) continue;
                    id = PF16[r * C::WPR];
                } else {
                    const uint32_t r = i - n3;
                    const uint32_t wl = M[r * C::WPR + C::WPR - 1];
                    if (!(wl >> 31)) continue;
                    const uint32_t wll = C::WPR > 1 ? M[r * C::WPR + C::WPR - 2] : 0u;
                    id = node_of(PF16[r * C::WPR + C::WPR - 1], word_starts<RUNS>(wl, wll), 31);
                }
                uint32_t x = id, p = P[id];
                while (!(p & kRoot)) {
                    mc.step();
                    x = p;
                    p = P[x];
                }
                const uint32_t bit = 1u << (x & 31);
                if (!(atomicOr(&FB[x >> 5], bit) & bit)) {  // the root's entry still holds its position
                    const uint32_t k = atomicAdd(FR, 1u);
                    const uint32_t n = t * uint32_t(C::MAXF) + k;  // compact global node
                    fst.f[2 * size_t(n)] = n;
                    fst.f[2 * size_t(n) + 1] = pos_gidx<C>(p & kCode, x0, y0, g);
                    FR[1 + k] = n;
                    P[x] = node_t(kRoot | kSeam | k);
                }
            }
        }
        __syncthreads();
        CCL_PH(5);

        // ---- unification + node table in one pass: every node's entry becomes
        // its root's code.  A walk stops at the first code it meets, so nodes
        // already rewritten (parents always have smaller ids) end walks early.
        {
            volatile node_t* vP = P;
            // two hops without branches (selects; most nodes are within two hops of
            // their root after the jump round), a loop only for deeper chains
            for (uint32_t id = tid; id < nodes; id += C::NT) {
                const uint32_t p = vP[id];
                const uint32_t q = (p & kRoot) ? p : uint32_t(vP[p & 0x7FFFu]);
                uint32_t r = (q & kRoot) ? q : uint32_t(vP[q & 0x7FFFu]);
                if (!(r & kRoot)) {
                    do {
                        mc.step();
                        r = vP[r];
                    } while (!(r & kRoot));
                }
                if (!(p & kRoot)) vP[id] = node_t(r);
            }
        }
        const uint32_t nf = FR[0];
        if (tid == 0) {
            wt[C::W_HEAD + 0] = nf;
            wt[C::W_HEAD + 1] = nodes;
        }
        fence_proxy_async_smem();
        __syncthreads();
        CCL_PH(7);
        if (tid == 0) {
            const uint64_t keep = CCL_HINTS ? policy_evict_last() : policy_evict_normal();  // hand-off to (e)
            bulk_store_hint(wt + C::W_MASK, M, C::MW * 6, keep);  // masks + u16 prefixes (contiguous)
            if (nodes) bulk_store_hint(wt + C::W_TBL, P, (nodes * 2 + 15) & ~15u, keep);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }

        // ---- seam records (every border pixel: its root's compact global node
        // or background) for kernel (d); strip-edge rows also into the strip
        // area for the strip seam export
        const uint16_t* T = P;
        for (int i = tid; i < 2 * C::TW + 2 * C::TH; i += C::NT) {
            int r, c;
            if (i < C::TW) { r = 0; c = i; }
            else if (i < 2 * C::TW) { r = C::TH - 1; c = i - C::TW; }
            else if (i < 2 * C::TW + C::TH) { r = i - 2 * C::TW; c = 0; }
            else { r = i - 2 * C::TW - C::TH; c = C::TW - 1; }
            const int w = c >> 5, b = c & 31;
            const uint32_t wm = M[r * C::WPR + w];
            uint32_t v = kBG;
            if ((wm >> b) & 1u) {
                const uint32_t wl = w > 0 ? M[r * C::WPR + w - 1] : 0u;
                const uint32_t code = T[node_of(PF16[r * C::WPR + w], word_starts<RUNS>(wm, wl), uint32_t(b))];
                if (code & kSeam) v = FR[1 + (code & kCode)];  // sides facing the image edge are not seams
            }
            wt[C::W_REC + i] = v;
            if (i < 2 * C::TW) {
                const bool top = i < C::TW;
                const bool edge = top ? (ty == 0 && g.edge_above) : (ty + 1 == g.nty && g.edge_below);
                const uint32_t gx = x0 + c;
                if (edge && gx < g.W) SE[(top ? 0u : g.W) + gx] = v;
            }
        }
        metrics_tile(g, t, mc);
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    CCL_PH_DONE();
    pdl_trigger();
}

// ------------------------------------------------------------------ kernel (a), 2-row bands (C2FL)
// Same phases as k_local, on 2-row BAND RUNS instead of row runs: within rows
// (2b, 2b+1) the 4-connected pieces are column intervals where every column
// has a foreground pixel and consecutive columns share a foreground row
// (lk = t & t>>1 | u & u>>1), so a band run's start mask is pure bit work and
// the prefix / node_of machinery carries over unchanged with about half the
// nodes of row runs (at d = 0.5).  A band run's minimum pixel -- its code when
// it is a root -- is its first top-row pixel, else its first column in the
// bottom row; node ids are not in code order inside a band, so unions compare
// root codes (the class root is the node of the component's minimum pixel,
// forest.hpp:98-111 restated on positions).  Lane = band, one word per lane.
__device__ __forceinline__ uint32_t band_starts(uint32_t t, uint32_t u, uint32_t tl, uint32_t ul) {
    const uint32_t lk = (t & (t >> 1)) | (u & (u >> 1));          // column c linked to c + 1
    const uint32_t cl = (((tl >> 31) & t) | ((ul >> 31) & u)) & 1u;  // bit 0 linked to the word on the left
    return (t | u) & ~((lk << 1) | cl);
}
// Segments of a word start at the bits of `starts` and run up to the next
// start.  seg_first: the first set bit of x in every segment (bits below the
// first start belong to the word on the left and yield none).  A carry
// injected at every start runs through the zeros of x and stops at the
// segment's first set bit; the bit before each start is forced to 0 in ~x, so
// no carry crosses into the next segment.
__device__ __forceinline__ uint32_t seg_first(uint32_t x, uint32_t starts) {
    return x & ((~x & ~(starts >> 1)) + starts);
}
// seg_back: the bits of every segment that hold a set bit of x at or after
// them (the region below the first start is a segment too).  On the
// bit-reversed word this is a segmented prefix-OR: the bits before a segment's
// first set bit are the carry chain of the same addition (carry-in bits
// shifted down), and an empty segment's chain ends on its last bit.  rs =
// (brev(starts) << 1) | 1 and re = brev(starts) | bit 31: segment starts and
// ends of the reversed word (shared by every scan over the same starts).
__device__ __forceinline__ uint32_t seg_back(uint32_t x, uint32_t rs, uint32_t re) {
    const uint32_t xr = __brev(x), y = ~xr & ~re, r = y + rs;
    const uint32_t chain = (r ^ y ^ rs) >> 1, emp = r & ~xr & re;
    return __brev(~(chain | emp));
}
template <class C>
__device__ __forceinline__ uint32_t band_starts_at(const uint32_t* M, int band, int w) {
    const uint32_t t = M[(2 * band) * C::WPR + w], u = M[(2 * band + 1) * C::WPR + w];
    const uint32_t tl = w > 0 ? M[(2 * band) * C::WPR + w - 1] : 0u, ul = w > 0 ? M[(2 * band + 1) * C::WPR + w - 1] : 0u;
    return band_starts(t, u, tl, ul);
}
// Min-union on root codes (positions): the root whose code is larger is
// linked below the other with a CAS on its entry.
__device__ __forceinline__ void nunion_pos(node_t* P, uint32_t a, uint32_t b, Ctr& m) {
    for (;;) {
        uint32_t ca, cb;
        a = nfind_code(P, a, ca, m);
        b = nfind_code(P, b, cb, m);
        if (a == b) return;
        if ((ca & kCode) < (cb & kCode)) {
            const uint32_t t = a; a = b; b = t;
            const uint32_t tc = ca; ca = cb; cb = tc;
        }
        m.cas();
        if (atomicCAS(const_cast<unsigned short*>(reinterpret_cast<volatile unsigned short*>(nslot(P, a))), static_cast<unsigned short>(ca),
                      static_cast<unsigned short>(b)) == ca)
            return;
    }
}

// Kernel (a) on band runs: CTA `cta` of `ncta` labels tiles cta, cta + ncta, ...
// (the body of the persistent kernel below).
template <class C, bool TMA>
__device__ __forceinline__ void local_band_tiles(const CUtensorMap* tmap, const uint8_t* img, uint32_t* work,
                                                 const Geo& g, uint32_t ntiles, uint32_t cta, uint32_t ncta) {
    static_assert(C::RPL == 2, "lane = 2-row band");
    using A = ALayout<C, true, true>;
    constexpr int WPL = C::WPL, WPR = C::WPR;
    uint8_t* smem = aligned_smem<A::ALIGN>();
    node_t* P = reinterpret_cast<node_t*>(smem + A::P_OFF);
    uint32_t* FB = reinterpret_cast<uint32_t*>(smem + A::FB_OFF);
    uint32_t* M = reinterpret_cast<uint32_t*>(smem + A::M_OFF);
    uint16_t* PF16 = reinterpret_cast<uint16_t*>(smem + A::PF16_OFF);  // per (band, word)
    uint32_t* BS = reinterpret_cast<uint32_t*>(smem + A::BS_OFF);      // band starts per (band, word)
    uint32_t* CNT = reinterpret_cast<uint32_t*>(smem + A::CNT_OFF);
    uint32_t* BT = reinterpret_cast<uint32_t*>(smem + A::BT_OFF);
    uint32_t* FR = reinterpret_cast<uint32_t*>(smem + A::FR_OFF);
    uint8_t* IMG = smem + A::IMG_OFF;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + A::BAR_OFF);
    uint16_t* BN = reinterpret_cast<uint16_t*>(smem + A::BN_OFF);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wx = warp % C::WX, wy = warp / C::WX;
    const int band = wy * 32 + lane;  // rows 2*band, 2*band + 1
    const int r0 = 2 * band, r1 = r0 + 1;
    const int wc0 = wx * WPL;         // first word column of this lane
    const Forest fst = forest_of<C>(work, ntiles);
    uint32_t* SE = strip_area<C>(work, ntiles);

    auto issue_at = [&](const TileId& q) {
        mbar_expect_tx(bar, C::PX);
        tma_load_3d_hint(IMG, tmap, int(q.tx * C::TW), int(q.ty * C::TH), int(q.fz), bar, policy_evict_first());
    };
    if (TMA && tid == 0) {
        prefetch_tmap(tmap);
        mbar_init(bar, 1);
        if (cta < ntiles) issue_at(tile_of(cta, g));
    }

    uint32_t it = 0;
    CCL_PH_INIT();
    Ctr mc;  // instrumented builds: this thread's find steps / CAS attempts of the current tile
    TileWalk walk(cta, ncta, g);
    for (uint32_t t = cta; t < ntiles; t += ncta, ++it, walk.advance()) {
        const TileId ti = walk.cur;
        const uint32_t tx = ti.tx, ty = ti.ty;
        const uint32_t x0 = tx * C::TW, y0 = ty * C::TH;
        uint32_t* wt = work_tile<C>(work, t);

        if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncthreads();
        CCL_PH(8);
#pragma unroll
        for (int k = 0; k < (A::MAXN / 32 + C::NT - 1) / C::NT; ++k)  // fixed trip count (tid < NT)
            if (k * C::NT + tid < A::MAXN / 32) FB[k * C::NT + tid] = 0u;
        if (tid == 0) FR[0] = 0u;

        // ---- row-word foreground masks (byte == 1)
        if (TMA) {
            mbar_wait(bar, it & 1u);
            constexpr int CPR = C::TW / 16;
            uint16_t* M16 = reinterpret_cast<uint16_t*>(M);
            static_assert((C::TH * CPR) % C::NT == 0, "whole mask-build rounds");
            constexpr int KK = C::TH * CPR / C::NT;
            uint4 q[KK];
            uint32_t big = 0u;  // any byte > 1 in this thread's chunks
#pragma unroll
            for (int kk = 0; kk < KK; ++kk) {
                q[kk] = *reinterpret_cast<const uint4*>(IMG + (kk * C::NT + tid) * 16);
                big |= (q[kk].x | q[kk].y | q[kk].z | q[kk].w) & 0xFEFEFEFEu;
            }
            if (CCL_BINFAST && !__any_sync(0xffffffffu, big)) {  // 0/1 images: one multiply per word
#pragma unroll
                for (int kk = 0; kk < KK; ++kk) M16[kk * C::NT + tid] = static_cast<uint16_t>(bin_mask16(q[kk]));
            } else {
#pragma unroll
                for (int kk = 0; kk < KK; ++kk) M16[kk * C::NT + tid] = static_cast<uint16_t>(eq1_mask16(q[kk]));
            }
        } else {  // unaligned pitch: byte loads, one mask word per thread and step
            for (int i = tid; i < C::MW; i += C::NT) {
                const int r = i / WPR, w = i - r * WPR;
                const uint32_t gy = y0 + r;
                uint32_t mm = 0u;
                if (gy < g.H) {
                    const uint8_t* src = img + size_t(ti.fz) * g.frame_pitch + size_t(gy) * g.img_pitch;
                    for (int b = 0; b < 32; ++b) {
                        const uint32_t gx = x0 + 32 * w + b;
                        if (gx < g.W && src[gx] == 1) mm |= 1u << b;
                    }
                }
                M[i] = mm;
            }
        }
        __syncthreads();
        CCL_PH(9);
        if (TMA && !A::OVL && tid == 0 && t + ncta < ntiles) {
            TileWalk nx = walk;
            nx.advance();
            issue_at(nx.cur);
        }

        // ---- band runs of this lane's words: coarse row scan in raster (band, word) order
        uint32_t tm[WPL], um[WPL], bs[WPL], ul0;
        uint32_t cnt = 0;
#pragma unroll
        for (int k = 0; k < WPL; ++k) {
            const int wc = wc0 + k;
            tm[k] = M[r0 * WPR + wc];
            um[k] = M[r1 * WPR + wc];
            const uint32_t tl = k > 0 ? tm[k - 1] : (wc > 0 ? M[r0 * WPR + wc - 1] : 0u);
            const uint32_t ul = k > 0 ? um[k - 1] : (wc > 0 ? M[r1 * WPR + wc - 1] : 0u);
            if (k == 0) ul0 = ul;
            bs[k] = band_starts(tm[k], um[k], tl, ul);
            cnt += __popc(bs[k]);
        }
        uint32_t nodes;
        const uint32_t pfx0 = tile_prefix<C>(cnt, CNT, BT, band, wx, wy, lane, &nodes);
        uint32_t pfx[WPL];
#pragma unroll
        for (int k = 0; k < WPL; ++k) {
            pfx[k] = k > 0 ? pfx[k - 1] + __popc(bs[k - 1]) : pfx0;
            PF16[band * WPR + wc0 + k] = uint16_t(pfx[k]);
            BS[band * WPR + wc0 + k] = bs[k];
        }
        {   // node of every border pixel, in seam-record order [top | bottom | left | right]
            // (0xFFFF = background): top / bottom rows from bands 0 / last by shuffles
            static_assert(WPL == 1 && C::WY == 1, "border nodes: one word per lane, one warp row");
            const uint32_t t0 = __shfl_sync(0xffffffffu, tm[0], 0), s0 = __shfl_sync(0xffffffffu, bs[0], 0);
            const uint32_t p0 = __shfl_sync(0xffffffffu, pfx[0], 0);
            const uint32_t u1 = __shfl_sync(0xffffffffu, um[0], 31), s1 = __shfl_sync(0xffffffffu, bs[0], 31);
            const uint32_t p1 = __shfl_sync(0xffffffffu, pfx[0], 31);
            const int c = 32 * wc0 + lane;
            BN[c] = ((t0 >> lane) & 1u) ? uint16_t(node_of(p0, s0, lane) << kNS) : uint16_t(0xFFFFu);
            BN[C::TW + c] = ((u1 >> lane) & 1u) ? uint16_t(node_of(p1, s1, lane) << kNS) : uint16_t(0xFFFFu);
            if (wc0 == 0) {  // column 0 starts a band run
                BN[2 * C::TW + r0] = (tm[0] & 1u) ? uint16_t(pfx[0] << kNS) : uint16_t(0xFFFFu);
                BN[2 * C::TW + r1] = (um[0] & 1u) ? uint16_t(pfx[0] << kNS) : uint16_t(0xFFFFu);
            }
            if (wc0 == WPR - 1) {  // column TW-1 is in the word's last band run
                const uint16_t last = uint16_t((pfx[0] + __popc(bs[0]) - 1u) << kNS);
                BN[2 * C::TW + C::TH + r0] = (tm[0] >> 31) ? last : uint16_t(0xFFFFu);
                BN[2 * C::TW + C::TH + r1] = (um[0] >> 31) ? last : uint16_t(0xFFFFu);
            }
        }
        if (C::WY > 1) __syncthreads();  // lane 0 of a lower warp row reads the band above from smem
        // the band above (lane - 1, or the warp row above): bottom row, starts, prefixes
        uint32_t ua[WPL], ubs[WPL], upfx[WPL], ual0;
        {
            const uint32_t ual_sh = __shfl_up_sync(0xffffffffu, ul0, 1);
#pragma unroll
            for (int k = 0; k < WPL; ++k) {
                ua[k] = __shfl_up_sync(0xffffffffu, um[k], 1);
                ubs[k] = __shfl_up_sync(0xffffffffu, bs[k], 1);
                upfx[k] = __shfl_up_sync(0xffffffffu, pfx[k], 1);
            }
            ual0 = ual_sh;
            if (lane == 0) {
                if (band == 0) {  // the tile's top side: a seam, handled by kernel (d)
#pragma unroll
                    for (int k = 0; k < WPL; ++k) ua[k] = ubs[k] = upfx[k] = 0u;
                    ual0 = 0u;
                } else {
#pragma unroll
                    for (int k = 0; k < WPL; ++k) {
                        ua[k] = M[(r0 - 1) * WPR + wc0 + k];
                        ubs[k] = BS[(band - 1) * WPR + wc0 + k];
                        upfx[k] = PF16[(band - 1) * WPR + wc0 + k];
                    }
                    ual0 = wc0 > 0 ? M[(r0 - 1) * WPR + wc0 - 1] : 0u;
                }
            }
        }

        // ---- init + coarse column scan: each band run links to the band run
        // above that holds its first overlap in its word (plain stores); a root
        // band run carries its minimum pixel as its code
        uint32_t U[WPL];
        uint32_t nlink = 0;  // this lane's linked runs
#pragma unroll
        for (int k = 0; k < WPL; ++k) {
            const int wc = wc0 + k;
            const uint32_t tl = k > 0 ? tm[k - 1] : (wc > 0 ? M[r0 * WPR + wc - 1] : 0u);
            const uint32_t ual = k > 0 ? ua[k - 1] : ual0;
            const uint32_t o = tm[k] & ua[k];
            const uint32_t ocont = (o & 1u) & ((tl & ual) >> 31);  // overlap continuing from the left word
            const uint32_t os = (o & ~(o << 1)) & ~ocont;
            const uint32_t rowpos0 = uint32_t(r0 * C::TW + 32 * wc);  // the bottom row's: + TW
            // (seg_first yields nothing below the word's first band start: that
            // part belongs to a band run of the word on the left, whose lane owns the node)
            const uint32_t firstm = seg_first(o, bs[k]);      // first overlap of each band run
            const uint32_t tfirst = seg_first(tm[k], bs[k]);  // first top-row pixel of each band run
            const uint32_t rbs = __brev(bs[k]), rss = (rbs << 1) | 1u, rse = rbs | 0x80000000u;
            {   // one marker bit per band run, in run order: its first overlap
                // (the run links to the band run above holding it), else its first
                // top-row pixel (a root, coded by it), else its start (a root
                // without a top-row pixel here, coded by its first bottom
                // column); the i-th marker is node pfx + i, so one loop whose
                // trip count is the lane's run count (not the sum of three
                // per-loop warp maxima) and no rank popcount for the node
                const uint32_t top_root = tfirst & ~seg_back(firstm, rss, rse);
                const uint32_t rb = bs[k] & ~seg_back(tfirst, rss, rse);
                uint32_t mk = firstm | top_root | rb;
                const uint32_t c0 = kRoot | rowpos0, c1 = c0 + uint32_t(C::TW);
                const uint32_t uh = (upfx[k] - 1u) << kNS;  // + (starts at or below the bit above) << kNS
                uint32_t hd = pfx[k] << kNS;  // handle of the next node
                while (mk) {
                    const uint32_t lb = mk & (0u - mk);
                    const uint32_t code = ((rb & lb) ? c1 : c0) + (31u - __clz(lb));
                    const uint32_t up = uh + (uint32_t(__popc(ubs[k] << __clz(lb))) << kNS);
                    *nslot(P, hd) = node_t((firstm & lb) ? up : code);
                    hd += 1u << kNS;
                    mk ^= lb;
                }
            }
            const bool last_has_top = bs[k] && (tfirst & (0xFFFFFFFFu << (31u - __clz(bs[k]))));
            if (bs[k] && (((tm[k] | um[k]) >> 31) & 1u) && !last_has_top) {
                // the last band run reaches the word's end with no top-row pixel
                // here: its top-row pixel may lie in a later word
                for (int w = wc + 1; w < WPR; ++w) {
                    const uint32_t tw = M[r0 * WPR + w], uw = M[r1 * WPR + w];
                    const uint32_t bw = band_starts(tw, uw, M[r0 * WPR + w - 1], M[r1 * WPR + w - 1]);
                    const uint32_t below = (bw & (0u - bw)) - 1u;  // bits before the first start (all if none)
                    const uint32_t cont = (tw | uw) & below;       // the part continuing from the left
                    const uint32_t tc = tw & cont;
                    if (tc) {
                        P[pfx[k] + __popc(bs[k]) - 1] =
                            node_t(kRoot | (uint32_t(r0 * C::TW + 32 * w) + 31u - __clz(tc & (0u - tc))));
                        break;
                    }
                    if (bw || cont != 0xFFFFFFFFu) break;  // the run ends in this word
                }
            }
            U[k] = os & ~firstm;  // remaining overlaps
            nlink += __popc(firstm);
        }
        // remaining overlaps -> this warp's union list
        uint32_t* UL = reinterpret_cast<uint32_t*>(smem + A::UL_OFF) + warp * A::UL_CAP;
        uint32_t nul;
        {
            uint32_t cu = 0;
#pragma unroll
            for (int k = 0; k < WPL; ++k) cu += __popc(U[k]);
            const uint32_t inc = warp_incl_scan(cu);
            const bool fits = inc <= uint32_t(A::UL_CAP);
            nul = __reduce_max_sync(0xffffffffu, fits ? inc : 0u);
            if (fits) {
                uint32_t* dst = UL + (inc - cu);
#pragma unroll
                for (int k = 0; k < WPL; ++k) {
                    // pair of handles {this band's node, the node above} of every
                    // remaining overlap bit (node_of as a popcount of the starts
                    // shifted up to the bit, on handle bases)
                    const uint32_t ph = (pfx[k] - 1u) << kNS, uhh = ((upfx[k] - 1u) << kNS) << 16;
                    while (U[k]) {
                        const uint32_t lb = U[k] & (0u - U[k]);
                        const uint32_t sh = __clz(lb);
                        *dst++ = (ph + (uint32_t(__popc(bs[k] << sh)) << kNS)) +
                                 (uhh + (uint32_t(__popc(ubs[k] << sh)) << (16 + kNS)));
                        U[k] ^= lb;
                    }
                }
            }
        }
        // the jump round pays where chains form: tiles where most lanes link
        // at least a third of their runs (lanes without runs count as linking);
        // sparse tiles and tiles of isolated runs (checkerboards) skip it
        // (output-invariant either way: a jump only shortens a path)
        const bool do_jump = __syncthreads_count(3u * nlink >= cnt) > C::NT / 2;
        CCL_PH(10);

        // ---- one pointer-jump round (no barrier after it: jumps and unions only
        // replace an entry by an ancestor, unions CAS root entries only)
#pragma unroll 1
        for (int j = 0; j < (do_jump ? CCL_BJUMP : 0); ++j) {
            for (uint32_t h = uint32_t(tid) << kNS; h < (nodes << kNS); h += uint32_t(C::NT) << kNS) {
                const uint32_t p = *nslot(P, h);
                const uint32_t pp = (p & kRoot) ? p : uint32_t(*nslot(P, p));
                if (!(p & kRoot)) mc.step();
                if (!(pp & kRoot)) *nslot(P, h) = node_t(pp);
            }
            if (j + 1 < CCL_BJUMP) __syncthreads();
        }
        // ---- refinement unions on root codes
        for (uint32_t k = lane; k < nul; k += 32) {
            const uint32_t pr = UL[k];
            nunion_pos(P, pr & 0xFFFFu, pr >> 16, mc);
        }
#pragma unroll
        for (int k = 0; k < WPL; ++k) {
            while (U[k]) {  // pairs that did not fit in the list
                const uint32_t b = lowbit(U[k]);
                U[k] &= U[k] - 1;
                nunion_pos(P, node_of(pfx[k], bs[k], b) << kNS, node_of(upfx[k], ubs[k], b) << kNS, mc);
            }
        }
        __syncthreads();
        CCL_PH(11);

        // ---- seam-touching roots: every foreground pixel on a side facing a
        // neighbour tile / strip marks its root once (balanced over threads)
        const bool has_top = ty > 0 || g.edge_above;
        const bool has_bot = ty + 1 < g.nty || g.edge_below;
        const bool has_left = tx > 0, has_right = tx + 1 < g.ntx;
        static_assert(C::NT == C::TW && C::NT == 2 * C::TH, "one top, one bottom and one side item per thread");
        auto mark = [&](uint32_t x) {  // x: the node (handle) of a foreground pixel on a facing side
            uint32_t p = *nslot(P, x);
            while (!(p & kRoot)) {
                mc.step();
                x = p;
                p = *nslot(P, x);
            }
            const uint32_t id = x >> kNS, bit = 1u << (id & 31);
            if (!(atomicOr(&FB[id >> 5], bit) & bit)) {
                const uint32_t k = atomicAdd(FR, 1u);
                const uint32_t n = t * uint32_t(C::MAXF) + k;
                fst.f[2 * size_t(n)] = n;
                fst.f[2 * size_t(n) + 1] = pos_gidx<C>(p & kCode, x0, y0, g);
                FR[1 + k] = n;
                *nslot(P, x) = node_t(kRoot | kSeam | k);
            }
        };
        {   // one item per RUN of foreground pixels along a facing side (the run's
            // pixels are adjacent, so they share the root): each warp lists its
            // run starts (ballots), then the whole CTA walks the dense list
            // (~100 items instead of 384 pixel slots, 3 per thread)
            uint32_t* WL = reinterpret_cast<uint32_t*>(smem + A::UL_OFF) + warp * A::UL_CAP;  // dead after the unions
            uint16_t* WLi = reinterpret_cast<uint16_t*>(WL + 1);
            static_assert(2 * (A::UL_CAP - 1) >= 3 * 32, "one warp's run starts fit in its union list");
            uint32_t nw = 0;
#pragma unroll
            for (int s3 = 0; s3 < 3; ++s3) {
                const int i = s3 * C::NT + tid;  // top, bottom, then left / right
                const bool act = s3 == 0 ? has_top : s3 == 1 ? has_bot : (tid < C::TH ? has_left : has_right);
                const bool first = s3 < 2 ? tid == 0 : (tid & (C::TH - 1)) == 0;  // first pixel of its side
                const bool st = act && BN[i] != 0xFFFFu && (first || BN[i - 1] == 0xFFFFu);
                const uint32_t bal = __ballot_sync(0xffffffffu, st);
                if (st) WLi[nw + __popc(bal & ((1u << lane) - 1u))] = uint16_t(i);
                nw += __popc(bal);
            }
            if (lane == 0) WL[0] = nw;
            __syncthreads();
            static_assert(C::NWARP == 4, "four warp lists");
            const uint32_t* UL0 = reinterpret_cast<const uint32_t*>(smem + A::UL_OFF);
            const uint32_t e1 = UL0[0], e2 = e1 + UL0[A::UL_CAP], e3 = e2 + UL0[2 * A::UL_CAP],
                           e4 = e3 + UL0[3 * A::UL_CAP];  // list ends (exclusive prefix of the warp counts)
            for (uint32_t j = tid; j < e4; j += C::NT) {
                const uint32_t w = uint32_t(j >= e1) + uint32_t(j >= e2) + uint32_t(j >= e3);
                const uint32_t b = w == 0 ? 0u : w == 1 ? e1 : w == 2 ? e2 : e3;
                const uint16_t* li = reinterpret_cast<const uint16_t*>(UL0 + w * A::UL_CAP + 1);
                mark(BN[li[j - b]]);
            }
        }
        __syncthreads();
        CCL_PH(12);

        // ---- node table: every entry becomes its root's code
        {
            volatile node_t* vP = P;
            // two hops without branches (selects; most nodes are within two hops of
            // their root after the jump round), a loop only for deeper chains
            (void)vP;
            for (uint32_t h = uint32_t(tid) << kNS; h < (nodes << kNS); h += uint32_t(C::NT) << kNS) {
                const uint32_t p = *nslot(P, h);
                const uint32_t q = (p & kRoot) ? p : uint32_t(*nslot(P, p & 0x7FFFu));
                uint32_t r = (q & kRoot) ? q : uint32_t(*nslot(P, q & 0x7FFFu));
                if (!(r & kRoot)) {
                    do {
                        mc.step();
                        r = *nslot(P, r);
                    } while (!(r & kRoot));
                }
                if (!(p & kRoot)) *nslot(P, h) = node_t(r);
            }
        }
        const uint32_t nf = FR[0];
        if (tid == 0) {
            wt[C::W_HEAD + 0] = nf;
            wt[C::W_HEAD + 1] = nodes;
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
            const uint64_t keep = policy_evict_last();
            bulk_store_hint(wt + C::W_MASK, M, C::MW * 6 + C::BSW * 4, keep);  // row masks, band prefixes, band starts
            if (nodes) bulk_store_hint(wt + C::W_TBL, P, (nodes * 2 + 15) & ~15u, keep);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }

        CCL_PH(13);
        // ---- seam records + strip-edge rows
        const bool edge_top = ty == 0 && g.edge_above, edge_bot = ty + 1 == g.nty && g.edge_below;
#pragma unroll
        for (int s3 = 0; s3 < 3; ++s3) {
            const int i = s3 * C::NT + tid;  // top, bottom, then left / right
            const uint32_t x = BN[i];
            uint32_t v = kBG;
            if (x != 0xFFFFu) {
                const uint32_t code = *nslot(P, x);
                if (code & kSeam) v = FR[1 + (code & kCode)];
            }
            wt[C::W_REC + i] = v;
            if (s3 < 2 && (s3 == 0 ? edge_top : edge_bot)) {  // strip-edge tiles only
                const uint32_t gx = x0 + uint32_t(tid);
                if (gx < g.W) SE[(s3 == 0 ? 0u : g.W) + gx] = v;
            }
        }
        metrics_tile(g, t, mc);
        if (TMA && A::OVL) {  // next tile into the node table once every reader is done with it
            fence_proxy_async_smem();
            __syncthreads();
            if (tid == 0) {
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                if (t + ncta < ntiles) {
                    TileWalk nx = walk;
                    nx.advance();
                    issue_at(nx.cur);
                }
            }
        }
        CCL_PH(14);
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    CCL_PH_DONE();
}

template <class C, bool TMA>
__global__ void __launch_bounds__(C::NT, CCL_BMINB)
    k_local_band(const __grid_constant__ CUtensorMap tm_img, const uint8_t* img, uint32_t* work, Geo g,
                 uint32_t ntiles) {
    local_band_tiles<C, TMA>(&tm_img, img, work, g, ntiles, blockIdx.x, gridDim.x);
    pdl_trigger();
}

// ------------------------------------------------------------------ kernel (d)
// Algorithm 2 over the compact seam records: one warp per 32 pixel pairs of a
// tile seam (coalesced record loads); a pair whose predecessor along the seam
// is also foreground on both sides joins the same two local components and is
// skipped (one union per overlapping run).  Global atomicMin union-find in L.
// One warp's share of kernel (d): K consecutive 32-pair chunks starting at
// chunk gw * K of frame fz; `list` = this warp's 32 K union slots (smem).
template <class C>
__device__ __forceinline__ void seams_warp(uint32_t* work, const Geo& g, uint32_t ntiles, uint32_t gw, uint32_t fz,
                                           uint2* list) {
    constexpr uint32_t HC = C::TW / 32, VC = C::TH / 32;  // 32-pair chunks per seam
    constexpr int K = CCL_SEAM_K;                          // chunks per warp
    const Forest fst = forest_of<C>(work, ntiles);
    const int lane = threadIdx.x & 31;
    Ctr mc;
    const uint32_t nh = (g.nty - 1) * g.ntx * HC;
    const uint32_t nv = (g.ntx - 1) * g.nty * VC;
    // records of K consecutive chunks, all loads in flight together
    uint32_t va[K], vb[K], c[K];
    bool prev0[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const uint32_t gc = gw * K + k;
        const uint32_t *ra = nullptr, *rb = nullptr;
        c[k] = 0;
        if (gc < nh) {  // horizontal seam: bottom record of (tx, ty) vs top record of (tx, ty + 1)
            const uint32_t s = gc / HC;
            c[k] = gc - s * HC;
            const uint32_t ty = s / g.ntx, tx = s - ty * g.ntx;
            const size_t ta = (size_t(fz) * g.nty + ty) * g.ntx + tx;
            ra = work + ta * C::TILE_WORDS + C::W_REC + C::TW;
            rb = work + (ta + g.ntx) * C::TILE_WORDS + C::W_REC;
        } else if (gc < nh + nv) {  // vertical seam: right record of (tx, ty) vs left record of (tx + 1, ty)
            const uint32_t u = gc - nh, s = u / VC;
            c[k] = u - s * VC;
            const uint32_t ty = s / (g.ntx - 1), tx = s - ty * (g.ntx - 1);
            const size_t ta = (size_t(fz) * g.nty + ty) * g.ntx + tx;
            ra = work + ta * C::TILE_WORDS + C::W_REC + 2 * C::TW + C::TH;
            rb = work + (ta + 1) * C::TILE_WORDS + C::W_REC + 2 * C::TW;
        }
        const uint32_t i = c[k] * 32 + lane;
        va[k] = ra ? ra[i] : kBG;
        vb[k] = ra ? rb[i] : kBG;
        prev0[k] = lane == 0 && ra && c[k] > 0 && ra[i - 1] != kBG && rb[i - 1] != kBG;
    }
    // Algorithm 2 per pair; a pair whose predecessor along the seam is also
    // foreground on both sides joins the same two local components and is
    // skipped; one union per distinct (a, b) pair of a chunk; the unions are
    // compacted so that every lane of the warp climbs
    uint32_t n = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const bool fg = (va[k] != kBG) && (vb[k] != kBG);
        bool prev = __shfl_up_sync(0xffffffffu, fg, 1);
        if (lane == 0) prev = prev0[k];
        bool act = fg && !prev;
#if CCL_SEAM_MATCH == 1
        const uint64_t key = act ? (uint64_t(va[k]) << 32 | vb[k]) : ~0ull;
        const uint32_t same = __match_any_sync(0xffffffffu, key);
        act = act && (__ffs(same) - 1 == lane);
#elif CCL_SEAM_MATCH == 2
        {   // drop a pair equal to the previous active pair of the chunk (the
            // same two components meeting again: dense images, long components)
            const uint32_t ab = __ballot_sync(0xffffffffu, act);
            const uint32_t below = ab & ((1u << lane) - 1u);
            const int pl = below ? 31 - __clz(below) : lane;
            const uint32_t pa = __shfl_sync(0xffffffffu, va[k], pl), pb = __shfl_sync(0xffffffffu, vb[k], pl);
            act = act && !(below && pa == va[k] && pb == vb[k]);
        }
#endif
        const uint32_t bal = __ballot_sync(0xffffffffu, act);
        if (act) list[n + __popc(bal & ((1u << lane) - 1u))] = make_uint2(va[k], vb[k]);
        n += __popc(bal);
    }
    __syncwarp();
    for (uint32_t j = lane; j < n; j += 32) {
        const uint2 pr = list[j];
#if CCL_SEAM_NOUNION  // timing probe only: wrong labels
        if (pr.x == 0xFFFFFFF0u) fst.f[0] = pr.y;
#else
        fst.unite(pr.x, pr.y, mc);
#endif
    }
    __syncwarp();  // the list is reused by this warp's next share (fused kernel)
    metrics_phase(g, 0, mc);
}

template <class C>
__global__ void __launch_bounds__(256) k_seams(uint32_t* work, Geo g, uint32_t ntiles) {
    __shared__ uint2 list[8][32 * CCL_SEAM_K];  // each warp's unions
    pdl_wait();
    pdl_trigger();
    seams_warp<C>(work, g, ntiles, (blockIdx.x * blockDim.x + threadIdx.x) >> 5, blockIdx.y, list[threadIdx.x >> 5]);
}

// ------------------------------------------------------------------ kernel (d2)
// After every union (and, in strip mode, after the strip seam resolve): the
// final label of each tile's seam-touching roots, written over the tile's
// root list, so kernel (e) needs no forest walks.  One warp per tile.
template <class C>
__device__ __forceinline__ void resolve_tile(uint32_t* work, const Geo& g, uint32_t ntiles, uint32_t t) {
    const int lane = threadIdx.x & 31;
    uint32_t* wt = work_tile<C>(work, t);
    const uint32_t nf = wt[C::W_HEAD];
    const Forest fst = forest_of<C>(work, ntiles);
    Ctr mc;
    // up to R roots of this lane climb at once (all first loads in flight
    // together, then lockstep hops): ~1-2 dependent L2 round trips per group
    // of 32 R roots instead of one chain per root
    constexpr int R = 4;
    const uint32_t base = t * uint32_t(C::MAXF);
    for (uint32_t k0 = 0; k0 < nf; k0 += 32u * R) {
        uint32_t cur[R];
        uint2 v[R];
#pragma unroll
        for (int i = 0; i < R; ++i) {
            cur[i] = base + k0 + lane + 32u * i;
            if (k0 + lane + 32u * i < nf) v[i] = fst.node(cur[i]);
        }
        for (;;) {
            bool more = false;
#pragma unroll
            for (int i = 0; i < R; ++i)
                if (k0 + lane + 32u * i < nf && v[i].x != cur[i]) {
                    mc.step();
                    cur[i] = v[i].x;
                    v[i] = fst.node_ca(cur[i]);
                    more = true;
                }
            if (!more) break;
        }
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const uint32_t k = k0 + lane + 32u * i;
            if (k < nf) {
                if (cur[i] != base + k) fst.f[2 * size_t(base + k)] = cur[i];  // path compression
                wt[C::W_LIST + k] = v[i].y;
            }
        }
    }
    metrics_phase(g, 2, mc);
}

template <class C>
__global__ void __launch_bounds__(256, 8) k_resolve(uint32_t* work, Geo g, uint32_t ntiles) {
    const uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    pdl_wait();
    pdl_trigger();
    if (t < ntiles) resolve_tile<C>(work, g, ntiles, t);
}

// ------------------------------------------------------------------ kernel (e)
// Persistent, 3-stage pipeline per CTA: while tile i is expanded, the node
// table + resolved seam labels of tile i+1 and the head/masks of tile i+2 are
// in flight (bulk copies).  Each warp expands its 32x32 block into a 128B-
// swizzled staging tile and writes it with one TMA store: every label is
// written exactly once and the image is never re-read.
template <class C, bool RUNS, bool TMA_ST, bool BAND>
__device__ __forceinline__ void final_tiles(const CUtensorMap* tmap, uint32_t* L, const uint32_t* work, const Geo& g,
                                            uint32_t ntiles, uint32_t cta, uint32_t ncta) {
    using E = ELayout<C, RUNS, BAND>;
    uint8_t* smem = aligned_smem();
    uint64_t* b1 = reinterpret_cast<uint64_t*>(smem + E::BAR_OFF);
    uint64_t* b2 = b1 + 3;
    uint64_t* b3 = b1 + 5;  // second half of an oversized band table
    uint32_t b3par = 0;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wx = warp % C::WX, wy = warp / C::WX;
    const int row = wy * 32 + lane;
    const uint32_t G = ncta;
    auto s1buf = [&](uint32_t j) { return reinterpret_cast<uint32_t*>(smem + E::S1_OFF + j * E::S1); };
    auto s2buf = [&](uint32_t j) { return reinterpret_cast<uint32_t*>(smem + E::S2_OFF + j * E::S2); };
    auto s1 = [&](uint32_t t, uint32_t j) {
        mbar_expect_tx(&b1[j], E::S1B);
        bulk_load(s1buf(j), work_tile<C>(const_cast<uint32_t*>(work), t), E::S1B, &b1[j]);
    };
    // a band tile with more nodes than the stage holds (checkerboard-like) is
    // staged in two halves: bands 0-15 first, bands 16-31 after them
    // (<= 16 x 4 x 32 = 2048 nodes each)
    static_assert(!BAND || 16 * C::WPR * 32 + 8 <= E::TBLN, "half a band tile's table fits the stage");
    auto half_nodes = [&](const uint32_t* head) -> uint32_t {
        return reinterpret_cast<const uint16_t*>(head + 4 + C::MW)[16 * C::WPR];  // prefix of band 16
    };
    auto s2 = [&](uint32_t t, uint32_t j, const uint32_t* head) {
        const uint32_t lb = (head[0] * 4 + 15) & ~15u;
        const uint32_t tb = head[1] <= uint32_t(E::TBLN) ? (head[1] * 2 + 15) & ~15u
                            : BAND ? (half_nodes(head) * 2 + 15) & ~15u : 0u;
        const uint32_t* wt = work_tile<C>(const_cast<uint32_t*>(work), t);
        mbar_expect_tx(&b2[j], lb + tb);
        if (lb) bulk_load(s2buf(j), wt + C::W_LIST, lb, &b2[j]);
        if (tb) bulk_load(s2buf(j) + C::MAXF, wt + C::W_TBL, tb, &b2[j]);
    };
    if (tid == 0 && TMA_ST) prefetch_tmap(tmap);
    if (tid == 0) {
        for (int j = 0; j < 3; ++j) mbar_init(&b1[j], 1);
        for (int j = 0; j < 2; ++j) mbar_init(&b2[j], 1);
        mbar_init(b3, 1);
        const uint32_t t0 = cta;
        // heads / masks come from kernel (a), complete before (d2) let this grid
        // launch; only the seam labels of (d2) need the dependency wait.  Every
        // other thread reads global data only through thread 0's copies.
        if (t0 < ntiles) s1(t0, 0);
        if (t0 + G < ntiles) s1(t0 + G, 1);
        pdl_wait();
        if (t0 < ntiles) {
            mbar_wait(&b1[0], 0);
            s2(t0, 0, s1buf(0));
        }
    }
    __syncthreads();

    const int sw = lane & 7;
    uint32_t it = 0;
    TileWalk walk(cta, G, g);
    for (uint32_t t = cta; t < ntiles; t += G, ++it, walk.advance()) {
        const uint32_t j1 = it % 3, j2 = it & 1u;
        if (tid == 0) {
            if (t + 2 * G < ntiles) s1(t + 2 * G, (it + 2) % 3);
            if (t + G < ntiles) {
                const uint32_t jn = (it + 1) % 3;
                mbar_wait(&b1[jn], ((it + 1) / 3) & 1u);
                s2(t + G, (it + 1) & 1u, s1buf(jn));
            }
        }
        mbar_wait(&b1[j1], (it / 3) & 1u);
        mbar_wait(&b2[j2], (it >> 1) & 1u);
        const uint32_t* M = s1buf(j1) + 4;
        const uint16_t* PF16 = reinterpret_cast<const uint16_t*>(M + C::MW);
        const uint32_t* BSt = M + C::MW + C::MW / 2;  // band starts (band mode)
        const uint32_t* FT = s2buf(j2);
        const uint16_t* TBL = reinterpret_cast<const uint16_t*>(FT + C::MAXF);
        const TileId ti = walk.cur;
        const uint32_t x0 = ti.tx * C::TW, y0 = ti.ty * C::TH;

        // label of a root code: a seam root's resolved label, else the global
        // raster index of its tile position (pos_gidx as one multiply-add:
        // y * W + x = pos + (pos / TW) * (W - TW))
        const uint32_t gbase = (g.row0 + y0) * g.W + x0, wm = g.W - uint32_t(C::TW);
        auto lab_of = [&](uint32_t v) -> uint32_t {
            const uint32_t pos = v & kCode;
            return (v & kSeam) ? FT[pos] : gbase + pos + (pos >> __builtin_ctz(C::TW)) * wm;
        };
        if (TMA_ST) {  // this warp's previous TMA stores must have read the staging tiles
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
        }
        uint32_t* Lf = L + size_t(ti.fz) * g.frame_px;
        if constexpr (C::RPL == 2) {
            // (a lambda called once per table location, so the shared-memory
            // table keeps LDS and the global fallback uses LDG)
            auto expand = [&](const uint16_t* tbl, int lo, int hi) {
            // lane = band (rows 2b, 2b+1) of word column wx: the band starts are
            // walked once and both rows are filled (two 32x32 staging tiles per
            // warp); lanes [lo, hi) only, then their staging tiles are stored
            static_assert(C::WY == 1, "lane = band of the whole tile");
            // bands whose runs start at the same columns (spirals, stripes,
            // checkerboards: neighbouring bands with equal start masks) would hit
            // one shared-memory bank all at once in the run-start scatter below;
            // such warps walk their starts from a lane-rotated column (whole
            // warp, before the lane range split)
            const uint32_t st_w = BSt[(wy * 32 + lane) * C::WPR + wx];
            const uint32_t st_n = __shfl_xor_sync(0xffffffffu, st_w, 1);  // every lane (no short circuit)
            const bool rotw = __popc(__ballot_sync(0xffffffffu, st_w != 0u && st_n == st_w)) > 8;
            if (lane >= lo && lane < hi) {
            const int b = wy * 32 + lane, wc = wx;
            const int r0 = 2 * b, r1 = r0 + 1;
            const int k = (r0 >> 5) & 1;  // staging tile of both rows (this warp covers rows 64 wy .. 64 wy + 63)
            uint8_t* stg = smem + E::STG_OFF + (warp * 2 + k) * 4096;
            uint8_t* row0 = stg + (r0 & 31) * 128;
            uint8_t* row1 = stg + (r1 & 31) * 128;
            const int sw0 = r0 & 7, sw1 = r1 & 7;
            const uint32_t swz0 = uint32_t(sw0) << 4;  // 128B swizzle: 16-byte chunk index ^= row & 7
            const uint32_t tm = M[r0 * C::WPR + wc], um = M[r1 * C::WPR + wc];
            const uint32_t st = BSt[b * C::WPR + wc];
            const uint32_t pfx = PF16[b * C::WPR + wc];
            uint32_t cur = (!(st & 1u) && ((tm | um) & 1u)) ? lab_of(tbl[pfx - 1]) : kBG;
            // run-start scatter into the staging row: rotated warps start at
            // column 4 (lane & 7) and index the table by rank; the others keep
            // the plain in-order walk (cheaper per run)
            if (rotw) {
                const uint32_t rot = 4u * (lane & 7);
                uint32_t tt = __funnelshift_r(st, st, rot);
                while (tt) {
                    const uint32_t bb = ((__ffs(tt) - 1) + rot) & 31u;
                    tt &= tt - 1;
                    const uint32_t e = pfx + __popc(st & ((1u << bb) - 1u));
                    *reinterpret_cast<uint32_t*>(row0 + ((bb << 2) ^ swz0)) = lab_of(tbl[e]);
                }
            } else {
                const uint16_t* e = tbl + pfx;
                uint32_t tt = st;
                while (tt) {
                    const uint32_t bb = __ffs(tt) - 1;
                    tt &= tt - 1;
                    *reinterpret_cast<uint32_t*>(row0 + ((bb << 2) ^ swz0)) = lab_of(*e++);
                }
            }
            uint4 vv[8];  // all read-backs first: the stores below may not be hoisted over
#pragma unroll
            for (int c = 0; c < 8; ++c) vv[c] = *reinterpret_cast<const uint4*>(row0 + ((c ^ sw0) << 4));
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                uint4* p0 = reinterpret_cast<uint4*>(row0 + ((c ^ sw0) << 4));
                uint4* p1 = reinterpret_cast<uint4*>(row1 + ((c ^ sw1) << 4));
                const uint4 v = vv[c];
                uint32_t a[4] = {v.x, v.y, v.z, v.w}, a1[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int i = 4 * c + q;
                    cur = ((st >> i) & 1u) ? a[q] : cur;
                    a[q] = ((tm >> i) & 1u) ? cur : kBG;
                    a1[q] = ((um >> i) & 1u) ? cur : kBG;
                }
                if (TMA_ST) {
                    *p0 = make_uint4(a[0], a[1], a[2], a[3]);
                    *p1 = make_uint4(a1[0], a1[1], a1[2], a1[3]);
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint32_t gx = x0 + wc * 32 + 4 * c + q;
                        if (gx < g.W && y0 + r0 < g.H) Lf[size_t(y0 + r0) * g.W + gx] = a[q];
                        if (gx < g.W && y0 + r1 < g.H) Lf[size_t(y0 + r1) * g.W + gx] = a1[q];
                    }
                }
            }
            }
            if (TMA_ST) {
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    for (int kk = lo / 16; kk < (hi + 15) / 16; ++kk) {
                        uint8_t* sk = smem + E::STG_OFF + (warp * 2 + kk) * 4096;
                        tma_store_3d_hint(tmap, int(x0 + wx * 32), int(y0 + 64 * wy + 32 * kk), int(ti.fz), sk,
                                          policy_evict_first());
                    }
                }
            }
            };
            if (M[-4 + 1] <= uint32_t(E::TBLN)) {
                expand(TBL, 0, 32);
            } else {  // two halves through the stage: bands 0-15, then bands 16-31
                expand(TBL, 0, 16);
                const uint32_t h = half_nodes(M - 4), a0 = (h * 2) & ~15u;  // 16-byte aligned source
                __syncthreads();  // every warp is done with the first half
                if (tid == 0) {
                    const uint32_t bytes = (M[-4 + 1] * 2 - a0 + 15) & ~15u;
                    mbar_expect_tx(b3, bytes);
                    bulk_load(const_cast<uint16_t*>(TBL),
                              reinterpret_cast<const uint8_t*>(work_tile<C>(const_cast<uint32_t*>(work), t) + C::W_TBL) + a0,
                              bytes, b3);
                }
                mbar_wait(b3, b3par);
                b3par ^= 1u;
                expand(TBL - a0 / 2, 16, 32);
            }
        } else {
#pragma unroll 1
        for (int k = 0; k < C::WPL; ++k) {  // this lane's row words, one 32x32 staging tile each
            const int wc = wx * C::WPL + k;
            uint8_t* stg = smem + E::STG_OFF + (warp * C::WPL + k) * 4096;  // 32 x 32 u32, 128B-swizzled
            uint8_t* myrow = stg + lane * 128;
            const uint32_t m = M[row * C::WPR + wc];
            uint32_t st, pfx;
            bool cont;  // the word starts inside a node continuing from the word on its left
            if (BAND) {  // node starts are the band starts of rows (2b, 2b+1); prefixes per (band, word)
                const int b = row >> 1;
                st = BSt[b * C::WPR + wc];
                pfx = PF16[b * C::WPR + wc];
                const uint32_t partner = __shfl_xor_sync(0xffffffffu, m, 1);  // the other row of the band
                cont = !(st & 1u) && ((m | partner) & 1u);
            } else {
                const uint32_t lm = wc > 0 ? M[row * C::WPR + wc - 1] : 0u;
                st = word_starts<RUNS>(m, lm);
                pfx = PF16[row * C::WPR + wc];
                cont = !(st & 1u) && (m & 1u);
            }
            uint32_t cur = cont ? lab_of(TBL[pfx - 1]) : kBG;  // node continuing from the left
            {
                const uint16_t* e = TBL + pfx;
                uint32_t tt = st;
                while (tt) {
                    const uint32_t b = __ffs(tt) - 1;
                    tt &= tt - 1;
                    *reinterpret_cast<uint32_t*>(myrow + ((((b >> 2) ^ sw) << 4) | ((b & 3) << 2))) = lab_of(*e++);
                }
            }
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                uint4* p = reinterpret_cast<uint4*>(myrow + ((c ^ sw) << 4));
                uint4 v = *p;
                uint32_t a[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int i = 4 * c + q;
                    cur = ((st >> i) & 1u) ? a[q] : cur;
                    a[q] = ((m >> i) & 1u) ? cur : kBG;
                }
                if (TMA_ST) {
                    *p = make_uint4(a[0], a[1], a[2], a[3]);
                } else {
                    const uint32_t gy = y0 + row;
                    if (gy < g.H) {
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const uint32_t gx = x0 + wc * 32 + 4 * c + q;
                            if (gx < g.W) Lf[size_t(gy) * g.W + gx] = a[q];
                        }
                    }
                }
            }
            if (TMA_ST) {
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    if (CCL_HINTS)
                        tma_store_3d_hint(tmap, int(x0 + wc * 32), int(y0 + wy * 32), int(ti.fz), stg,
                                          policy_evict_first());  // OOB clipped; labels stream out
                    else
                        tma_store_3d(tmap, int(x0 + wc * 32), int(y0 + wy * 32), int(ti.fz), stg);
                }
            }
        }
        }
        if (TMA_ST && lane == 0) asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        __syncthreads();  // stage buffers j1 / j2 are free for thread 0's next copies
    }
    if (TMA_ST && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

template <class C, bool RUNS, bool TMA_ST, bool BAND>
__global__ void __launch_bounds__(C::NT, CCL_EMINB) k_final(const __grid_constant__ CUtensorMap tm_lab, uint32_t* L,
                                                    const uint32_t* work, Geo g, uint32_t ntiles) {
    final_tiles<C, RUNS, TMA_ST, BAND>(&tm_lab, L, work, g, ntiles, blockIdx.x, gridDim.x);
}

// ================================================================== host side
// Persistent grid: every SM filled to the kernel's occupancy, cached per
// (kernel, device, block, smem) -- each template instantiation has its own
// entry -- under a mutex (strip workers call this from several host threads).
template <class K>
static unsigned persistent_grid(K kernel, int threads, int smem, uint32_t ntiles, int cap_per_sm = 0) {
    static std::mutex mu;
    static std::map<std::tuple<const void*, int, int, int>, std::pair<int, int>> cache;  // {CTAs/SM, SMs}
    int dev = 0;
    cudaGetDevice(&dev);
    const auto key = std::make_tuple(reinterpret_cast<const void*>(kernel), dev, threads, smem);
    std::pair<int, int> occ;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it == cache.end()) {
            int n = 0, sms = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            it = cache.emplace(key, std::make_pair(n > 0 ? n : 1, sms > 0 ? sms : 1)).first;
        }
        occ = it->second;
    }
    const int per = (cap_per_sm > 0 && cap_per_sm < occ.first ? cap_per_sm : occ.first) * occ.second;
    return unsigned(per < int(ntiles) ? per : int(ntiles));
}

static uint32_t tile_count(const LaunchArgs& a) { return a.g.ntx * a.g.nty * a.nframes; }


// Launch (optionally) with programmatic stream serialization: the kernel calls
// pdl_wait() before reading what the previous kernel in the stream produced.
template <class K, class... Args>
static cudaError_t launch_ex(K kernel, dim3 grid, int threads, int smem, cudaStream_t s, bool pdl, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = CCL_PDL;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}
template <class K, class... Args>
static cudaError_t launch_pdl(K kernel, dim3 grid, int threads, int smem, cudaStream_t s, Args... args) {
    return launch_ex(kernel, grid, threads, smem, s, true, args...);
}

template <int VAR>
static cudaError_t launch_local_v(const LaunchArgs& a) {
    using C = TileCfg;
    using A = ALayout<C, (VAR == 0 || VAR == 1)>;
    const uint32_t nt = tile_count(a);
    if (a.tma_load) {
        auto k = k_local<C, VAR, true>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, A::SMEM);
        cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, CCL_CARVEOUT);
        const cudaError_t e = launch_ex(k, dim3(persistent_grid(k, C::NT, A::SMEM, nt)), C::NT, A::SMEM,
                                        a.stream, false, a.tm_img, a.img, a.labels, a.work, a.g, nt);
        if (e != cudaSuccess) return e;
    } else {
        auto k = k_local<C, VAR, false>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, A::SMEM);
        k<<<persistent_grid(k, C::NT, A::SMEM, nt), C::NT, A::SMEM, a.stream>>>(a.tm_img, a.img, a.labels,
                                                                                           a.work, a.g, nt);
    }
    return cudaGetLastError();
}

static bool uses_band(const LaunchArgs& a) { return CCL_BAND && a.variant == 0; }

static cudaError_t launch_local_band(const LaunchArgs& a) {
    using C = BandCfg;
    using A = ALayout<C, true, true>;
    const uint32_t nt = tile_count(a);
    cudaError_t e;
    if (a.tma_load) {
        auto k = k_local_band<C, true>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, A::SMEM);
        cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, CCL_CARVEOUT);
        e = launch_ex(k, dim3(persistent_grid(k, C::NT, A::SMEM, nt, a.a_cap_per_sm)), C::NT, A::SMEM,
                      a.stream, false,
                      a.tm_img, a.img, a.work, a.g, nt);
    } else {
        auto k = k_local_band<C, false>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, A::SMEM);
        e = launch_ex(k, dim3(persistent_grid(k, C::NT, A::SMEM, nt)), C::NT, A::SMEM, a.stream, false, a.tm_img,
                      a.img, a.work, a.g, nt);
    }
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_local(const LaunchArgs& a) {
    if (uses_band(a)) return launch_local_band(a);
    switch (a.variant) {
        case 0: return launch_local_v<0>(a);
        case 1: return launch_local_v<1>(a);
        case 2: return launch_local_v<2>(a);
        default: return launch_local_v<3>(a);
    }
}

int debug_skip() {
    static const int v = [] {
        const char* e = std::getenv("CCL_DEBUG_SKIP");
        return e && *e ? std::atoi(e) : 0;
    }();
    return v;
}

template <bool RUNS, bool BAND>
static cudaError_t launch_final_v(const LaunchArgs& a) {
    using C = typename std::conditional<BAND, BandECfg, ECfg>::type;
    using E = ELayout<C, RUNS, BAND>;
    const uint32_t nt = tile_count(a);
    constexpr int NTH = C::NT;
    cudaError_t e = cudaSuccess;
    if (!(debug_skip() & 4))
        e = launch_ex(k_resolve<TileCfg>, dim3(unsigned((uint64_t(nt) * 32 + 255) / 256)), 256, 0, a.stream,
                      !a.no_pdl_first, a.work, a.g, nt);
    if (e != cudaSuccess) return e;
    if (debug_skip() & 8) return cudaGetLastError();
    if (a.tma_store) {
        auto k = k_final<C, RUNS, true, BAND>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, E::SMEM);
        cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, CCL_CARVEOUT);
        e = launch_pdl(k, dim3(persistent_grid(k, NTH, E::SMEM, nt, a.e_cap_per_sm)), NTH, E::SMEM, a.stream,
                       a.tm_lab, a.labels, const_cast<const uint32_t*>(a.work), a.g, nt);
    } else {
        auto k = k_final<C, RUNS, false, BAND>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, E::SMEM);
        e = launch_pdl(k, dim3(persistent_grid(k, NTH, E::SMEM, nt)), NTH, E::SMEM, a.stream,
                       a.tm_lab, a.labels, const_cast<const uint32_t*>(a.work), a.g, nt);
    }
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_final(const LaunchArgs& a) {
    if (uses_band(a)) return launch_final_v<true, true>(a);
    return (a.variant == 0 || a.variant == 1) ? launch_final_v<true, false>(a) : launch_final_v<false, false>(a);
}

cudaError_t launch_seams(const LaunchArgs& a) {
    using C = TileCfg;
    const uint64_t chunks = uint64_t(a.g.nty - 1) * a.g.ntx * (C::TW / 32) + uint64_t(a.g.ntx - 1) * a.g.nty * (C::TH / 32);
    if (chunks == 0) return cudaSuccess;
    const uint64_t warps = (chunks + CCL_SEAM_K - 1) / CCL_SEAM_K;
    const dim3 grid(unsigned((warps * 32 + 255) / 256), a.nframes);
    const cudaError_t e = launch_pdl(k_seams<C>, grid, 256, 0, a.stream, a.work, a.g, tile_count(a));
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

size_t work_bytes(uint32_t w, uint32_t h, uint32_t nframes) {
    using C = TileCfg;
    const size_t ntiles = size_t((w + C::TW - 1) / C::TW) * ((h + C::TH - 1) / C::TH) * nframes;
    return (ntiles * (size_t(C::TILE_WORDS) + 2 * size_t(C::MAXF)) + 4 * size_t(w)) * 4;
}

uint32_t* strip_area_ptr(uint32_t* work, const Geo& g) {
    using C = TileCfg;
    return work + size_t(g.ntx) * g.nty * (size_t(C::TILE_WORDS) + 2 * size_t(C::MAXF));
}
uint32_t* forest_ptr(uint32_t* work, const Geo& g) {
    using C = TileCfg;
    return work + size_t(g.ntx) * g.nty * size_t(C::TILE_WORDS);
}
int tile_maxf() { return TileCfg::MAXF; }

int tile_w() { return TileCfg::TW; }
#if CCL_PHASES
extern "C" int ccl_debug_phases(unsigned long long* out16, int reset) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out16, g_phase_cycles, 16 * 8);
    if (reset) {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
    }
    return 0;
}
#endif
int tile_h() { return TileCfg::TH; }

}  // namespace cclk
