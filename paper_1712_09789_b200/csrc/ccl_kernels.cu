// ccl_kernels.cu — the hand-written sm_100a kernels of the labeler.
//
//   (a)+(b)+(c)  k_local  : TMA-stage a TW x TH tile, warp-bit run detection
//                           (coarse row scan), coarse column link, smem
//                           min-union refinement, flatten (unification).
//                           Exports, per tile, a compact RUN TABLE (one u16
//                           local root per row run), the row-word masks and
//                           the list of seam-touching roots; writes the tile's
//                           seam pixels and registers the seam-touching roots
//                           as nodes of the global forest in the label buffer.
//   (d)          k_seams  : boundary-only pass (Algorithm 2): one thread per
//                           interior tile-seam pixel pair, global atomicMin
//                           union-find directly in the label buffer.
//   (e)          k_final  : resolves each seam-touching root ONCE through the
//                           global forest, expands the run table to pixels and
//                           writes every label exactly once (swizzled TMA
//                           stores).  It never re-reads the image: masks
//                           (0.125 B/px) + run table (~0.5 B/px at d=0.5).
//
// The reference's block config / variant are honoured for validation and
// strategy selection; the GPU tile is an internal constant (labels are
// tile-shape invariant: SPEC.md "Variant equivalence", "Scheduler independence").
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ccl_device.cuh"
#include "ccl_internal.h"

namespace cclk {

template <int WX_, int WY_>
struct Cfg {
    static constexpr int WX = WX_, WY = WY_;
    static constexpr int TW = 32 * WX, TH = 32 * WY, NT = 32 * WX * WY, NWARP = WX * WY;
    static constexpr int PS = TW + 1;  // padded node row stride: node id order == raster order
    static constexpr int NODES = TH * PS;
    static constexpr int FW = (NODES + 31) / 32;
    static constexpr int P_BYTES = ((NODES * 2 + 1023) / 1024) * 1024;  // u16 parents
    static constexpr int F_OFF = P_BYTES;
    static constexpr int M_OFF = F_OFF + ((FW * 4 + 127) / 128) * 128;
    static constexpr int IMG_OFF = M_OFF + ((TH * WX * 4 + 127) / 128) * 128;
    static constexpr int FR_OFF = IMG_OFF + TW * TH;
    static constexpr int BAR_OFF = FR_OFF + ((4 * (1 + TW + 2 * TH) + 127) / 128) * 128;
    static constexpr int SMEM = BAR_OFF + 64 + 1024;  // +1024: runtime base alignment slack
    // work buffer (global) per tile
    static constexpr int MASK_WORDS = TH * WX;                    // row-word masks
    static constexpr int MAXF = TW + 2 * TH;                      // bound on seam-touching roots
    static constexpr int HDR_WORDS = ((1 + NWARP + MAXF) + 3) / 4 * 4;  // nF, run count per warp, F list
    static constexpr int TBL_PER_WARP = 512;                      // u16 run entries (<= 16 runs x 32 rows)
    // kernel (e) smem
    static constexpr int E_M_OFF = 0;
    static constexpr int E_HDR_OFF = E_M_OFF + MASK_WORDS * 4;
    static constexpr int E_FT_OFF = E_HDR_OFF + HDR_WORDS * 4;
    static constexpr int E_TBL_OFF = E_FT_OFF + MAXF * 4;
    static constexpr int E_STG_OFF = ((E_TBL_OFF + NWARP * TBL_PER_WARP * 2) + 1023) / 1024 * 1024;
    static constexpr int E_BAR_OFF = E_STG_OFF + NWARP * 4096;
    static constexpr int E_SMEM = E_BAR_OFF + 64 + 1024;
    static_assert(TW <= 256 && TH <= 256, "TMA box dims are limited to 256");
    static_assert(NWARP * TBL_PER_WARP * 2 <= TW * TH, "run-table staging must fit in the image area");
    static_assert(NODES < 0x8000, "node ids must leave bit 15 free for the seam-root tag");
};

using TileCfg = Cfg<CCL_TILE_WX, CCL_TILE_WY>;

// Node parents are u16 (node ids < 2^15; bit 15 tags seam roots): half the
// shared memory of u32 parents -> more resident CTAs for this latency-bound
// phase.  Unions are CAS min-unions on the 16-bit entries.
using node_t = uint16_t;
constexpr uint32_t kTag = 0x8000u;
__device__ __forceinline__ uint32_t nfind(node_t* P, uint32_t x) {
    volatile node_t* vP = P;
    uint32_t p = vP[x];
    while (p != x) {
        const uint32_t gp = vP[p];
        if (gp == p) return p;
        vP[x] = node_t(gp);  // path halving (ancestor only)
        x = gp;
        p = vP[x];
    }
    return x;
}
__device__ __forceinline__ void nunion(node_t* P, uint32_t a, uint32_t b) {
    for (;;) {
        a = nfind(P, a);
        b = nfind(P, b);
        if (a == b) return;
        if (a < b) { const uint32_t t = a; a = b; b = t; }
        if (atomicCAS(reinterpret_cast<unsigned short*>(P + a), static_cast<unsigned short>(a),
                      static_cast<unsigned short>(b)) == a)
            return;
    }
}

__device__ __forceinline__ uint8_t* aligned_smem() {
    extern __shared__ uint8_t smem_raw[];
    return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
}

// Work-buffer views of one tile (tile index tg over frames x tile rows x tile cols).
template <class C>
struct Work {
    uint32_t* masks;
    uint32_t* hdr;
    uint16_t* tbl;
    __device__ __forceinline__ Work(uint32_t* work, size_t ntiles, size_t tg) {
        masks = work + tg * C::MASK_WORDS;
        hdr = work + ntiles * C::MASK_WORDS + tg * C::HDR_WORDS;
        tbl = reinterpret_cast<uint16_t*>(work + ntiles * (C::MASK_WORDS + C::HDR_WORDS)) +
              tg * size_t(C::NWARP * C::TBL_PER_WARP);
    }
};

__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_load(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(sdst)),
                 "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// Per-lane result of the tile-local phase.
struct LaneState {
    uint32_t m;         // foreground bits of this lane's 32-px row word
    uint32_t st;        // segment (node) starts in the word
    uint32_t rootmask;  // segment starts that are local roots
};

// Steps 1-3 of Algorithm 1 for one tile, fully in shared memory.  On return
// (after a __syncthreads): P[s] == local root for every segment start s, and
// the F bitmap flags every local root whose component touches a tile side
// that faces another tile (or another strip).
template <class C, int VAR, bool TMA>
__device__ __forceinline__ LaneState tile_local(const CUtensorMap* tm, const uint8_t* img, const Geo& g,
                                                uint32_t tx, uint32_t ty, uint32_t fz, uint8_t* smem) {
    node_t* P = reinterpret_cast<node_t*>(smem);
    uint32_t* F = reinterpret_cast<uint32_t*>(smem + C::F_OFF);
    uint32_t* M = reinterpret_cast<uint32_t*>(smem + C::M_OFF);
    uint8_t* IMG = smem + C::IMG_OFF;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wx = warp % C::WX, wy = warp / C::WX;
    const int row = wy * 32 + lane;
    const int col0 = wx * 32;
    const uint32_t x0 = tx * C::TW, y0 = ty * C::TH;

    // ---- stage the tile and build the row-word foreground masks
    if (TMA) {
        if (tid == 0) {
            mbar_init(bar, 1);
            mbar_expect_tx(bar, C::TW * C::TH);
            tma_load_3d(IMG, tm, int(x0), int(y0), int(fz), bar);  // OOB -> 0 == background
        }
    }
    for (int i = tid; i < C::FW; i += C::NT) F[i] = 0u;
    if (tid == 0) *reinterpret_cast<uint32_t*>(smem + C::FR_OFF) = 0u;
    uint32_t m;
    if (TMA) {
        __syncthreads();  // mbarrier init visible before anyone polls it
        mbar_wait(bar, 0);
        constexpr int CPR = C::TW / 16;
        uint16_t* M16 = reinterpret_cast<uint16_t*>(M);
#pragma unroll
        for (int c = tid; c < C::TH * CPR; c += C::NT) {
            const uint4 q = *reinterpret_cast<const uint4*>(IMG + c * 16);
            M16[c] = static_cast<uint16_t>(eq1_mask16(q));
        }
        __syncthreads();
        m = M[row * C::WX + wx];
    } else {
        m = 0u;
        const uint32_t gy = y0 + row;
        if (gy < g.H) {
            const uint8_t* src = img + size_t(fz) * g.frame_pitch + size_t(gy) * g.img_pitch;
            for (int b = 0; b < 32; ++b) {
                const uint32_t gx = x0 + col0 + b;
                if (gx < g.W && src[gx] == 1) m |= 1u << b;
            }
        }
        M[row * C::WX + wx] = m;
        __syncthreads();
    }

    // ---- coarse row scan: word-local runs are the nodes (pixel nodes for CC2FL/NC2FL)
    constexpr bool RUNS = (VAR == 0 || VAR == 1);
    const uint32_t st = RUNS ? (m & ~(m << 1)) : m;
    uint32_t um = __shfl_up_sync(0xffffffffu, m, 1);
    if (lane == 0) um = (wy > 0) ? M[(row - 1) * C::WX + wx] : 0u;
    const uint32_t ust = RUNS ? (um & ~(um << 1)) : um;
    const uint32_t nbase = uint32_t(row * C::PS + col0);

    // ---- init + coarse column scan (no atomics: plain parent links upward).
    // C2FL links a run to the first run above it that it overlaps -- and, since
    // the masks of the rows above are at hand (shuffles), keeps climbing that
    // first-overlap path up to CLIMB rows in registers, linking straight to the
    // highest ancestor reached: vertical coarse chains come out CLIMB x shorter.
    {
        constexpr int CLIMB = CCL_CLIMB;
        uint32_t ups[CLIMB];
        ups[0] = um;
#pragma unroll
        for (int k = 1; k < CLIMB; ++k) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, m, k + 1);
            ups[k] = lane > k ? v : 0u;  // rows above this warp's band are not climbed
        }
        uint32_t t = st;
        while (t) {
            const uint32_t b = __ffs(t) - 1;
            t &= t - 1;
            uint32_t par = nbase + b;
            if (VAR == 0) {  // C2FL: run -> the run at the top of the vertical fg run
                             // through its first overlap column (<= CLIMB rows up)
                const uint32_t mb = m >> b;
                const uint32_t ov = ((mb & ~(mb + 1u)) << b) & um;
                if (ov) {
                    const uint32_t f = __ffs(ov) - 1;
                    uint32_t u = um, k = 0;
#pragma unroll
                    for (int j = 1; j < CLIMB; ++j) {
                        const bool up = (k == uint32_t(j - 1)) && ((ups[j] >> f) & 1u);
                        k = up ? uint32_t(j) : k;
                        u = up ? ups[j] : u;
                    }
                    par = nbase - (k + 1) * C::PS + hi_bit_le(u & ~(u << 1), f);
                }
            } else if (VAR == 2) {  // CC2FL: pixel -> pixel above
                if ((um >> b) & 1u) par = nbase + b - C::PS;
            }
            P[nbase + b] = node_t(par);
        }
    }
    __syncthreads();

    // ---- refinement: min-union of the adjacencies the coarse scans did not link
    if (RUNS) {
        const uint32_t o = m & um;
        uint32_t U = o & ~(o << 1);                   // one pair per overlapping (run, upper run)
        if (VAR == 0) U &= has_lower_in_run(m, o);   // first overlap already linked by the column scan
        while (U) {
            const uint32_t b = __ffs(U) - 1;
            U &= U - 1;
            nunion(P, nbase + hi_bit_le(st, b), nbase - C::PS + hi_bit_le(ust, b));
        }
    } else {
        if (VAR == 3) {  // NC2FL: every vertical pair
            uint32_t U = m & um;
            while (U) {
                const uint32_t b = __ffs(U) - 1;
                U &= U - 1;
                nunion(P, nbase + b, nbase + b - C::PS);
            }
        }
        uint32_t hp = (m & (m << 1)) & ~(um & (um << 1));  // row pairs, minus closed 2x2 squares
        while (hp) {
            const uint32_t b = __ffs(hp) - 1;
            hp &= hp - 1;
            nunion(P, nbase + b, nbase + b - 1);
        }
    }
    if (wx > 0 && (m & 1u)) {  // run continuing across the word boundary
        const uint32_t lm = M[row * C::WX + wx - 1];
        if (lm >> 31) {
            const uint32_t lst = RUNS ? (lm & ~(lm << 1)) : lm;
            nunion(P, nbase, nbase - 32 + (31 - __clz(lst)));
        }
    }
    __syncthreads();

    // ---- seam-touching roots (components reaching a side that faces a
    // neighbour tile/strip): marked once via the F bitmap, ranked by arrival
    // and TAGGED in their own entry (0x8000 | rank) after a barrier, so a
    // single read-only walk per run later yields either an interior root or
    // the rank of a seam root.  No whole-tile flatten pass is needed.
    const bool has_top = ty > 0 || g.edge_above;
    const bool has_bot = ty + 1 < g.nty || g.edge_below;
    const bool has_left = tx > 0, has_right = tx + 1 < g.ntx;
    uint32_t* FR = reinterpret_cast<uint32_t*>(smem + C::FR_OFF);  // [0] = count, [1..] = roots
    auto mark = [&](uint32_t n) {
        const uint32_t x = nfind(P, n);
        const uint32_t bit = 1u << (x & 31);
        if (!(atomicOr(&F[x >> 5], bit) & bit)) FR[1 + atomicAdd(FR, 1u)] = x;
    };
    if (wy == 0 && has_top) {
        const uint32_t s0 = __shfl_sync(0xffffffffu, st, 0);
        if ((s0 >> lane) & 1u) mark(col0 + lane);
    }
    if (wy == C::WY - 1 && has_bot) {
        const uint32_t sl = __shfl_sync(0xffffffffu, st, 31);
        if ((sl >> lane) & 1u) mark((C::TH - 1) * C::PS + col0 + lane);
    }
    if (wx == 0 && has_left && (m & 1u)) mark(nbase);
    if (wx == C::WX - 1 && has_right && (m >> 31)) mark(nbase + hi_bit_le(st, 31));
    __syncthreads();
    const uint32_t nf = FR[0];
    for (uint32_t k = tid; k < nf; k += C::NT) P[FR[1 + k]] = node_t(kTag | k);
    __syncthreads();
    const uint32_t rootmask = 0u;
    return LaneState{m, st, rootmask};
}

template <class C>
__device__ __forceinline__ uint32_t node_gidx(uint32_t node, uint32_t x0, uint32_t y0, const Geo& g) {
    const uint32_t r = node / C::PS;
    const uint32_t c = node - r * C::PS;
    return (g.row0 + y0 + r) * g.W + x0 + c;  // global raster index (convert_ids)
}

// Read-only walk to a run's root after tagging: returns the root node id and
// sets `tag` to 0x8000|rank for seam-touching roots (0 otherwise).
// (Path halving here was measured: it shortens spiral chains but costs more
// than it saves on random d=0.5 tiles, whose chains are short.)
__device__ __forceinline__ uint32_t walk_root(const node_t* P, uint32_t x, uint32_t& tag) {
    uint32_t p = P[x];
    while (p != x && !(p & kTag)) {
        x = p;
        p = P[x];
    }
    tag = (p & kTag) ? p : 0u;
    return x;
}

// ------------------------------------------------------------------ kernel (a)(b)(c)
template <class C, int VAR, bool TMA>
__global__ void __launch_bounds__(C::NT, CCL_MINB) k_local(const __grid_constant__ CUtensorMap tm_img, const uint8_t* img,
                                                    uint32_t* L, uint32_t* work, Geo g) {
    uint8_t* smem = aligned_smem();
    const uint32_t tx = blockIdx.x, ty = blockIdx.y, fz = blockIdx.z;
    if (TMA && threadIdx.x == 0) prefetch_tmap(&tm_img);
    const LaneState s = tile_local<C, VAR, TMA>(&tm_img, img, g, tx, ty, fz, smem);
    node_t* P = reinterpret_cast<node_t*>(smem);
    const uint32_t* M = reinterpret_cast<const uint32_t*>(smem + C::M_OFF);
    uint16_t* STG = reinterpret_cast<uint16_t*>(smem + C::IMG_OFF);  // image tile is dead: run-table staging
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wx = warp % C::WX, wy = warp / C::WX;
    const int row = wy * 32 + lane, col0 = wx * 32;
    const uint32_t x0 = tx * C::TW, y0 = ty * C::TH;
    const uint32_t nbase = uint32_t(row * C::PS + col0);
    uint32_t* Lf = L + size_t(fz) * g.frame_px;  // strip/frame-local index = global - base
    const size_t ntiles = size_t(g.ntx) * g.nty * gridDim.z;
    const Work<C> wk(work, ntiles, (size_t(fz) * g.nty + ty) * g.ntx + tx);

    const uint32_t* FR = reinterpret_cast<const uint32_t*>(smem + C::FR_OFF);
    const uint32_t nf = FR[0];
    if (tid == 0) wk.hdr[0] = nf;
    // run table: one u16 per row run, in (row, run) order per warp; seam-touching
    // roots carry 0x8000 | rank (the index into this tile's seam-root list)
    const uint32_t rst = s.m & ~(s.m << 1);
    const uint32_t cnt = __popc(rst);
    uint32_t inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
    {
        uint16_t* dst = STG + warp * C::TBL_PER_WARP + (inc - cnt);
        uint32_t t = rst;
        while (t) {
            const uint32_t b = __ffs(t) - 1;
            t &= t - 1;
            uint32_t tag;
            const uint32_t r = walk_root(P, nbase + b, tag);
            *dst++ = tag ? uint16_t(0x8000u | (tag & 0x7FFFu)) : uint16_t(r);
        }
    }
    if (lane == 0) wk.hdr[1 + warp] = total;
    // seam-root list (global raster indices, rank order) + forest registration L[g] = g
    for (uint32_t k = tid; k < nf; k += C::NT) {
        const uint32_t gi = node_gidx<C>(FR[1 + k], x0, y0, g);
        wk.hdr[1 + C::NWARP + k] = gi;
        Lf[gi - g.base] = gi;
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0 && total) bulk_store(wk.tbl + warp * C::TBL_PER_WARP, STG + warp * C::TBL_PER_WARP, (total * 2 + 15) & ~15u);
    __syncthreads();
    if (tid == 0) bulk_store(wk.masks, M, C::MASK_WORDS * 4);
    if (lane == 0) asm volatile("cp.async.bulk.commit_group;" ::: "memory");

    // seam pixels: their local root (global index) or background
    const bool has_top = ty > 0 || g.edge_above;
    const bool has_bot = ty + 1 < g.nty || g.edge_below;
    const uint32_t gx = x0 + col0 + lane;
    if (wy == 0 && has_top) {
        const uint32_t m0 = __shfl_sync(0xffffffffu, s.m, 0), s0 = __shfl_sync(0xffffffffu, s.st, 0);
        if (gx < g.W) {
            uint32_t v = kBG;
            if ((m0 >> lane) & 1u) { uint32_t tg; v = node_gidx<C>(walk_root(P, col0 + hi_bit_le(s0, lane), tg), x0, y0, g); }
            Lf[size_t(y0) * g.W + gx] = v;
        }
    }
    if (wy == C::WY - 1 && has_bot) {
        const uint32_t ml = __shfl_sync(0xffffffffu, s.m, 31), sl = __shfl_sync(0xffffffffu, s.st, 31);
        if (gx < g.W) {
            uint32_t v = kBG;
            if ((ml >> lane) & 1u) { uint32_t tg; v = node_gidx<C>(walk_root(P, (C::TH - 1) * C::PS + col0 + hi_bit_le(sl, lane), tg), x0, y0, g); }
            Lf[size_t(y0 + C::TH - 1) * g.W + gx] = v;
        }
    }
    const uint32_t gy = y0 + row;
    if (gy < g.H) {
        if (wx == 0 && tx > 0) {
            uint32_t tg; const uint32_t v = (s.m & 1u) ? node_gidx<C>(walk_root(P, nbase, tg), x0, y0, g) : kBG;
            Lf[size_t(gy) * g.W + x0] = v;
        }
        if (wx == C::WX - 1 && tx + 1 < g.ntx) {
            uint32_t tg; const uint32_t v = (s.m >> 31) ? node_gidx<C>(walk_root(P, nbase + hi_bit_le(s.st, 31), tg), x0, y0, g) : kBG;
            Lf[size_t(gy) * g.W + x0 + C::TW - 1] = v;
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// ------------------------------------------------------------------ kernel (d)
// One thread per interior seam pixel pair; pairs whose left (resp. upper)
// neighbour pair is also foreground on both sides join the same two local
// components and are skipped (one union per overlapping run).
template <class C>
__global__ void __launch_bounds__(256) k_seams(uint32_t* L, Geo g) {
    const uint32_t fz = blockIdx.y;
    uint32_t* Lf = L + size_t(fz) * g.frame_px;
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t nh = uint64_t(g.W) * (g.nty - 1);
    const uint64_t nv = uint64_t(g.H) * (g.ntx - 1);
    const int lane = threadIdx.x & 31;
    uint32_t a = kBG, b = kBG;
    bool can_dedup = false;
    size_t p = 0, step = 0;
    if (t < nh) {
        const uint32_t k = uint32_t(t / g.W), x = uint32_t(t - uint64_t(k) * g.W);
        p = size_t((k + 1) * C::TH) * g.W + x;
        step = 1;  // neighbour pair along the seam is at x-1
        a = Lf[p];
        b = Lf[p - g.W];
        can_dedup = (x % C::TW) != 0;
    } else if (t - nh < nv) {
        const uint64_t u = t - nh;
        const uint32_t k = uint32_t(u / g.H), y = uint32_t(u - uint64_t(k) * g.H);
        p = size_t(y) * g.W + size_t(k + 1) * C::TW;
        step = g.W;  // neighbour pair along the seam is at y-1
        a = Lf[p];
        b = Lf[p - 1];
        can_dedup = (y % C::TH) != 0;
    }
    const bool fg = (a != kBG) && (b != kBG);
    bool prev = __shfl_up_sync(0xffffffffu, fg, 1);
    if (fg && can_dedup && lane == 0) {
        const size_t q = p - step;
        prev = (Lf[q] != kBG) && (Lf[q - (step == 1 ? size_t(g.W) : size_t(1))] != kBG);
    }
    if (fg && !(can_dedup && prev)) gunion(Lf, g.base, a, b);
}

// ------------------------------------------------------------------ kernel (e)
// Reads only the tile's masks + run table + seam-root list (written by (a)),
// resolves each seam-touching root once through the global forest, expands
// runs to pixels and writes every label exactly once.
template <class C, bool TMA_ST>
__global__ void __launch_bounds__(C::NT, 4) k_final(const __grid_constant__ CUtensorMap tm_lab, uint32_t* L,
                                                    const uint32_t* work, Geo g) {
    uint8_t* smem = aligned_smem();
    uint32_t* M = reinterpret_cast<uint32_t*>(smem + C::E_M_OFF);
    uint32_t* HDR = reinterpret_cast<uint32_t*>(smem + C::E_HDR_OFF);
    uint32_t* FT = reinterpret_cast<uint32_t*>(smem + C::E_FT_OFF);
    uint16_t* TBL = reinterpret_cast<uint16_t*>(smem + C::E_TBL_OFF);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::E_BAR_OFF);
    const uint32_t tx = blockIdx.x, ty = blockIdx.y, fz = blockIdx.z;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wx = warp % C::WX, wy = warp / C::WX;
    const int row = wy * 32 + lane;
    const uint32_t x0 = tx * C::TW, y0 = ty * C::TH;
    uint32_t* Lf = L + size_t(fz) * g.frame_px;
    const size_t ntiles = size_t(g.ntx) * g.nty * gridDim.z;
    const Work<C> wk(const_cast<uint32_t*>(work), ntiles, (size_t(fz) * g.nty + ty) * g.ntx + tx);

    if (tid == 0) {
        if (TMA_ST) prefetch_tmap(&tm_lab);
        mbar_init(bar, 1);
        mbar_expect_tx(bar, (C::MASK_WORDS + C::HDR_WORDS) * 4);
        bulk_load(M, wk.masks, C::MASK_WORDS * 4, bar);
        bulk_load(HDR, wk.hdr, C::HDR_WORDS * 4, bar);
    }
    __syncthreads();
    mbar_wait(bar, 0);
    const uint32_t m = M[row * C::WX + wx];
    const uint32_t st = m & ~(m << 1);
    const uint32_t cnt = __popc(st);
    uint32_t inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
    {   // this warp's run entries -> smem (coalesced 16-byte loads)
        const uint4* src = reinterpret_cast<const uint4*>(wk.tbl + warp * C::TBL_PER_WARP);
        uint4* dst = reinterpret_cast<uint4*>(TBL + warp * C::TBL_PER_WARP);
        for (uint32_t i = lane; i < (total * 2 + 15) / 16; i += 32) dst[i] = __ldg(src + i);
    }
    // each seam-touching root resolved once through the global forest
    const uint32_t nF = HDR[0];
    for (uint32_t k = tid; k < nF; k += C::NT) FT[k] = gfind_ro(Lf, g.base, HDR[1 + C::NWARP + k]);
    __syncthreads();

    // run labels at the run starts of this lane's staging row, then expand
    uint8_t* stg = smem + C::E_STG_OFF + warp * 4096;  // 32 x 32 u32, 128B-swizzled
    uint8_t* myrow = stg + lane * 128;
    const int sw = lane & 7;
    {
        const uint16_t* e = TBL + warp * C::TBL_PER_WARP + (inc - cnt);
        uint32_t t = st;
        while (t) {
            const uint32_t b = __ffs(t) - 1;
            t &= t - 1;
            const uint32_t v = *e++;
            const uint32_t lab = (v & 0x8000u) ? FT[v & 0x7FFFu] : node_gidx<C>(v, x0, y0, g);
            *reinterpret_cast<uint32_t*>(myrow + ((((b >> 2) ^ sw) << 4) | ((b & 3) << 2))) = lab;
        }
    }
    uint32_t cur = kBG;
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
                    const uint32_t gx = x0 + wx * 32 + 4 * c + q;
                    if (gx < g.W) Lf[size_t(gy) * g.W + gx] = a[q];
                }
            }
        }
    }
    if (TMA_ST) {
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
            tma_store_3d(&tm_lab, int(x0 + wx * 32), int(y0 + wy * 32), int(fz), stg);  // OOB clipped
            tma_store_commit_and_wait();
        }
    }
}

// ================================================================== host side
template <int VAR>
static cudaError_t launch_local_v(const LaunchArgs& a) {
    using C = TileCfg;
    const dim3 grid(a.g.ntx, a.g.nty, a.nframes);
    if (a.tma_load) {
        auto k = k_local<C, VAR, true>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        k<<<grid, C::NT, C::SMEM, a.stream>>>(a.tm_img, a.img, a.labels, a.work, a.g);
    } else {
        auto k = k_local<C, VAR, false>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        k<<<grid, C::NT, C::SMEM, a.stream>>>(a.tm_img, a.img, a.labels, a.work, a.g);
    }
    return cudaGetLastError();
}

cudaError_t launch_local(const LaunchArgs& a) {
    switch (a.variant) {
        case 0: return launch_local_v<0>(a);
        case 1: return launch_local_v<1>(a);
        case 2: return launch_local_v<2>(a);
        default: return launch_local_v<3>(a);
    }
}

cudaError_t launch_final(const LaunchArgs& a) {
    using C = TileCfg;
    const dim3 grid(a.g.ntx, a.g.nty, a.nframes);
    if (a.tma_store) {
        auto k = k_final<C, true>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::E_SMEM);
        k<<<grid, C::NT, C::E_SMEM, a.stream>>>(a.tm_lab, a.labels, a.work, a.g);
    } else {
        auto k = k_final<C, false>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::E_SMEM);
        k<<<grid, C::NT, C::E_SMEM, a.stream>>>(a.tm_lab, a.labels, a.work, a.g);
    }
    return cudaGetLastError();
}

cudaError_t launch_seams(const LaunchArgs& a) {
    const uint64_t n = uint64_t(a.g.W) * (a.g.nty - 1) + uint64_t(a.g.H) * (a.g.ntx - 1);
    if (n == 0) return cudaSuccess;
    const dim3 grid(unsigned((n + 255) / 256), a.nframes);
    k_seams<TileCfg><<<grid, 256, 0, a.stream>>>(a.labels, a.g);
    return cudaGetLastError();
}

size_t work_bytes(uint32_t w, uint32_t h, uint32_t nframes) {
    using C = TileCfg;
    const size_t ntiles = size_t((w + C::TW - 1) / C::TW) * ((h + C::TH - 1) / C::TH) * nframes;
    return ntiles * (size_t(C::MASK_WORDS + C::HDR_WORDS) * 4 + size_t(C::NWARP) * C::TBL_PER_WARP * 2);
}

int tile_w() { return TileCfg::TW; }
int tile_h() { return TileCfg::TH; }

}  // namespace cclk
