// ccl_kernels.cu — the five hand-written sm_100a kernels of the labeler.
//
//   (a)+(b)+(c)  k_local  : TMA-stage a TW x TH tile, warp-bit run detection
//                           (coarse row scan), coarse column link, smem
//                           min-union refinement, flatten (unification);
//                           exports only the tile's seam labels + registers
//                           the seam-touching local roots in the label buffer.
//   (d)          k_seams  : boundary-only pass (Algorithm 2): one thread per
//                           interior tile-seam pixel pair, global atomicMin
//                           union-find directly in the label buffer.
//   (e)          k_final  : recomputes the tile's local labels (cheaper than a
//                           4 B/px round trip), resolves seam-touching roots
//                           through the global forest, and writes every
//                           label exactly once with swizzled TMA stores.
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
    static constexpr int P_BYTES = ((NODES * 4 + 1023) / 1024) * 1024;
    static constexpr int F_OFF = P_BYTES;
    static constexpr int M_OFF = F_OFF + ((FW * 4 + 127) / 128) * 128;
    static constexpr int IMG_OFF = M_OFF + ((TH * WX * 4 + 127) / 128) * 128;
    static constexpr int BAR_OFF = IMG_OFF + TW * TH;
    static constexpr int SMEM = BAR_OFF + 64 + 1024;  // +1024: runtime base alignment slack
    static_assert(NWARP * 4096 <= NODES * 4, "output staging must fit in the node array");
    static_assert(TW <= 256 && TH <= 256, "TMA box dims are limited to 256");
};

using TileCfg = Cfg<CCL_TILE_WX, CCL_TILE_WY>;

__device__ __forceinline__ uint8_t* aligned_smem() {
    extern __shared__ uint8_t smem_raw[];
    return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
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
    uint32_t* P = reinterpret_cast<uint32_t*>(smem);
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

    // ---- init + coarse column scan (no atomics: plain parent links to the row above)
    {
        uint32_t t = st;
        while (t) {
            const uint32_t b = __ffs(t) - 1;
            t &= t - 1;
            uint32_t par = nbase + b;
            if (VAR == 0) {  // C2FL: run -> upper run under its first overlap
                const uint32_t mb = m >> b;
                const uint32_t ov = ((mb & ~(mb + 1u)) << b) & um;
                if (ov) par = nbase - C::PS + hi_bit_le(ust, __ffs(ov) - 1);
            } else if (VAR == 2) {  // CC2FL: pixel -> pixel above
                if ((um >> b) & 1u) par = nbase + b - C::PS;
            }
            P[nbase + b] = par;
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
            sunion(P, nbase + hi_bit_le(st, b), nbase - C::PS + hi_bit_le(ust, b));
        }
    } else {
        if (VAR == 3) {  // NC2FL: every vertical pair
            uint32_t U = m & um;
            while (U) {
                const uint32_t b = __ffs(U) - 1;
                U &= U - 1;
                sunion(P, nbase + b, nbase + b - C::PS);
            }
        }
        uint32_t hp = (m & (m << 1)) & ~(um & (um << 1));  // row pairs, minus closed 2x2 squares
        while (hp) {
            const uint32_t b = __ffs(hp) - 1;
            hp &= hp - 1;
            sunion(P, nbase + b, nbase + b - 1);
        }
    }
    if (wx > 0 && (m & 1u)) {  // run continuing across the word boundary
        const uint32_t lm = M[row * C::WX + wx - 1];
        if (lm >> 31) {
            const uint32_t lst = RUNS ? (lm & ~(lm << 1)) : lm;
            sunion(P, nbase, nbase - 32 + (31 - __clz(lst)));
        }
    }
    __syncthreads();

    // ---- unification: every node points at its root.  Two passes: path-halving
    // stores of other lanes may still overwrite an entry this lane has already
    // flattened (with a valid but non-root ancestor), so pass 1 compresses and
    // pass 2, after a barrier, re-reads the now short chains without writing
    // anything but the node's own entry.
    uint32_t rootmask = 0u;
    {
        uint32_t t = st;
        while (t) {
            const uint32_t b = __ffs(t) - 1;
            t &= t - 1;
            const uint32_t n = nbase + b;
            const uint32_t r = sfind(P, n);
            P[n] = r;
            if (r == n) rootmask |= 1u << b;
        }
    }
    __syncthreads();
    {
        volatile uint32_t* vP = P;
        uint32_t t = st & ~rootmask;
        while (t) {
            const uint32_t b = __ffs(t) - 1;
            t &= t - 1;
            const uint32_t n = nbase + b;
            uint32_t r = vP[n];
            for (uint32_t q = vP[r]; q != r; q = vP[r]) r = q;
            vP[n] = r;
        }
    }
    __syncthreads();

    // ---- flag roots of components touching a side that faces a neighbour
    const bool has_top = ty > 0 || g.edge_above;
    const bool has_bot = ty + 1 < g.nty || g.edge_below;
    const bool has_left = tx > 0, has_right = tx + 1 < g.ntx;
    auto mark = [&](uint32_t r) { atomicOr(&F[r >> 5], 1u << (r & 31)); };
    if (wy == 0 && has_top) {
        const uint32_t s0 = __shfl_sync(0xffffffffu, st, 0);
        if ((s0 >> lane) & 1u) mark(P[col0 + lane]);
    }
    if (wy == C::WY - 1 && has_bot) {
        const uint32_t sl = __shfl_sync(0xffffffffu, st, 31);
        if ((sl >> lane) & 1u) mark(P[(C::TH - 1) * C::PS + col0 + lane]);
    }
    if (wx == 0 && has_left && (m & 1u)) mark(P[nbase]);
    if (wx == C::WX - 1 && has_right && (m >> 31)) mark(P[nbase + hi_bit_le(st, 31)]);
    __syncthreads();
    return LaneState{m, st, rootmask};
}

template <class C>
__device__ __forceinline__ uint32_t node_gidx(uint32_t node, uint32_t x0, uint32_t y0, const Geo& g) {
    const uint32_t r = node / C::PS;
    const uint32_t c = node - r * C::PS;
    return (g.row0 + y0 + r) * g.W + x0 + c;  // global raster index (convert_ids)
}

// ------------------------------------------------------------------ kernel (a)(b)(c)
template <class C, int VAR, bool TMA>
__global__ void __launch_bounds__(C::NT, 3) k_local(const __grid_constant__ CUtensorMap tm_img, const uint8_t* img,
                                                 uint32_t* L, Geo g) {
    uint8_t* smem = aligned_smem();
    const uint32_t tx = blockIdx.x, ty = blockIdx.y, fz = blockIdx.z;
    if (TMA && threadIdx.x == 0) prefetch_tmap(&tm_img);
    const LaneState s = tile_local<C, VAR, TMA>(&tm_img, img, g, tx, ty, fz, smem);
    const uint32_t* P = reinterpret_cast<const uint32_t*>(smem);
    const uint32_t* F = reinterpret_cast<const uint32_t*>(smem + C::F_OFF);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wx = warp % C::WX, wy = warp / C::WX;
    const int row = wy * 32 + lane, col0 = wx * 32;
    const uint32_t x0 = tx * C::TW, y0 = ty * C::TH;
    const uint32_t nbase = uint32_t(row * C::PS + col0);
    uint32_t* Lf = L + size_t(fz) * g.frame_px;  // strip/frame-local index = global - base

    // register seam-touching roots as global forest nodes: L[g] = g
    uint32_t t = s.rootmask;
    while (t) {
        const uint32_t b = __ffs(t) - 1;
        t &= t - 1;
        const uint32_t n = nbase + b;
        if ((F[n >> 5] >> (n & 31)) & 1u) {
            const uint32_t gi = node_gidx<C>(n, x0, y0, g);
            Lf[gi - g.base] = gi;
        }
    }
    // seam pixels: their local root (global index) or background
    const bool has_top = ty > 0 || g.edge_above;
    const bool has_bot = ty + 1 < g.nty || g.edge_below;
    const uint32_t gx = x0 + col0 + lane;
    if (wy == 0 && has_top) {
        const uint32_t m0 = __shfl_sync(0xffffffffu, s.m, 0), s0 = __shfl_sync(0xffffffffu, s.st, 0);
        if (gx < g.W) {
            uint32_t v = kBG;
            if ((m0 >> lane) & 1u) v = node_gidx<C>(P[col0 + hi_bit_le(s0, lane)], x0, y0, g);
            Lf[size_t(y0) * g.W + gx] = v;
        }
    }
    if (wy == C::WY - 1 && has_bot) {
        const uint32_t ml = __shfl_sync(0xffffffffu, s.m, 31), sl = __shfl_sync(0xffffffffu, s.st, 31);
        if (gx < g.W) {
            uint32_t v = kBG;
            if ((ml >> lane) & 1u) v = node_gidx<C>(P[(C::TH - 1) * C::PS + col0 + hi_bit_le(sl, lane)], x0, y0, g);
            Lf[size_t(y0 + C::TH - 1) * g.W + gx] = v;
        }
    }
    const uint32_t gy = y0 + row;
    if (gy < g.H) {
        if (wx == 0 && tx > 0) {
            const uint32_t v = (s.m & 1u) ? node_gidx<C>(P[nbase], x0, y0, g) : kBG;
            Lf[size_t(gy) * g.W + x0] = v;
        }
        if (wx == C::WX - 1 && tx + 1 < g.ntx) {
            const uint32_t v = (s.m >> 31) ? node_gidx<C>(P[nbase + hi_bit_le(s.st, 31)], x0, y0, g) : kBG;
            Lf[size_t(gy) * g.W + x0 + C::TW - 1] = v;
        }
    }
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
template <class C, int VAR, bool TMA, bool TMA_ST>
__global__ void __launch_bounds__(C::NT, 3) k_final(const __grid_constant__ CUtensorMap tm_img,
                                                 const __grid_constant__ CUtensorMap tm_lab, const uint8_t* img,
                                                 uint32_t* L, Geo g) {
    uint8_t* smem = aligned_smem();
    const uint32_t tx = blockIdx.x, ty = blockIdx.y, fz = blockIdx.z;
    if (threadIdx.x == 0) {
        if (TMA) prefetch_tmap(&tm_img);
        if (TMA_ST) prefetch_tmap(&tm_lab);
    }
    const LaneState s = tile_local<C, VAR, TMA>(&tm_img, img, g, tx, ty, fz, smem);
    uint32_t* P = reinterpret_cast<uint32_t*>(smem);
    const uint32_t* F = reinterpret_cast<const uint32_t*>(smem + C::F_OFF);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wx = warp % C::WX, wy = warp / C::WX;
    const int row = wy * 32 + lane, col0 = wx * 32;
    const uint32_t x0 = tx * C::TW, y0 = ty * C::TH;
    const uint32_t nbase = uint32_t(row * C::PS + col0);
    uint32_t* Lf = L + size_t(fz) * g.frame_px;

    // (e1) final label of each local root; seam-touching roots walk the global forest
    {
        uint32_t t = s.rootmask;
        while (t) {
            const uint32_t b = __ffs(t) - 1;
            t &= t - 1;
            const uint32_t n = nbase + b;
            const uint32_t gi = node_gidx<C>(n, x0, y0, g);
            P[n] = ((F[n >> 5] >> (n & 31)) & 1u) ? gfind_ro(Lf, g.base, gi) : gi;
        }
    }
    __syncthreads();
    // (e2) expand to pixels: root segments hold the label, others point at their root
    uint32_t lab[32];
    uint32_t cur = kBG;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        if ((s.st >> i) & 1u) {
            const uint32_t v = P[nbase + i];
            if ((s.rootmask >> i) & 1u) cur = v;
            else cur = P[v];
        }
        lab[i] = ((s.m >> i) & 1u) ? cur : kBG;
    }
    __syncthreads();  // node array is dead from here on: reuse it as the store staging
    if (TMA_ST) {
        uint8_t* stg = smem + warp * 4096;  // 32x32 u32, 128B-swizzled (1024B-aligned)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const uint4 v = make_uint4(lab[4 * c], lab[4 * c + 1], lab[4 * c + 2], lab[4 * c + 3]);
            *reinterpret_cast<uint4*>(stg + lane * 128 + ((c ^ (lane & 7)) << 4)) = v;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
            tma_store_3d(&tm_lab, int(x0 + col0), int(y0 + wy * 32), int(fz), stg);  // OOB clipped
            tma_store_commit_and_wait();
        }
    } else {
        const uint32_t gy = y0 + row;
        if (gy < g.H) {
            uint32_t* dst = Lf + size_t(gy) * g.W;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const uint32_t gx = x0 + col0 + i;
                if (gx < g.W) dst[gx] = lab[i];
            }
        }
    }
}

// ================================================================== host side
template <int VAR>
static cudaError_t launch_variant(const LaunchArgs& a, int phase) {
    using C = TileCfg;
    const dim3 grid(a.g.ntx, a.g.nty, a.nframes);
    const dim3 block(C::NT);
    if (phase == 0) {
        if (a.tma_load) {
            auto k = k_local<C, VAR, true>;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
            k<<<grid, block, C::SMEM, a.stream>>>(a.tm_img, a.img, a.labels, a.g);
        } else {
            auto k = k_local<C, VAR, false>;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
            k<<<grid, block, C::SMEM, a.stream>>>(a.tm_img, a.img, a.labels, a.g);
        }
    } else {
#define CCL_LAUNCH_FINAL(TL, TS)                                                             \
    {                                                                                        \
        auto k = k_final<C, VAR, TL, TS>;                                                    \
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);       \
        k<<<grid, block, C::SMEM, a.stream>>>(a.tm_img, a.tm_lab, a.img, a.labels, a.g);     \
    }
        if (a.tma_load && a.tma_store) CCL_LAUNCH_FINAL(true, true)
        else if (a.tma_load) CCL_LAUNCH_FINAL(true, false)
        else if (a.tma_store) CCL_LAUNCH_FINAL(false, true)
        else CCL_LAUNCH_FINAL(false, false)
#undef CCL_LAUNCH_FINAL
    }
    return cudaGetLastError();
}

cudaError_t launch_local(const LaunchArgs& a) {
    switch (a.variant) {
        case 0: return launch_variant<0>(a, 0);
        case 1: return launch_variant<1>(a, 0);
        case 2: return launch_variant<2>(a, 0);
        default: return launch_variant<3>(a, 0);
    }
}

cudaError_t launch_final(const LaunchArgs& a) {
    switch (a.variant) {
        case 0: return launch_variant<0>(a, 1);
        case 1: return launch_variant<1>(a, 1);
        case 2: return launch_variant<2>(a, 1);
        default: return launch_variant<3>(a, 1);
    }
}

cudaError_t launch_seams(const LaunchArgs& a) {
    const uint64_t n = uint64_t(a.g.W) * (a.g.nty - 1) + uint64_t(a.g.H) * (a.g.ntx - 1);
    if (n == 0) return cudaSuccess;
    const dim3 grid(unsigned((n + 255) / 256), a.nframes);
    k_seams<TileCfg><<<grid, 256, 0, a.stream>>>(a.labels, a.g);
    return cudaGetLastError();
}

int tile_w() { return TileCfg::TW; }
int tile_h() { return TileCfg::TH; }

}  // namespace cclk
