// ccl_device.cuh — device-side building blocks of the sm_100a labeler.
//
// Reference mapping (arXiv 1712.09789 as restated in /root/reference/proj):
//   foreground predicate byte == 1 ......... local_labeler.cpp:59,64 / oracle.cpp:41-43
//   parent[i] <= i forest, min-union ........ forest.hpp:44-111
//   find_root / flatten ..................... forest.hpp:72-92
//   coarse row scan (runs) .................. local_labeler.cpp:30-38  -> word-level run starts
//   coarse column scan ...................... local_labeler.cpp:40-48  -> link run to first upper overlap
//   refine (min-union merges) ............... local_labeler.cpp:55-68  -> smem atomicMin union
//   convert_ids (local -> global raster idx). local_labeler.cpp:102-112
//   merge_borders ........................... boundary.cpp:22-35       -> global atomicMin union
//   resolve_global .......................... boundary.cpp:37-55       -> path-compressing relabel
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#ifndef CCL_METRICS
#define CCL_METRICS 0
#endif
#ifndef CCL_UNITE_COMPRESS
#define CCL_UNITE_COMPRESS 2  // kernel (d): after a union both start nodes (and the node above each, when not already one hop below) point at the root
#endif

namespace cclk {

constexpr uint32_t kBG = 0xFFFFFFFFu;

// Per-thread cost counters of an instrumented build (-DCCL_METRICS=1, a
// separate library): the two cost drivers the reference reports per block
// (BlockMetrics, forest.hpp:12-29) -- parent-link steps taken while finding
// roots, and CAS attempts (successful or failed) of unions.  Empty otherwise.
struct Ctr {
#if CCL_METRICS
    uint32_t f = 0, c = 0;
    __device__ __forceinline__ void step(uint32_t n = 1) { f += n; }
    __device__ __forceinline__ void cas() { ++c; }
#else
    __device__ __forceinline__ void step(uint32_t = 1) {}
    __device__ __forceinline__ void cas() {}
#endif
};

// ---------------------------------------------------------------- bit helpers
// Foreground bits of 4 bytes: bit k set iff byte k == 1 (exact for any byte value).
__device__ __forceinline__ uint32_t eq1_nibble(uint32_t v) {
    const uint32_t x = v ^ 0x01010101u;                 // zero bytes where v == 1
    uint32_t y = (x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu;       // high bit set where low 7 bits != 0
    y = ~(y | x | 0x7F7F7F7Fu);                         // 0x80 exactly in the zero bytes of x
    // gather bits 7,15,23,31 -> nibble: the partial products land on distinct
    // bits (7,14,15,21,22,23 below the nibble), so no carry reaches bits 28-31
    return (y * 0x00204081u) >> 28;
}
__device__ __forceinline__ uint32_t eq1_mask16(uint4 q) {
    return eq1_nibble(q.x) | (eq1_nibble(q.y) << 4) | (eq1_nibble(q.z) << 8) | (eq1_nibble(q.w) << 12);
}
// Same for a chunk whose bytes are all 0 or 1 (the caller checks): byte k's
// low bit gathered to bit k of each nibble by one multiply per word
// (bits 21-24 of v * 0x00204081 are exactly b0..b3; the cross terms land on
// bits 0-16 and 29-31 and cannot carry into them).
__device__ __forceinline__ uint32_t bin_mask16(uint4 q) {
    constexpr uint32_t G = 0x00204081u;
    return (((q.x * G) >> 21) & 0xFu) | (((q.y * G) >> 17) & 0xF0u) | (((q.z * G) >> 13) & 0xF00u) |
           (((q.w * G) >> 9) & 0xF000u);
}
// Highest set bit of s at or below bit b (caller guarantees one exists).
__device__ __forceinline__ uint32_t hi_bit_le(uint32_t s, uint32_t b) {
    return 31u - __clz(s & (0xFFFFFFFFu >> (31u - b)));
}
// Bits b of o such that some bit of o lies strictly below b inside the same
// run of m (o must be a subset of m): the carry-in vector of m + o, within m.
__device__ __forceinline__ uint32_t has_lower_in_run(uint32_t m, uint32_t o) {
    return ((m + o) ^ m ^ o) & m;
}

// ----------------------------------------------------------- smem union-find
// Lock-free min-union over a shared-memory parent array (forest.hpp:98-111
// semantics: the larger root is linked below the smaller one, so every class
// is rooted at its minimum node).  atomicMin instead of CAS: a lost race is
// repaired by continuing with the returned parent (Playne-Hawick style).
__device__ __forceinline__ uint32_t sfind(volatile uint32_t* P, uint32_t x) {
    uint32_t p = P[x];
    while (p != x) {
        const uint32_t gp = P[p];
        if (gp == p) return p;
        P[x] = gp;  // path halving; only ever writes an ancestor
        x = gp;
        p = P[x];
    }
    return x;
}
__device__ __forceinline__ void sunion(uint32_t* P, uint32_t a, uint32_t b) {
    volatile uint32_t* vP = P;
    for (;;) {
        a = sfind(vP, a);
        b = sfind(vP, b);
        if (a == b) return;
        if (a < b) { const uint32_t t = a; a = b; b = t; }
        const uint32_t old = atomicMin(&P[a], b);
        if (old == a) return;
        a = old;
    }
}

// --------------------------------------------------------- global union-find
__device__ __forceinline__ uint32_t gload(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Compact global forest (kernels (a) register, (d) unions, (d2) resolves).
// Parents are node ids; the class root is the node with the smallest key, so
// its key is the component's minimum raster index (forest.hpp:98-111 min-union
// semantics, restated over seam-touching roots only).  ~10 MB touched at 8192^2:
// the walks hit L2 instead of scattered HBM sectors of the label buffer.
struct Forest {
    uint32_t* f;  // f[2n] = parent, f[2n+1] = key (one 8-byte load gives both)
    __device__ __forceinline__ uint2 node(uint32_t n) const {
        uint2 v;
        asm volatile("ld.relaxed.gpu.global.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(f + 2 * size_t(n))
                     : "memory");
        return v;
    }
    // L1-cached read for kernel (d2), which runs after every union (after its
    // griddepcontrol.wait): a parent read stale from L1 -- another warp's path
    // compression not yet seen -- is still an ancestor, keys never change.
    // Near the percolation threshold every seam root of the spanning cluster
    // climbs to the same few nodes; through L1 those lines are read once per
    // SM instead of once per warp at one L2 slice (d=0.6: -7 us per step).
    __device__ __forceinline__ uint2 node_ca(uint32_t n) const {
        uint2 v;
        asm volatile("ld.global.ca.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(f + 2 * size_t(n)) : "memory");
        return v;
    }
    __device__ __forceinline__ uint32_t key(uint32_t n) const { return node(n).y; }
    // Root of x and the root's {parent, key}.
    __device__ __forceinline__ uint32_t find(uint32_t x, uint2& v, Ctr& m) const {
        v = node(x);
        while (v.x != x) {
            m.step();
            x = v.x;
            v = node(x);
        }
        return x;
    }
    __device__ __forceinline__ uint32_t find(uint32_t x) const {
        uint2 v;
        Ctr m;
        return find(x, v, m);
    }
    // find + path compression of x itself (later walks through x take one hop)
    __device__ __forceinline__ uint2 find_compress(uint32_t x, Ctr& m) const {
        uint2 v;
        const uint32_t r = find(x, v, m);
        if (r != x) f[2 * size_t(x)] = r;
        return v;
    }
    // Min-key union: the root with the larger key is linked below the other
    // one with a CAS on its parent; both sides climb in lockstep so their
    // loads overlap (the common case is one load per side, then the CAS).
    __device__ __forceinline__ void unite(uint32_t a, uint32_t b, Ctr& m) const {
#if CCL_UNITE_COMPRESS
        const uint32_t a0 = a, b0 = b;
        // afterwards both start nodes point at the class root they reached: a
        // tile's seam root meets many seams, and these are its own (cold) lines
#if CCL_UNITE_COMPRESS >= 2
        // ... and so does the first node above each start when it is not one
        // hop below the root already (written once per node and change: a node
        // that points at the root is never rewritten, so hot nodes stay cold)
        uint32_t a1 = 0xFFFFFFFFu, a1p = 0, b1 = 0xFFFFFFFFu, b1p = 0;
#endif
        auto done = [&](uint32_t r) {
            if (a0 != r && a0 != a) f[2 * size_t(a0)] = r;
            if (b0 != r && b0 != b) f[2 * size_t(b0)] = r;
#if CCL_UNITE_COMPRESS >= 2
            if (a1 != 0xFFFFFFFFu && a1 != r && a1p != r) f[2 * size_t(a1)] = r;
            if (b1 != 0xFFFFFFFFu && b1 != r && b1p != r) f[2 * size_t(b1)] = r;
#endif
        };
#else
        auto done = [](uint32_t) {};
#endif
        uint2 A = node(a), B = node(b);
        for (;;) {
            bool ca = A.x != a, cb = B.x != b;
            while (ca || cb) {
                uint2 An = A, Bn = B;
                if (ca) An = node(A.x);
                if (cb) Bn = node(B.x);
#if CCL_UNITE_COMPRESS >= 2
                if (ca && a1 == 0xFFFFFFFFu) { a1 = A.x; a1p = An.x; }
                if (cb && b1 == 0xFFFFFFFFu) { b1 = B.x; b1p = Bn.x; }
#endif
                // (no path halving here: at high density every union climbs
                // through the same few hot nodes and the extra stores thrash)
                m.step(uint32_t(ca) + uint32_t(cb));
                if (ca) { a = A.x; A = An; ca = A.x != a; }
                if (cb) { b = B.x; B = Bn; cb = B.x != b; }
            }
            if (a == b) {
                done(a);
                return;
            }
            if (A.y < B.y) {  // a: the root with the larger key
                const uint32_t t = a; a = b; b = t;
                const uint2 T = A; A = B; B = T;
            }
            m.cas();
            const uint32_t old = atomicCAS(f + 2 * size_t(a), a, b);
            if (old == a) {
                done(b);
                return;
            }
            a = old;  // a was linked meanwhile: continue from its new parent
            A = node(a);
            B = node(b);
        }
    }
};
// --------------------------------------------------------------- TMA / mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    const uint32_t a = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(a),
        "r"(phase)
        : "memory");
}
// L2 cache policies (createpolicy): streaming data is evicted first so the
// small hand-off buffers between kernels stay L2-resident.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void tma_load_3d_hint(void* dst, const CUtensorMap* tm, int x, int y, int z, uint64_t* bar,
                                                 uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, "
        "%4}], [%5], %6;" ::"r"(smem_u32(dst)),
        "l"(tm), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void tma_store_3d_hint(const CUtensorMap* tm, int x, int y, int z, const void* src,
                                                  uint64_t pol) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2, %3}], [%4], %5;" ::
                     "l"(tm),
                 "r"(x), "r"(y), "r"(z), "r"(smem_u32(src)), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int x, int y, int z, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
            "r"(smem_u32(dst)),
        "l"(tm), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* tm, int x, int y, int z, const void* src) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(tm), "r"(x),
                 "r"(y), "r"(z), "r"(smem_u32(src))
                 : "memory");
}
__device__ __forceinline__ void tma_store_commit_and_wait() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* tm) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(tm) : "memory");
}

}  // namespace cclk
