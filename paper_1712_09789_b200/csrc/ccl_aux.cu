// ccl_aux.cu — strip-mode seam kernels and GPU compaction.
//
// Strip mode: every strip labels its rows in GLOBAL raster
// space with kernels (a)-(d); then a seam step merges components across the
// horizontal strip boundaries:
//   export  : k_strip_roots -> k_strip_repmin -> k_strip_reps
//   exchange: every strip's 4*W seam words into every rank's exchange area
//             (ccl_strips.cu strip groups; a device-local copy for virtual strips)
//   resolve : k_seam_init -> k_seam_union (identical on every strip) -> k_seam_apply
// (all six PDL-chained: each waits for its predecessor before reading)
// Kernel (a) leaves, in the strip area of the work buffer, the compact forest
// node of every top/bottom-row pixel; k_strip_roots resolves them to the
// strip-local roots (exported by key = global raster index) and remembers the
// compact root per column, and k_seam_apply overwrites that root's key with
// the component's final label f <= key (possibly another strip's pixel), which
// kernel (d2) then hands to kernel (e) like any other root label.
// Compaction (pipeline.cpp:54-70): compacted label =
// 1 + rank of the component root among all roots (roots are component minima,
// so raster order of first appearance == ascending root order).
#include <cuda_runtime.h>
#include <stdint.h>

#include "ccl_device.cuh"
#include "ccl_internal.h"

namespace cclk {

// Programmatic dependent launch (as in ccl_kernels.cu): the small strip-seam
// kernels are chained so that each one's launch overlaps its predecessor's
// drain; every kernel waits for its predecessor before reading its output.
__device__ __forceinline__ void aux_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void aux_pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <class K, class... Args>
static cudaError_t aux_launch_pdl(K kernel, unsigned grid, unsigned block, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = CCL_PDL;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// ------------------------------------------------------------ strip export
__global__ void k_strip_roots(const uint32_t* se, Forest fst, uint32_t* L, Geo g, uint32_t* out, uint32_t* croot) {
    aux_pdl_wait();
    aux_pdl_trigger();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 2 * g.W) return;
    const bool top = i < g.W;
    uint32_t r = kBG, cr = kBG;
    if (top ? g.edge_above : g.edge_below) {
        const uint32_t v = se[i];  // compact node of the edge pixel's tile-local root
        if (v != kBG) {
            cr = fst.find(v);      // strip-local root after kernel (d)
            r = fst.key(cr);
            L[r - g.base] = r;     // scratch for k_strip_repmin (L is rewritten by kernel (e))
        }
    }
    out[i] = r;
    croot[i] = cr;
}

// Bottom-row roots that are not on the top row: the first (min x) bottom node
// carrying the root is found with an atomicMin on the root's scratch entry in
// L, encoded as base + x (< base + W <= root, so the root value itself loses).
__global__ void k_strip_repmin(uint32_t* L, Geo g, const uint32_t* out) {
    aux_pdl_wait();
    aux_pdl_trigger();
    const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= g.W) return;
    const uint32_t r = out[g.W + x];
    if (r == kBG) return;
    const uint32_t rl = r - g.base;
    if (rl < g.W) return;  // root pixel is on the (always exported) top row
    atomicMin(L + rl, g.base + x);
}

__global__ void k_strip_reps(const uint32_t* L, Geo g, uint32_t k, uint32_t* out) {
    aux_pdl_wait();
    aux_pdl_trigger();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 2 * g.W) return;
    const uint32_t r = out[i];
    uint32_t rep = kBG;
    if (r != kBG) {
        const uint32_t rl = r - g.base;
        const uint32_t local = rl < g.W ? rl : g.W + (L[rl] - g.base);
        rep = k * 2 * g.W + local;
    }
    out[2 * g.W + i] = rep;
}

// ------------------------------------------------------------ seam resolve
// Nodes: strip s, slot i in [0, 2W) -> s*2W + i (i < W: top row x=i, else
// bottom row x=i-W).  Key = the node's strip root (global raster index); the
// class root is the node with the smallest key, so its key is the component's
// global minimum.  Parents start at the exported reps.
__device__ __forceinline__ uint32_t seam_key(const uint32_t* all, uint32_t W, uint32_t j) {
    const uint32_t s = j / (2 * W);
    return all[size_t(s) * 4 * W + (j - s * 2 * W)];
}
__device__ __forceinline__ uint32_t seam_find(uint32_t* par, uint32_t j) {
    uint32_t p = par[j];
    while (p != j) {
        const uint32_t gp = par[p];
        if (gp == p) return p;
        par[j] = gp;
        j = gp;
        p = par[j];
    }
    return j;
}
__global__ void k_seam_init(const uint32_t* all, uint32_t N, uint32_t W, uint32_t* par) {
    aux_pdl_wait();
    aux_pdl_trigger();
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= uint64_t(N) * 2 * W) return;
    const uint32_t s = uint32_t(t / (2 * W)), i = uint32_t(t - uint64_t(s) * 2 * W);
    par[t] = all[size_t(s) * 4 * W + 2 * W + i];  // every node starts at its exported representative
}
__global__ void k_seam_union(const uint32_t* all, uint32_t N, uint32_t W, uint32_t* par) {
    aux_pdl_wait();
    aux_pdl_trigger();
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= uint64_t(N - 1) * W) return;
    const uint32_t s = uint32_t(t / W), x = uint32_t(t - uint64_t(s) * W);
    const uint32_t* up = all + size_t(s) * 4 * W;  // strip s: bottom roots at [W, 2W)
    const uint32_t* dn = up + 4 * size_t(W);       // strip s+1: top roots at [0, W)
    if (up[W + x] == kBG || dn[x] == kBG) return;
    if (x > 0 && up[W + x - 1] != kBG && dn[x - 1] != kBG) return;  // same strip components as x-1
    uint32_t a = s * 2 * W + W + x, b = (s + 1) * 2 * W + x;
    for (;;) {
        a = seam_find(par, a);
        b = seam_find(par, b);
        if (a == b) return;
        if (seam_key(all, W, a) > seam_key(all, W, b)) {
            const uint32_t tt = a;
            a = b;
            b = tt;
        }
        if (atomicCAS(par + b, b, a) == b) return;  // link larger-key root below smaller-key root
    }
}
__global__ void k_seam_apply(const uint32_t* all, uint32_t W, uint32_t k, uint32_t* par, const uint32_t* croot,
                             Forest fst) {
    aux_pdl_wait();
    aux_pdl_trigger();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 2 * W) return;
    const uint32_t j = k * 2 * W + i;
    const uint32_t r = seam_key(all, W, j);
    if (r == kBG) return;
    const uint32_t q = seam_find(par, j);  // path halving: all unions are done
    fst.f[2 * size_t(croot[i]) + 1] = seam_key(all, W, q);  // final label of this strip root
}

cudaError_t launch_strip_export(const Geo& g, uint32_t* labels, uint32_t* work, uint32_t* seam_out, uint32_t k,
                                cudaStream_t s) {
    const unsigned nb2 = (2 * g.W + 255) / 256, nb1 = (g.W + 255) / 256;
    uint32_t* se = strip_area_ptr(work, g);
    cudaError_t e = aux_launch_pdl(k_strip_roots, nb2, 256, s, static_cast<const uint32_t*>(se),
                                   Forest{forest_ptr(work, g)}, labels, g, seam_out, se + 2 * size_t(g.W));
    if (e == cudaSuccess) e = aux_launch_pdl(k_strip_repmin, nb1, 256, s, labels, g, static_cast<const uint32_t*>(seam_out));
    if (e == cudaSuccess)
        e = aux_launch_pdl(k_strip_reps, nb2, 256, s, static_cast<const uint32_t*>(labels), g, k, seam_out);
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_strip_resolve(const Geo& g, const uint32_t* all, uint32_t N, uint32_t k, uint32_t* labels,
                                 uint32_t* work, uint32_t* scratch, cudaStream_t s) {
    (void)labels;
    const size_t W = g.W;
    cudaError_t e = aux_launch_pdl(k_seam_init, unsigned((uint64_t(N) * 2 * W + 255) / 256), 256, s, all, N, g.W,
                                   scratch);
    if (e == cudaSuccess && N > 1) {
        const uint64_t n = uint64_t(N - 1) * W;
        e = aux_launch_pdl(k_seam_union, unsigned((n + 255) / 256), 256, s, all, N, g.W, scratch);
    }
    if (e == cudaSuccess)
        e = aux_launch_pdl(k_seam_apply, unsigned((2 * W + 255) / 256), 256, s, all, g.W, k,
                           scratch, static_cast<const uint32_t*>(strip_area_ptr(work, g) + 2 * W),
                           Forest{forest_ptr(work, g)});
    return e != cudaSuccess ? e : cudaGetLastError();
}

// ------------------------------------------------------------ compaction
constexpr int kScanBlock = 1024;  // words per scan block (256 threads x 4)

__global__ void k_root_bits(const uint32_t* raw, size_t n, uint32_t* bits, uint32_t* cnt) {
    const size_t p = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool root = p < n && raw[p] == uint32_t(p);
    const uint32_t word = __ballot_sync(0xffffffffu, root);
    if ((threadIdx.x & 31) == 0 && p < n) {
        bits[p >> 5] = word;
        cnt[p >> 5] = __popc(word);
    }
}

// In-place exclusive scan of kScanBlock words per block; block total -> sums.
__global__ void __launch_bounds__(256) k_scan_block(uint32_t* v, size_t n, uint32_t* sums) {
    __shared__ uint32_t warp_tot[8];
    const size_t base = size_t(blockIdx.x) * kScanBlock + threadIdx.x * 4;
    uint32_t x[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = (base + i < n) ? v[base + i] : 0u;
    const uint32_t loc = x[0] + x[1] + x[2] + x[3];
    uint32_t inc = loc;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    uint32_t woff = 0;
    for (int w = 0; w < warp; ++w) woff += warp_tot[w];
    uint32_t run = woff + inc - loc;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (base + i < n) v[base + i] = run;
        run += x[i];
    }
    if (threadIdx.x == 255) sums[blockIdx.x] = woff + inc;
}

// Single-block exclusive scan of the block sums (sequential chunks of 1024).
__global__ void __launch_bounds__(1024) k_scan_sums(uint32_t* sums, uint32_t nb, uint32_t* total) {
    __shared__ uint32_t warp_tot[32];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t b0 = 0; b0 < nb; b0 += 1024) {
        const uint32_t i = b0 + threadIdx.x;
        const uint32_t x = i < nb ? sums[i] : 0u;
        uint32_t inc = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) warp_tot[warp] = inc;
        __syncthreads();
        uint32_t woff = 0;
        for (int w = 0; w < warp; ++w) woff += warp_tot[w];
        const uint32_t c = carry;
        if (i < nb) sums[i] = c + woff + inc - x;
        __syncthreads();
        if (threadIdx.x == 1023) carry = c + woff + inc;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

__global__ void k_scan_add(uint32_t* v, size_t n, const uint32_t* sums) {
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) v[i] += sums[i / kScanBlock];
}

__global__ void k_compact_apply(const uint32_t* raw, size_t n, const uint32_t* bits, const uint32_t* pre,
                                uint32_t* out) {
    const size_t p = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const uint32_t r = raw[p];
    uint32_t v = 0;
    if (r != kBG) v = 1u + pre[r >> 5] + __popc(bits[r >> 5] & ((1u << (r & 31)) - 1u));
    out[p] = v;
}

size_t compact_scratch_words(size_t n) {
    const size_t words = (n + 31) / 32;
    const size_t nb = (words + kScanBlock - 1) / kScanBlock;
    return 2 * words + nb + 32;
}

// scratch: [bits words][prefix words][block sums nb][total]
cudaError_t launch_compact(const uint32_t* raw, size_t n, uint32_t* out, uint32_t* scratch, cudaStream_t s) {
    const size_t words = (n + 31) / 32;
    const size_t nb = (words + kScanBlock - 1) / kScanBlock;
    uint32_t* bits = scratch;
    uint32_t* pre = scratch + words;
    uint32_t* sums = pre + words;
    uint32_t* total = sums + nb;
    k_root_bits<<<unsigned((words * 32 + 255) / 256), 256, 0, s>>>(raw, n, bits, pre);
    k_scan_block<<<unsigned(nb), 256, 0, s>>>(pre, words, sums);
    k_scan_sums<<<1, 1024, 0, s>>>(sums, uint32_t(nb), total);
    k_scan_add<<<unsigned((words + 255) / 256), 256, 0, s>>>(pre, words, sums);
    k_compact_apply<<<unsigned((n + 255) / 256), 256, 0, s>>>(raw, n, bits, pre, out);
    return cudaGetLastError();
}

}  // namespace cclk
