// ccl_internal.h — shared between the kernel TUs and the C-ABI TU (not installed).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

// GPU tile = CCL_TILE_WX x CCL_TILE_WY warps, each warp a 32x32 pixel sub-tile.
#ifndef CCL_JUMP
#define CCL_JUMP 1  // pointer-jumping rounds over the coarse forest in kernel (a)
#endif
#ifndef CCL_ULCAP
#define CCL_ULCAP 128  // union-list entries per warp in kernel (a)
#endif
#ifndef CCL_HINTS
#define CCL_HINTS 1  // L2 evict-first / evict-last policies on streams vs hand-off data
#endif
#ifndef CCL_PDL
#define CCL_PDL 1  // programmatic dependent launch of kernels (d), (d2), (e)
#endif
#ifndef CCL_SEAM_MATCH
#define CCL_SEAM_MATCH 2  // kernel (d) dedup of a chunk's pairs: 1 = __match_any (distinct pairs), 2 = previous active pair
#endif
#ifndef CCL_CARVEOUT
#define CCL_CARVEOUT 100  // preferred shared-memory carveout (%) of kernels (a) and (e)
#endif
#ifndef CCL_EMINB
#define CCL_EMINB 2
#endif
#ifndef CCL_BULCAP
#define CCL_BULCAP 160  // band kernel (a): union pairs per warp (dense tiles overflow 96: d=0.7 -20 us)
#endif
#ifndef CCL_ETBL
#define CCL_ETBL 3072  // band kernel (e): node-table stage capacity (sized for 4 CTAs/SM)
#endif
#ifndef CCL_SEAM_K
#define CCL_SEAM_K 4  // kernel (d): 32-pair seam chunks per warp (unions compacted over the warp)
#endif
#ifndef CCL_BJUMP
#define CCL_BJUMP 1  // band kernel (a): pointer-jumping rounds before the unions
#endif
#ifndef CCL_METRICS
#define CCL_METRICS 0  // instrumented build: per-tile find / CAS counters (separate library)
#endif
#ifndef CCL_AIMG_OVERLAY
#define CCL_AIMG_OVERLAY 1  // band kernel (a): TMA tile staged in the node table (no prefetch, -8 KB smem)
#endif
#ifndef CCL_BAND
#define CCL_BAND 1  // C2FL kernel (a) on 2-row band runs
#endif
#ifndef CCL_BWPL
#define CCL_BWPL 1  // 32-px row words per lane in the band kernel (a)
#endif
#ifndef CCL_BMINB
#define CCL_BMINB 12  // min resident CTAs of the band kernel (a)
#endif
#ifndef CCL_BINFAST
#define CCL_BINFAST 1  // kernel (a): multiply-gather masks when every byte of a warp's chunks is 0 or 1
#endif
#ifndef CCL_SEAM_NOUNION
#define CCL_SEAM_NOUNION 0  // timing probe: kernel (d) skips its unions (wrong labels)
#endif
#ifndef CCL_PHASES
#define CCL_PHASES 0
#endif
#ifndef CCL_MINB
#define CCL_MINB 10  // min resident CTAs of kernel (a) (register cap)
#endif
#ifndef CCL_WPL
#define CCL_WPL 2  // 32-px row words per lane in kernels (a) and (e)
#endif
#ifndef CCL_TILE_WX
#define CCL_TILE_WX 2
#endif
#ifndef CCL_TILE_WY
#define CCL_TILE_WY 2
#endif

namespace cclk {

// Geometry of one labeling problem (a frame, a batch of frames or one strip).
struct Geo {
    uint32_t W, H;          // width, rows held by this buffer (strip height in strip mode)
    uint32_t ntx, nty;      // tile grid
    uint32_t row0;          // global row of the buffer's first row (strip mode), else 0
    uint32_t base;          // row0 * W: global raster index of L[0]
    uint32_t edge_above;    // strip has a neighbour strip above / below
    uint32_t edge_below;
    size_t img_pitch;       // bytes between image rows
    size_t frame_pitch;     // bytes between frames (batch)
    size_t frame_px;        // labels per frame (W*H)
    uint32_t epoch;         // per-launch id (never 0): fused seam flags of kernel (a)
    // instrumented builds (CCL_METRICS=1) only, else null: u64[4] phase totals
    // {border find steps, border CAS attempts, resolve find steps, 0}, then
    // u32[2] {find steps, CAS attempts} per tile of kernel (a)
    uint32_t* metrics;
};

struct LaunchArgs {
    Geo g;
    uint32_t nframes;
    int variant;
    bool tma_load, tma_store;
    CUtensorMap tm_img;     // u8 {W, H, F}, box {TW, TH, 1}
    CUtensorMap tm_lab;     // u32 {W, H, F}, box {32, 32, 1}, 128B swizzle
    const uint8_t* img;
    uint32_t* labels;
    uint32_t* work;         // per-tile masks / run table / seam-root list (work_bytes)
    cudaStream_t stream;
    // pipelined batches (ccl_label_batch): persistent grids capped at this many
    // CTAs per SM (0 = full occupancy) so kernel (a) of one chunk and kernel (e)
    // of the previous one share the SMs; the first launch of a group follows a
    // cross-stream event, so it must not be a programmatic dependent launch
    int a_cap_per_sm, e_cap_per_sm;
    bool no_pdl_first;
};

cudaError_t launch_local(const LaunchArgs& a);
// timing ablations only (env CCL_DEBUG_SKIP, bits: 1 (a), 2 (d), 4 (d2), 8 (e)); labels are wrong when set
int debug_skip();
cudaError_t launch_seams(const LaunchArgs& a);
cudaError_t launch_final(const LaunchArgs& a);

// strip-mode and compaction kernels (ccl_aux.cu)
cudaError_t launch_strip_export(const Geo& g, uint32_t* labels, uint32_t* work, uint32_t* seam_out,
                                uint32_t strip_index, cudaStream_t s);
cudaError_t launch_strip_resolve(const Geo& g, const uint32_t* seam_all, uint32_t n_strips, uint32_t strip_index,
                                 uint32_t* labels, uint32_t* work, uint32_t* scratch, cudaStream_t s);
cudaError_t launch_compact(const uint32_t* raw, size_t n, uint32_t* out, uint32_t* scratch, cudaStream_t s);
size_t compact_scratch_words(size_t n);
cudaError_t launch_gen_random(uint8_t* out, uint64_t n, uint64_t first, double density, uint64_t seed,
                              cudaStream_t s);

size_t work_bytes(uint32_t w, uint32_t h, uint32_t nframes);
uint32_t* strip_area_ptr(uint32_t* work, const Geo& g);  // strip mode: [edge nodes 2W | edge roots 2W]
uint32_t* forest_ptr(uint32_t* work, const Geo& g);      // compact global forest
int tile_maxf();
// records the thread-local message ccl_last_error() returns (ccl_capi.cu); returns status
int set_error(int status, const char* msg);
int tile_w();
int tile_h();

}  // namespace cclk
