/*
 * ccl_cuda.h — C-ABI of the B200-native connected-components labeler.
 *
 * This is the drop-in boundary under the reference's C++ entry point
 * `ccl::label_image` (/root/reference/proj/include/ccl/pipeline.hpp:33-34,
 * implemented at /root/reference/proj/src/pipeline.cpp:11-52).  The host C++
 * in include/ccl/pipeline.hpp keeps that signature verbatim and calls down
 * through these functions; any FFI (ctypes, cgo, JNI, N-API) can bind them
 * directly: plain pointers and sizes, no C++ or torch types, no exceptions.
 *
 * Output convention (identical to the reference, image.hpp:11-15,41-43):
 *   labels[x + y*W] = minimum raster index of the pixel's 4-connected
 *   foreground component, foreground iff image byte == 1, background
 *   CCL_BACKGROUND (0xFFFFFFFF).  Bit-exact with ccl::sequential_ccl and
 *   ccl::label_image of the reference for every block config and variant.
 *
 * Every function returns a ccl_status; on failure ccl_last_error() returns a
 * thread-local message.  All functions are thread-safe; a ccl_ctx must not be
 * used by two host threads at the same time (create one per thread).
 */
#ifndef CCL_CUDA_H
#define CCL_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CCL_BACKGROUND 0xFFFFFFFFu

typedef enum {
    CCL_OK = 0,
    CCL_EINVAL = 1,  /* bad argument: size 0 / > 2^32-2 px, bad variant, null ptr (pipeline.cpp:13-15) */
    CCL_ENOMEM = 2,  /* device or pinned-host allocation failed */
    CCL_ECUDA = 3,   /* CUDA runtime / launch error (message has the CUDA error string) */
    CCL_ENODEV = 4   /* no usable sm_100 device */
} ccl_status;

/* Variant (image.hpp:68-73).  All four produce identical labels; they select
 * the kernel's local-labeling strategy (template instantiation). */
typedef enum { CCL_C2FL = 0, CCL_RC2FL = 1, CCL_CC2FL = 2, CCL_NC2FL = 3 } ccl_variant;

typedef struct ccl_ctx ccl_ctx;  /* device, stream, pinned + device workspace cache */

/* Per-kernel device times (ms) of the last call on a context, from CUDA events. */
typedef struct {
    float local_ms;  /* kernel (a)(b)(c): tile-local labeling + seam export        */
    float merge_ms;  /* kernel (d): boundary-only global union-find                 */
    float final_ms;  /* kernel (e): recompute + path-compressed global relabel      */
    float total_ms;  /* first launch start to last launch end (== RunReport.wall_time) */
} ccl_timing;

ccl_status ccl_ctx_create(int device, ccl_ctx** out);
void ccl_ctx_destroy(ccl_ctx* ctx);
/* The context's stream (cudaStream_t) as an opaque pointer. */
void* ccl_ctx_stream(ccl_ctx* ctx);

/* Device-resident path (the timed roofline path).  d_img: H rows of
 * `img_pitch` bytes (pitch >= w).  d_labels: W*H u32, row-major, stride W.
 * The context owns the kernel (a)->(e) work buffer (grown on first use), so
 * calls sharing a context must be ordered on one stream.
 * Enqueued on `stream` exactly as given (NULL = the legacy default stream;
 * pass ccl_ctx_stream(ctx) for the context's own stream); asynchronous.
 * `timing` (may be NULL) is filled after the call only if `sync` != 0. */
ccl_status ccl_label_device(ccl_ctx* ctx, const uint8_t* d_img, size_t img_pitch, uint32_t w, uint32_t h,
                            uint32_t* d_labels, int variant, void* stream, int sync, ccl_timing* timing);

/* Host path used by ccl::label_image: H2D, the kernels, D2H.  Blocking.
 * Page-locked img / labels are copied directly; pageable ones (std::vector,
 * numpy) are staged through the context's page-locked double buffer in 16 MiB
 * chunks, the host-side copy of one chunk (split over a small thread pool)
 * overlapping the DMA of the other, in both directions.
 * `kernel_ms` (may be NULL) = device time of the kernels only. */
ccl_status ccl_label_host(ccl_ctx* ctx, const uint8_t* img, uint32_t w, uint32_t h, uint32_t* labels,
                          int variant, float* kernel_ms);
/* The same, asynchronous: H2D, kernels and D2H are enqueued on ctx's stream
 * and the call returns at once; img / labels must stay valid (and should be
 * page-locked for the copies to overlap) until ccl_ctx_sync(ctx).  A caller
 * alternating two contexts overlaps an image's upload with the previous
 * image's label download. */
ccl_status ccl_label_host_async(ccl_ctx* ctx, const uint8_t* img, uint32_t w, uint32_t h, uint32_t* labels,
                                int variant);
ccl_status ccl_ctx_sync(ccl_ctx* ctx);

/* Batch of n frames of w*h, frame f at d_frames + f*frame_pitch (rows of
 * img_pitch bytes).  Labels are per-frame raster indices at d_labels + f*w*h.
 * One launch per kernel for the whole batch.  Asynchronous on `stream`. */
ccl_status ccl_label_batch(ccl_ctx* ctx, const uint8_t* d_frames, size_t img_pitch, size_t frame_pitch,
                           uint32_t n, uint32_t w, uint32_t h, uint32_t* d_labels, int variant, void* stream);

/* One image over several devices in one process (the additive C++ entry point
 * ccl::label_image_strips): devices[k] labels strip k (near-equal row bands,
 * all but the last a multiple of the tile height) with the strip protocol
 * below; each strip's seam export is stored straight into every strip's
 * exchange area (NVLink peer stores between distinct devices) and the strips'
 * streams are ordered by cross-device events -- one host thread, no joins.
 * A device may be listed more than once (virtual strips).  Contexts and
 * buffers are cached for the next call with the same devices and shape.
 * Host buffers; labels are global raster indices, bit-exact with
 * ccl_label_host.  *kernel_ms = max over strips of the device time from the
 * first kernel to the last (exchange included). */
ccl_status ccl_label_strips(const int* devices, int ndev, const uint8_t* img, uint32_t w, uint32_t h,
                            uint32_t* labels, int variant, float* kernel_ms);
/* Frees the contexts and buffers ccl_label_strips keeps for repeated shapes
 * (call before exit for a leak-free teardown; later calls re-create them). */
void ccl_release_caches(void);

/* ---- Strip groups: one image over N GPUs, one process (rank) per GPU ----
 * The seam exchange is inside the library and needs no host round trip per
 * step: every rank owns an exchange area in its HBM, shared through a CUDA IPC
 * handle; a rank's step stores its 16*W-byte seam export into every rank's
 * area over NVLink and raises its epoch flag there (release, system scope);
 * each rank's seam resolve waits on its LOCAL flags (acquire, system scope),
 * then runs the same union-find over all N exports (no broadcast).  Setup:
 *   1. ccl_strip_group_create on every rank -> CCL_IPC_HANDLE_BYTES of handle
 *   2. all-gather the handles (any host channel, e.g. torch.distributed), rank order
 *   3. ccl_strip_group_connect(group, all_handles)
 * Then every step: ccl_strip_group_label on each rank with its strip
 * (ccl_strip_group_rows: rows [row0, row0+h) of the full image; d_labels holds
 * global raster indices for those rows).  Steps must be issued in the same
 * order on all ranks.  A rank whose peers never arrive traps after 20 s. */
typedef struct ccl_strip_group ccl_strip_group;
#define CCL_IPC_HANDLE_BYTES 64
size_t ccl_strip_group_handle_bytes(void);
ccl_status ccl_strip_group_create(ccl_ctx* ctx, uint32_t rank, uint32_t n_ranks, uint32_t w, uint32_t full_h,
                                  ccl_strip_group** out, void* handle_out);
ccl_status ccl_strip_group_connect(ccl_strip_group* group, const void* all_handles);
ccl_status ccl_strip_group_rows(const ccl_strip_group* group, uint32_t* row0, uint32_t* h);
ccl_status ccl_strip_group_label(ccl_strip_group* group, const uint8_t* d_img, size_t img_pitch, uint32_t* d_labels,
                                 int variant, void* stream);
/* kernel launches (and copies) one ccl_strip_group_label enqueues */
int ccl_strip_group_launches(const ccl_strip_group* group);
void ccl_strip_group_destroy(ccl_strip_group* group);

/* ---- Strip mode (image split into horizontal strips, one per GPU/rank) ----
 * A strip holds rows [row0, row0+h) of a full image of `full_h` rows, width w;
 * every strip but the last must have h a multiple of the tile height
 * (ccl_tile_shape).  Labels are GLOBAL raster indices x + (row0+y)*w; the
 * strip's label buffer holds indices [row0*w, (row0+h)*w).  Protocol:
 *   1. ccl_strip_local        kernels (a)(b)(c)(d) on the strip
 *   2. ccl_strip_seam_export  4*w u32 to d_seam_out: the strip-local roots of
 *                             its top and bottom rows (2*w, background =
 *                             CCL_BACKGROUND) and, per seam node, the global
 *                             node index of the first seam node of the same
 *                             strip root (2*w)
 *   3. all-gather the n_strips*4*w words (NCCL / peer copies) in strip order
 *   4. ccl_strip_seam_resolve union-find over all strips' seam nodes, run
 *                             identically on every strip (no broadcast), then
 *                             each own seam root's final label is written into
 *                             the strip's compact forest (in d_work)
 *   5. ccl_strip_final        kernel (e) on the strip (same variant as step 1)
 * Steps 2-4 must all run before step 5; d_work (the strip's work buffer from
 * step 1) carries the forest between the steps, and the label buffer is
 * scratch until step 5 writes it. */
ccl_status ccl_strip_local(ccl_ctx* ctx, const uint8_t* d_img, size_t img_pitch, uint32_t w, uint32_t h,
                           uint32_t row0, uint32_t full_h, uint32_t* d_labels, void* d_work, int variant,
                           void* stream);
ccl_status ccl_strip_seam_export(ccl_ctx* ctx, uint32_t w, uint32_t h, uint32_t row0, uint32_t full_h,
                                 uint32_t strip_index, uint32_t* d_labels, void* d_work, uint32_t* d_seam_out,
                                 void* stream);
ccl_status ccl_strip_seam_resolve(ccl_ctx* ctx, const uint32_t* d_seam_all, uint32_t n_strips,
                                  uint32_t strip_index, uint32_t w, uint32_t h, uint32_t row0, uint32_t full_h,
                                  uint32_t* d_labels, void* d_work, uint32_t* d_scratch, void* stream);
ccl_status ccl_strip_final(ccl_ctx* ctx, uint32_t w, uint32_t h, uint32_t row0, uint32_t full_h,
                           uint32_t* d_labels, const void* d_work, int variant, void* stream);
/* d_scratch for ccl_strip_seam_resolve must hold ccl_strip_scratch_words(n_strips, w) u32;
 * d_work (kernel (a) -> kernel (e) hand-off: per-tile masks, run table and
 * seam-root list) must hold ccl_work_bytes(w, h, 1) bytes and stay untouched
 * between ccl_strip_local and ccl_strip_final of the same strip.  Zero-fill it
 * once after allocating it (it carries kernel (a)'s per-seam flags, which
 * are tagged with a per-launch id, so it can be reused without clearing). */
size_t ccl_strip_scratch_words(uint32_t n_strips, uint32_t w);
size_t ccl_work_bytes(uint32_t w, uint32_t h, uint32_t nframes);

/* GPU compaction (pipeline.cpp:54-70, "next" row (f)1): labels 1..K in raster
 * order of first appearance, background 0; K written to *k_out (host).
 * d_scratch must hold ccl_compact_scratch_words(w, h) u32. Blocking. */
ccl_status ccl_compact_device(ccl_ctx* ctx, const uint32_t* d_raw, uint32_t w, uint32_t h, uint32_t* d_out,
                              uint32_t* d_scratch, uint64_t* k_out, void* stream);
size_t ccl_compact_scratch_words(uint32_t w, uint32_t h);

/* random_image generated on the device: rows
 * [row0, row0+h) of random_image(w, *, density, seed) as w*h bytes at d_out
 * (pitch w, 16-byte aligned), byte-identical with ccl_gen_random / the
 * reference generate.cpp:9-18 (xoshiro256** jump-ahead per chunk; row0 > 0
 * gives one strip of a taller image).  Returns once the image is written. */
ccl_status ccl_gen_random_device(ccl_ctx* ctx, uint8_t* d_out, uint32_t w, uint32_t h, uint32_t row0, double density,
                                 uint64_t seed, void* stream);

/* ---- Label-map files (reference proj/src/label_io.cpp:27-94) ----
 * ccl_label_to_cclm: label `img` (host, w*h bytes) on the device, compact on
 * the device and write a CCLM file ("CCLM", version 1, W, H as u32 LE, then
 * W*H compacted u32 LE labels); device->host copies overlap the file writes.
 * *k_out (may be NULL) = number of components.  Blocking. */
ccl_status ccl_label_to_cclm(ccl_ctx* ctx, const uint8_t* img, uint32_t w, uint32_t h, int variant, const char* path,
                             uint64_t* k_out);
/* Host-only (no device needed): the reference's write_label_map (compacts
 * first; format 0 raw CCLM, 1 csv, 2 pgm16) and read_label_map (CCLM).  On
 * error they return CCL_EINVAL and ccl_io_last_error() says why. */
ccl_status ccl_write_label_map(const uint32_t* labels, uint32_t w, uint32_t h, int compacted, int format,
                               const char* path);
ccl_status ccl_read_label_map(const char* path, uint32_t* labels, size_t capacity, uint32_t* w, uint32_t* h);
const char* ccl_io_last_error(void);

/* Tile geometry used by the kernels (for docs / tests). */
void ccl_tile_shape(uint32_t* tile_w, uint32_t* tile_h);
/* Number of kernel launches one ccl_label_device call makes. */
int ccl_launches_per_label(void);

/* Instrumented metrics mode (reference BlockMetrics and
 * RunReport, forest.hpp:12-29, pipeline.hpp:15-26, pipeline.cpp:72-91): a
 * separate build of this library with -DCCL_METRICS=1
 * (libccl_b200_metrics1.so) counts, per 128x64 tile of kernel (a), the
 * parent-link steps taken while finding roots and the CAS attempts of unions,
 * plus the border-merge (kernel (d)) and resolve (kernel (d2)) totals.
 * ccl_metrics_build() is 1 in that build; ccl_read_metrics() copies the
 * counters of the last labeling call on ctx (single image or batch; strips are
 * not instrumented): tile_find / tile_cas get tiles_x*tiles_y*n_frames u32 in
 * row-major tile order (either may be null), phase4 = {border find steps,
 * border CAS attempts, resolve find steps, 0}.  CCL_EINVAL in the product build. */
int ccl_metrics_build(void);
ccl_status ccl_read_metrics(ccl_ctx* ctx, uint32_t* tile_find, uint32_t* tile_cas, size_t n_tiles, uint64_t* phase4,
                            uint32_t* tiles_x, uint32_t* tiles_y, uint32_t* n_frames);

/* Host-side synthetic inputs, byte-identical to the reference generators
 * (generate.cpp:9-106).  kind: 0 stripes, 1 spiral, 2 blobs, 3 checkerboard. */
ccl_status ccl_gen_random(uint8_t* out, uint32_t w, uint32_t h, double density, uint64_t seed);
ccl_status ccl_gen_pattern(uint8_t* out, int kind, uint32_t w, uint32_t h, uint32_t period, double density,
                           uint64_t seed);

const char* ccl_last_error(void);
const char* ccl_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CCL_CUDA_H */
