// ccl_capi.cu — the extern "C" boundary (include/ccl_cuda.h): contexts,
// argument validation with the reference's error semantics
// (pipeline.cpp:13-15, image.hpp:31-38), TMA descriptor setup, staging and
// timing.  No exception crosses this boundary; every CUDA failure becomes a
// status code plus a thread-local message.
#include <atomic>
#include <cstdlib>
#include <algorithm>
#include <thread>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <condition_variable>
#include <mutex>
#include <string>

#include "ccl/generate.hpp"
#include "ccl_cuda.h"
#include "ccl_internal.h"

namespace {

thread_local std::string g_err;

ccl_status fail(ccl_status s, const std::string& msg) {
    g_err = msg;
    return s;
}
ccl_status cuda_fail(cudaError_t e, const char* where) {
    return fail(e == cudaErrorMemoryAllocation ? CCL_ENOMEM : CCL_ECUDA,
                std::string(where) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
}
#define CCL_CHECK(call)                                   \
    do {                                                  \
        cudaError_t e__ = (call);                         \
        if (e__ != cudaSuccess) return cuda_fail(e__, #call); \
    } while (0)

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
    static std::once_flag once;
    static EncodeFn fn = nullptr;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    return fn;
}

}  // namespace

struct ccl_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    // host-path workspace (grown on demand)
    uint8_t* d_img = nullptr;
    size_t d_img_bytes = 0;
    uint32_t* d_lab = nullptr;
    size_t d_lab_bytes = 0;
    uint8_t* h_img = nullptr;  // pinned
    size_t h_img_bytes = 0;
    uint32_t* h_lab = nullptr;  // pinned
    size_t h_lab_bytes = 0;
    void* d_work = nullptr;     // kernel (a) -> (e) hand-off buffer
    uint32_t* d_aux = nullptr;  // compacted labels + compaction scratch (CCLM path)
    size_t d_aux_bytes = 0;
    uint8_t* h_ring = nullptr;  // pinned double buffer for chunked device->file copies
    cudaEvent_t ring_ev[2] = {nullptr, nullptr};
    size_t d_work_bytes = 0;
    // CUDA graphs of the device path, keyed by the call's buffers and shape
    struct Graph {
        const void* img;
        size_t pitch;
        uint32_t w, h;
        const void* lab;
        int variant;
        const void* work;
        cudaGraphExec_t exec;
    };
    std::vector<Graph> graphs;
    uint32_t* d_metrics = nullptr;  // instrumented builds: counters of the last call (Geo::metrics)
    size_t d_metrics_bytes = 0;
    uint32_t m_tx = 0, m_ty = 0, m_frames = 0;
    ccl_timing last{};
    bool last_split = false;
    // pipelined batches: second stream for kernels (d2)+(e) of chunk j while
    // kernels (a)+(d) of chunk j+1 run on the call's stream
    cudaStream_t stream2 = nullptr;
    cudaEvent_t pev[2] = {nullptr, nullptr};
};

namespace {

// Launch ids for kernel (a)'s fused seam flags: unique in the process (work
// buffers may be shared between contexts), never 0 (a zero-filled buffer).
uint32_t next_epoch() {
    static std::atomic<uint32_t> counter{0};
    uint32_t e;
    do {
        e = ++counter;
    } while (e == 0);
    return e;
}

ccl_status check_dims(uint32_t w, uint32_t h) {
    if (w == 0 || h == 0) return fail(CCL_EINVAL, "image dimensions must be at least 1x1");
    if (uint64_t(w) * h > uint64_t(CCL_BACKGROUND) - 1) return fail(CCL_EINVAL, "image exceeds 2^32-2 pixels");
    return CCL_OK;
}

ccl_status make_geo(uint32_t w, uint32_t h, uint32_t row0, size_t img_pitch, size_t frame_pitch, bool above,
                    bool below, cclk::Geo* g) {
    const uint32_t tw = uint32_t(cclk::tile_w()), th = uint32_t(cclk::tile_h());
    g->W = w;
    g->H = h;
    g->ntx = (w + tw - 1) / tw;
    g->nty = (h + th - 1) / th;
    g->row0 = row0;
    g->base = row0 * w;
    g->edge_above = above ? 1u : 0u;
    g->edge_below = below ? 1u : 0u;
    g->img_pitch = img_pitch;
    g->frame_pitch = frame_pitch;
    g->frame_px = size_t(w) * h;
    if (below && (h % th) != 0) return fail(CCL_EINVAL, "strip height must be a multiple of the tile height");
    return CCL_OK;
}

ccl_status prepare(cclk::LaunchArgs* a, const uint8_t* img, size_t pitch, size_t frame_pitch, uint32_t nframes,
                   uint32_t* labels, int variant, cudaStream_t s) {
    if (variant < 0 || variant > 3) return fail(CCL_EINVAL, "unknown variant");
    a->nframes = nframes;
    a->variant = variant;
    a->img = img;
    a->labels = labels;
    a->stream = s;
    std::memset(&a->tm_img, 0, sizeof(a->tm_img));
    std::memset(&a->tm_lab, 0, sizeof(a->tm_lab));
    const cclk::Geo& g = a->g;
    // CCL_NO_TMA=1 (diagnostics only, e.g. compute-sanitizer initcheck, which
    // does not see bulk-tensor stores as initialising writes): generic loads /
    // stores instead of the TMA tile paths.  Same labels, slower.
    static const bool no_tma = [] {
        const char* v = std::getenv("CCL_NO_TMA");
        return v && v[0] == '1';
    }();
    EncodeFn enc = no_tma ? nullptr : encode_fn();
    a->tma_load = enc && (reinterpret_cast<uintptr_t>(img) % 16 == 0) && (pitch % 16 == 0) &&
                  (frame_pitch % 16 == 0) && pitch < (uint64_t(1) << 40);
    a->tma_store = enc && (reinterpret_cast<uintptr_t>(labels) % 16 == 0) && (uint64_t(g.W) * 4 % 16 == 0);
    if (a->tma_load) {
        const cuuint64_t dims[3] = {g.W, g.H, nframes};
        const cuuint64_t strides[2] = {pitch, frame_pitch};
        const cuuint32_t box[3] = {uint32_t(cclk::tile_w()), uint32_t(cclk::tile_h()), 1};
        const cuuint32_t es[3] = {1, 1, 1};
        CUresult r = enc(&a->tm_img, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(img), dims, strides, box,
                         es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) a->tma_load = false;
    }
    if (a->tma_store) {
        const cuuint64_t dims[3] = {g.W, g.H, nframes};
        const cuuint64_t strides[2] = {cuuint64_t(g.W) * 4, cuuint64_t(g.frame_px) * 4};
        const cuuint32_t box[3] = {32, 32, 1};
        const cuuint32_t es[3] = {1, 1, 1};
        CUresult r = enc(&a->tm_lab, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, labels, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) a->tma_store = false;
    }
    return CCL_OK;
}

// CUDA graphs for repeated device-path calls (off with CCL_GRAPHS=0; never in
// instrumented builds: per-call memsets).
bool graphs_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("CCL_GRAPHS");
        return !(v && v[0] == '0') && !CCL_METRICS;
    }();
    return on;
}

// One replay, bracketed by the context's events (the total time of the call,
// as run_pipeline records it for direct launches).
ccl_status launch_graph(ccl_ctx* ctx, cudaGraphExec_t exec, cudaStream_t st) {
    ctx->last_split = false;
    CCL_CHECK(cudaEventRecord(ctx->ev[0], st));
    CCL_CHECK(cudaGraphLaunch(exec, st));
    CCL_CHECK(cudaEventRecord(ctx->ev[3], st));
    return CCL_OK;
}

// `split`: also time each kernel group (events between the launches break the
// programmatic-dependent-launch chaining, so only timed calls pay for them).
ccl_status run_pipeline(ccl_ctx* ctx, cclk::LaunchArgs& a, bool events, bool split = false) {
    ctx->last_split = events && split;
#if CCL_METRICS
    {   // instrumented build: zeroed counters for this call
        const size_t bytes = 32 + size_t(a.g.ntx) * a.g.nty * a.nframes * 8;
        if (ctx->d_metrics_bytes < bytes) {
            if (ctx->d_metrics) cudaFree(ctx->d_metrics);
            ctx->d_metrics = nullptr;
            ctx->d_metrics_bytes = 0;
            CCL_CHECK(cudaMalloc(&ctx->d_metrics, bytes));
            ctx->d_metrics_bytes = bytes;
        }
        CCL_CHECK(cudaMemsetAsync(ctx->d_metrics, 0, bytes, a.stream));
        a.g.metrics = ctx->d_metrics;
        ctx->m_tx = a.g.ntx;
        ctx->m_ty = a.g.nty;
        ctx->m_frames = a.nframes;
    }
#endif
    if (events) CCL_CHECK(cudaEventRecord(ctx->ev[0], a.stream));
    a.g.epoch = next_epoch();
    const int skip = cclk::debug_skip();
    if (!(skip & 1)) CCL_CHECK(cclk::launch_local(a));
    if (ctx->last_split) CCL_CHECK(cudaEventRecord(ctx->ev[1], a.stream));
    if (!(skip & 2)) CCL_CHECK(cclk::launch_seams(a));
    if (ctx->last_split) CCL_CHECK(cudaEventRecord(ctx->ev[2], a.stream));
    CCL_CHECK(cclk::launch_final(a));
    if (events) CCL_CHECK(cudaEventRecord(ctx->ev[3], a.stream));
    return CCL_OK;
}

ccl_status read_timing(ccl_ctx* ctx, ccl_timing* t) {
    CCL_CHECK(cudaEventSynchronize(ctx->ev[3]));
    ccl_timing r{};
    if (ctx->last_split) {
        CCL_CHECK(cudaEventElapsedTime(&r.local_ms, ctx->ev[0], ctx->ev[1]));
        CCL_CHECK(cudaEventElapsedTime(&r.merge_ms, ctx->ev[1], ctx->ev[2]));
        CCL_CHECK(cudaEventElapsedTime(&r.final_ms, ctx->ev[2], ctx->ev[3]));
    }
    CCL_CHECK(cudaEventElapsedTime(&r.total_ms, ctx->ev[0], ctx->ev[3]));
    ctx->last = r;
    if (t) *t = r;
    return CCL_OK;
}

// Grows the context's work buffer; the zero fill is ordered on the stream of
// the call that uses the buffer next.
ccl_status ensure_work(ccl_ctx* ctx, size_t bytes, cudaStream_t st) {
    if (ctx->d_work_bytes >= bytes) return CCL_OK;
    for (auto& gr : ctx->graphs) cudaGraphExecDestroy(gr.exec);  // they point at the old buffer
    ctx->graphs.clear();
    if (ctx->d_work) cudaFree(ctx->d_work);
    ctx->d_work = nullptr;
    ctx->d_work_bytes = 0;
    CCL_CHECK(cudaMalloc(&ctx->d_work, bytes));
    CCL_CHECK(cudaMemsetAsync(ctx->d_work, 0, bytes, st));  // seam flags start clear
    ctx->d_work_bytes = bytes;
    return CCL_OK;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

}  // namespace

extern "C" {

ccl_status ccl_ctx_create(int device, ccl_ctx** out) {
    if (!out) return fail(CCL_EINVAL, "null out pointer");
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0) return fail(CCL_ENODEV, "no CUDA device visible");
    if (device < 0 || device >= n) return fail(CCL_ENODEV, "device index out of range");
    cudaDeviceProp prop;
    CCL_CHECK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) return fail(CCL_ENODEV, std::string("built for sm_100a; device is ") + prop.name);
    DeviceGuard dg(device);
    ccl_ctx* c = new ccl_ctx();
    c->device = device;
    cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    for (int i = 0; e == cudaSuccess && i < 4; ++i) e = cudaEventCreate(&c->ev[i]);
    if (e != cudaSuccess) {
        ccl_ctx_destroy(c);
        return cuda_fail(e, "ccl_ctx_create");
    }
    *out = c;
    return CCL_OK;
}

void ccl_ctx_destroy(ccl_ctx* c) {
    if (!c) return;
    DeviceGuard dg(c->device);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    if (c->stream) cudaStreamDestroy(c->stream);
    if (c->stream2) cudaStreamDestroy(c->stream2);
    for (auto& e : c->pev)
        if (e) cudaEventDestroy(e);
    if (c->d_img) cudaFree(c->d_img);
    if (c->d_lab) cudaFree(c->d_lab);
    if (c->h_img) cudaFreeHost(c->h_img);
    if (c->h_lab) cudaFreeHost(c->h_lab);
    for (auto& gr : c->graphs) cudaGraphExecDestroy(gr.exec);
    if (c->d_work) cudaFree(c->d_work);
    if (c->d_metrics) cudaFree(c->d_metrics);
    if (c->d_aux) cudaFree(c->d_aux);
    if (c->h_ring) cudaFreeHost(c->h_ring);
    for (auto& e : c->ring_ev)
        if (e) cudaEventDestroy(e);
    delete c;
}

void* ccl_ctx_stream(ccl_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

ccl_status ccl_label_device(ccl_ctx* ctx, const uint8_t* d_img, size_t img_pitch, uint32_t w, uint32_t h,
                            uint32_t* d_labels, int variant, void* stream, int sync, ccl_timing* timing) {
    if (!ctx || !d_img || !d_labels) return fail(CCL_EINVAL, "null argument");
    if (ccl_status s = check_dims(w, h)) return s;
    if (img_pitch < w) return fail(CCL_EINVAL, "image pitch smaller than width");
    DeviceGuard dg(ctx->device);
    cclk::LaunchArgs a{};
    if (ccl_status s = make_geo(w, h, 0, img_pitch, img_pitch * h, false, false, &a.g)) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (variant < 0 || variant > 3) return fail(CCL_EINVAL, "unknown variant");
    if (ccl_status s = ensure_work(ctx, cclk::work_bytes(w, h, 1), static_cast<cudaStream_t>(stream))) return s;
    if (!sync && graphs_enabled()) {
        // repeated calls on the same buffers replay one CUDA graph of the
        // (PDL-chained) launches: no per-call host work between the kernels
        for (auto& gr : ctx->graphs)
            if (gr.img == d_img && gr.pitch == img_pitch && gr.w == w && gr.h == h && gr.lab == d_labels &&
                gr.variant == variant && gr.work == ctx->d_work)
                return launch_graph(ctx, gr.exec, st);
    }
    if (ccl_status s = prepare(&a, d_img, img_pitch, img_pitch * h, 1, d_labels, variant, st)) return s;
    a.work = static_cast<uint32_t*>(ctx->d_work);
    if (!sync && graphs_enabled()) {
        // capture on the context's own stream (the legacy default stream cannot be captured)
        cclk::LaunchArgs c = a;
        c.stream = ctx->stream;
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        if (cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeRelaxed) == cudaSuccess) {
            // no context events inside the graph: they would no longer be usable
            // by later timed calls (this path reads no timing)
            const ccl_status s = run_pipeline(ctx, c, false, false);
            const cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
            if (s == CCL_OK && e == cudaSuccess && graph && cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess) {
                cudaGraphDestroy(graph);
                if (ctx->graphs.size() >= 8) {
                    cudaGraphExecDestroy(ctx->graphs.front().exec);
                    ctx->graphs.erase(ctx->graphs.begin());
                }
                ctx->graphs.push_back({d_img, img_pitch, w, h, d_labels, variant, ctx->d_work, exec});
                return launch_graph(ctx, exec, st);
            }
            if (graph) cudaGraphDestroy(graph);
            cudaGetLastError();  // capture failed: launch directly below
        }
    }
    if (ccl_status s = run_pipeline(ctx, a, true, sync != 0)) return s;
    if (sync) return read_timing(ctx, timing);
    return CCL_OK;
}

namespace {
int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v && *v ? std::atoi(v) : dflt;
}
}  // namespace

ccl_status ccl_label_batch(ccl_ctx* ctx, const uint8_t* d_frames, size_t img_pitch, size_t frame_pitch, uint32_t n,
                           uint32_t w, uint32_t h, uint32_t* d_labels, int variant, void* stream) {
    if (!ctx || !d_frames || !d_labels) return fail(CCL_EINVAL, "null argument");
    if (n == 0) return CCL_OK;
    if (n > 65535) return fail(CCL_EINVAL, "at most 65535 frames per batch call");
    if (ccl_status s = check_dims(w, h)) return s;
    if (img_pitch < w || frame_pitch < img_pitch * h) return fail(CCL_EINVAL, "bad pitch");
    if (variant < 0 || variant > 3) return fail(CCL_EINVAL, "unknown variant");
    DeviceGuard dg(ctx->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // Frames are independent, so a big batch is labeled as a PIPELINE of
    // chunks over two streams: kernels (a)+(d) of chunk j+1 (issue-bound) run
    // while kernels (d2)+(e) of chunk j (HBM-bound: the label stores) drain,
    // with the persistent grids capped so both fit on every SM.  Each chunk
    // has its own work region, so the chunks share nothing.
    const uint32_t tiles_per_frame = ((w + cclk::tile_w() - 1) / cclk::tile_w()) * ((h + cclk::tile_h() - 1) / cclk::tile_h());
    const uint32_t min_chunk_tiles = uint32_t(env_int("CCL_PIPE_TILES", 24576));
    const uint32_t chunk = std::max(1u, (min_chunk_tiles + tiles_per_frame - 1) / tiles_per_frame);
    const bool pipe = env_int("CCL_PIPE", 1) != 0 && n >= 3 * chunk && !CCL_METRICS;
    if (!pipe) {
        cclk::LaunchArgs a{};
        if (ccl_status s = make_geo(w, h, 0, img_pitch, frame_pitch, false, false, &a.g)) return s;
        if (ccl_status s = prepare(&a, d_frames, img_pitch, frame_pitch, n, d_labels, variant, st)) return s;
        if (ccl_status s = ensure_work(ctx, cclk::work_bytes(w, h, n), st)) return s;
        a.work = static_cast<uint32_t*>(ctx->d_work);
        return run_pipeline(ctx, a, true);
    }
    const uint32_t nchunks = (n + chunk - 1) / chunk;
    const size_t wb = (cclk::work_bytes(w, h, chunk) + 255) / 256 * 256;  // per chunk
    if (ccl_status s = ensure_work(ctx, wb * nchunks, st)) return s;
    if (!ctx->stream2) {
        CCL_CHECK(cudaStreamCreateWithFlags(&ctx->stream2, cudaStreamNonBlocking));
        for (auto& e : ctx->pev) CCL_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    cudaStream_t s2 = ctx->stream2;
    ctx->last_split = false;
    CCL_CHECK(cudaEventRecord(ctx->ev[0], st));
    CCL_CHECK(cudaStreamWaitEvent(s2, ctx->ev[0], 0));  // inputs / previous work on the caller's stream
    const int acap = env_int("CCL_PIPE_A", 6), ecap = env_int("CCL_PIPE_E", 4);  // tuned: scripts/batch_sweep.py (r2n)
    for (uint32_t j = 0; j < nchunks; ++j) {
        const uint32_t f0 = j * chunk, nj = std::min(chunk, n - f0);
        cclk::LaunchArgs a{};
        if (ccl_status s = make_geo(w, h, 0, img_pitch, frame_pitch, false, false, &a.g)) return s;
        if (ccl_status s = prepare(&a, d_frames + size_t(f0) * frame_pitch, img_pitch, frame_pitch, nj,
                                   d_labels + size_t(f0) * w * h, variant, st))
            return s;
        a.work = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(ctx->d_work) + wb * j);
        a.a_cap_per_sm = acap;
        a.e_cap_per_sm = ecap;
        a.g.epoch = next_epoch();
        CCL_CHECK(cclk::launch_local(a));
        CCL_CHECK(cclk::launch_seams(a));
        CCL_CHECK(cudaEventRecord(ctx->pev[j & 1], st));
        CCL_CHECK(cudaStreamWaitEvent(s2, ctx->pev[j & 1], 0));
        a.stream = s2;
        a.no_pdl_first = true;
        CCL_CHECK(cclk::launch_final(a));
    }
    CCL_CHECK(cudaEventRecord(ctx->pev[0], s2));
    CCL_CHECK(cudaStreamWaitEvent(st, ctx->pev[0], 0));  // the caller's stream sees every label
    CCL_CHECK(cudaEventRecord(ctx->ev[3], st));
    return CCL_OK;
}

namespace {

bool page_locked(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

// Host memcpy split over a small persistent worker pool (the pageable side of
// the staged copies below: one thread copies ~10 GB/s, PCIe moves ~50 GB/s).
class CopyPool {
public:
    static CopyPool& get() {
        static CopyPool* pool = new CopyPool();  // never destroyed (workers are detached)
        return *pool;
    }
    void copy(void* dst, const void* src, size_t n) {
        const size_t parts = n < (size_t(1) << 20) ? 1 : workers_ + 1;
        if (parts == 1) {
            std::memcpy(dst, src, n);
            return;
        }
        const size_t step = (n / parts + 63) & ~size_t(63);
        std::unique_lock<std::mutex> lk(mu_);
        for (size_t k = 1; k < parts; ++k) {
            const size_t off = std::min(n, k * step), len = std::min(step, n - off);
            jobs_.push_back({static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, len});
        }
        pending_ += parts - 1;
        lk.unlock();
        cv_.notify_all();
        std::memcpy(dst, src, std::min(step, n));  // the caller's own share
        lk.lock();
        done_.wait(lk, [&] { return pending_ == 0; });
    }

private:
    struct Job {
        char* d;
        const char* s;
        size_t n;
    };
    CopyPool() {
        const unsigned hw = std::thread::hardware_concurrency();
        workers_ = std::max(1u, std::min(7u, hw > 2 ? hw / 2 : 1u));
        for (unsigned i = 0; i < workers_; ++i) std::thread([this] { run(); }).detach();
    }
    void run() {
        std::unique_lock<std::mutex> lk(mu_);
        for (;;) {
            cv_.wait(lk, [&] { return !jobs_.empty(); });
            const Job j = jobs_.back();
            jobs_.pop_back();
            lk.unlock();
            std::memcpy(j.d, j.s, j.n);
            lk.lock();
            if (--pending_ == 0) done_.notify_all();
        }
    }
    unsigned workers_ = 1;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    std::vector<Job> jobs_;
    size_t pending_ = 0;
};

}  // namespace

// Blocking host path of ccl::label_image.  Page-locked buffers go straight to
// the copy engines; PAGEABLE ones (std::vector, numpy) are staged through the
// context's page-locked double buffer in 16 MiB chunks, the host copy of one
// chunk overlapping the DMA of the other (both directions).
ccl_status ccl_label_host(ccl_ctx* ctx, const uint8_t* img, uint32_t w, uint32_t h, uint32_t* labels, int variant,
                          float* kernel_ms) {
    if (!ctx || !img || !labels) return fail(CCL_EINVAL, "null argument");
    if (ccl_status s = check_dims(w, h)) return s;
    if (variant < 0 || variant > 3) return fail(CCL_EINVAL, "unknown variant");
    DeviceGuard dg(ctx->device);
    if (page_locked(img) && page_locked(labels)) {
        if (ccl_status s = ccl_label_host_async(ctx, img, w, h, labels, variant)) return s;
    } else {
        const size_t pitch = (size_t(w) + 15) / 16 * 16;
        const size_t img_bytes = pitch * h, lab_bytes = size_t(w) * h * 4;
        if (ctx->d_img_bytes < img_bytes) {
            if (ctx->d_img) cudaFree(ctx->d_img);
            ctx->d_img = nullptr;
            ctx->d_img_bytes = 0;
            CCL_CHECK(cudaMalloc(&ctx->d_img, img_bytes));
            ctx->d_img_bytes = img_bytes;
        }
        if (ctx->d_lab_bytes < lab_bytes) {
            if (ctx->d_lab) cudaFree(ctx->d_lab);
            ctx->d_lab = nullptr;
            ctx->d_lab_bytes = 0;
            CCL_CHECK(cudaMalloc(&ctx->d_lab, lab_bytes));
            ctx->d_lab_bytes = lab_bytes;
        }
        constexpr size_t CH = size_t(16) << 20;
        if (!ctx->h_ring) {
            CCL_CHECK(cudaMallocHost(&ctx->h_ring, 2 * CH));
            for (auto& e : ctx->ring_ev) CCL_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        CopyPool& pool = CopyPool::get();
        cudaStream_t st = ctx->stream;
        // H2D: rows_per_chunk rows per slot
        const uint32_t rpc = uint32_t(std::max<size_t>(1, CH / w));
        bool slot_busy[2] = {false, false};
        for (uint32_t r0 = 0, i = 0; r0 < h; r0 += rpc, ++i) {
            const uint32_t rows = std::min(rpc, h - r0);
            const int k = int(i & 1u);
            if (slot_busy[k]) CCL_CHECK(cudaEventSynchronize(ctx->ring_ev[k]));  // its previous DMA has read it
            pool.copy(ctx->h_ring + k * CH, img + size_t(r0) * w, size_t(rows) * w);
            CCL_CHECK(cudaMemcpy2DAsync(ctx->d_img + size_t(r0) * pitch, pitch, ctx->h_ring + k * CH, w, w, rows,
                                        cudaMemcpyHostToDevice, st));
            CCL_CHECK(cudaEventRecord(ctx->ring_ev[k], st));
            slot_busy[k] = true;
        }
        if (ccl_status s = ccl_label_device(ctx, ctx->d_img, pitch, w, h, ctx->d_lab, variant, st, 0, nullptr))
            return s;
        // D2H: the DMA of chunk j+1 runs while chunk j is copied out
        const size_t nch = (lab_bytes + CH - 1) / CH;
        auto issue = [&](size_t j) -> cudaError_t {
            const size_t off = j * CH, n = std::min(CH, lab_bytes - off);
            cudaError_t e = cudaMemcpyAsync(ctx->h_ring + (j & 1) * CH, reinterpret_cast<uint8_t*>(ctx->d_lab) + off, n,
                                            cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaEventRecord(ctx->ring_ev[j & 1], st);
            return e;
        };
        CCL_CHECK(cudaEventSynchronize(ctx->ring_ev[0]));  // the H2D slots are free again
        CCL_CHECK(cudaEventSynchronize(ctx->ring_ev[1]));
        CCL_CHECK(issue(0));
        for (size_t j = 0; j < nch; ++j) {
            if (j + 1 < nch) CCL_CHECK(issue(j + 1));
            CCL_CHECK(cudaEventSynchronize(ctx->ring_ev[j & 1]));
            const size_t off = j * CH, n = std::min(CH, lab_bytes - off);
            pool.copy(reinterpret_cast<uint8_t*>(labels) + off, ctx->h_ring + (j & 1) * CH, n);
        }
    }
    CCL_CHECK(cudaStreamSynchronize(ctx->stream));
    ccl_timing t{};
    if (ccl_status s = read_timing(ctx, &t)) return s;
    if (kernel_ms) *kernel_ms = t.total_ms;
    return CCL_OK;
}

ccl_status ccl_ctx_sync(ccl_ctx* ctx) {
    if (!ctx) return fail(CCL_EINVAL, "null context");
    DeviceGuard dg(ctx->device);
    CCL_CHECK(cudaStreamSynchronize(ctx->stream));
    return CCL_OK;
}

// H2D, kernels and D2H enqueued on the context's stream; returns at once.
// With page-locked img / labels the copies are asynchronous, so a caller that
// alternates two contexts overlaps one image's upload with the previous
// image's label download (PCIe is full duplex).
ccl_status ccl_label_host_async(ccl_ctx* ctx, const uint8_t* img, uint32_t w, uint32_t h, uint32_t* labels,
                                int variant) {
    if (!ctx || !img || !labels) return fail(CCL_EINVAL, "null argument");
    if (ccl_status s = check_dims(w, h)) return s;
    if (variant < 0 || variant > 3) return fail(CCL_EINVAL, "unknown variant");
    DeviceGuard dg(ctx->device);
    const size_t pitch = (size_t(w) + 15) / 16 * 16;  // 16B-aligned rows for the TMA tile loads
    const size_t img_bytes = pitch * h, lab_bytes = size_t(w) * h * 4;
    if (ctx->d_img_bytes < img_bytes) {
        if (ctx->d_img) cudaFree(ctx->d_img);
        ctx->d_img = nullptr;
        ctx->d_img_bytes = 0;
        CCL_CHECK(cudaMalloc(&ctx->d_img, img_bytes));
        ctx->d_img_bytes = img_bytes;
    }
    if (ctx->d_lab_bytes < lab_bytes) {
        if (ctx->d_lab) cudaFree(ctx->d_lab);
        ctx->d_lab = nullptr;
        ctx->d_lab_bytes = 0;
        CCL_CHECK(cudaMalloc(&ctx->d_lab, lab_bytes));
        ctx->d_lab_bytes = lab_bytes;
    }
    CCL_CHECK(cudaMemcpy2DAsync(ctx->d_img, pitch, img, w, w, h, cudaMemcpyHostToDevice, ctx->stream));
    if (ccl_status s = ccl_label_device(ctx, ctx->d_img, pitch, w, h, ctx->d_lab, variant, ctx->stream, 0, nullptr))
        return s;
    CCL_CHECK(cudaMemcpyAsync(labels, ctx->d_lab, lab_bytes, cudaMemcpyDeviceToHost, ctx->stream));
    return CCL_OK;
}

// ---------------------------------------------------------------- strip mode
namespace {
ccl_status strip_geo(uint32_t w, uint32_t h, uint32_t row0, uint32_t full_h, size_t pitch, cclk::Geo* g) {
    if (ccl_status s = check_dims(w, full_h)) return s;
    if (h == 0 || uint64_t(row0) + h > full_h) return fail(CCL_EINVAL, "strip rows outside the image");
    // the top row of every strip is exported (also strip 0: keeps seam reps uniform)
    return make_geo(w, h, row0, pitch, pitch * h, true, row0 + h < full_h, g);
}
}  // namespace

ccl_status ccl_strip_local(ccl_ctx* ctx, const uint8_t* d_img, size_t img_pitch, uint32_t w, uint32_t h,
                           uint32_t row0, uint32_t full_h, uint32_t* d_labels, void* d_work, int variant,
                           void* stream) {
    if (!ctx || !d_img || !d_labels || !d_work) return fail(CCL_EINVAL, "null argument");
    if (img_pitch < w) return fail(CCL_EINVAL, "image pitch smaller than width");
    DeviceGuard dg(ctx->device);
    cclk::LaunchArgs a{};
    if (ccl_status s = strip_geo(w, h, row0, full_h, img_pitch, &a.g)) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (ccl_status s = prepare(&a, d_img, img_pitch, img_pitch * h, 1, d_labels, variant, st)) return s;
    a.work = static_cast<uint32_t*>(d_work);
    a.g.epoch = next_epoch();
    CCL_CHECK(cclk::launch_local(a));
    CCL_CHECK(cclk::launch_seams(a));
    return CCL_OK;
}

ccl_status ccl_strip_seam_export(ccl_ctx* ctx, uint32_t w, uint32_t h, uint32_t row0, uint32_t full_h,
                                 uint32_t strip_index, uint32_t* d_labels, void* d_work, uint32_t* d_seam_out,
                                 void* stream) {
    if (!ctx || !d_labels || !d_work || !d_seam_out) return fail(CCL_EINVAL, "null argument");
    DeviceGuard dg(ctx->device);
    cclk::Geo g{};
    if (ccl_status s = strip_geo(w, h, row0, full_h, w, &g)) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    CCL_CHECK(cclk::launch_strip_export(g, d_labels, static_cast<uint32_t*>(d_work), d_seam_out, strip_index, st));
    return CCL_OK;
}

ccl_status ccl_strip_seam_resolve(ccl_ctx* ctx, const uint32_t* d_seam_all, uint32_t n_strips, uint32_t strip_index,
                                  uint32_t w, uint32_t h, uint32_t row0, uint32_t full_h, uint32_t* d_labels,
                                  void* d_work, uint32_t* d_scratch, void* stream) {
    if (!ctx || !d_seam_all || !d_labels || !d_work || !d_scratch) return fail(CCL_EINVAL, "null argument");
    if (n_strips == 0 || strip_index >= n_strips) return fail(CCL_EINVAL, "bad strip index");
    if (uint64_t(n_strips) * 2 * w >= 0xFFFFFFFFull) return fail(CCL_EINVAL, "too many seam nodes");
    DeviceGuard dg(ctx->device);
    cclk::Geo g{};
    if (ccl_status s = strip_geo(w, h, row0, full_h, w, &g)) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    CCL_CHECK(cclk::launch_strip_resolve(g, d_seam_all, n_strips, strip_index, d_labels,
                                         static_cast<uint32_t*>(d_work), d_scratch, st));
    return CCL_OK;
}

ccl_status ccl_strip_final(ccl_ctx* ctx, uint32_t w, uint32_t h, uint32_t row0, uint32_t full_h, uint32_t* d_labels,
                           const void* d_work, int variant, void* stream) {
    if (!ctx || !d_labels || !d_work) return fail(CCL_EINVAL, "null argument");
    DeviceGuard dg(ctx->device);
    cclk::LaunchArgs a{};
    if (ccl_status s = strip_geo(w, h, row0, full_h, w, &a.g)) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // kernel (e) never reads the image; any 16B-aligned pointer satisfies prepare().
    // `variant` must be the one ccl_strip_local used: it selects the node
    // layout kernel (e) expands (band runs, row runs or pixels).
    if (ccl_status s =
            prepare(&a, reinterpret_cast<const uint8_t*>(d_work), 16, 16 * size_t(h), 1, d_labels, variant, st))
        return s;
    a.work = static_cast<uint32_t*>(const_cast<void*>(d_work));
    CCL_CHECK(cclk::launch_final(a));
    return CCL_OK;
}

size_t ccl_strip_scratch_words(uint32_t n_strips, uint32_t w) { return size_t(n_strips) * 2 * w; }

size_t ccl_work_bytes(uint32_t w, uint32_t h, uint32_t nframes) { return cclk::work_bytes(w, h, nframes); }

// ---------------------------------------------------------------- compaction
ccl_status ccl_compact_device(ccl_ctx* ctx, const uint32_t* d_raw, uint32_t w, uint32_t h, uint32_t* d_out,
                              uint32_t* d_scratch, uint64_t* k_out, void* stream) {
    if (!ctx || !d_raw || !d_out || !d_scratch) return fail(CCL_EINVAL, "null argument");
    if (ccl_status s = check_dims(w, h)) return s;
    DeviceGuard dg(ctx->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t n = size_t(w) * h;
    CCL_CHECK(cclk::launch_compact(d_raw, n, d_out, d_scratch, st));
    if (k_out) {
        const size_t words = (n + 31) / 32, nb = (words + 1023) / 1024;
        uint32_t k = 0;
        CCL_CHECK(cudaMemcpyAsync(&k, d_scratch + 2 * words + nb, 4, cudaMemcpyDeviceToHost, st));
        CCL_CHECK(cudaStreamSynchronize(st));
        *k_out = k;
    }
    return CCL_OK;
}

size_t ccl_compact_scratch_words(uint32_t w, uint32_t h) { return cclk::compact_scratch_words(size_t(w) * h); }

// ---------------------------------------------------------------- generators
ccl_status ccl_gen_random(uint8_t* out, uint32_t w, uint32_t h, double density, uint64_t seed) {
    if (!out) return fail(CCL_EINVAL, "null argument");
    try {
        const ccl::BinaryImage img = ccl::random_image(w, h, density, seed);
        std::memcpy(out, img.data.data(), img.data.size());
        return CCL_OK;
    } catch (const std::invalid_argument& e) {
        return fail(CCL_EINVAL, e.what());
    } catch (const std::exception& e) {
        return fail(CCL_ENOMEM, e.what());
    }
}

ccl_status ccl_gen_random_device(ccl_ctx* ctx, uint8_t* d_out, uint32_t w, uint32_t h, uint32_t row0, double density,
                                 uint64_t seed, void* stream) {
    if (!ctx || !d_out) return fail(CCL_EINVAL, "null argument");
    if (ccl_status s = check_dims(w, h)) return s;
    if (!(density >= 0.0 && density <= 1.0)) return fail(CCL_EINVAL, "density must be in [0, 1]");
    if (reinterpret_cast<uintptr_t>(d_out) % 16) return fail(CCL_EINVAL, "d_out must be 16-byte aligned");
    DeviceGuard dg(ctx->device);
    CCL_CHECK(cclk::launch_gen_random(d_out, uint64_t(w) * h, uint64_t(row0) * w, density, seed,
                                      static_cast<cudaStream_t>(stream)));
    return CCL_OK;
}

ccl_status ccl_gen_pattern(uint8_t* out, int kind, uint32_t w, uint32_t h, uint32_t period, double density,
                           uint64_t seed) {
    if (!out) return fail(CCL_EINVAL, "null argument");
    if (kind < 0 || kind > 3) return fail(CCL_EINVAL, "unknown pattern kind");
    try {
        ccl::PatternParams pp;
        pp.period = period;
        pp.density = density;
        pp.seed = seed;
        const ccl::BinaryImage img = ccl::pattern_image(static_cast<ccl::PatternKind>(kind), w, h, pp);
        std::memcpy(out, img.data.data(), img.data.size());
        return CCL_OK;
    } catch (const std::invalid_argument& e) {
        return fail(CCL_EINVAL, e.what());
    } catch (const std::exception& e) {
        return fail(CCL_ENOMEM, e.what());
    }
}

// ---------------------------------------------------------------- CCLM stream
// Label on the device, compact on the device (pipeline.cpp:54-70), then copy
// the compacted labels to a CCLM file (label_io.cpp:27-33 format) in chunks
// through a pinned double buffer: the copy of chunk i+1 overlaps the write of
// chunk i.
ccl_status ccl_label_to_cclm(ccl_ctx* ctx, const uint8_t* img, uint32_t w, uint32_t h, int variant, const char* path,
                             uint64_t* k_out) {
    if (!ctx || !img || !path) return fail(CCL_EINVAL, "null argument");
    if (ccl_status s = check_dims(w, h)) return s;
    if (variant < 0 || variant > 3) return fail(CCL_EINVAL, "unknown variant");
    DeviceGuard dg(ctx->device);
    const size_t px = size_t(w) * h;
    const size_t pitch = (size_t(w) + 15) / 16 * 16;
    if (ctx->d_img_bytes < pitch * h) {
        if (ctx->d_img) cudaFree(ctx->d_img);
        ctx->d_img = nullptr;
        ctx->d_img_bytes = 0;
        CCL_CHECK(cudaMalloc(&ctx->d_img, pitch * h));
        ctx->d_img_bytes = pitch * h;
    }
    if (ctx->d_lab_bytes < px * 4) {
        if (ctx->d_lab) cudaFree(ctx->d_lab);
        ctx->d_lab = nullptr;
        ctx->d_lab_bytes = 0;
        CCL_CHECK(cudaMalloc(&ctx->d_lab, px * 4));
        ctx->d_lab_bytes = px * 4;
    }
    const size_t aux = (px + cclk::compact_scratch_words(px)) * 4;
    if (ctx->d_aux_bytes < aux) {
        if (ctx->d_aux) cudaFree(ctx->d_aux);
        ctx->d_aux = nullptr;
        ctx->d_aux_bytes = 0;
        CCL_CHECK(cudaMalloc(&ctx->d_aux, aux));
        ctx->d_aux_bytes = aux;
    }
    constexpr size_t CH = size_t(16) << 20;  // bytes per chunk
    if (!ctx->h_ring) {
        CCL_CHECK(cudaMallocHost(&ctx->h_ring, 2 * CH));
        for (auto& e : ctx->ring_ev) CCL_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    CCL_CHECK(cudaMemcpy2DAsync(ctx->d_img, pitch, img, w, w, h, cudaMemcpyHostToDevice, ctx->stream));
    if (ccl_status s = ccl_label_device(ctx, ctx->d_img, pitch, w, h, ctx->d_lab, variant, ctx->stream, 0, nullptr))
        return s;
    uint32_t* d_out = ctx->d_aux;
    uint32_t* d_scr = ctx->d_aux + px;
    CCL_CHECK(cclk::launch_compact(ctx->d_lab, px, d_out, d_scr, ctx->stream));
    const size_t words = (px + 31) / 32, nb = (words + 1023) / 1024;
    uint32_t k = 0;
    CCL_CHECK(cudaMemcpyAsync(&k, d_scr + 2 * words + nb, 4, cudaMemcpyDeviceToHost, ctx->stream));

    FILE* f = std::fopen(path, "wb");
    if (!f) return fail(CCL_EINVAL, std::string("cannot open ") + path + " for writing");
    unsigned char hdr[13] = {'C', 'C', 'L', 'M', 1};
    for (int i = 0; i < 4; ++i) {
        hdr[5 + i] = uint8_t(w >> (8 * i));
        hdr[9 + i] = uint8_t(h >> (8 * i));
    }
    bool ok = std::fwrite(hdr, 1, 13, f) == 13;
    const size_t total = px * 4, nchunks = (total + CH - 1) / CH;
    auto issue = [&](size_t i) {
        const size_t off = i * CH, n = std::min(CH, total - off);
        cudaError_t e = cudaMemcpyAsync(ctx->h_ring + (i & 1) * CH, reinterpret_cast<uint8_t*>(d_out) + off, n,
                                        cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaEventRecord(ctx->ring_ev[i & 1], ctx->stream);
        return e;
    };
    cudaError_t e = issue(0);
    for (size_t i = 0; ok && e == cudaSuccess && i < nchunks; ++i) {
        if (i + 1 < nchunks) e = issue(i + 1);  // next copy in flight while this chunk is written
        if (e != cudaSuccess) break;
        e = cudaEventSynchronize(ctx->ring_ev[i & 1]);
        if (e != cudaSuccess) break;
        const size_t n = std::min(CH, total - i * CH);
        ok = std::fwrite(ctx->h_ring + (i & 1) * CH, 1, n, f) == n;
    }
    ok = (std::fclose(f) == 0) && ok;
    if (e != cudaSuccess) return cuda_fail(e, "ccl_label_to_cclm");
    CCL_CHECK(cudaStreamSynchronize(ctx->stream));
    if (!ok) return fail(CCL_EINVAL, std::string("write failed: ") + path);
    if (k_out) *k_out = k;
    return CCL_OK;
}

void ccl_tile_shape(uint32_t* tw, uint32_t* th) {
    if (tw) *tw = uint32_t(cclk::tile_w());
    if (th) *th = uint32_t(cclk::tile_h());
}

int ccl_launches_per_label(void) { return 4; }  // (a), (d), (d2) resolve, (e)

int ccl_metrics_build(void) { return CCL_METRICS; }

ccl_status ccl_read_metrics(ccl_ctx* ctx, uint32_t* tile_find, uint32_t* tile_cas, size_t n_tiles, uint64_t* phase4,
                            uint32_t* tiles_x, uint32_t* tiles_y, uint32_t* n_frames) {
    if (!ctx) return fail(CCL_EINVAL, "null context");
    if (!CCL_METRICS) return fail(CCL_EINVAL, "not an instrumented build (compile with CCL_METRICS=1)");
    if (!ctx->d_metrics) return fail(CCL_EINVAL, "no labeling call on this context yet");
    if (tiles_x) *tiles_x = ctx->m_tx;
    if (tiles_y) *tiles_y = ctx->m_ty;
    if (n_frames) *n_frames = ctx->m_frames;
    const size_t nt = size_t(ctx->m_tx) * ctx->m_ty * ctx->m_frames;
    if ((tile_find || tile_cas) && n_tiles < nt) return fail(CCL_EINVAL, "tile buffers smaller than the tile grid");
    DeviceGuard dg(ctx->device);
    std::vector<uint32_t> h(8 + 2 * nt);
    CCL_CHECK(cudaStreamSynchronize(ctx->stream));
    CCL_CHECK(cudaDeviceSynchronize());
    CCL_CHECK(cudaMemcpy(h.data(), ctx->d_metrics, h.size() * 4, cudaMemcpyDeviceToHost));
    if (phase4) std::memcpy(phase4, h.data(), 32);
    for (size_t t = 0; t < nt; ++t) {
        if (tile_find) tile_find[t] = h[8 + 2 * t];
        if (tile_cas) tile_cas[t] = h[8 + 2 * t + 1];
    }
    return CCL_OK;
}

const char* ccl_last_error(void) { return g_err.c_str(); }

const char* ccl_version(void) { return "ccl-b200 0.1 (sm_100a)"; }

}  // extern "C"

// ccl_label_strips (one image over several devices of this process) and the
// multi-process strip groups live in ccl_strips.cu.

namespace cclk {
int set_error(int status, const char* msg) {
    g_err = msg ? msg : "";
    return status;
}
}  // namespace cclk
