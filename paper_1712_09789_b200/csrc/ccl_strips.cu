// ccl_strips.cu — one image over several GPUs in horizontal strips, with the
// seam exchange inside the library.
//
// A strip group is one rank (one GPU) of an N-strip labeling.  Every rank owns
// an EXCHANGE AREA in its own HBM:
//     [flags: 64 u32, flag k = last epoch rank k published here]
//     [exports: 2 parities x N slots x 4W u32]
// and one step of a rank is, all enqueued on its stream with no host round trip:
//   1. ccl_strip_local            kernels (a)(b)(c)(d) on the strip (global raster space)
//   2. ccl_strip_seam_export      the strip's 4W seam words (roots of the top / bottom
//                                 rows + their seam reps, ccl_aux.cu)
//   3. k_strip_push               those words stored into slot `rank` of EVERY rank's
//                                 area (NVLink peer stores; the area is mapped with a
//                                 CUDA IPC handle across processes, or a plain peer
//                                 pointer in-process); the last CTA to finish raises
//                                 flag `rank` = epoch in every area (release, system scope)
//   4. k_strip_wait               one thread per peer spins on its LOCAL flag until it
//                                 reaches this epoch or a later one (acquire, system scope)
//   5. ccl_strip_seam_resolve     the same union-find over all N exports on every rank
//                                 (no broadcast: the local area already holds them)
//   6. ccl_strip_final            kernels (d2)+(e)
// Exports alternate between two parities: a rank can only reach step s+2 after
// its step s+1 wait saw every peer's s+1 flag, i.e. after every peer finished
// reading step s -- so parity (s & 1) is free again.
//
// The reference's counterpart is the boundary merge of Algorithm 2
// (proj/src/boundary.cpp:22-35) applied to the strip seams, then the global
// resolve (boundary.cpp:37-55); the reference itself is single-process.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "ccl_cuda.h"
#include "ccl_internal.h"

namespace {

constexpr uint32_t kFlagWords = 64;  // flags region (n_ranks <= 64)
constexpr uint64_t kWaitTimeoutNs = 20ull * 1000 * 1000 * 1000;

ccl_status err(ccl_status s, const std::string& m) { return ccl_status(cclk::set_error(int(s), m.c_str())); }
ccl_status cuda_err(cudaError_t e, const char* where) {
    return err(e == cudaErrorMemoryAllocation ? CCL_ENOMEM : CCL_ECUDA,
               std::string(where) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
}
#define SG_CHECK(call)                                     \
    do {                                                   \
        const cudaError_t e__ = (call);                    \
        if (e__ != cudaSuccess) return cuda_err(e__, #call); \
    } while (0)

struct DevScope {
    int prev = -1;
    explicit DevScope(int d) {
        cudaGetDevice(&prev);
        if (prev != d) cudaSetDevice(d);
    }
    ~DevScope() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Step 3: this rank's export -> slot `rank` of every area (blockIdx.y = the
// destination), then the last CTA publishes the epoch flag in every area.
__global__ void __launch_bounds__(256) k_strip_push(const uint4* __restrict__ src, uint32_t n4,
                                                     uint32_t* const* __restrict__ areas, uint32_t n_ranks,
                                                     size_t slot_words, uint32_t rank, uint32_t epoch,
                                                     uint32_t* counter) {
    uint4* dst = reinterpret_cast<uint4*>(areas[blockIdx.y] + slot_words);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x) dst[i] = src[i];
    __threadfence_system();  // this CTA's peer stores before its arrival
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t total = gridDim.x * gridDim.y;
        if (atomicAdd(counter, 1u) == total - 1) {  // every CTA's stores are fenced
            __threadfence_system();
            for (uint32_t k = 0; k < n_ranks; ++k) st_release_sys(areas[k] + rank, epoch);
            *counter = 0;  // ready for the next step (stream order)
        }
    }
}

// Step 4: one thread per peer waits for that peer's flag in the local area.
__global__ void k_strip_wait(const uint32_t* flags, uint32_t n_ranks, uint32_t rank, uint32_t epoch) {
    const uint32_t k = threadIdx.x;
    if (k >= n_ranks || k == rank) return;
    const uint64_t t0 = globaltimer();
    // >=, not ==: a fast peer may already have published a LATER epoch here
    // (it only needs this rank's current export, which is still in its parity
    // slot: the peer cannot run two steps ahead, see the header)
    while (int32_t(ld_acquire_sys(flags + k) - epoch) < 0) {
        if (globaltimer() - t0 > kWaitTimeoutNs) __trap();  // a peer never arrived: fail loudly
        __nanosleep(64);
    }
}

}  // namespace

namespace {
// ccl_label_strips' per-shape resources.  Never destroyed by a static
// destructor (CUDA must not be called after the runtime's own teardown at
// exit); ccl_release_caches() frees them explicitly.
std::mutex& strips_mu() {
    static std::mutex mu;
    return mu;
}
using StripsKey = std::tuple<std::vector<int>, uint32_t, uint32_t>;
struct CacheBase {
    virtual ~CacheBase() = default;
};
std::map<StripsKey, std::unique_ptr<CacheBase>>& strips_cache_base() {
    static auto* m = new std::map<StripsKey, std::unique_ptr<CacheBase>>();
    return *m;
}
}  // namespace

struct ccl_strip_group {
    ccl_ctx* ctx = nullptr;
    int device = 0;
    uint32_t rank = 0, n = 1, w = 0, full_h = 0, row0 = 0, h = 0;
    uint32_t* area = nullptr;  // own exchange area
    size_t area_words = 0;
    std::vector<uint32_t*> peers;  // every rank's area as seen from this device (peers[rank] == area)
    std::vector<bool> ipc_opened;
    uint32_t** d_peers = nullptr;  // device copy of `peers`
    void* work = nullptr;          // kernel (a) -> (e) hand-off of the strip
    uint32_t* scratch = nullptr;   // seam union-find parents (n * 2W)
    uint32_t* seam = nullptr;      // this strip's export (4W)
    uint32_t* counter = nullptr;   // k_strip_push arrivals
    uint32_t epoch = 0;
    bool host_ordered = false;     // in-process: steps ordered by events, no flag wait
};

namespace {

void strip_split(uint32_t full_h, uint32_t n, uint32_t k, uint32_t* row0, uint32_t* h) {
    // strips.split_rows: near-equal heights, all but the last a multiple of the tile height
    const uint32_t th = uint32_t(cclk::tile_h()), tiles = (full_h + th - 1) / th;
    uint32_t acc = 0;
    for (uint32_t j = 0; j <= k; ++j) {
        const uint32_t t = tiles / n + (j < tiles % n ? 1u : 0u);
        const uint32_t hh = j + 1 < n ? std::min(t * th, full_h - acc) : full_h - acc;
        if (j == k) {
            *row0 = acc;
            *h = hh;
        }
        acc += hh;
    }
}

ccl_status upload_peers(ccl_strip_group* g) {
    DevScope ds(g->device);
    SG_CHECK(cudaMemcpy(g->d_peers, g->peers.data(), g->n * sizeof(uint32_t*), cudaMemcpyHostToDevice));
    return CCL_OK;
}

// Steps 1-3 (local pass, export, push + publish).
ccl_status group_phase1(ccl_strip_group* g, const uint8_t* d_img, size_t pitch, uint32_t* d_labels, int variant,
                        cudaStream_t st) {
    ++g->epoch;
    if (g->epoch == 0) g->epoch = 1;  // 0 is the "never published" flag value
    if (ccl_status s = ccl_strip_local(g->ctx, d_img, pitch, g->w, g->h, g->row0, g->full_h, d_labels, g->work, variant,
                                       st))
        return s;
    if (ccl_status s =
            ccl_strip_seam_export(g->ctx, g->w, g->h, g->row0, g->full_h, g->rank, d_labels, g->work, g->seam, st))
        return s;
    DevScope ds(g->device);
    const uint32_t n4 = g->w;  // 4W u32 = W uint4
    const size_t slot = kFlagWords + (size_t((g->epoch & 1u) * g->n + g->rank)) * 4 * g->w;
    const unsigned bx = std::max(1u, std::min(64u, (n4 + 255) / 256));
    k_strip_push<<<dim3(bx, g->n), 256, 0, st>>>(reinterpret_cast<const uint4*>(g->seam), n4, g->d_peers, g->n, slot,
                                                  g->rank, g->epoch, g->counter);
    SG_CHECK(cudaGetLastError());
    return CCL_OK;
}

// Steps 4-6 (wait for the peers, seam resolve, kernels (d2)+(e)).
ccl_status group_phase2(ccl_strip_group* g, uint32_t* d_labels, int variant, cudaStream_t st) {
    {
        DevScope ds(g->device);
        if (!g->host_ordered && g->n > 1) {
            k_strip_wait<<<1, 64, 0, st>>>(g->area, g->n, g->rank, g->epoch);
            SG_CHECK(cudaGetLastError());
        }
    }
    const uint32_t* all = g->area + kFlagWords + size_t(g->epoch & 1u) * g->n * 4 * g->w;
    if (ccl_status s = ccl_strip_seam_resolve(g->ctx, all, g->n, g->rank, g->w, g->h, g->row0, g->full_h, d_labels,
                                              g->work, g->scratch, st))
        return s;
    return ccl_strip_final(g->ctx, g->w, g->h, g->row0, g->full_h, d_labels, g->work, variant, st);
}

ccl_status group_alloc(ccl_ctx* ctx, uint32_t rank, uint32_t n, uint32_t w, uint32_t full_h, ccl_strip_group** out) {
    if (!ctx || !out) return err(CCL_EINVAL, "null argument");
    *out = nullptr;
    if (n == 0 || n > kFlagWords || rank >= n) return err(CCL_EINVAL, "need 1 <= n_ranks <= 64 and rank < n_ranks");
    if (w == 0 || full_h == 0 || uint64_t(w) * full_h > uint64_t(CCL_BACKGROUND) - 1)
        return err(CCL_EINVAL, "image must be 1x1 .. 2^32-2 pixels");
    const uint32_t th = uint32_t(cclk::tile_h());
    if ((full_h + th - 1) / th < n) return err(CCL_EINVAL, "image has fewer tile rows than strips");
    if (uint64_t(n) * 2 * w >= 0xFFFFFFFFull) return err(CCL_EINVAL, "too many seam nodes");
    auto g = std::make_unique<ccl_strip_group>();
    g->ctx = ctx;
    // the context's device: its stream was created there
    cudaStream_t cst = static_cast<cudaStream_t>(ccl_ctx_stream(ctx));
    int dev = 0;
    SG_CHECK(cudaStreamGetDevice(cst, &dev));
    g->device = dev;
    g->rank = rank;
    g->n = n;
    g->w = w;
    g->full_h = full_h;
    strip_split(full_h, n, rank, &g->row0, &g->h);
    DevScope ds(dev);
    g->area_words = kFlagWords + size_t(2) * n * 4 * w;
    SG_CHECK(cudaMalloc(&g->area, g->area_words * 4));
    SG_CHECK(cudaMemset(g->area, 0, g->area_words * 4));
    SG_CHECK(cudaMalloc(&g->d_peers, n * sizeof(uint32_t*)));
    const size_t wb = ccl_work_bytes(w, g->h, 1);
    SG_CHECK(cudaMalloc(&g->work, wb));
    SG_CHECK(cudaMemset(g->work, 0, wb));
    SG_CHECK(cudaMalloc(&g->scratch, ccl_strip_scratch_words(n, w) * 4));
    SG_CHECK(cudaMalloc(&g->seam, size_t(4) * w * 4));
    SG_CHECK(cudaMalloc(&g->counter, 4));
    SG_CHECK(cudaMemset(g->counter, 0, 4));
    SG_CHECK(cudaDeviceSynchronize());  // areas zeroed before any peer can push
    g->peers.assign(n, nullptr);
    g->ipc_opened.assign(n, false);
    g->peers[rank] = g->area;
    *out = g.release();
    return CCL_OK;
}

void group_free(ccl_strip_group* g) {
    if (!g) return;
    DevScope ds(g->device);
    cudaDeviceSynchronize();
    for (uint32_t k = 0; k < g->peers.size(); ++k)
        if (g->ipc_opened[k] && g->peers[k]) cudaIpcCloseMemHandle(g->peers[k]);
    cudaFree(g->area);
    cudaFree(g->d_peers);
    cudaFree(g->work);
    cudaFree(g->scratch);
    cudaFree(g->seam);
    cudaFree(g->counter);
    delete g;
}

}  // namespace

extern "C" {

size_t ccl_strip_group_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

ccl_status ccl_strip_group_create(ccl_ctx* ctx, uint32_t rank, uint32_t n_ranks, uint32_t w, uint32_t full_h,
                                  ccl_strip_group** out, void* handle_out) {
    if (ccl_status s = group_alloc(ctx, rank, n_ranks, w, full_h, out)) return s;
    if (handle_out) {
        DevScope ds((*out)->device);
        cudaIpcMemHandle_t h;
        const cudaError_t e = cudaIpcGetMemHandle(&h, (*out)->area);
        if (e != cudaSuccess) {
            group_free(*out);
            *out = nullptr;
            return cuda_err(e, "cudaIpcGetMemHandle");
        }
        std::memcpy(handle_out, &h, sizeof(h));
    }
    return CCL_OK;
}

ccl_status ccl_strip_group_connect(ccl_strip_group* g, const void* handles) {
    if (!g || (!handles && g->n > 1)) return err(CCL_EINVAL, "null argument");
    DevScope ds(g->device);
    const auto* hs = static_cast<const cudaIpcMemHandle_t*>(handles);
    for (uint32_t k = 0; k < g->n; ++k) {
        if (k == g->rank || g->peers[k]) continue;
        void* p = nullptr;
        SG_CHECK(cudaIpcOpenMemHandle(&p, hs[k], cudaIpcMemLazyEnablePeerAccess));
        g->peers[k] = static_cast<uint32_t*>(p);
        g->ipc_opened[k] = true;
    }
    return upload_peers(g);
}

ccl_status ccl_strip_group_rows(const ccl_strip_group* g, uint32_t* row0, uint32_t* h) {
    if (!g) return err(CCL_EINVAL, "null group");
    if (row0) *row0 = g->row0;
    if (h) *h = g->h;
    return CCL_OK;
}

ccl_status ccl_strip_group_label(ccl_strip_group* g, const uint8_t* d_img, size_t img_pitch, uint32_t* d_labels,
                                 int variant, void* stream) {
    if (!g || !d_img || !d_labels) return err(CCL_EINVAL, "null argument");
    for (auto* p : g->peers)
        if (!p) return err(CCL_EINVAL, "strip group not connected (ccl_strip_group_connect)");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (ccl_status s = group_phase1(g, d_img, img_pitch, d_labels, variant, st)) return s;
    return group_phase2(g, d_labels, variant, st);
}

int ccl_strip_group_launches(const ccl_strip_group* g) {
    // (a) (d) | roots repmin reps | push | wait | seam union + apply (+ the
    // parents copy) | (d2) (e)
    return g ? 2 + 3 + 1 + (g->n > 1 ? 1 : 0) + 2 + 2 : 0;
}

void ccl_strip_group_destroy(ccl_strip_group* g) { group_free(g); }

// ---------------------------------------------------------------------------
// One image over several devices of this process (ccl::label_image_strips):
// strip k on devices[k] as a strip group connected with plain peer pointers.
// One host thread enqueues everything: phase 1 of every strip, an event per
// strip, every strip's stream waits on all of them (cross-device events), then
// phase 2 -- no host joins, no flag spinning.  Contexts, groups and buffers are
// cached per (devices, w, h) and reused by the next call with the same shape.
ccl_status ccl_label_strips(const int* devices, int ndev, const uint8_t* img, uint32_t w, uint32_t h,
                            uint32_t* labels, int variant, float* kernel_ms) {
    if (!devices || ndev <= 0 || !img || !labels) return err(CCL_EINVAL, "null argument or no devices");
    if (w == 0 || h == 0 || uint64_t(w) * h > uint64_t(CCL_BACKGROUND) - 1)
        return err(CCL_EINVAL, "image dimensions must be 1x1 .. 2^32-2 pixels");
    if (variant < 0 || variant > 3) return err(CCL_EINVAL, "unknown variant");
    const uint32_t n = uint32_t(ndev), th = uint32_t(cclk::tile_h());
    if (n > kFlagWords) return err(CCL_EINVAL, "at most 64 strips");
    if ((h + th - 1) / th < n) return err(CCL_EINVAL, "image has fewer tile rows than strips");

    struct Strip {
        int dev = 0;
        ccl_ctx* ctx = nullptr;
        ccl_strip_group* g = nullptr;
        uint8_t* d_img = nullptr;
        uint32_t* d_lab = nullptr;
        cudaEvent_t e0 = nullptr, e1 = nullptr, mid = nullptr;
    };
    struct Setup : CacheBase {
        std::vector<Strip> s;
        ~Setup() override {
            for (auto& x : s) {
                DevScope ds(x.dev);
                if (x.g) group_free(x.g);
                cudaFree(x.d_img);
                cudaFree(x.d_lab);
                for (auto e : {x.e0, x.e1, x.mid})
                    if (e) cudaEventDestroy(e);
                if (x.ctx) ccl_ctx_destroy(x.ctx);
            }
        }
    };
    std::lock_guard<std::mutex> lk(strips_mu());
    auto& cache = strips_cache_base();
    const StripsKey key{std::vector<int>(devices, devices + n), w, h};
    auto it = cache.find(key);
    if (it == cache.end()) {
        if (cache.size() >= 2) cache.clear();  // bound the device memory kept alive
        auto su = std::make_unique<Setup>();
        su->s.resize(n);
        const size_t pitch = (size_t(w) + 15) / 16 * 16;
        for (uint32_t k = 0; k < n; ++k) {
            Strip& s = su->s[k];
            s.dev = devices[k];
            if (ccl_status r = ccl_ctx_create(s.dev, &s.ctx)) return r;
            if (ccl_status r = group_alloc(s.ctx, k, n, w, h, &s.g)) return r;
            DevScope ds(s.dev);
            SG_CHECK(cudaMalloc(&s.d_img, pitch * s.g->h));
            SG_CHECK(cudaMalloc(&s.d_lab, size_t(w) * s.g->h * 4));
            SG_CHECK(cudaEventCreate(&s.e0));
            SG_CHECK(cudaEventCreate(&s.e1));
            SG_CHECK(cudaEventCreateWithFlags(&s.mid, cudaEventDisableTiming));
        }
        for (uint32_t k = 0; k < n; ++k) {  // plain peer pointers (NVLink P2P between distinct devices)
            Strip& s = su->s[k];
            DevScope ds(s.dev);
            for (uint32_t j = 0; j < n; ++j) {
                const int dj = su->s[j].dev;
                if (dj != s.dev) {
                    int ok = 0;
                    SG_CHECK(cudaDeviceCanAccessPeer(&ok, s.dev, dj));
                    if (!ok) return err(CCL_ENODEV, "devices without peer access cannot share a strip image");
                    const cudaError_t e = cudaDeviceEnablePeerAccess(dj, 0);
                    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                    else if (e != cudaSuccess) return cuda_err(e, "cudaDeviceEnablePeerAccess");
                }
                s.g->peers[j] = su->s[j].g->area;
            }
            s.g->host_ordered = true;
            if (ccl_status r = upload_peers(s.g)) return r;
        }
        it = cache.emplace(key, std::move(su)).first;
    }
    std::vector<Strip>& S = static_cast<Setup*>(it->second.get())->s;
    const size_t pitch = (size_t(w) + 15) / 16 * 16;
    for (uint32_t k = 0; k < n; ++k) {  // phase 1 everywhere
        Strip& s = S[k];
        DevScope ds(s.dev);
        cudaStream_t q = static_cast<cudaStream_t>(ccl_ctx_stream(s.ctx));
        SG_CHECK(cudaMemcpy2DAsync(s.d_img, pitch, img + size_t(s.g->row0) * w, w, w, s.g->h, cudaMemcpyHostToDevice,
                                   q));
        SG_CHECK(cudaEventRecord(s.e0, q));
        if (ccl_status r = group_phase1(s.g, s.d_img, pitch, s.d_lab, variant, q)) return r;
        SG_CHECK(cudaEventRecord(s.mid, q));
    }
    for (uint32_t k = 0; k < n; ++k) {  // every stream waits for every push, then phase 2
        Strip& s = S[k];
        DevScope ds(s.dev);
        cudaStream_t q = static_cast<cudaStream_t>(ccl_ctx_stream(s.ctx));
        for (uint32_t j = 0; j < n; ++j)
            if (j != k) SG_CHECK(cudaStreamWaitEvent(q, S[j].mid, 0));
        if (ccl_status r = group_phase2(s.g, s.d_lab, variant, q)) return r;
        SG_CHECK(cudaEventRecord(s.e1, q));
        SG_CHECK(cudaMemcpyAsync(labels + size_t(s.g->row0) * w, s.d_lab, size_t(w) * s.g->h * 4,
                                 cudaMemcpyDeviceToHost, q));
    }
    float worst = 0.f;
    for (uint32_t k = 0; k < n; ++k) {
        Strip& s = S[k];
        DevScope ds(s.dev);
        SG_CHECK(cudaStreamSynchronize(static_cast<cudaStream_t>(ccl_ctx_stream(s.ctx))));
        float ms = 0.f;
        SG_CHECK(cudaEventElapsedTime(&ms, s.e0, s.e1));
        worst = std::max(worst, ms);
    }
    if (kernel_ms) *kernel_ms = worst;
    return CCL_OK;
}

void ccl_release_caches(void) {
    std::lock_guard<std::mutex> lk(strips_mu());
    strips_cache_base().clear();
}

}  // extern "C"
