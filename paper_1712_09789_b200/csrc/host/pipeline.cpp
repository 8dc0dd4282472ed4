// pipeline.cpp — host C++ drop-in for ccl::label_image
// (/root/reference/proj/src/pipeline.cpp:11-52) on top of the C-ABI.
//
// Same validation order and exceptions as the reference:
//   !cfg.valid()  -> std::invalid_argument        (pipeline.cpp:13-14)
//   workers == 0  -> std::invalid_argument        (pipeline.cpp:15)
//   0x0 image     -> std::invalid_argument via LabelMap/check_size (image.hpp:31-33)
// plus ccl::DeviceError (a std::runtime_error) for CUDA failures.
// Each host thread owns its own ccl_ctx (stream + workspace), so concurrent
// calls on distinct images are safe.
#include <cuda_runtime.h>

#include <algorithm>
#include <memory>
#include <string>
#include <vector>

#include "ccl/generate.hpp"
#include "ccl/label_io.hpp"
#include "ccl/pipeline.hpp"
#include "ccl_cuda.h"

namespace ccl {

namespace {

thread_local int t_device = 0;

struct CtxDeleter {
    void operator()(ccl_ctx* c) const { ccl_ctx_destroy(c); }
};

ccl_ctx* thread_ctx() {
    thread_local std::unique_ptr<ccl_ctx, CtxDeleter> ctx;
    thread_local int ctx_dev = -1;
    if (!ctx || ctx_dev != t_device) {
        ctx.reset();
        ccl_ctx* c = nullptr;
        const ccl_status s = ccl_ctx_create(t_device, &c);
        if (s != CCL_OK) throw DeviceError(int(s), ccl_last_error());
        ctx.reset(c);
        ctx_dev = t_device;
    }
    return ctx.get();
}

void check(ccl_status s) {
    if (s == CCL_EINVAL) throw std::invalid_argument(ccl_last_error());
    if (s != CCL_OK) throw DeviceError(int(s), ccl_last_error());
}

void cuda_check(cudaError_t e, const char* where) {
    if (e != cudaSuccess)
        throw DeviceError(e == cudaErrorMemoryAllocation ? CCL_ENOMEM : CCL_ECUDA,
                          std::string(where) + ": " + cudaGetErrorString(e));
}

// Makes `dev` current for the scope (restores the caller's device after).
struct DeviceScope {
    int prev = -1;
    explicit DeviceScope(int dev) {
        cuda_check(cudaGetDevice(&prev), "cudaGetDevice");
        if (prev != dev) cuda_check(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~DeviceScope() {
        int cur = -1;
        if (cudaGetDevice(&cur) == cudaSuccess && prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// Device allocation freed on scope exit (also when a later step throws).
struct DeviceBuffer {
    void* p = nullptr;
    explicit DeviceBuffer(std::size_t bytes) { cuda_check(cudaMalloc(&p, bytes), "cudaMalloc"); }
    ~DeviceBuffer() { cudaFree(p); }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
};

}  // namespace

void set_device(int device) { t_device = device; }

RunReport label_image(const BinaryImage& img, const BlockConfig& cfg, Variant variant, unsigned workers) {
    if (!cfg.valid()) throw std::invalid_argument("block configuration invalid or over the scratch ceiling");
    if (workers == 0) throw std::invalid_argument("workers must be >= 1");

    RunReport rep;
    rep.variant = variant;
    rep.cfg = cfg;
    rep.worker_count = workers;
    rep.blocks_x = (img.width + cfg.block_w - 1) / cfg.block_w;
    rep.blocks_y = (img.height + cfg.block_h - 1) / cfg.block_h;
    rep.per_block.resize(std::size_t(rep.blocks_x) * rep.blocks_y);
    for (std::size_t i = 0; i < rep.per_block.size(); ++i) rep.per_block[i].block_id = std::uint32_t(i);

    rep.label_map = LabelMap(img.width, img.height);  // throws invalid_argument for 0x0 like the reference
    if (img.data.size() != rep.label_map.labels.size())
        throw std::invalid_argument("image data size does not match width*height");

    float ms = 0.f;
    check(ccl_label_host(thread_ctx(), img.data.data(), img.width, img.height, rep.label_map.labels.data(),
                         int(variant), &ms));
    rep.wall_time = std::chrono::duration<double, std::milli>(double(ms));
    if (ccl_metrics_build()) {
        // instrumented build: the counters are per GPU tile (the GPU's block),
        // so per_block / blocks_x / blocks_y describe the tile grid
        std::uint32_t tx = 0, ty = 0, nfr = 0;
        std::uint64_t ph[4] = {0, 0, 0, 0};
        check(ccl_read_metrics(thread_ctx(), nullptr, nullptr, 0, nullptr, &tx, &ty, &nfr));
        std::vector<std::uint32_t> f(std::size_t(tx) * ty), c(f.size());
        check(ccl_read_metrics(thread_ctx(), f.data(), c.data(), f.size(), ph, &tx, &ty, &nfr));
        rep.blocks_x = tx;
        rep.blocks_y = ty;
        rep.per_block.assign(f.size(), BlockMetrics{});
        for (std::size_t i = 0; i < f.size(); ++i) {
            rep.per_block[i].block_id = std::uint32_t(i);
            rep.per_block[i].findroot_iterations = f[i];
            rep.per_block[i].atomic_ops = c[i];
        }
        rep.border_phase.findroot_iterations = ph[0];
        rep.border_phase.atomic_ops = ph[1];
        rep.resolve_phase.findroot_iterations = ph[2];
    }
    return rep;
}

std::uint64_t label_to_cclm(const BinaryImage& img, const std::string& path, Variant variant) {
    if (img.data.size() != BinaryImage::check_size(img.width, img.height))
        throw std::invalid_argument("image data size does not match width*height");
    std::uint64_t k = 0;
    check(ccl_label_to_cclm(thread_ctx(), img.data.data(), img.width, img.height, int(variant), path.c_str(), &k));
    return k;
}

LabelMap compact_labels(const LabelMap& lm) {
    if (lm.compacted) return lm;
    LabelMap out(lm.width, lm.height, 0);
    out.compacted = true;
    // roots are component minima, so "order of first appearance" == ascending
    // root order; one sweep with a dense remap (pipeline.cpp:54-70)
    std::vector<Label> remap(lm.labels.size(), 0);
    Label next = 0;
    for (std::size_t i = 0; i < lm.labels.size(); ++i) {
        const Label raw = lm.labels[i];
        if (raw == kBackground) continue;
        if (remap[raw] == 0) remap[raw] = ++next;
        out.labels[i] = remap[raw];
    }
    return out;
}

MetricsSummary aggregate_metrics(const RunReport& report) {
    MetricsSummary s;
    s.grid_w = report.blocks_x;
    s.grid_h = report.blocks_y;
    std::uint64_t it = 0, at = 0;
    for (const auto& m : report.per_block) {
        s.iterations_grid.push_back(m.findroot_iterations);
        s.atomics_grid.push_back(m.atomic_ops);
        it += m.findroot_iterations;
        at += m.atomic_ops;
    }
    if (!report.per_block.empty()) {
        s.mean_iterations = double(it) / double(report.per_block.size());
        s.mean_atomics = double(at) / double(report.per_block.size());
    }
    return s;
}

RunReport label_image_strips(const BinaryImage& img, const std::vector<int>& devices, Variant variant) {
    if (devices.empty()) throw std::invalid_argument("label_image_strips: no devices");
    RunReport rep;
    rep.variant = variant;
    rep.worker_count = unsigned(devices.size());
    rep.blocks_x = (img.width + rep.cfg.block_w - 1) / rep.cfg.block_w;
    rep.blocks_y = (img.height + rep.cfg.block_h - 1) / rep.cfg.block_h;
    rep.per_block.resize(std::size_t(rep.blocks_x) * rep.blocks_y);
    for (std::size_t i = 0; i < rep.per_block.size(); ++i) rep.per_block[i].block_id = std::uint32_t(i);
    rep.label_map = LabelMap(img.width, img.height);
    if (img.data.size() != rep.label_map.labels.size())
        throw std::invalid_argument("image data size does not match width*height");
    float ms = 0.f;
    check(ccl_label_strips(devices.data(), int(devices.size()), img.data.data(), img.width, img.height,
                           rep.label_map.labels.data(), int(variant), &ms));
    rep.wall_time = std::chrono::duration<double, std::milli>(double(ms));
    return rep;
}

std::vector<LabelMap> label_batch(const std::vector<BinaryImage>& frames, Variant variant) {
    std::vector<LabelMap> out;
    if (frames.empty()) return out;
    const std::uint32_t w = frames[0].width, h = frames[0].height;
    for (const auto& f : frames)
        if (f.width != w || f.height != h) throw std::invalid_argument("label_batch: frames differ in size");
    ccl_ctx* ctx = thread_ctx();
    // the staging buffers live on the context's device, not on whatever device
    // the calling thread happens to have current
    DeviceScope on(t_device);
    const std::size_t px = BinaryImage::check_size(w, h);
    const std::size_t pitch = (std::size_t(w) + 15) / 16 * 16, fpitch = pitch * h;
    const std::uint32_t n = std::uint32_t(frames.size());
    std::vector<std::uint8_t> host(fpitch * n, 0);
    for (std::uint32_t f = 0; f < n; ++f)
        for (std::uint32_t y = 0; y < h; ++y)
            std::copy_n(frames[f].data.data() + std::size_t(y) * w, w, host.data() + f * fpitch + y * pitch);
    DeviceBuffer d_img(host.size()), d_lab(px * n * 4);
    cudaStream_t st = static_cast<cudaStream_t>(ccl_ctx_stream(ctx));
    cuda_check(cudaMemcpyAsync(d_img.p, host.data(), host.size(), cudaMemcpyHostToDevice, st), "label_batch H2D");
    check(ccl_label_batch(ctx, static_cast<std::uint8_t*>(d_img.p), pitch, fpitch, n, w, h,
                          static_cast<std::uint32_t*>(d_lab.p), int(variant), st));
    out.reserve(n);
    for (std::uint32_t f = 0; f < n; ++f) {
        out.emplace_back(w, h);
        cuda_check(cudaMemcpyAsync(out.back().labels.data(), static_cast<std::uint32_t*>(d_lab.p) + f * px, px * 4,
                                   cudaMemcpyDeviceToHost, st),
                   "label_batch D2H");
    }
    cuda_check(cudaStreamSynchronize(st), "label_batch");
    return out;
}

}  // namespace ccl
