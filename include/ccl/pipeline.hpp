// ccl/pipeline.hpp — the drop-in labeling entry point.
//
// `label_image` keeps the reference signature verbatim
// (/root/reference/proj/include/ccl/pipeline.hpp:33-34) and its contract
// (pipeline.cpp:11-52): raw-root label map identical to the reference for any
// cfg / variant / workers, std::invalid_argument for an invalid cfg or
// workers == 0, wall_time covering only the labeling steps (here: CUDA-event
// device time of the kernels, "kernel-only GPU timings").
// Implemented in paper_1712_09789_b200/csrc/host/pipeline.cpp on top of the
// C-ABI in include/ccl_cuda.h.
#pragma once

#include <chrono>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "ccl/forest.hpp"
#include "ccl/image.hpp"

namespace ccl {

// BlockMetrics (reference forest.hpp:15-29) comes from ccl/forest.hpp, included
// here as the reference pipeline.hpp:7 does.  The product build leaves its
// counters 0; the instrumented build fills them per GPU tile.

// pipeline.hpp:15-26
struct RunReport {
    LabelMap label_map;  // raw-root form
    std::vector<BlockMetrics> per_block;
    std::uint32_t blocks_x = 0;
    std::uint32_t blocks_y = 0;
    BlockMetrics border_phase;
    BlockMetrics resolve_phase;
    std::chrono::duration<double, std::milli> wall_time{0};
    Variant variant = Variant::C2FL;
    BlockConfig cfg;
    unsigned worker_count = 1;
};

// A CUDA failure below the C-ABI.  Derives from std::runtime_error, so a CLI
// mapping exceptions to exit codes (tools/ccl.cpp:310-325) must catch it.
class DeviceError : public std::runtime_error {
public:
    DeviceError(int status, const std::string& msg) : std::runtime_error(msg), status_(status) {}
    int status() const { return status_; }

private:
    int status_;
};

// The drop-in (pipeline.hpp:33-34).  `workers` is validated (>= 1) and
// recorded; the GPU ignores it (output is identical for any count).
RunReport label_image(const BinaryImage& img, const BlockConfig& cfg, Variant variant, unsigned workers = 1);

// Renumber to 1..K in raster order of first appearance, background 0
// (pipeline.cpp:54-70).  Idempotent.
LabelMap compact_labels(const LabelMap& lm);

struct MetricsSummary {
    double mean_iterations = 0.0;
    double mean_atomics = 0.0;
    std::uint32_t grid_w = 0;
    std::uint32_t grid_h = 0;
    std::vector<std::uint64_t> iterations_grid;
    std::vector<std::uint64_t> atomics_grid;
};

// pipeline.cpp:72-91 (counters are zero on the GPU path).
MetricsSummary aggregate_metrics(const RunReport& report);

// ---- additive B200 entry points -------------------------------------------
// Batch of equally sized frames, one launch per kernel for all of them;
// labels are per-frame raster indices.
std::vector<LabelMap> label_batch(const std::vector<BinaryImage>& frames, Variant variant = Variant::C2FL);

// One image over several GPUs of this process (horizontal strips, seams
// exchanged by peer copies; a device may repeat).  Same label map as
// label_image; wall_time = max over strips of the device time.
RunReport label_image_strips(const BinaryImage& img, const std::vector<int>& devices,
                             Variant variant = Variant::C2FL);

// CUDA device used by this host thread's implicit context (default 0).
void set_device(int device);

}  // namespace ccl
