// ref_adapter.cpp — TEST INFRASTRUCTURE ONLY.
//
// Exposes the UNMODIFIED reference CPU labeler (compiled straight from
// /root/reference/proj/src by oracle/Makefile, namespace renamed with
// -Dccl=ccl_ref so it can never clash with the product's ccl::) through a
// plain C ABI for ctypes.  Output goes to oracle/_ref/ only.  Used by the
// tests to pin oracle/ccl_oracle.c and by bench.py's reference / cpu_baseline
// arm.  Nothing here is linked into the product library.
#include <cstdint>
#include <cstring>
#include <exception>
#include <thread>

#include "ccl/generate.hpp"
#include "ccl/label_io.hpp"
#include "ccl/oracle.hpp"
#include "ccl/pipeline.hpp"

namespace {
ccl::BinaryImage wrap(const std::uint8_t* img, std::uint32_t w, std::uint32_t h) {
    ccl::BinaryImage b(w, h);
    std::memcpy(b.data.data(), img, b.data.size());
    return b;
}
}  // namespace

extern "C" {

int ref_random_image(std::uint8_t* out, std::uint32_t w, std::uint32_t h, double density,
                     std::uint64_t seed) {
    try {
        auto img = ccl::random_image(w, h, density, seed);
        std::memcpy(out, img.data.data(), img.data.size());
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

int ref_pattern_image(std::uint8_t* out, int kind, std::uint32_t w, std::uint32_t h,
                      std::uint32_t period, double density, std::uint64_t seed) {
    try {
        ccl::PatternParams pp;
        pp.period = period;
        pp.density = density;
        pp.seed = seed;
        auto img = ccl::pattern_image(static_cast<ccl::PatternKind>(kind), w, h, pp);
        std::memcpy(out, img.data.data(), img.data.size());
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// labels_out: W*H u32 raw-root map; wall_ms: RunReport.wall_time (steps 1-3 only).
int ref_label_image(const std::uint8_t* img, std::uint32_t w, std::uint32_t h, std::uint32_t bw,
                    std::uint32_t bh, int variant, unsigned workers, std::uint32_t* labels_out,
                    double* wall_ms) {
    try {
        auto b = wrap(img, w, h);
        ccl::BlockConfig cfg;
        cfg.block_w = bw;
        cfg.block_h = bh;
        auto rep = ccl::label_image(b, cfg, static_cast<ccl::Variant>(variant), workers);
        std::memcpy(labels_out, rep.label_map.labels.data(), rep.label_map.labels.size() * 4);
        if (wall_ms) *wall_ms = rep.wall_time.count();
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    } catch (const std::exception&) {
        return -2;
    }
}

int ref_sequential_ccl(const std::uint8_t* img, std::uint32_t w, std::uint32_t h,
                       std::uint32_t* labels_out) {
    try {
        auto b = wrap(img, w, h);
        auto lm = ccl::sequential_ccl(b);
        std::memcpy(labels_out, lm.labels.data(), lm.labels.size() * 4);
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

unsigned ref_hardware_concurrency() { return std::thread::hardware_concurrency(); }

// write_label_map (label_io.cpp:66-76): format 0 raw, 1 csv, 2 pgm16
int ref_write_label_map(const std::uint32_t* labels, std::uint32_t w, std::uint32_t h, int compacted, int format,
                        const char* path) {
    try {
        ccl::LabelMap lm(w, h);
        std::memcpy(lm.labels.data(), labels, lm.labels.size() * 4);
        lm.compacted = compacted != 0;
        ccl::write_label_map(lm, path, format == 1 ? ccl::LabelMapFormat::csv
                                                   : format == 2 ? ccl::LabelMapFormat::pgm16
                                                                 : ccl::LabelMapFormat::raw);
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

}  // extern "C"
