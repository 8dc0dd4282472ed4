// label_io.cpp — label-map files.  Formats follow the
// reference spec (proj/src/label_io.cpp:27-94); the CCLM
// stream path overlaps device->host copies with file writes.
#include "ccl/label_io.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <fstream>
#include <vector>

#include "ccl_cuda.h"

namespace ccl {

namespace {

void put_le32(std::ostream& os, std::uint32_t v) {
    const char b[4] = {char(v), char(v >> 8), char(v >> 16), char(v >> 24)};
    os.write(b, 4);
}

void cclm_header(std::ostream& os, std::uint32_t w, std::uint32_t h) {
    os.write("CCLM", 4);
    os.put(char(1));
    put_le32(os, w);
    put_le32(os, h);
}

// u32 little-endian payload in bounded chunks (the host is little-endian x86,
// so a chunk is written as is)
void le32_block(std::ostream& os, const std::uint32_t* v, std::size_t n) {
    os.write(reinterpret_cast<const char*>(v), std::streamsize(n * 4));
}

}  // namespace

LabelMapFormat parse_label_format(const std::string& s) {
    if (s == "raw") return LabelMapFormat::raw;
    if (s == "csv") return LabelMapFormat::csv;
    if (s == "pgm16") return LabelMapFormat::pgm16;
    throw std::invalid_argument("unknown label map format: " + s);
}

void write_label_map(const LabelMap& lm, const std::string& path, LabelMapFormat format) {
    const LabelMap c = compact_labels(lm);
    std::ofstream os(path, std::ios::binary);
    if (!os) throw IoError("cannot open " + path + " for writing");
    if (format == LabelMapFormat::raw) {
        cclm_header(os, c.width, c.height);
        le32_block(os, c.labels.data(), c.labels.size());
    } else if (format == LabelMapFormat::csv) {
        std::string line;
        for (std::uint32_t y = 0; y < c.height; ++y) {
            line.clear();
            for (std::uint32_t x = 0; x < c.width; ++x) {
                if (x) line.push_back(',');
                line += std::to_string(c.labels[std::size_t(y) * c.width + x]);
            }
            line.push_back('\n');
            os << line;
        }
    } else {
        const Label kmax = c.labels.empty() ? 0 : *std::max_element(c.labels.begin(), c.labels.end());
        if (kmax > 65535) throw std::overflow_error("pgm16 cannot represent more than 65535 components");
        os << "P5\n" << c.width << ' ' << c.height << '\n' << std::max<Label>(kmax, 1) << '\n';
        std::vector<char> row(std::size_t(c.width) * 2);
        for (std::uint32_t y = 0; y < c.height; ++y) {
            for (std::uint32_t x = 0; x < c.width; ++x) {
                const Label v = c.labels[std::size_t(y) * c.width + x];
                row[2 * x] = char(v >> 8);
                row[2 * x + 1] = char(v);
            }
            os.write(row.data(), std::streamsize(row.size()));
        }
    }
    if (!os) throw IoError("write failed: " + path);
}

LabelMap read_label_map(const std::string& path) {
    using K = ParseError::Kind;
    std::ifstream is(path, std::ios::binary);
    if (!is) throw IoError("cannot open " + path);
    char magic[4] = {};
    is.read(magic, 4);
    if (is.gcount() != 4 || std::string(magic, 4) != "CCLM") throw ParseError(K::unsupported_magic, "not a CCLM file: " + path);
    if (is.get() != 1) throw ParseError(K::bad_header, "unsupported CCLM version");
    unsigned char hb[8];
    is.read(reinterpret_cast<char*>(hb), 8);
    if (is.gcount() != 8) throw ParseError(K::truncated, "truncated CCLM header");
    const std::uint32_t w = hb[0] | hb[1] << 8 | hb[2] << 16 | std::uint32_t(hb[3]) << 24;
    const std::uint32_t h = hb[4] | hb[5] << 8 | hb[6] << 16 | std::uint32_t(hb[7]) << 24;
    if (w == 0 || h == 0) throw ParseError(K::bad_header, "zero dimension in CCLM header");
    LabelMap lm(w, h, 0);
    lm.compacted = true;
    is.read(reinterpret_cast<char*>(lm.labels.data()), std::streamsize(lm.labels.size() * 4));
    if (std::size_t(is.gcount()) != lm.labels.size() * 4) throw ParseError(K::truncated, "truncated CCLM file");
    return lm;
}

// Reference label_io.cpp:97-128: the counter grids of aggregate_metrics, then
// one summary row (none for an empty report).
void write_metrics_csv(const RunReport& report, const std::string& path, std::optional<double> density) {
    std::ofstream os(path, std::ios::binary);
    if (!os) throw IoError("cannot open " + path + " for writing");
    const MetricsSummary s = aggregate_metrics(report);
    for (const auto* grid : {&s.iterations_grid, &s.atomics_grid}) {
        os << (grid == &s.iterations_grid ? "iterations" : "atomics") << '\n';
        for (std::uint32_t by = 0; by < s.grid_h; ++by) {
            for (std::uint32_t bx = 0; bx < s.grid_w; ++bx)
                os << (bx ? "," : "") << (*grid)[std::size_t(by) * s.grid_w + bx];
            os << '\n';
        }
    }
    os << "width,height,block_w,block_h,density,variant,mean_iterations,mean_atomics,wall_ms\n";
    if (!report.per_block.empty()) {
        os << report.label_map.width << ',' << report.label_map.height << ',' << report.cfg.block_w << ','
           << report.cfg.block_h << ',';
        if (density) os << *density;
        os << ',' << to_string(report.variant) << ',' << s.mean_iterations << ',' << s.mean_atomics << ','
           << report.wall_time.count() << '\n';
    }
    if (!os) throw IoError("write failed: " + path);
}

}  // namespace ccl

// ------------------------------------------------------------------ C-ABI
namespace {
thread_local std::string t_io_err;
}

extern "C" {

ccl_status ccl_write_label_map(const uint32_t* labels, uint32_t w, uint32_t h, int compacted, int format,
                               const char* path) {
    try {
        ccl::LabelMap lm(w, h);
        std::copy_n(labels, lm.labels.size(), lm.labels.begin());
        lm.compacted = compacted != 0;
        ccl::write_label_map(lm, path, format == 1 ? ccl::LabelMapFormat::csv
                                                   : format == 2 ? ccl::LabelMapFormat::pgm16
                                                                 : ccl::LabelMapFormat::raw);
        return CCL_OK;
    } catch (const std::exception& e) {
        t_io_err = e.what();
        return CCL_EINVAL;
    }
}

ccl_status ccl_read_label_map(const char* path, uint32_t* labels, size_t capacity, uint32_t* w, uint32_t* h) {
    try {
        const ccl::LabelMap lm = ccl::read_label_map(path);
        if (w) *w = lm.width;
        if (h) *h = lm.height;
        if (labels) {
            if (capacity < lm.labels.size()) {
                t_io_err = "label buffer too small";
                return CCL_EINVAL;
            }
            std::copy(lm.labels.begin(), lm.labels.end(), labels);
        }
        return CCL_OK;
    } catch (const std::exception& e) {
        t_io_err = e.what();
        return CCL_EINVAL;
    }
}

const char* ccl_io_last_error(void) { return t_io_err.c_str(); }

}  // extern "C"
