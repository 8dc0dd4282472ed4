// label_io.hpp — label-map files (reference: /root/reference/proj/include/ccl/label_io.hpp,
// proj/src/label_io.cpp:27-94).
//
//   write_label_map / read_label_map / parse_label_format: same names, formats
//   and errors as the reference (maps are compacted before writing):
//     raw   "CCLM", version byte 1, width, height (u32 LE), W*H u32 LE labels
//     csv   one line per row, comma-separated, LF endings
//     pgm16 P5 with 16-bit big-endian samples; std::overflow_error past 65535
//   label_to_cclm (additive): the GPU path straight to a CCLM file — label,
//   compact on the device, and stream the compacted labels to the file in
//   chunks so the device->host copy of one chunk overlaps the write of the last.
#pragma once

#include <cstdint>
#include <optional>
#include <string>

#include "ccl/errors.hpp"
#include "ccl/image.hpp"
#include "ccl/pipeline.hpp"

namespace ccl {

enum class LabelMapFormat { raw, csv, pgm16 };

LabelMapFormat parse_label_format(const std::string& s);  // std::invalid_argument on unknown names

void write_label_map(const LabelMap& lm, const std::string& path, LabelMapFormat format);

LabelMap read_label_map(const std::string& path);  // compacted map from a CCLM file

// Per-block counter grids ("iterations", then "atomics", one CSV row per block
// row) and the summary row width,height,block_w,block_h,density,variant,
// mean_iterations,mean_atomics,wall_ms (density empty when unknown; no summary
// row for an empty report) -- reference label_io.hpp / label_io.cpp:97-128.
void write_metrics_csv(const RunReport& report, const std::string& path,
                       std::optional<double> density = std::nullopt);

// Labels `img` on the calling thread's GPU and writes the compacted map as a
// CCLM file; returns the number of components K.
std::uint64_t label_to_cclm(const BinaryImage& img, const std::string& path, Variant variant = Variant::C2FL);

}  // namespace ccl
