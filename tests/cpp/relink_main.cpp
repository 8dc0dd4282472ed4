// relink_main.cpp — proves INTEGRATION.md §1: reference-side code compiled
// against THIS repo's include/ (ccl/image.hpp, pipeline.hpp, forest.hpp,
// label_io.hpp, errors.hpp, generate.hpp first on the include path; the
// reference's own include/ supplies the headers this repo does not ship, e.g.
// ccl/oracle.hpp) and linked with libccl_b200.so.  oracle/Makefile builds it
// together with the reference's UNMODIFIED proj/src/oracle.cpp and
// proj/src/label_io.cpp (namespace ccl, no renaming) into oracle/_ref/relink_test.
//
// Exercises what the reference CLI touches (proj/tools/ccl.cpp run_label /
// run_verify): label_image (now on the GPU), sequential_ccl (reference
// oracle.cpp), compact_labels, write_label_map / read_label_map /
// write_metrics_csv (reference label_io.cpp), and the forest.hpp primitives.
// `--no-gpu` skips the labeling calls (the container that builds it has no GPU).
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>

#include "ccl/forest.hpp"
#include "ccl/generate.hpp"
#include "ccl/label_io.hpp"
#include "ccl/oracle.hpp"
#include "ccl/pipeline.hpp"

static int fails = 0;
#define CHECK(c)                                                    \
    do {                                                            \
        if (!(c)) {                                                 \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
            ++fails;                                                \
        }                                                           \
    } while (0)

int main(int argc, char** argv) {
    const bool gpu = !(argc > 1 && std::strcmp(argv[1], "--no-gpu") == 0);
    const std::string dir = argc > 2 ? argv[2] : "/tmp";

    // forest.hpp (reference forest.hpp:44-111 semantics)
    ccl::LabelForest f(8);
    ccl::BlockMetrics m;
    ccl::merge(f, 5, 3, m);
    ccl::merge(f, 7, 5, m);
    ccl::merge(f, 6, 2, m);
    CHECK(ccl::find_root(f, 7, m) == 3 && ccl::find_root(f, 6, m) == 2 && f.is_root(0));
    ccl::flatten(f, 7, m);
    CHECK(f.parent(7) == 3 && m.atomic_ops == 3 && m.findroot_iterations > 0);

    const ccl::BinaryImage img = ccl::random_image(777, 513, 0.55, 17);
    const ccl::LabelMap want = ccl::sequential_ccl(img);  // reference oracle.cpp
    ccl::RunReport rep;
    if (gpu) {
        rep = ccl::label_image(img, ccl::BlockConfig{}, ccl::Variant::C2FL, 4);
        CHECK(rep.label_map.labels == want.labels);
        CHECK(rep.per_block.size() == std::size_t(rep.blocks_x) * rep.blocks_y);
    } else {
        rep.label_map = want;
        rep.blocks_x = rep.blocks_y = 1;
        rep.per_block.resize(1);
    }
    // reference label_io.cpp against this repo's label_io.hpp / errors.hpp
    const std::string raw = dir + "/relink_test.cclm", csv = dir + "/relink_test_metrics.csv";
    ccl::write_label_map(rep.label_map, raw, ccl::parse_label_format("raw"));
    const ccl::LabelMap back = ccl::read_label_map(raw);
    CHECK(back.compacted && back.labels == ccl::compact_labels(want).labels);
    ccl::write_metrics_csv(rep, csv, 0.55);
    bool threw = false;
    try {
        (void)ccl::read_label_map(dir + "/does_not_exist.cclm");
    } catch (const ccl::IoError&) {
        threw = true;
    }
    CHECK(threw);
    threw = false;
    try {
        (void)ccl::label_image(img, ccl::BlockConfig{0, 0}, ccl::Variant::C2FL, 1);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    CHECK(threw);
    std::remove(raw.c_str());
    std::remove(csv.c_str());
    if (fails == 0) std::printf("RELINK OK (%s)\n", gpu ? "gpu" : "no-gpu");
    return fails ? 1 : 0;
}
