// dropin_test.cpp — code written against the reference C++ API
// (proj/include/ccl/pipeline.hpp:33-34) compiled unchanged against this
// library's headers, checked against the unmodified reference labeler
// (oracle/_ref/libccl_ref.so, test infrastructure, via its C adapter).
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

#include "ccl/generate.hpp"
#include "ccl/image.hpp"
#include "ccl/pipeline.hpp"

extern "C" int ref_label_image(const std::uint8_t*, std::uint32_t, std::uint32_t, std::uint32_t, std::uint32_t, int,
                               unsigned, std::uint32_t*, double*);

static int fails = 0;
#define CHECK(c)                                                  \
    do {                                                          \
        if (!(c)) {                                               \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
            ++fails;                                              \
        }                                                         \
    } while (0)

int main() {
    struct Case { std::uint32_t w, h; double d; std::uint64_t seed; };
    const Case cases[] = {{512, 512, 0.5, 0}, {97, 131, 0.3, 1}, {1, 1, 1.0, 2}, {1000, 37, 0.62, 3},
                          {2048, 2048, 0.7, 4}, {1920, 1080, 0.5, 5}};
    const ccl::Variant vs[] = {ccl::Variant::C2FL, ccl::Variant::RC2FL, ccl::Variant::CC2FL, ccl::Variant::NC2FL};
    for (const auto& c : cases) {
        const ccl::BinaryImage img = ccl::random_image(c.w, c.h, c.d, c.seed);
        std::vector<std::uint32_t> want(img.pixel_count());
        double ms = 0;
        CHECK(ref_label_image(img.data.data(), c.w, c.h, 32, 32, 0, 4, want.data(), &ms) == 0);
        for (auto v : vs) {
            ccl::BlockConfig cfg;
            cfg.block_w = 16;
            cfg.block_h = 8;
            const ccl::RunReport rep = ccl::label_image(img, cfg, v, 8);
            CHECK(rep.label_map.labels == want);
            CHECK(rep.blocks_x == (c.w + 15) / 16 && rep.blocks_y == (c.h + 7) / 8);
            CHECK(rep.per_block.size() == std::size_t(rep.blocks_x) * rep.blocks_y);
            CHECK(rep.per_block.empty() || rep.per_block.back().block_id == rep.per_block.size() - 1);
            CHECK(rep.variant == v && rep.worker_count == 8 && !rep.label_map.compacted);
            CHECK(rep.wall_time.count() > 0.0);
        }
        const ccl::LabelMap comp = ccl::compact_labels(ccl::label_image(img, ccl::BlockConfig{}, ccl::Variant::C2FL).label_map);
        CHECK(comp.compacted);
    }
    // error behaviour identical to pipeline.cpp:13-15 / image.hpp:31-33
    const ccl::BinaryImage small(4, 4, 1);
    bool threw = false;
    try { ccl::label_image(small, ccl::BlockConfig{0, 32, 4096}, ccl::Variant::C2FL); } catch (const std::invalid_argument&) { threw = true; }
    CHECK(threw);
    threw = false;
    try { ccl::label_image(small, ccl::BlockConfig{128, 64, 4096}, ccl::Variant::C2FL); } catch (const std::invalid_argument&) { threw = true; }
    CHECK(threw);
    threw = false;
    try { ccl::label_image(small, ccl::BlockConfig{}, ccl::Variant::C2FL, 0); } catch (const std::invalid_argument&) { threw = true; }
    CHECK(threw);
    threw = false;
    try { ccl::label_image(ccl::BinaryImage{}, ccl::BlockConfig{}, ccl::Variant::C2FL); } catch (const std::invalid_argument&) { threw = true; }
    CHECK(threw);
    // concurrent callers on distinct images: one context per thread
    std::vector<std::thread> th;
    std::vector<int> ok(4, 0);
    for (int t = 0; t < 4; ++t)
        th.emplace_back([t, &ok] {
            const ccl::BinaryImage im = ccl::random_image(777, 555, 0.55, 100 + t);
            std::vector<std::uint32_t> w(im.pixel_count());
            double ms;
            ref_label_image(im.data.data(), 777, 555, 32, 32, 0, 1, w.data(), &ms);
            ok[t] = ccl::label_image(im, ccl::BlockConfig{}, ccl::Variant::C2FL).label_map.labels == w;
        });
    for (auto& x : th) x.join();
    for (int t = 0; t < 4; ++t) CHECK(ok[t]);
    // batch entry point
    std::vector<ccl::BinaryImage> frames;
    for (int f = 0; f < 5; ++f) frames.push_back(ccl::random_image(320, 200, 0.5, 50 + f));
    const auto maps = ccl::label_batch(frames);
    for (int f = 0; f < 5; ++f) {
        std::vector<std::uint32_t> w(frames[f].pixel_count());
        double ms;
        ref_label_image(frames[f].data.data(), 320, 200, 32, 32, 0, 1, w.data(), &ms);
        CHECK(maps[f].labels == w);
    }
    // multi-device strips in one process (device 0 listed three times: virtual strips)
    {
        const ccl::BinaryImage im = ccl::random_image(1000, 700, 0.58, 77);
        std::vector<std::uint32_t> w(im.pixel_count());
        double ms;
        ref_label_image(im.data.data(), 1000, 700, 32, 32, 0, 1, w.data(), &ms);
        const ccl::RunReport r = ccl::label_image_strips(im, {0, 0, 0});
        CHECK(r.label_map.labels == w);
        CHECK(r.worker_count == 3);
        bool threw = false;
        try {
            ccl::label_image_strips(im, {});
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
    }
    std::printf(fails ? "dropin_test: %d failures\n" : "dropin_test: OK\n", fails);
    return fails ? 1 : 0;
}
