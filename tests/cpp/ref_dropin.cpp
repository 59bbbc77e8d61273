// Drop-in check: the reference's own caller-side code, with fwa::backbone::run_backbone
// swapped for fwa::b200::run_backbone (include/fwa_b200.hpp).  Built by
// oracle/Makefile (target ref_dropin) against the UNMODIFIED reference headers; run by
// tests/test_gpu_integration.py on the GPU box.  Prints one JSON line.
#include <cmath>
#include <cstdio>
#include <vector>

#include "fwa/backbone.hpp"
#include "fwa/geometry.hpp"
#include "fwa_b200.hpp"

int main() {
    using namespace fwa;
    // tests/test_backbone.cpp-style fixture: clustered scene -> pillarize at 0.32 m
    geometry::SceneSpec spec{6, 200, 300, 2.0, 60.0, 60.0, 500, 2};
    const auto cloud = geometry::generate_synthetic(spec, 42);
    const auto pillars = geometry::pillarize(cloud, 0.32, geometry::random_pillar_params(2, 128, 42));
    backbone::FwaConfig cfg;  // defaults: 0.32 m, 9x9, G 69, 8 blocks, D 128, H 8, D_ff 256
    const auto params = backbone::init_backbone_params(cfg, 128, 7);
    const auto want = backbone::run_backbone(pillars, cfg, params, 4);
    const auto got = b200::run_backbone(pillars, cfg, params, 4);
    double max_abs = 0, max_ref = 0;
    for (std::size_t i = 0; i < want.features.data.size(); ++i) {
        max_abs = std::fmax(max_abs, std::fabs(double(got.features.data[i]) - double(want.features.data[i])));
        max_ref = std::fmax(max_ref, std::fabs(double(want.features.data[i])));
    }
    const bool ints = got.kept_indices == want.kept_indices && got.dropped_indices == want.dropped_indices &&
                      got.coords == want.coords && got.stats.cache.computed == want.stats.cache.computed &&
                      got.stats.cache.hits == want.stats.cache.hits &&
                      got.stats.dropped_per_block == want.stats.dropped_per_block;
    bool threw = false;
    try {  // error taxonomy: fewer pillars than the group size -> numeric_error
        geometry::PillarSet tiny;
        tiny.coords = {{0.16, 0.16}, {0.48, 0.16}};
        tiny.features = Dense2<double>(2, 128);
        b200::run_backbone(tiny, cfg, params);
    } catch (const fwa::numeric_error&) {
        threw = true;
    }
    // a frame sequence through the streamed entry point: each output == its own single call
    std::vector<geometry::PillarSet> frames;
    for (std::uint64_t sd : {43ull, 44ull, 45ull})
        frames.push_back(geometry::pillarize(geometry::generate_synthetic(spec, sd), 0.32,
                                             geometry::random_pillar_params(2, 128, sd)));
    b200::Backbone dev(0);
    const auto outs = dev.run_frames(frames, cfg, params);
    bool stream_equal = outs.size() == frames.size();
    for (std::size_t i = 0; stream_equal && i < frames.size(); ++i) {
        const auto one = dev.run(frames[i], cfg, params);
        stream_equal = outs[i].features.data == one.features.data && outs[i].kept_indices == one.kept_indices &&
                       outs[i].dropped_indices == one.dropped_indices && outs[i].coords == one.coords &&
                       outs[i].stats.dropped_per_block == one.stats.dropped_per_block;
    }
    std::printf("{\"n\": %zu, \"n_kept\": %zu, \"ints_equal\": %s, \"rel_err\": %.3e, \"numeric_error\": %s, "
                "\"cache\": [%d, %d], \"stream_equal\": %s}\n",
                pillars.size(), got.kept_indices.size(), ints ? "true" : "false", max_abs / max_ref,
                threw ? "true" : "false", got.stats.cache.computed, got.stats.cache.hits,
                stream_equal ? "true" : "false");
    return ints && threw && stream_equal && max_abs / max_ref <= 1e-2 ? 0 : 1;
}
