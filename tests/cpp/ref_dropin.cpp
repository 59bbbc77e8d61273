// Drop-in check: the reference's own caller-side code, with fwa::backbone::run_backbone
// swapped for fwa::b200::run_backbone (include/fwa_b200.hpp).  Built by
// oracle/Makefile (target ref_dropin) against the UNMODIFIED reference headers; run by
// tests/test_gpu_integration.py on the GPU box.  Prints one JSON line.
#include <cmath>
#include <cstdio>
#include <thread>
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
    bool empty_numeric = false;
    try {  // an EMPTY PillarSet is the same numeric_error (backbone.hpp:218-222), not a shape error
        geometry::PillarSet empty;
        empty.features = Dense2<double>(0, 128);
        b200::run_backbone(empty, cfg, params);
    } catch (const fwa::numeric_error&) {
        empty_numeric = true;
    }
    // bench_group (bench.hpp:222-241) reads RunStats.stages after every run
    const auto& st = got.stats.stages;
    const bool stages_ok = st.sort_ms > 0 && st.group_ms > 0 && st.attention_ms > 0 && st.ffn_ms > 0 &&
                           st.gather_ms >= 0 && st.scatter_ms >= 0 && st.total() > 0;
    // BackboneParams::input_proj (backbone.hpp:74-81, 179-190): 16-wide pillars, the seed
    // initialiser draws the projection; the b200 path projects on the device
    const auto pillars16 = geometry::pillarize(cloud, 0.32, geometry::random_pillar_params(2, 16, 42));
    const auto params16 = backbone::init_backbone_params(cfg, 16, 9);
    const auto want16 = backbone::run_backbone(pillars16, cfg, params16, 4);
    const auto got16 = b200::run_backbone(pillars16, cfg, params16, 4);
    double pa = 0, pr = 0;
    for (std::size_t i = 0; i < want16.features.data.size(); ++i) {
        pa = std::fmax(pa, std::fabs(double(got16.features.data[i]) - double(want16.features.data[i])));
        pr = std::fmax(pr, std::fabs(double(want16.features.data[i])));
    }
    const bool proj_ok = params16.input_proj.has_value() && got16.kept_indices == want16.kept_indices &&
                         got16.dropped_indices == want16.dropped_indices && pa / pr <= 1e-2;
    bool width_shape_error = false;
    try {  // a projection whose width differs from the pillars' -> shape_error, as the reference
        b200::run_backbone(pillars, cfg, params16);
    } catch (const fwa::shape_error&) {
        width_shape_error = true;
    }
    // concurrent callers of the free function on one device: serialised, same results
    std::vector<backbone::BackboneOutput> par(2);
    {
        std::thread t0([&] { par[0] = b200::run_backbone(pillars, cfg, params, 1); });
        std::thread t1([&] { par[1] = b200::run_backbone(pillars16, cfg, params16, 1); });
        t0.join();
        t1.join();
    }
    const bool concurrent_ok = par[0].features.data == got.features.data &&
                               par[1].features.data == got16.features.data;
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
                "\"cache\": [%d, %d], \"stream_equal\": %s, \"empty_numeric_error\": %s, "
                "\"stages_ms\": [%.4f, %.4f, %.4f, %.4f, %.4f, %.4f], \"stages_ok\": %s, "
                "\"proj_rel_err\": %.3e, \"proj_ok\": %s, \"proj_width_shape_error\": %s, "
                "\"concurrent_ok\": %s}\n",
                pillars.size(), got.kept_indices.size(), ints ? "true" : "false", max_abs / max_ref,
                threw ? "true" : "false", got.stats.cache.computed, got.stats.cache.hits,
                stream_equal ? "true" : "false", empty_numeric ? "true" : "false", st.sort_ms, st.group_ms,
                st.gather_ms, st.attention_ms, st.ffn_ms, st.scatter_ms, stages_ok ? "true" : "false", pa / pr,
                proj_ok ? "true" : "false", width_shape_error ? "true" : "false", concurrent_ok ? "true" : "false");
    return ints && threw && stream_equal && max_abs / max_ref <= 1e-2 && empty_numeric && stages_ok && proj_ok &&
                   width_shape_error && concurrent_ok
               ? 0
               : 1;
}
