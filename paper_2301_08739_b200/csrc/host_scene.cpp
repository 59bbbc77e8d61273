// Host-side synthetic input generators, bit-identical to the reference's
// (paths relative to /root/reference/proj):
//
//   DetRng                 include/fwa/rng.hpp:12-52   (pinned std::mt19937_64, hand-rolled
//                                                       uniform / Box-Muller normal)
//   generate_synthetic     include/fwa/geometry.hpp:355-386
//   random_pillar_params   include/fwa/geometry.hpp:71-79
//   pillarize              include/fwa/geometry.hpp:246-300 (cells in lexicographic
//                          (x-cell, y-cell) order, pairwise mean in ingestion order,
//                          linear + exact-erf GELU in fp64)
//   init_backbone_params   include/fwa/backbone.hpp:83-102 + init_attn_params
//                          include/fwa/kernels.hpp:116-130, serialised as FWAP records
//                          (kernels.hpp:149-175)
//
// These sit upstream of the drop-in boundary: they make
// the pillars-in / params-in inputs that both the GPU path and the reference
// consume.  Compiled with -ffp-contract=off (fp64 rounding must match).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#include "fwa_b200.h"

namespace fwa_b200 {

class DetRng {
public:
    explicit DetRng(uint64_t seed) : eng_(seed) {}
    uint64_t next_u64() { return eng_(); }
    double uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    uint64_t uniform_int(uint64_t n) { return next_u64() % n; }
    double normal() {
        if (has_spare_) {
            has_spare_ = false;
            return spare_;
        }
        const double u1 = (static_cast<double>(next_u64() >> 11) + 1.0) * 0x1.0p-53;
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double theta = 2.0 * 3.14159265358979323846 * u2;
        spare_ = r * std::sin(theta);
        has_spare_ = true;
        return r * std::cos(theta);
    }
    double normal(double mean, double sd) { return mean + sd * normal(); }

private:
    std::mt19937_64 eng_;
    double spare_ = 0.0;
    bool has_spare_ = false;
};

static double pairwise_sum(const double* v, size_t n) {
    if (n == 0) return 0.0;
    if (n <= 8) {
        double s = 0.0;
        for (size_t i = 0; i < n; ++i) s += v[i];
        return s;
    }
    const size_t h = n / 2;
    return pairwise_sum(v, h) + pairwise_sum(v + h, n - h);
}

static double gelu64(double x) {
    return 0.5 * x * (1.0 + std::erf(x / 1.4142135623730951));
}

struct Cloud {
    std::vector<double> x, y, f; // f: n x f_in
    int f_in = 0;
};

static Cloud generate_synthetic(const fwa_scene_spec_t& s, uint64_t seed) {
    DetRng rng(seed);
    Cloud pc;
    pc.f_in = s.f_in;
    const double hx = s.extent_x / 2.0, hy = s.extent_y / 2.0;
    auto emit = [&](double x, double y) {
        pc.x.push_back(x);
        pc.y.push_back(y);
        for (int c = 0; c < s.f_in; ++c) pc.f.push_back(rng.normal());
    };
    for (int c = 0; c < s.n_clusters; ++c) {
        const double cx = rng.uniform(-hx, hx);
        const double cy = rng.uniform(-hy, hy);
        const uint64_t span =
            static_cast<uint64_t>(s.points_per_cluster_max - s.points_per_cluster_min + 1);
        const int count = s.points_per_cluster_min + static_cast<int>(rng.uniform_int(span));
        for (int i = 0; i < count; ++i) {
            // The reference writes emit(cx + sigma*normal(), cy + sigma*normal());
            // g++ (x86-64 SysV) evaluates those arguments right to left, so the
            // y draw comes first.  Pinned against the reference in tests/test_host.py.
            const double py = cy + s.cluster_sigma * rng.normal();
            const double px = cx + s.cluster_sigma * rng.normal();
            emit(px, py);
        }
    }
    for (int i = 0; i < s.n_background; ++i) {
        const double py = rng.uniform(-hy, hy); // same right-to-left order
        const double px = rng.uniform(-hx, hx);
        emit(px, py);
    }
    return pc;
}

} // namespace fwa_b200

using namespace fwa_b200;

// FNV-1a-64 (bench.hpp:62-72): the `fwa attend` feature_hash over the f32 feature bytes
extern "C" uint64_t fwa_b200_fnv1a64(const void* bytes, size_t n) {
    const unsigned char* p = static_cast<const unsigned char*>(bytes);
    uint64_t h = 0xcbf29ce484222325ull;
    for (size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

extern "C" int64_t fwa_b200_generate_points(const fwa_scene_spec_t* spec, uint64_t seed, double* xy,
                                            double* feats) {
    if (!spec) return -FWA_ERR_CONFIG;
    const auto& s = *spec;
    if (s.extent_x <= 0.0 || s.extent_y <= 0.0 || s.n_clusters < 0 || s.n_background < 0 ||
        s.points_per_cluster_min < 1 || s.points_per_cluster_max < s.points_per_cluster_min ||
        s.cluster_sigma < 0.0 || s.f_in < 0)
        return -FWA_ERR_CONFIG;
    const Cloud pc = generate_synthetic(s, seed);
    const size_t n = pc.x.size();
    if (xy) {
        for (size_t i = 0; i < n; ++i) {
            xy[2 * i] = pc.x[i];
            xy[2 * i + 1] = pc.y[i];
        }
        if (feats) std::copy(pc.f.begin(), pc.f.end(), feats);
    }
    return static_cast<int64_t>(n);
}

extern "C" int64_t fwa_b200_pillar_params(int32_t f_in, int32_t d_out, uint64_t seed, double* weight) {
    if (f_in < 0 || d_out < 1) return -FWA_ERR_CONFIG;
    // random_pillar_params (geometry.hpp:71-79): weight d_out x f_in ~ N(0, 0.5^2), bias 0
    DetRng prng(seed);
    const size_t k = static_cast<size_t>(d_out) * static_cast<size_t>(f_in);
    for (size_t i = 0; i < k; ++i) weight[i] = prng.normal(0.0, 0.5);
    return static_cast<int64_t>(k);
}

extern "C" int64_t fwa_b200_generate_pillars(const fwa_scene_spec_t* spec, uint64_t seed,
                                             double resolution, int32_t d_out,
                                             uint64_t param_seed, double* coords, double* feats) {
    if (!spec) return -FWA_ERR_CONFIG;
    const auto& s = *spec;
    if (s.extent_x <= 0.0 || s.extent_y <= 0.0 || s.n_clusters < 0 || s.n_background < 0 ||
        s.points_per_cluster_min < 1 || s.points_per_cluster_max < s.points_per_cluster_min ||
        s.cluster_sigma < 0.0 || s.f_in < 0)
        return -FWA_ERR_CONFIG;
    if (resolution <= 0.0 || d_out < 1) return -FWA_ERR_CONFIG;
    const Cloud pc = generate_synthetic(s, seed);
    const size_t n = pc.x.size();
    // cells, lexicographic order, members in ingestion order (std::map semantics)
    std::vector<int64_t> cx(n), cy(n);
    for (size_t i = 0; i < n; ++i) {
        cx[i] = static_cast<int64_t>(std::floor(pc.x[i] / resolution));
        cy[i] = static_cast<int64_t>(std::floor(pc.y[i] / resolution));
    }
    std::vector<size_t> order(n);
    std::iota(order.begin(), order.end(), size_t(0));
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
        if (cx[a] != cx[b]) return cx[a] < cx[b];
        return cy[a] < cy[b];
    });
    int64_t n_cells = 0;
    for (size_t i = 0; i < n; ++i)
        if (i == 0 || cx[order[i]] != cx[order[i - 1]] || cy[order[i]] != cy[order[i - 1]]) ++n_cells;
    if (!coords) return n_cells;

    // random_pillar_params(f_in, d_out, param_seed): weight d_out x f_in ~ N(0, 0.5^2)
    DetRng prng(param_seed);
    std::vector<double> w(static_cast<size_t>(d_out) * static_cast<size_t>(s.f_in));
    for (auto& v : w) v = prng.normal(0.0, 0.5);

    std::vector<double> channel, pooled(static_cast<size_t>(s.f_in));
    int64_t row = 0;
    for (size_t i = 0; i < n;) {
        size_t j = i;
        while (j < n && cx[order[j]] == cx[order[i]] && cy[order[j]] == cy[order[i]]) ++j;
        const size_t m = j - i;
        for (int c = 0; c < s.f_in; ++c) {
            channel.resize(m);
            for (size_t k = 0; k < m; ++k)
                channel[k] = pc.f[order[i + k] * static_cast<size_t>(s.f_in) + static_cast<size_t>(c)];
            pooled[static_cast<size_t>(c)] = pairwise_sum(channel.data(), m) / static_cast<double>(m);
        }
        for (int o = 0; o < d_out; ++o) {
            double acc = 0.0; // bias is zero (geometry.hpp:77)
            const double* wr = w.data() + static_cast<size_t>(o) * static_cast<size_t>(s.f_in);
            for (int c = 0; c < s.f_in; ++c) acc += wr[c] * pooled[static_cast<size_t>(c)];
            feats[row * d_out + o] = gelu64(acc);
        }
        coords[2 * row] = (static_cast<double>(cx[order[i]]) + 0.5) * resolution;
        coords[2 * row + 1] = (static_cast<double>(cy[order[i]]) + 0.5) * resolution;
        ++row;
        i = j;
    }
    return n_cells;
}

// init_backbone_params(cfg, f_in, seed) (backbone.hpp:83-102): when f_in != d_model the
// input projection (d_model x f_in ~ N(0, 0.1^2), bias 0) is drawn first, then the blocks
extern "C" int64_t fwa_b200_init_params_fin(const fwa_config_t* cfg, int32_t f_in, uint64_t seed, void* out,
                                            size_t cap, float* proj_weight) {
    if (!cfg) return -FWA_ERR_CONFIG;
    const int d = cfg->d_model, h = cfg->n_heads, f = cfg->d_ff;
    if (cfg->resolution <= 0.0 || cfg->window_px < 1 || cfg->window_py < 1 ||
        cfg->group_size < 1 || cfg->n_blocks < 1 || d < 4 || d % 4 != 0 || h < 1 || d % h != 0 ||
        f < 1)
        return -FWA_ERR_CONFIG;
    const size_t n_floats = static_cast<size_t>(3 * d * d + 3 * d + d * d + d + 4 * d + f * d + f +
                                                d * f + d);
    const size_t rec = 16 + 4 * n_floats;
    const size_t total = rec * static_cast<size_t>(cfg->n_blocks);
    if (!out) return static_cast<int64_t>(total);
    if (cap < total) return -FWA_ERR_CONFIG;
    if (f_in < 0) return -FWA_ERR_SHAPE;
    DetRng rng(seed);
    if (f_in != d) {  // backbone.hpp:89-96
        if (!proj_weight) return -FWA_ERR_SHAPE;
        for (int i = 0; i < d * f_in; ++i) proj_weight[i] = static_cast<float>(rng.normal(0.0, 0.1));
    }
    uint8_t* p = static_cast<uint8_t*>(out);
    for (int b = 0; b < cfg->n_blocks; ++b) {
        std::memcpy(p, "FWAP", 4);
        const uint32_t dims[3] = {static_cast<uint32_t>(d), static_cast<uint32_t>(h),
                                  static_cast<uint32_t>(f)};
        std::memcpy(p + 4, dims, 12);
        std::vector<float> t(n_floats, 0.0f);
        float* w_qkv = t.data();
        float* w_out = w_qkv + 3 * d * d + 3 * d;
        float* ln1_g = w_out + d * d + d;
        float* ln2_g = ln1_g + 2 * d;
        float* w1 = ln2_g + 2 * d;
        float* w2 = w1 + f * d + f;
        // init_attn_params fill order: w_qkv, w_out, ffn_w1, ffn_w2 ~ N(0, 0.02^2)
        for (int i = 0; i < 3 * d * d; ++i) w_qkv[i] = static_cast<float>(rng.normal(0.0, 0.02));
        for (int i = 0; i < d * d; ++i) w_out[i] = static_cast<float>(rng.normal(0.0, 0.02));
        for (int i = 0; i < f * d; ++i) w1[i] = static_cast<float>(rng.normal(0.0, 0.02));
        for (int i = 0; i < d * f; ++i) w2[i] = static_cast<float>(rng.normal(0.0, 0.02));
        for (int i = 0; i < d; ++i) ln1_g[i] = 1.0f;
        for (int i = 0; i < d; ++i) ln2_g[i] = 1.0f;
        std::memcpy(p + 16, t.data(), 4 * n_floats);
        p += rec;
    }
    return static_cast<int64_t>(total);
}

extern "C" int64_t fwa_b200_init_params(const fwa_config_t* cfg, uint64_t seed, void* out, size_t cap) {
    return fwa_b200_init_params_fin(cfg, cfg ? cfg->d_model : 0, seed, out, cap, nullptr);
}
