// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (header-only C++20,
// /root/reference/proj/include/fwa/*.hpp).  `oracle/Makefile` compiles this
// file against the reference headers where they lie and writes the result to
// oracle/_ref/libfwa_ref.so.  Nothing from the reference is copied here; every
// function below only marshals plain pointers into the reference's own API:
//
//   fwa::geometry::generate_synthetic / pillarize / random_pillar_params
//       (proj/include/fwa/geometry.hpp:355-386, 246-300, 71-79)
//   fwa::backbone::init_backbone_params / run_backbone
//       (proj/include/fwa/backbone.hpp:83-102, 159-325)
//   fwa::kernels::save_params / fwa_block_forward / positional_embedding
//       (proj/include/fwa/kernels.hpp:151-175, 636-650, 364-393)
//   fwa::flatten::sort / block_schedule (proj/include/fwa/flatten.hpp:97-120, 150-161)
//   fwa::oracle::oracle_sort (proj/include/fwa/oracle.hpp:35-61)
//
// Status codes mirror the reference error taxonomy (proj/include/fwa/error.hpp:11-33)
// with the same numbering the product C-ABI uses (include/fwa_b200.h).

#include <cstdint>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "fwa/backbone.hpp"
#include "fwa/bench.hpp"
#include "fwa/flatten.hpp"
#include "fwa/geometry.hpp"
#include "fwa/kernels.hpp"
#include "fwa/oracle.hpp"

using namespace fwa;

namespace {

thread_local std::string g_err;

template <class Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const config_error& e) {
        g_err = e.what();
        return 1;
    } catch (const parse_error& e) {
        g_err = e.what();
        return 2;
    } catch (const schema_error& e) {
        g_err = e.what();
        return 3;
    } catch (const shape_error& e) {
        g_err = e.what();
        return 4;
    } catch (const numeric_error& e) {
        g_err = e.what();
        return 5;
    } catch (const contract_error& e) {
        g_err = e.what();
        return 6;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 7;
    }
}

struct CfgC {
    double resolution;
    int32_t window_px, window_py, group_size, n_blocks, d_model, n_heads, d_ff;
};

backbone::FwaConfig to_cfg(const CfgC* c) {
    backbone::FwaConfig cfg;
    cfg.resolution = c->resolution;
    cfg.window_px = c->window_px;
    cfg.window_py = c->window_py;
    cfg.group_size = c->group_size;
    cfg.n_blocks = c->n_blocks;
    cfg.d_model = c->d_model;
    cfg.n_heads = c->n_heads;
    cfg.d_ff = c->d_ff;
    return cfg;
}

struct PillarsHandle {
    geometry::PillarSet ps;
};

std::vector<kernels::AttnParams<float>> parse_blob(const void* blob, size_t len) {
    std::string bytes(static_cast<const char*>(blob), len);
    std::istringstream in(bytes);
    std::vector<kernels::AttnParams<float>> out;
    while (in.peek() != std::char_traits<char>::eof()) out.push_back(kernels::load_params(in));
    return out;
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// generate_synthetic(spec, seed) -> pillarize(cloud, resolution, random_pillar_params(f_in, d_out, param_seed))
void* ref_make_pillars(int n_clusters, int ppc_min, int ppc_max, double sigma, double ext_x,
                       double ext_y, int n_background, int f_in, uint64_t seed,
                       double resolution, int d_out, uint64_t param_seed, int64_t* n_out) {
    auto* h = new PillarsHandle;
    int rc = guarded([&] {
        geometry::SceneSpec s;
        s.n_clusters = n_clusters;
        s.points_per_cluster_min = ppc_min;
        s.points_per_cluster_max = ppc_max;
        s.cluster_sigma = sigma;
        s.extent_x = ext_x;
        s.extent_y = ext_y;
        s.n_background = n_background;
        s.f_in = f_in;
        const auto cloud = geometry::generate_synthetic(s, seed);
        h->ps = geometry::pillarize(
            cloud, resolution,
            geometry::random_pillar_params(static_cast<std::size_t>(f_in),
                                           static_cast<std::size_t>(d_out), param_seed));
    });
    if (rc != 0) {
        delete h;
        *n_out = -rc;
        return nullptr;
    }
    *n_out = static_cast<int64_t>(h->ps.size());
    return h;
}

void ref_pillars_get(void* handle, double* coords, double* feats) {
    auto* h = static_cast<PillarsHandle*>(handle);
    for (std::size_t i = 0; i < h->ps.size(); ++i) {
        coords[2 * i] = h->ps.coords[i][0];
        coords[2 * i + 1] = h->ps.coords[i][1];
    }
    std::memcpy(feats, h->ps.features.data.data(), h->ps.features.data.size() * sizeof(double));
}

void ref_pillars_free(void* handle) { delete static_cast<PillarsHandle*>(handle); }

// Raw point cloud of generate_synthetic (x, y, f0..f_{k-1} per point).
int64_t ref_generate_points(int n_clusters, int ppc_min, int ppc_max, double sigma, double ext_x,
                            double ext_y, int n_background, int f_in, uint64_t seed,
                            double* out, int64_t cap) {
    int64_t n = -1;
    int rc = guarded([&] {
        geometry::SceneSpec s{n_clusters, ppc_min, ppc_max, sigma, ext_x, ext_y, n_background, f_in};
        const auto cloud = geometry::generate_synthetic(s, seed);
        n = static_cast<int64_t>(cloud.size());
        if (out && n <= cap) {
            const std::size_t stride = 2 + static_cast<std::size_t>(f_in);
            for (std::size_t i = 0; i < cloud.size(); ++i) {
                out[i * stride] = cloud.points[i].x;
                out[i * stride + 1] = cloud.points[i].y;
                for (int c = 0; c < f_in; ++c) out[i * stride + 2 + c] = cloud.points[i].feature[c];
            }
        }
    });
    return rc ? -rc : n;
}

// `fwa attend` output-contract pieces (tools/fwa_cli.cpp:71-73, 204-241; bench.hpp:62-72):
// the config JSON (nlohmann dump) and its FNV-1a digest, FNV-1a of arbitrary bytes, and
// the point-file writers (geometry.hpp:202-237) for the ingest parity tests.
int64_t ref_config_json(const CfgC* c, char* out, int64_t cap) {
    int64_t n = -1;
    int rc = guarded([&] {
        const std::string s = nlohmann::json(to_cfg(c)).dump();
        n = static_cast<int64_t>(s.size());
        if (out && n < cap) std::memcpy(out, s.c_str(), s.size() + 1);
    });
    return rc ? -rc : n;
}

// bench.hpp:75-143 (percentile, 3x IQR exclusion, summarize) for the `fwa bench` protocol
// parity: out = {mean, p50, p95, outliers_excluded}
int ref_bench_summarize(const double* samples, int64_t n, int runs, int warmup, double* out4) {
    return guarded([&] {
        const std::vector<double> v(samples, samples + n);
        const auto r = bench::summarize("x", 0, "", v, runs, warmup);
        out4[0] = r.mean_ms;
        out4[1] = r.p50_ms;
        out4[2] = r.p95_ms;
        out4[3] = r.outliers_excluded;
    });
}

void ref_fnv1a64_hex(const void* bytes, int64_t n, char* out19) {
    const std::string h = bench::fnv1a64_hex(std::string(static_cast<const char*>(bytes), static_cast<size_t>(n)));
    std::memcpy(out19, h.c_str(), h.size() + 1);
}

int ref_write_points(int n_clusters, int ppc_min, int ppc_max, double sigma, double ext_x, double ext_y,
                     int n_background, int f_in, uint64_t seed, const char* path, int binary) {
    return guarded([&] {
        geometry::SceneSpec s{n_clusters, ppc_min, ppc_max, sigma, ext_x, ext_y, n_background, f_in};
        const auto cloud = geometry::generate_synthetic(s, seed);
        std::ofstream f(path, binary ? std::ios::binary : std::ios::out);
        if (binary) geometry::write_binary(f, cloud);
        else geometry::write_csv(f, cloud);
    });
}

// init_backbone_params(cfg, f_in, seed) serialised as back-to-back FWAP records.
// Returns the blob length (call with out=nullptr to size).
int64_t ref_init_params_fwap(const CfgC* c, int64_t f_in, uint64_t seed, void* out, int64_t cap) {
    int64_t len = -1;
    int rc = guarded([&] {
        const auto p = backbone::init_backbone_params(to_cfg(c), static_cast<std::size_t>(f_in), seed);
        std::ostringstream os;
        for (const auto& b : p.blocks) kernels::save_params(os, b);
        const std::string s = os.str();
        len = static_cast<int64_t>(s.size());
        if (out && len <= cap) std::memcpy(out, s.data(), s.size());
    });
    return rc ? -rc : len;
}

// Zero-weight params (kernels::zero_attn_params) for the identity checks.
int64_t ref_zero_params_fwap(const CfgC* c, void* out, int64_t cap) {
    int64_t len = -1;
    int rc = guarded([&] {
        std::ostringstream os;
        for (int b = 0; b < c->n_blocks; ++b)
            kernels::save_params(os, kernels::zero_attn_params<float>(c->d_model, c->n_heads, c->d_ff));
        const std::string s = os.str();
        len = static_cast<int64_t>(s.size());
        if (out && len <= cap) std::memcpy(out, s.data(), s.size());
    });
    return rc ? -rc : len;
}

// run_backbone on (coords, f64 feats). Outputs are caller-allocated with
// capacity N (features N*d_model, kept N, dropped N, dropped_per_block n_blocks).
namespace {
void run_marshal(const double* coords, const double* feats, int64_t n, int64_t d_in, const CfgC* c,
                 const backbone::BackboneParams& params, int n_threads, float* out_feats, int32_t* out_kept,
                 int64_t* out_n_kept, int32_t* out_dropped, int32_t* out_dropped_per_block, int32_t* out_cache,
                 double* out_stage_ms) {
    geometry::PillarSet ps;
    ps.resolution = c->resolution;
    ps.coords.resize(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) ps.coords[i] = {coords[2 * i], coords[2 * i + 1]};
    ps.features = Dense2<double>(static_cast<std::size_t>(n), static_cast<std::size_t>(d_in));
    std::memcpy(ps.features.data.data(), feats, static_cast<std::size_t>(n * d_in) * sizeof(double));
    const auto out = backbone::run_backbone(ps, to_cfg(c), params, n_threads);
    *out_n_kept = static_cast<int64_t>(out.kept_indices.size());
    if (out_feats) std::memcpy(out_feats, out.features.data.data(), out.features.data.size() * sizeof(float));
    if (out_kept)
        for (std::size_t i = 0; i < out.kept_indices.size(); ++i) out_kept[i] = out.kept_indices[i];
    std::size_t w = 0;
    for (std::size_t b = 0; b < out.dropped_indices.size(); ++b) {
        if (out_dropped_per_block) out_dropped_per_block[b] = static_cast<int32_t>(out.dropped_indices[b].size());
        for (const int id : out.dropped_indices[b])
            if (out_dropped) out_dropped[w++] = id;
    }
    if (out_cache) {
        out_cache[0] = out.stats.cache.computed;
        out_cache[1] = out.stats.cache.hits;
    }
    if (out_stage_ms) {
        const auto& s = out.stats.stages;
        out_stage_ms[0] = s.sort_ms;
        out_stage_ms[1] = s.group_ms;
        out_stage_ms[2] = s.gather_ms;
        out_stage_ms[3] = s.attention_ms;
        out_stage_ms[4] = s.ffn_ms;
        out_stage_ms[5] = s.scatter_ms;
    }
}
}  // namespace

int ref_run_backbone(const double* coords, const double* feats, int64_t n, int64_t d_in,
                     const CfgC* c, const void* blob, int64_t blob_len, int n_threads,
                     float* out_feats, int32_t* out_kept, int64_t* out_n_kept,
                     int32_t* out_dropped, int32_t* out_dropped_per_block, int32_t* out_cache,
                     double* out_stage_ms) {
    return guarded([&] {
        backbone::BackboneParams params;
        params.blocks = parse_blob(blob, static_cast<std::size_t>(blob_len));
        run_marshal(coords, feats, n, d_in, c, params, n_threads, out_feats, out_kept, out_n_kept, out_dropped,
                    out_dropped_per_block, out_cache, out_stage_ms);
    });
}

// The seed overload (backbone.hpp:328-334): init_backbone_params(cfg, d_in, seed), which
// draws the input projection when d_in != d_model, then run_backbone.  proj_weight_out
// (d_model x d_in, may be null) receives the drawn projection weight.
int ref_run_backbone_seeded(const double* coords, const double* feats, int64_t n, int64_t d_in, const CfgC* c,
                            uint64_t seed, int n_threads, float* out_feats, int32_t* out_kept, int64_t* out_n_kept,
                            int32_t* out_dropped, int32_t* out_dropped_per_block, int32_t* out_cache,
                            float* proj_weight_out) {
    return guarded([&] {
        const auto params = backbone::init_backbone_params(to_cfg(c), static_cast<std::size_t>(d_in), seed);
        if (proj_weight_out && params.input_proj)
            std::memcpy(proj_weight_out, params.input_proj->weight.data.data(),
                        params.input_proj->weight.data.size() * sizeof(float));
        run_marshal(coords, feats, n, d_in, c, params, n_threads, out_feats, out_kept, out_n_kept, out_dropped,
                    out_dropped_per_block, out_cache, nullptr);
    });
}

// Replays the per-block plans run_backbone computes internally: block b's
// permutation (local indices into that block's active list), re-derived with
// flatten::sort on the compacted active coordinates exactly as
// backbone.hpp:215-316 does.  perms_out: n_blocks x n (row b holds n_active_b
// entries); n_active_out[b] = n_active at block b.
int ref_block_plans(const double* coords, int64_t n, const CfgC* c, int32_t* perms_out,
                    int32_t* n_active_out) {
    return guarded([&] {
        const auto cfg = to_cfg(c);
        backbone::validate(cfg);
        std::vector<std::array<double, 2>> cur(static_cast<std::size_t>(n));
        for (int64_t i = 0; i < n; ++i) cur[i] = {coords[2 * i], coords[2 * i + 1]};
        const auto schedule = flatten::block_schedule(cfg.n_blocks, cfg.window_x_m(), cfg.window_y_m());
        for (int b = 0; b < cfg.n_blocks; ++b) {
            if (cur.size() < static_cast<std::size_t>(cfg.group_size))
                throw numeric_error("fewer active pillars than group size");
            const auto plan = flatten::sort(cur, schedule[static_cast<std::size_t>(b)]);
            const auto grouping = flatten::group(plan, cfg.group_size);
            n_active_out[b] = static_cast<int32_t>(cur.size());
            for (std::size_t i = 0; i < plan.permutation.size(); ++i)
                perms_out[static_cast<std::size_t>(b) * static_cast<std::size_t>(n) + i] = plan.permutation[i];
            if (!grouping.dropped.empty()) {
                std::vector<bool> keep(cur.size(), true);
                for (const int l : grouping.dropped) keep[static_cast<std::size_t>(l)] = false;
                std::vector<std::array<double, 2>> nxt;
                for (std::size_t i = 0; i < cur.size(); ++i)
                    if (keep[i]) nxt.push_back(cur[i]);
                cur = std::move(nxt);
            }
        }
    });
}

int ref_sort(const double* coords, int64_t n, double w_x, double w_y, int shift, int axis_y,
             int32_t* perm_out) {
    return guarded([&] {
        std::vector<std::array<double, 2>> cs(static_cast<std::size_t>(n));
        for (int64_t i = 0; i < n; ++i) cs[i] = {coords[2 * i], coords[2 * i + 1]};
        flatten::WindowSpec spec;
        spec.w_x = w_x;
        spec.w_y = w_y;
        spec.shift = shift != 0;
        spec.major_axis = axis_y ? flatten::Axis::Y : flatten::Axis::X;
        const auto plan = flatten::sort(cs, spec);
        std::memcpy(perm_out, plan.permutation.data(), plan.permutation.size() * sizeof(int));
    });
}

int ref_oracle_sort(const double* coords, int64_t n, double w_x, double w_y, int shift, int axis_y,
                    int32_t* perm_out) {
    return guarded([&] {
        std::vector<std::array<double, 2>> cs(static_cast<std::size_t>(n));
        for (int64_t i = 0; i < n; ++i) cs[i] = {coords[2 * i], coords[2 * i + 1]};
        flatten::WindowSpec spec;
        spec.w_x = w_x;
        spec.w_y = w_y;
        spec.shift = shift != 0;
        spec.major_axis = axis_y ? flatten::Axis::Y : flatten::Axis::X;
        const auto perm = oracle::oracle_sort(cs, spec);
        std::memcpy(perm_out, perm.data(), perm.size() * sizeof(int));
    });
}

// Eq. 1 key of one point (flatten::make_sort_key), for golden key vectors.
void ref_sort_key(double x, double y, double w_x, double w_y, int shift, int axis_y,
                  int64_t* win, double* loc) {
    flatten::WindowSpec spec;
    spec.w_x = w_x;
    spec.w_y = w_y;
    spec.shift = shift != 0;
    spec.major_axis = axis_y ? flatten::Axis::Y : flatten::Axis::X;
    const auto k = flatten::make_sort_key({x, y}, 0, spec);
    win[0] = k.win_major;
    win[1] = k.win_minor;
    loc[0] = k.loc_major;
    loc[1] = k.loc_minor;
}

int ref_positional_embedding(const double* coords, int64_t n, int d_model, float* out) {
    return guarded([&] {
        std::vector<std::array<double, 2>> cs(static_cast<std::size_t>(n));
        for (int64_t i = 0; i < n; ++i) cs[i] = {coords[2 * i], coords[2 * i + 1]};
        const auto pe = kernels::positional_embedding<float>(cs, d_model);
        std::memcpy(out, pe.data.data(), pe.data.size() * sizeof(float));
    });
}

// fwa_block_forward(f, pe, params(one FWAP record), n_groups) in f32.
int ref_block_forward(const float* f, const float* pe, int64_t rows, int64_t d, int n_groups,
                      const void* blob, int64_t blob_len, int n_threads, float* out) {
    return guarded([&] {
        const auto params = parse_blob(blob, static_cast<std::size_t>(blob_len));
        if (params.size() != 1) throw config_error("expected exactly one FWAP record");
        Dense2<float> F(static_cast<std::size_t>(rows), static_cast<std::size_t>(d));
        Dense2<float> P(static_cast<std::size_t>(rows), static_cast<std::size_t>(d));
        std::memcpy(F.data.data(), f, F.data.size() * sizeof(float));
        std::memcpy(P.data.data(), pe, P.data.size() * sizeof(float));
        const auto o = kernels::fwa_block_forward(F, P, params[0], n_groups, static_cast<kernels::FwaBlockCache<float>*>(nullptr), n_threads);
        std::memcpy(out, o.data.data(), o.data.size() * sizeof(float));
    });
}

// fwa_block_forward with a cache, then fwa_block_backward (kernels.hpp:636-765): the input
// gradient (rows x d) and the parameter gradients serialised as one FWAP record.
int64_t ref_block_backward(const float* f, const float* pe, int64_t rows, int64_t d, int n_groups,
                           const void* blob, int64_t blob_len, const float* grad_out, float* grad_f,
                           void* grad_blob, int64_t cap) {
    int64_t len = -1;
    int rc = guarded([&] {
        const auto params = parse_blob(blob, static_cast<std::size_t>(blob_len));
        if (params.size() != 1) throw config_error("expected exactly one FWAP record");
        Dense2<float> F(static_cast<std::size_t>(rows), static_cast<std::size_t>(d));
        Dense2<float> P(static_cast<std::size_t>(rows), static_cast<std::size_t>(d));
        Dense2<float> G(static_cast<std::size_t>(rows), static_cast<std::size_t>(d));
        std::memcpy(F.data.data(), f, F.data.size() * sizeof(float));
        std::memcpy(P.data.data(), pe, P.data.size() * sizeof(float));
        std::memcpy(G.data.data(), grad_out, G.data.size() * sizeof(float));
        kernels::FwaBlockCache<float> cache;
        kernels::fwa_block_forward(F, P, params[0], n_groups, &cache, 1);
        const auto gr = kernels::fwa_block_backward(G, cache, params[0]);
        std::memcpy(grad_f, gr.grad_f.data.data(), gr.grad_f.data.size() * sizeof(float));
        std::ostringstream os;
        kernels::save_params(os, gr.params);
        const std::string sp = os.str();
        len = static_cast<int64_t>(sp.size());
        if (grad_blob && len <= cap) std::memcpy(grad_blob, sp.data(), sp.size());
    });
    return rc ? -rc : len;
}

// f64 dense-oracle attention + unfused FFN (oracle.hpp:90-173, 205-228).
int ref_oracle_block(const double* f, const double* pe, int64_t rows, int64_t d, int n_groups,
                     const void* blob, int64_t blob_len, double* out) {
    return guarded([&] {
        const auto params = parse_blob(blob, static_cast<std::size_t>(blob_len));
        const auto p64 = params.at(0).cast<double>();
        Dense2<double> F(static_cast<std::size_t>(rows), static_cast<std::size_t>(d));
        Dense2<double> P(static_cast<std::size_t>(rows), static_cast<std::size_t>(d));
        std::memcpy(F.data.data(), f, F.data.size() * sizeof(double));
        std::memcpy(P.data.data(), pe, P.data.size() * sizeof(double));
        const auto a = oracle::oracle_attention(F, P, p64, n_groups);
        const auto o = oracle::oracle_unfused_ffn(a, p64);
        std::memcpy(out, o.data.data(), o.data.size() * sizeof(double));
    });
}

} // extern "C"
