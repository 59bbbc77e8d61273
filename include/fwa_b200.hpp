// fwa_b200.hpp — drop-in C++ binding of the B200 backbone for callers of the
// reference library (/root/reference/proj/include/fwa).  Header-only; compiles
// against the reference's own types and forwards to the C ABI in fwa_b200.h.
//
//   fwa::b200::run_backbone(pillars, cfg, params, n_threads)
//       == fwa::backbone::run_backbone (backbone.hpp:159-325), same arguments,
//          same BackboneOutput (features in active order, coords, kept_indices,
//          dropped_indices per block, stats.cache / stats.dropped_per_block),
//          same exception taxonomy (error.hpp:11-33).
//
// A caller such as cmd_attend (tools/fwa_cli.cpp:195-243) or bench_group
// (bench.hpp:215-242) switches by replacing `fwa::backbone::run_backbone` with
// `fwa::b200::run_backbone` and linking libfwa_b200.so.
#pragma once

#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "fwa/backbone.hpp"
#include "fwa/error.hpp"
#include "fwa/kernels.hpp"
#include "fwa_b200.h"

namespace fwa::b200 {

inline void throw_status(int rc, const char* msg) {
    const std::string m = msg ? msg : "";
    switch (rc) {
        case FWA_OK: return;
        case FWA_ERR_CONFIG: throw fwa::config_error(m);
        case FWA_ERR_PARSE: throw fwa::parse_error(m);
        case FWA_ERR_SCHEMA: throw fwa::schema_error(m);
        case FWA_ERR_SHAPE: throw fwa::shape_error(m);
        case FWA_ERR_NUMERIC: throw fwa::numeric_error(m);
        case FWA_ERR_CONTRACT: throw fwa::contract_error(m);
        default: throw std::runtime_error("fwa_b200: " + m);
    }
}

inline fwa_config_t to_c(const backbone::FwaConfig& c) {
    return fwa_config_t{c.resolution, c.window_px, c.window_py, c.group_size,
                        c.n_blocks,   c.d_model,   c.n_heads,   c.d_ff};
}

// One device context (stream + HBM workspace + resident parameters).
class Backbone {
public:
    explicit Backbone(int device = 0, bool fp32_check_mode = false) {
        fwa_b200_ctx* c = nullptr;
        const int rc = fwa_b200_ctx_create(device, nullptr, &c);
        if (rc != FWA_OK) throw_status(rc, "fwa_b200_ctx_create failed");
        ctx_.reset(c);
        if (fp32_check_mode) throw_status(fwa_b200_set_precision(c, FWA_PREC_FP32), nullptr);
    }

    // Uploads params (FWAP records, kernels.hpp:151-175) when they differ from the
    // resident ones, then runs the backbone.
    backbone::BackboneOutput run(const geometry::PillarSet& pillars, const backbone::FwaConfig& cfg,
                                 const backbone::BackboneParams& params) {
        const fwa_config_t cc = upload(cfg, params);
        const std::size_t n = pillars.size();
        const std::size_t d = static_cast<std::size_t>(cfg.d_model);
        // Optional input projection (backbone.hpp:179-190): a host GEMV per pillar in
        // the reference's order; never used on the north-star path (f_in == d_model).
        std::vector<float> proj;
        const void* feats = pillars.features.data.data();
        int f64 = 1;
        if (params.input_proj) {
            const auto& pr = *params.input_proj;
            if (pr.weight.cols != pillars.features.cols)
                throw fwa::shape_error("backbone: input projection width mismatch");
            proj.resize(n * d);
            for (std::size_t r = 0; r < n; ++r)
                for (std::size_t j = 0; j < d; ++j) {
                    float acc = pr.bias[j];
                    const float* w = pr.weight.row(j);
                    for (std::size_t c = 0; c < pr.weight.cols; ++c)
                        acc += w[c] * static_cast<float>(pillars.features(r, c));
                    proj[r * d + j] = acc;
                }
            feats = proj.data();
            f64 = 0;
        } else if (pillars.features.cols != d) {
            throw fwa::shape_error("backbone: pillar width != d_model and no input projection");
        }
        std::vector<double> coords(2 * n);
        for (std::size_t i = 0; i < n; ++i) {
            coords[2 * i] = pillars.coords[i][0];
            coords[2 * i + 1] = pillars.coords[i][1];
        }
        Frame fr(pillars, cfg);
        throw_status(fwa_b200_backbone_forward(ctx_.get(), coords.data(), feats, f64,
                                               static_cast<int64_t>(n), &cc, &fr.o),
                     fwa_b200_last_error(ctx_.get()));
        return fr.finish(pillars, cfg);
    }

    // A sequence of frames, each exactly run(frames[i], cfg, params), with the PCIe copies of
    // neighbouring frames pipelined against the compute (fwa_b200_backbone_forward_frames).
    std::vector<backbone::BackboneOutput> run_frames(const std::vector<geometry::PillarSet>& frames,
                                                     const backbone::FwaConfig& cfg,
                                                     const backbone::BackboneParams& params) {
        std::vector<backbone::BackboneOutput> outs;
        if (params.input_proj) {  // host projection per frame: no streaming to gain
            for (const auto& f : frames) outs.push_back(run(f, cfg, params));
            return outs;
        }
        const fwa_config_t cc = upload(cfg, params);
        const std::size_t d = static_cast<std::size_t>(cfg.d_model);
        std::vector<std::vector<double>> coords(frames.size());
        std::vector<Frame> fr;
        fr.reserve(frames.size());
        std::vector<const double*> cp(frames.size());
        std::vector<const void*> fp(frames.size());
        std::vector<int64_t> ns(frames.size());
        std::vector<fwa_output_t> os(frames.size());
        for (std::size_t i = 0; i < frames.size(); ++i) {
            const auto& p = frames[i];
            if (p.features.cols != d) throw fwa::shape_error("backbone: pillar width != d_model and no input projection");
            coords[i].resize(2 * p.size());
            for (std::size_t j = 0; j < p.size(); ++j) {
                coords[i][2 * j] = p.coords[j][0];
                coords[i][2 * j + 1] = p.coords[j][1];
            }
            fr.emplace_back(p, cfg);
            cp[i] = coords[i].data();
            fp[i] = p.features.data.data();
            ns[i] = static_cast<int64_t>(p.size());
            os[i] = fr.back().o;
        }
        throw_status(fwa_b200_backbone_forward_frames(ctx_.get(), static_cast<int>(frames.size()), cp.data(), fp.data(),
                                                      1, ns.data(), &cc, os.data()),
                     fwa_b200_last_error(ctx_.get()));
        for (std::size_t i = 0; i < frames.size(); ++i) {
            fr[i].o = os[i];
            outs.push_back(fr[i].finish(frames[i], cfg));
        }
        return outs;
    }

private:
    // params -> FWAP records (kernels.hpp:151-175), uploaded when they differ from the resident ones
    fwa_config_t upload(const backbone::FwaConfig& cfg, const backbone::BackboneParams& params) {
        backbone::validate(cfg);
        const fwa_config_t cc = to_c(cfg);
        std::ostringstream os;
        for (const auto& b : params.blocks) kernels::save_params(os, b);
        const std::string blob = os.str();
        if (blob != blob_) {
            throw_status(fwa_b200_load_params(ctx_.get(), &cc, blob.data(), blob.size()),
                         fwa_b200_last_error(ctx_.get()));
            blob_ = blob;
        }
        return cc;
    }

    // one frame's output buffers and the BackboneOutput rebuilt from them
    struct Frame {
        backbone::BackboneOutput out;
        std::vector<int32_t> kept, dropped, dpb;
        fwa_output_t o{};
        Frame(const geometry::PillarSet& p, const backbone::FwaConfig& cfg)
            : kept(p.size()), dropped(p.size() ? p.size() : 1), dpb(static_cast<std::size_t>(cfg.n_blocks)) {
            out.n_input = p.size();
            out.features = Dense2<float>(p.size(), static_cast<std::size_t>(cfg.d_model));
            o = fwa_output_t{out.features.data.data(), kept.data(), dropped.data(), dpb.data(), nullptr, 0, 0, 0};
        }
        Frame(Frame&&) = default;
        backbone::BackboneOutput finish(const geometry::PillarSet& pillars, const backbone::FwaConfig& cfg) {
            const std::size_t d = static_cast<std::size_t>(cfg.d_model);
            const std::size_t k = static_cast<std::size_t>(o.n_kept);
            out.features.rows = k;
            out.features.data.resize(k * d);
            out.kept_indices.assign(kept.begin(), kept.begin() + static_cast<std::ptrdiff_t>(k));
            out.coords.reserve(k);
            for (std::size_t i = 0; i < k; ++i) out.coords.push_back(pillars.coords[static_cast<std::size_t>(kept[i])]);
            std::size_t w = 0;
            for (int b = 0; b < cfg.n_blocks; ++b) {
                const std::size_t m = static_cast<std::size_t>(dpb[static_cast<std::size_t>(b)]);
                out.dropped_indices.emplace_back(dropped.begin() + static_cast<std::ptrdiff_t>(w),
                                                 dropped.begin() + static_cast<std::ptrdiff_t>(w + m));
                out.stats.dropped_per_block.push_back(static_cast<int>(m));
                w += m;
            }
            out.stats.cache.computed = o.cache_computed;
            out.stats.cache.hits = o.cache_hits;
            return std::move(out);
        }
    };

    struct Del {
        void operator()(fwa_b200_ctx* c) const { fwa_b200_ctx_destroy(c); }
    };
    std::unique_ptr<fwa_b200_ctx, Del> ctx_;
    std::string blob_;
};

// Same signature as fwa::backbone::run_backbone; n_threads is accepted for API
// parity (the GPU result does not depend on it).  One context per device, reused.
inline backbone::BackboneOutput run_backbone(const geometry::PillarSet& pillars,
                                             const backbone::FwaConfig& cfg,
                                             const backbone::BackboneParams& params,
                                             int n_threads = 1) {
    (void)n_threads;
    static Backbone device0(0);
    return device0.run(pillars, cfg, params);
}

// Seed overload (backbone.hpp:328-334).
inline backbone::BackboneOutput run_backbone(const geometry::PillarSet& pillars,
                                             const backbone::FwaConfig& cfg, std::uint64_t seed,
                                             int n_threads = 1) {
    return ::fwa::b200::run_backbone(  // qualified: no ADL into fwa::backbone
        pillars, cfg, backbone::init_backbone_params(cfg, pillars.features.cols, seed), n_threads);
}

} // namespace fwa::b200
