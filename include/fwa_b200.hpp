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
#include <map>
#include <memory>
#include <mutex>
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

    // Uploads params (FWAP records, kernels.hpp:151-175, and the optional input projection,
    // backbone.hpp:74-81) when they differ from the resident ones, then runs the backbone.
    // The input projection (backbone.hpp:179-190) runs on the device, bit-exact.
    backbone::BackboneOutput run(const geometry::PillarSet& pillars, const backbone::FwaConfig& cfg,
                                 const backbone::BackboneParams& params) {
        const fwa_config_t cc = upload(cfg, params);
        check_width(pillars, cfg, params);
        const std::size_t n = pillars.size();
        std::vector<double> coords(2 * n);
        for (std::size_t i = 0; i < n; ++i) {
            coords[2 * i] = pillars.coords[i][0];
            coords[2 * i + 1] = pillars.coords[i][1];
        }
        Frame fr(pillars, cfg);
        throw_status(fwa_b200_backbone_forward(ctx_.get(), coords.data(), pillars.features.data.data(), 1,
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
            check_width(p, cfg, params);
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
        // BackboneParams::input_proj (backbone.hpp:74-81): resident on the device as well
        std::vector<float> pr;
        if (params.input_proj) {
            const auto& p = *params.input_proj;
            pr.push_back(static_cast<float>(p.weight.rows));
            pr.push_back(static_cast<float>(p.weight.cols));
            pr.insert(pr.end(), p.weight.data.begin(), p.weight.data.end());
            pr.insert(pr.end(), p.bias.begin(), p.bias.end());
        }
        if (pr != proj_) {
            if (params.input_proj) {
                const auto& p = *params.input_proj;
                if (p.weight.rows != static_cast<std::size_t>(cfg.d_model) ||
                    (!p.bias.empty() && p.bias.size() != p.weight.rows))
                    throw fwa::shape_error("backbone: input projection shape mismatch");
                throw_status(fwa_b200_load_input_proj(ctx_.get(), static_cast<int32_t>(p.weight.rows),
                                                      static_cast<int32_t>(p.weight.cols), p.weight.data.data(),
                                                      p.bias.empty() ? nullptr : p.bias.data()),
                             fwa_b200_last_error(ctx_.get()));
            } else {
                throw_status(fwa_b200_load_input_proj(ctx_.get(), 0, 0, nullptr, nullptr),
                             fwa_b200_last_error(ctx_.get()));
            }
            proj_ = pr;
        }
        return cc;
    }

    // backbone.hpp:179-194: the projection's width, or d_model without one
    static void check_width(const geometry::PillarSet& p, const backbone::FwaConfig& cfg,
                            const backbone::BackboneParams& params) {
        if (params.input_proj) {
            if (params.input_proj->weight.cols != p.features.cols)
                throw fwa::shape_error("backbone: input projection width mismatch");
        } else if (p.features.cols != static_cast<std::size_t>(cfg.d_model)) {
            throw fwa::shape_error("backbone: pillar width != d_model and no input projection");
        }
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
            o = fwa_output_t{};
            o.features = out.features.data.data();
            o.kept_indices = kept.data();
            o.dropped_ids = dropped.data();
            o.dropped_per_block = dpb.data();
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
            // StageTimes (backbone.hpp:109-126): device time per stage of this call
            out.stats.stages.sort_ms = o.stage_ms[FWA_STAGE_SORT];
            out.stats.stages.group_ms = o.stage_ms[FWA_STAGE_GROUP];
            out.stats.stages.gather_ms = o.stage_ms[FWA_STAGE_GATHER];
            out.stats.stages.attention_ms = o.stage_ms[FWA_STAGE_ATTENTION];
            out.stats.stages.ffn_ms = o.stage_ms[FWA_STAGE_FFN];
            out.stats.stages.scatter_ms = o.stage_ms[FWA_STAGE_SCATTER];
            return std::move(out);
        }
    };

    struct Del {
        void operator()(fwa_b200_ctx* c) const { fwa_b200_ctx_destroy(c); }
    };
    std::unique_ptr<fwa_b200_ctx, Del> ctx_;
    std::string blob_;
    std::vector<float> proj_;
};

// Same signature as fwa::backbone::run_backbone; n_threads is accepted for API
// parity (the GPU result does not depend on it).  One context per device (the caller's
// current CUDA device), created on first use and reused; concurrent callers on one device
// are serialised on its mutex (the reference function is reentrant), callers on
// different devices run concurrently.
inline backbone::BackboneOutput run_backbone(const geometry::PillarSet& pillars,
                                             const backbone::FwaConfig& cfg,
                                             const backbone::BackboneParams& params,
                                             int n_threads = 1) {
    (void)n_threads;
    struct Slot {
        std::mutex m;
        std::unique_ptr<Backbone> bb;
    };
    static std::mutex registry_m;
    static std::map<int, std::unique_ptr<Slot>> registry;
    const int dev = fwa_b200_current_device();
    Slot* slot;
    {
        std::lock_guard<std::mutex> g(registry_m);
        auto& p = registry[dev];
        if (!p) p = std::make_unique<Slot>();
        slot = p.get();
    }
    std::lock_guard<std::mutex> g(slot->m);
    if (!slot->bb) slot->bb = std::make_unique<Backbone>(dev);
    return slot->bb->run(pillars, cfg, params);
}

// Seed overload (backbone.hpp:328-334).
inline backbone::BackboneOutput run_backbone(const geometry::PillarSet& pillars,
                                             const backbone::FwaConfig& cfg, std::uint64_t seed,
                                             int n_threads = 1) {
    return ::fwa::b200::run_backbone(  // qualified: no ADL into fwa::backbone
        pillars, cfg, backbone::init_backbone_params(cfg, pillars.features.cols, seed), n_threads);
}

} // namespace fwa::b200
