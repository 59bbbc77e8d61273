// Host driver + C ABI for the B200 FlatFormer backbone forward.
//
// Mirrors fwa::backbone::run_backbone (/root/reference/proj/include/fwa/backbone.hpp:159-325):
// same inputs (pillar centres + features), config fields, FWAP parameters,
// outputs (features in ascending-id active order, kept ids, per-block dropped
// ids in tail order, sort-cache stats) and error taxonomy.
//
// B200-first structure:
//   * the whole index schedule (4 window sorts, groups, drops, kept set) depends
//     only on coordinates, so it is built ONCE per call in one batched device
//     sort (sort.cu) before any feature math; every block then is
//     gather -> LN1+PE -> QKV -> group attention -> out-proj+FFN -> scatter over
//     precomputed index arrays, with the residual stream kept in fp32 in HBM,
//     indexed by pillar id;
//   * the plan-cache statistics the reference reports (computed/hits) are
//     reproduced by simulating its cache rule (backbone.hpp:224-234, 314) on the host;
//   * frames of a batch are concatenated: windows carry the frame id, groups
//     never cross frames, one launch sequence serves all frames.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "fwa_b200.h"
#include "internal.h"

using namespace fwa_b200;

namespace {

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
};

struct StageRec;

struct BlockParams {
    // fp32 tensors (device), FWAP field order
    const float *w_qkv, *b_qkv, *w_out, *b_out, *ln1_g, *ln1_b, *ln2_g, *ln2_b, *w1, *b1, *w2, *b2;
    TcBlockWeights tc{};
};

} // namespace

struct fwa_b200_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    std::string err;
    int precision = FWA_PREC_BF16;
    int64_t launches = 0;
    bool have_params = false;
    fwa_config_t pcfg{};
    DevBuf params_f32, params_bf16;
    std::vector<BlockParams> blocks;
    std::map<std::string, DevBuf> ws;
    int freq_d = 0;
    DevBuf freq;
    cudaStream_t side = nullptr;             // PE overlaps the schedule's host round trip
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaStream_t copy = nullptr;             // host API: feature H2D overlaps the schedule
    cudaEvent_t ev_copy = nullptr, ev_feats = nullptr;
    cudaStream_t d2h = nullptr;              // pipelined frames: outputs back while the next computes
    cudaEvent_t fr_ev[10] = {};
    int* h_fr_flags = nullptr;               // pinned, 2 ints per frame
    size_t h_fr_cap = 0;
    int* d_flag = nullptr;     // [0] non-finite input, [1] window-bin capacity overflow
    int* h_flag = nullptr;     // pinned, 2 ints
    bool exact_bins = false;   // set for one call after an overflow: host-sized bins
    uint64_t ws_epoch = 0;     // bumped whenever a workspace buffer moves
    const void* hist_clean = nullptr;  // sync-free histogram buffer known to be zeroed
    const void* ticket_clean = nullptr;  // key-kernel CTA ticket known to be zeroed
    uint64_t params_version = 0;
    // CUDA graph of the device-resident forward (replayed while its key is unchanged)
    struct GraphKey {
        const void *coords = nullptr, *feats = nullptr, *out = nullptr, *kept = nullptr;
        std::vector<int64_t> off;
        fwa_config_t cfg{};
        int precision = -1;
        uint64_t params_version = 0, ws_epoch = 0;
        bool operator==(const GraphKey& o) const {
            return coords == o.coords && feats == o.feats && out == o.out && kept == o.kept && off == o.off &&
                   std::memcmp(&cfg, &o.cfg, sizeof(cfg)) == 0 && precision == o.precision &&
                   params_version == o.params_version && ws_epoch == o.ws_epoch;
        }
    };
    // a few captured graphs (a double-buffered frame stream alternates two keys), least
    // recently used first out; a key is captured on its second sighting among the last few
    struct GraphEntry {
        GraphKey key;
        cudaGraphExec_t exec = nullptr;
        int64_t launches = 0;
        int64_t* tab = nullptr;  // frame table owned by the captured graph
        uint64_t used = 0;
    };
    static constexpr int kGraphs = 4;
    std::vector<GraphEntry> graphs;
    std::vector<GraphKey> g_seen;  // recent keys run eagerly (at most kGraphs)
    uint64_t g_clock = 0;
    bool g_disabled = false;
    // group-range split of one scene across ranks (BASELINE config 4)
    struct Split {
        bool ready = false;
        fwa_config_t cfg{};
        int64_t ntot = 0, K = 0;
        int32_t *idx = nullptr, *out_pos = nullptr;  // into ws buffers of the last schedule
        float* pe = nullptr;
        __half* pe16 = nullptr;
        bool fast = false;
        uint64_t ws_epoch = 0;
        // peer-memory variant: this rank's group range, per-block rank-tagged scatter rows
        // (n_blocks x rows), device arrays of the 8 peer pointers (x buffers | outputs)
        int world = 0, rank = 0;
        int64_t g0 = 0, g1 = 0;
        int32_t* p2p_sidx = nullptr;
        float** p2p_x = nullptr;
        float** p2p_out = nullptr;
    } split;
    int64_t* h_tab = nullptr;  // pinned frame-table staging (2 slots)
    size_t h_tab_cap = 0;
    int h_tab_slot = 0;
    static constexpr int kTabSlots = 8;  // pinned frame-table staging ring (host run-ahead depth)
    cudaEvent_t ev_tab[kTabSlots] = {};
    long long* h_minmax = nullptr;  // pinned (16)
    // stage profiling (the analogue of the reference's StageTimer, backbone.hpp:139-151)
    bool profiling = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    struct Pending { int slot; cudaEvent_t a, b; };
    std::vector<Pending> pending;
    double prof_ms[FWA_PROF_SLOTS] = {};
    int64_t prof_n[FWA_PROF_SLOTS] = {};
    // BackboneParams::input_proj (backbone.hpp:74-81), resident; proj_in == 0: none
    int proj_in = 0;
    DevBuf proj_w, proj_b;
    bool proj_bias = false;
    // StageTimes of the host-API calls (fwa_output_t::stage_ms): event spans of the call
    // being enqueued (null: not recorded) and the event pool they come from
    StageRec* rec = nullptr;
    std::vector<cudaEvent_t> st_pool;
    size_t st_used = 0;
};

namespace {

struct FwaError {
    int code;
    std::string msg;
};

#define CUDA_OK(expr)                                                                      \
    do {                                                                                   \
        cudaError_t e_ = (expr);                                                           \
        if (e_ != cudaSuccess)                                                             \
            throw FwaError{FWA_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)}; \
    } while (0)

template <class T>
T* ws(fwa_b200_ctx* c, const char* name, size_t count) {
    DevBuf& b = c->ws[name];
    const size_t bytes = std::max<size_t>(count * sizeof(T), 256);
    if (b.cap < bytes) {
        ++c->ws_epoch;  // captured graphs hold the old pointers
        if (b.p) cudaFree(b.p);
        b.p = nullptr;
        size_t want = std::max(bytes, b.cap + b.cap / 2);
        CUDA_OK(cudaMalloc(&b.p, want));
        b.cap = want;
    }
    return static_cast<T*>(b.p);
}

cudaEvent_t prof_event(fwa_b200_ctx* c) {
    if (c->ev_used == c->ev_pool.size()) {
        cudaEvent_t e;
        CUDA_OK(cudaEventCreate(&e));
        c->ev_pool.push_back(e);
    }
    return c->ev_pool[c->ev_used++];
}

// RAII stage timer on the context stream (no-op unless profiling is enabled).
struct StageEv {
    fwa_b200_ctx* c;
    int slot;
    cudaEvent_t a = nullptr;
    StageEv(fwa_b200_ctx* c_, int slot_) : c(c_), slot(slot_) {
        if (c->profiling) {
            a = prof_event(c);
            cudaEventRecord(a, c->stream);
        }
    }
    ~StageEv() {
        if (a) {
            cudaEvent_t b = prof_event(c);
            cudaEventRecord(b, c->stream);
            c->pending.push_back({slot, a, b});
        }
    }
};

void prof_collect(fwa_b200_ctx* c) {
    if (c->pending.empty()) return;
    cudaStreamSynchronize(c->stream);
    for (auto& p : c->pending) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
            c->prof_ms[p.slot] += ms;
            c->prof_n[p.slot] += 1;
        }
    }
    c->pending.clear();
    c->ev_used = 0;
}

// ---- StageTimes (backbone.hpp:109-126) for the host-buffer entry points.  Spans of
// device work between two events on the context stream, per reference stage; a span of
// the fused block kernel (stage -1) is apportioned to gather / attention / ffn / scatter
// by the kernel's per-phase SM-clock sums (block_fused.cu FPH).
struct StageSpan {
    int stage;
    cudaEvent_t a, b;
    int phase_slot;
};
struct StageRec {
    std::vector<StageSpan> spans;
    unsigned long long* d_phase = nullptr;  // n_slots x 4, zeroed when the call starts
    int n_slots = 0, next_slot = 0;
    // the fused blocks of a call share phase slot 0 and ONE event span (set by forward_device):
    // no events between the block launches, whose programmatic dependent launches they
    // would serialise
    bool blocks_whole = false;
    std::vector<unsigned long long> h_phase;
};

cudaEvent_t st_event(fwa_b200_ctx* c) {
    if (c->st_used == c->st_pool.size()) {
        cudaEvent_t e;
        CUDA_OK(cudaEventCreate(&e));
        c->st_pool.push_back(e);
    }
    return c->st_pool[c->st_used++];
}

struct RecSpan {
    fwa_b200_ctx* c;
    StageRec* r;
    int stage, slot;
    cudaEvent_t a = nullptr;
    RecSpan(fwa_b200_ctx* c_, int stage_, int slot_ = -1) : c(c_), r(c_->rec), stage(stage_), slot(slot_) {
        if (r) {
            a = st_event(c);
            cudaEventRecord(a, c->stream);
        }
    }
    ~RecSpan() {
        if (!a) return;
        cudaEvent_t b = st_event(c);
        cudaEventRecord(b, c->stream);
        r->spans.push_back({stage, a, b, slot});
    }
};

// call after the stream work of `r` completed (and r.h_phase was copied back)
void stage_finish(const StageRec& r, double* out) {
    for (int i = 0; i < FWA_STAGES; ++i) out[i] = 0.0;
    for (const auto& sp : r.spans) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, sp.a, sp.b) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        if (sp.stage >= 0) {
            out[sp.stage] += ms;
            continue;
        }
        const unsigned long long* p = r.h_phase.data() + 4 * sp.phase_slot;
        const double tot = static_cast<double>(p[0]) + p[1] + p[2] + p[3];
        if (!(tot > 0)) {
            out[FWA_STAGE_ATTENTION] += ms;
            continue;
        }
        out[FWA_STAGE_GATHER] += ms * (p[0] / tot);
        out[FWA_STAGE_ATTENTION] += ms * (p[1] / tot);
        out[FWA_STAGE_FFN] += ms * (p[2] / tot);
        out[FWA_STAGE_SCATTER] += ms * (p[3] / tot);
    }
}

// record a host-API call's StageTimes: spans on the context stream + the fused kernel's
// phase counters (n_slots blocks); the guard detaches the record on every exit path
struct StageScope {
    fwa_b200_ctx* c;
    StageScope(fwa_b200_ctx* c_, StageRec& r, unsigned long long* d_phase, int n_slots) : c(c_) {
        r.d_phase = d_phase;
        r.n_slots = n_slots;
        r.next_slot = 0;
        CUDA_OK(cudaMemsetAsync(d_phase, 0, static_cast<size_t>(n_slots) * 4 * sizeof(unsigned long long), c->stream));
        c->rec = &r;
    }
    ~StageScope() { c->rec = nullptr; }
};

// FWA_B200_SYNC_DEBUG=1: synchronise after every launch group and name the failing stage.
bool sync_debug() {
    static const bool on = [] {
        const char* v = std::getenv("FWA_B200_SYNC_DEBUG");
        return v && v[0] == '1';
    }();
    return on;
}

void check_launch(const char* what = "kernel launch") {
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess && sync_debug()) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) throw FwaError{FWA_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}

// backbone.hpp:36-47
void validate_cfg(const fwa_config_t* c) {
    if (!c) throw FwaError{FWA_ERR_CONFIG, "config: null"};
    if (!(c->resolution > 0.0)) throw FwaError{FWA_ERR_CONFIG, "config: resolution must be > 0"};
    if (c->window_px < 1 || c->window_py < 1)
        throw FwaError{FWA_ERR_CONFIG, "config: window dims must be >= 1"};
    if (c->group_size < 1) throw FwaError{FWA_ERR_CONFIG, "config: group_size must be >= 1"};
    if (c->n_blocks < 1) throw FwaError{FWA_ERR_CONFIG, "config: n_blocks must be >= 1"};
    if (c->d_model < 4 || c->d_model % 4 != 0)
        throw FwaError{FWA_ERR_CONFIG, "config: d_model must be divisible by 4"};
    if (c->n_heads < 1 || c->d_model % c->n_heads != 0)
        throw FwaError{FWA_ERR_CONFIG, "config: d_model must be divisible by n_heads"};
    if (c->d_ff < 1) throw FwaError{FWA_ERR_CONFIG, "config: d_ff must be >= 1"};
}

bool fast_path_ok(const fwa_b200_ctx* c, int d, int h, int dff, int G) {
    return c->precision != FWA_PREC_FP32 && d == 128 && dff == 256 && h > 0 && d / h == 16 &&
           G >= 1 && G <= 128;
}

size_t record_floats(int d, int dff) {
    return static_cast<size_t>(3 * d * d + 3 * d + d * d + d + 4 * d + dff * d + dff + d * dff + d);
}

struct Record {
    int d, h, dff;
    const float* t;  // host pointer into the blob (may be unaligned -> copied)
};

// FWAP records (kernels.hpp:149-206).  Throws parse_error like load_params.
std::vector<Record> parse_fwap(const void* blob, size_t len, std::vector<std::vector<float>>& keep) {
    std::vector<Record> out;
    const uint8_t* p = static_cast<const uint8_t*>(blob);
    size_t off = 0;
    while (off < len) {
        if (len - off < 4 || std::memcmp(p + off, "FWAP", 4) != 0)
            throw FwaError{FWA_ERR_PARSE, "bad magic, expected FWAP"};
        if (len - off < 16) throw FwaError{FWA_ERR_PARSE, "truncated FWAP header"};
        uint32_t dims[3];
        std::memcpy(dims, p + off + 4, 12);
        const int d = static_cast<int>(dims[0]), h = static_cast<int>(dims[1]), f = static_cast<int>(dims[2]);
        // zero_attn_params -> validate (kernels.hpp:75-90, 92-114)
        if (d < 1 || h < 1 || f < 1) throw FwaError{FWA_ERR_CONFIG, "attn params: dims must be >= 1"};
        if (d % h != 0) throw FwaError{FWA_ERR_CONFIG, "attn params: d_model must be divisible by n_heads"};
        const size_t nf = record_floats(d, f);
        if (len - off - 16 < nf * 4) throw FwaError{FWA_ERR_PARSE, "truncated FWAP tensor"};
        keep.emplace_back(nf);
        std::memcpy(keep.back().data(), p + off + 16, nf * 4);
        out.push_back(Record{d, h, f, keep.back().data()});
        off += 16 + nf * 4;
    }
    return out;
}

__global__ void k_out_pos(const int32_t* __restrict__ idx, const uint32_t* __restrict__ rank,
                          int64_t n, int32_t* __restrict__ out) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r < n) out[r] = static_cast<int32_t>(rank[idx[r]]);
}


// peer-memory split tables.  inv[s][pid] = position of pillar pid in spec s's kept plan
__global__ void k_plan_inverse(const int32_t* __restrict__ idx, int64_t K, int32_t* __restrict__ inv) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k < K) inv[idx[k]] = static_cast<int32_t>(k);
}
// row r of this rank's block-b range: block b < last -> (rank owning the pillar's group in
// block b+1) << 28 | pillar id; the last block -> its output row (rank 0's buffer)
__global__ void k_p2p_rows(const int32_t* __restrict__ plan_b, const int32_t* __restrict__ inv_next,
                           const int32_t* __restrict__ out_pos, int64_t r0, int64_t rows, int64_t chunk, int last,
                           int32_t* __restrict__ sidx) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    if (last) {
        sidx[r] = out_pos[r0 + r];
        return;
    }
    const int32_t pid = plan_b[r0 + r];
    const int32_t dest = static_cast<int32_t>(inv_next[pid] / chunk);
    sidx[r] = (dest << 28) | pid;
}

std::vector<BlockParams> upload_block_params(const std::vector<Record>& recs, DevBuf& pf32,
                                             DevBuf& pbf16, cudaStream_t st) {
    const int d = recs[0].d, dff = recs[0].dff;
    const size_t nf = record_floats(d, dff);
    const size_t nb = recs.size();
    std::vector<float> host(nf * nb);
    for (size_t b = 0; b < nb; ++b) std::memcpy(host.data() + b * nf, recs[b].t, nf * 4);
    const size_t bytes = host.size() * 4;
    if (pf32.cap < bytes) {
        if (pf32.p) cudaFree(pf32.p);
        pf32.p = nullptr;
        CUDA_OK(cudaMalloc(&pf32.p, bytes));
        pf32.cap = bytes;
    }
    CUDA_OK(cudaMemcpyAsync(pf32.p, host.data(), bytes, cudaMemcpyHostToDevice, st));
    const float* base = static_cast<const float*>(pf32.p);
    std::vector<BlockParams> blocks(nb);
    const bool tc = d == 128 && dff == 256;
    const size_t tc_elems = 2 * (384 * 128 + 128 * 128 + 256 * 128 + 128 * 256);  // + pair images
    // per block, after the bf16 images: f32 [b_qkv 384 | b_out 128 | b2 128 | b1' 256]
    constexpr size_t kTcVec = 896, kPairVec = 1152;
    std::vector<uint16_t> sw;
    std::vector<float> tcv, pv;
    if (tc) {
        sw.assign(tc_elems * nb + (kTcVec + kPairVec) * 2 * nb, 0);
        tcv.assign(kTcVec * nb, 0.f);
        pv.assign(kPairVec * nb, 0.f);
        const size_t tb = sw.size() * 2;
        if (pbf16.cap < tb) {
            if (pbf16.p) cudaFree(pbf16.p);
            pbf16.p = nullptr;
            CUDA_OK(cudaMalloc(&pbf16.p, tb));
            pbf16.cap = tb;
        }
    }
    for (size_t b = 0; b < nb; ++b) {
        const float* t = base + b * nf;
        BlockParams& bp = blocks[b];
        bp.w_qkv = t; t += 3 * d * d;
        bp.b_qkv = t; t += 3 * d;
        bp.w_out = t; t += d * d;
        bp.b_out = t; t += d;
        bp.ln1_g = t; t += d;
        bp.ln1_b = t; t += d;
        bp.ln2_g = t; t += d;
        bp.ln2_b = t; t += d;
        bp.w1 = t; t += dff * d;
        bp.b1 = t; t += dff;
        bp.w2 = t; t += d * dff;
        bp.b2 = t;
        if (tc) {
            const float* h = host.data() + b * nf;
            const float* hw_qkv = h;
            const float* hw_out = h + 3 * d * d + 3 * d;
            const float* hw1 = hw_out + d * d + d + 4 * d;
            const float* hw2 = hw1 + dff * d + dff;
            uint16_t* o = sw.data() + b * tc_elems;
            swizzle_weight_bf16(hw_qkv, 384, 128, o);
            swizzle_weight_bf16(hw_out, 128, 128, o + 384 * 128);
            // LN2's affine folded into FFN1 (bf16 fast path only): U = (g*xhat + b) W1^T + b1
            //   = xhat (W1 diag g)^T + (b1 + W1 b)   -- exact in real arithmetic
            const float* hln2g = hw_out + d * d + d + 2 * d;
            const float* hln2b = hln2g + d;
            const float* hb1 = hw1 + dff * d;
            std::vector<float> w1f(static_cast<size_t>(dff) * d);
            for (int j = 0; j < dff; ++j) {
                double acc = hb1[j];
                for (int i = 0; i < d; ++i) {
                    w1f[static_cast<size_t>(j) * d + i] = hw1[static_cast<size_t>(j) * d + i] * hln2g[i];
                    acc += static_cast<double>(hw1[static_cast<size_t>(j) * d + i]) * hln2b[i];
                }
                tcv[b * kTcVec + 640 + j] = static_cast<float>(acc);
            }
            swizzle_weight_bf16(w1f.data(), 256, 128, o + 384 * 128 + 128 * 128);
            for (int i = 0; i < 384; ++i) tcv[b * kTcVec + i] = hw_qkv[3 * d * d + i];           // b_qkv
            for (int i = 0; i < 128; ++i) tcv[b * kTcVec + 384 + i] = hw_out[d * d + i];          // b_out
            for (int i = 0; i < 128; ++i) tcv[b * kTcVec + 512 + i] = hw2[static_cast<size_t>(d) * dff + i];  // b2
            swizzle_weight_bf16(hw2, 128, 256, o + 384 * 128 + 128 * 128 + 256 * 128);
            // fused kernel: LN1's beta into b_qkv (fp64), Q rows scaled to the base-2 exponent
            constexpr double kQScale = 0.25 * 1.4426950408889634;  // block_fused.cu kScaleLog2
            const float* hln1g = hw_out + d * d + d;
            const float* hln1b = hln1g + d;
            std::vector<float> wq(hw_qkv, hw_qkv + 3 * d * d);
            float* pvb = pv.data() + b * kPairVec;
            for (int j = 0; j < 3 * d; ++j) {
                double acc = hw_qkv[3 * d * d + j];
                for (int i = 0; i < d; ++i) acc += static_cast<double>(hw_qkv[static_cast<size_t>(j) * d + i]) * hln1b[i];
                pvb[j] = static_cast<float>(j < d ? acc * kQScale : acc);
            }
            for (size_t i = 0; i < static_cast<size_t>(d) * d; ++i) wq[i] = static_cast<float>(wq[i] * kQScale);
            for (int i = 0; i < 512; ++i) pvb[384 + i] = tcv[b * kTcVec + 384 + i];  // b_out | b2 | b1'
            for (int i = 0; i < d; ++i) pvb[896 + i] = hln1g[i];                      // ln1_g | (beta: 0)
            build_pair_images(wq.data(), hw_out, w1f.data(), hw2, o + tc_elems / 2);
            const __nv_bfloat16* dbase =
                static_cast<const __nv_bfloat16*>(pbf16.p) + b * tc_elems;
            bp.tc.w_qkv = dbase;
            bp.tc.w_out = dbase + 384 * 128;
            bp.tc.w1 = dbase + 384 * 128 + 128 * 128;
            bp.tc.w2 = dbase + 384 * 128 + 128 * 128 + 256 * 128;
            bp.tc.w_pair = reinterpret_cast<const uint8_t*>(dbase + tc_elems / 2);
            const float* vbase = reinterpret_cast<const float*>(
                                     static_cast<const __nv_bfloat16*>(pbf16.p) + tc_elems * nb) +
                                 b * kTcVec;
            bp.tc.vec = vbase;  // b_qkv | b_out | b2 | b1 (LN2-folded)
            bp.tc.vec_pair = reinterpret_cast<const float*>(static_cast<const __nv_bfloat16*>(pbf16.p) + tc_elems * nb +
                                                            kTcVec * 2 * nb) + b * kPairVec;
            bp.tc.ln1_g = bp.ln1_g;
            bp.tc.ln1_b = bp.ln1_b;
        }
    }
    if (tc) {
        std::memcpy(sw.data() + tc_elems * nb, tcv.data(), tcv.size() * 4);
        std::memcpy(sw.data() + tc_elems * nb + kTcVec * 2 * nb, pv.data(), pv.size() * 4);
        CUDA_OK(cudaMemcpyAsync(pbf16.p, sw.data(), sw.size() * 2, cudaMemcpyHostToDevice, st));
    }
    CUDA_OK(cudaStreamSynchronize(st));  // host staging vectors die on return
    return blocks;
}

const double* pe_freq(fwa_b200_ctx* c, int d) {
    if (c->freq_d != d) {
        const int nf = d / 4;
        std::vector<double> f(static_cast<size_t>(nf));
        const double f_min = 1.0 / 10000.0, f_max = 1.0;
        for (int k = 0; k < nf; ++k)  // kernels.hpp:373-377
            f[static_cast<size_t>(k)] =
                nf == 1 ? f_min : f_min * std::pow(f_max / f_min, static_cast<double>(k) / (nf - 1));
        // + the fp16 PE kernel's (hi, lo) float split of 2 f_k
        std::vector<float> f2(2 * static_cast<size_t>(nf));
        for (int k = 0; k < nf; ++k) {
            const double t = 2.0 * f[static_cast<size_t>(k)];
            f2[2 * k] = static_cast<float>(t);
            f2[2 * k + 1] = static_cast<float>(t - static_cast<double>(f2[2 * k]));
        }
        if (c->freq.p) cudaFree(c->freq.p);
        c->freq.p = nullptr;
        CUDA_OK(cudaMalloc(&c->freq.p, f.size() * 16));
        CUDA_OK(cudaMemcpyAsync(c->freq.p, f.data(), f.size() * 8, cudaMemcpyHostToDevice, c->stream));
        CUDA_OK(cudaMemcpyAsync(static_cast<double*>(c->freq.p) + nf, f2.data(), f2.size() * 4,
                                cudaMemcpyHostToDevice, c->stream));
        CUDA_OK(cudaStreamSynchronize(c->stream));
        c->freq_d = d;
    }
    return static_cast<const double*>(c->freq.p);
}

// ------------------------------------------------------------------ schedule

struct Schedule {
    int64_t ntot = 0, K = 0, n_drop = 0;
    int n_frames = 0, n_specs = 0;
    std::vector<int64_t> off, rows, drop, drop_off;
    int32_t* sorted = nullptr;     // n_specs x ntot, full-set plans
    int32_t* sorted_inv = nullptr; // n_specs x ntot, position of each pillar id in its plan
    int32_t* idx = nullptr;        // n_specs x K, kept-restricted plans
    uint8_t* dropped = nullptr;    // ntot
    uint32_t* kept_rank = nullptr; // ntot
    int32_t* kept_ids = nullptr;   // K
    int32_t* dropped_ids = nullptr;
    int32_t* out_pos = nullptr;    // K: output row of the last block's row r
};

void host_frames(const int64_t* off, int n_frames, int G, Schedule& S) {
    S.n_frames = n_frames;
    S.off.assign(off, off + n_frames + 1);
    S.rows.resize(static_cast<size_t>(n_frames));
    S.drop.resize(static_cast<size_t>(n_frames));
    S.drop_off.assign(static_cast<size_t>(n_frames) + 1, 0);
    S.ntot = S.off[static_cast<size_t>(n_frames)];
    S.K = 0;
    for (int f = 0; f < n_frames; ++f) {
        const int64_t n = S.off[f + 1] - S.off[f];
        if (n < 0) throw FwaError{FWA_ERR_SHAPE, "frame offsets must be non-decreasing"};
        if (n < G)  // backbone.hpp:218-222
            throw FwaError{FWA_ERR_NUMERIC, "backbone: block 0 has " + std::to_string(n) +
                                                " pillars, fewer than group size " + std::to_string(G) +
                                                "; refusing to emit empty output"};
        S.rows[f] = (n / G) * G;
        S.drop[f] = n - S.rows[f];
        S.drop_off[f + 1] = S.drop_off[f] + S.drop[f];
        S.K += S.rows[f];
    }
    S.n_drop = S.drop_off[static_cast<size_t>(n_frames)];
    if (S.ntot > INT32_MAX / 4) throw FwaError{FWA_ERR_SHAPE, "too many pillars for int32 ids"};
}

constexpr long long kBinCap = 1LL << 22;  // sync-free histogram capacity (window bins)

// K1..K4 for n_specs specs of nf frames: returns the n_specs x ntot full-set plans.
// Default: fully enqueued (device-side bin ranges, fixed-capacity histogram); an
// overflow sets d_flag[1] and the caller re-runs with exact = true (one host round trip
// to size the histogram exactly).
int32_t* sort_specs(fwa_b200_ctx* c, const double* d_coords, int64_t ntot, int n_specs, double w_x,
                    double w_y, const int64_t* d_off, int nf, bool exact = true) {
    cudaStream_t st = c->stream;
    const int64_t total = ntot * n_specs;
    long long* win = ws<long long>(c, "win", 2 * static_cast<size_t>(total));
    double* loc = ws<double>(c, "loc", 2 * static_cast<size_t>(total));
    long long* mm = ws<long long>(c, "minmax", 16);
    const int64_t n_part = sort_keys_partials(ntot);
    long long* partials = ws<long long>(c, "key_partials", static_cast<size_t>(n_part) * 4 * n_specs);
    if (!exact) {
        SpecBins* d_sb = ws<SpecBins>(c, "specbins", 4 * static_cast<size_t>(nf));
        uint32_t* d_nbins = ws<uint32_t>(c, "nbins", 4);
        unsigned* ticket = ws<unsigned>(c, "sort_ticket", 4);  // [0] key kernel, [1] bin scan
        uint32_t* large = ws<uint32_t>(c, "large_bins", static_cast<size_t>(kBinCap) + 1);
        if (ticket != c->ticket_clean) {  // fresh buffer: zero once; the key kernel resets it
            CUDA_OK(cudaMemsetAsync(ticket, 0, 4 * sizeof(unsigned), st));
            c->ticket_clean = ticket;
        }
        BinsFuse fz;
        fz.ticket = ticket; fz.nf = nf; fz.cap = kBinCap; fz.mm = mm; fz.specs = d_sb; fz.d_nbins = d_nbins;
        fz.overflow = c->d_flag + 1;
        fz.large = large;
        launch_sort_keys(d_coords, ntot, n_specs, w_x, w_y, win, loc, partials, st, &c->launches, fz);
        check_launch();
        uint32_t* hist = ws<uint32_t>(c, "hist", static_cast<size_t>(kBinCap));
        if (hist != c->hist_clean) {  // fresh buffer: zero once; the sort kernels keep it zeroed
            CUDA_OK(cudaMemsetAsync(hist, 0, c->ws["hist"].cap, st));
            c->hist_clean = hist;
        }
        uint32_t* bin_start = ws<uint32_t>(c, "bin_start", static_cast<size_t>(kBinCap));
        uint32_t* cursor = ws<uint32_t>(c, "cursor", static_cast<size_t>(kBinCap));
        uint32_t* tile_sums = ws<uint32_t>(c, "bin_tile_sums", 1024);
        uint32_t* bin_of = ws<uint32_t>(c, "bin_of", static_cast<size_t>(total));
        if (nf > 1) {
            // a batch: every frame's own window range (frames far apart in world coordinates cost
            // no empty bins between them); the union layout of the key kernel's setup is replaced
            long long* mmf = ws<long long>(c, "minmax_frame", 4 * static_cast<size_t>(n_specs) * nf);
            launch_frame_minmax(win, ntot, n_specs, d_off, nf, mmf, st, &c->launches);
            launch_bins_setup_frames(mmf, n_specs, nf, kBinCap, d_sb, d_nbins, c->d_flag + 1, st, &c->launches);
        }
        launch_bins_hist(win, ntot, n_specs, d_off, nf, d_sb, bin_of, hist, d_nbins, st, &c->launches, nf > 1);
        launch_scan_bins_dev(hist, bin_start, cursor, d_nbins, kBinCap, tile_sums, ticket + 1, st, &c->launches);
        int32_t* pre = ws<int32_t>(c, "pre", static_cast<size_t>(total));
        double* pre_loc = ws<double>(c, "pre_loc", 2 * static_cast<size_t>(total));
        uint32_t* pre_bin = ws<uint32_t>(c, "pre_bin", static_cast<size_t>(total));
        launch_bin_scatter(bin_of, loc, ntot, n_specs, cursor, pre, pre_loc, d_nbins, tile_sums, pre_bin, st,
                           &c->launches);
        int32_t* sorted = ws<int32_t>(c, "sorted", static_cast<size_t>(total));
        int32_t* inv = ws<int32_t>(c, "sorted_inv", static_cast<size_t>(total));
        int32_t* scratch = ws<int32_t>(c, "sort_scratch", 2 * static_cast<size_t>(total));
        launch_bin_sort(bin_start, hist, 0u, pre, pre_loc, pre_bin, loc, ntot, n_specs, sorted, inv, scratch,
                        large, d_nbins, tile_sums, st, &c->launches);
        check_launch();
        return sorted;
    }
    // exact path (one host round trip): every frame's own window range per spec, so frames
    // far apart (world coordinates) cost no empty bins; window sets too wide for a dense bin
    // per window (a far outlier) are rank-compressed by a radix sort instead -- any finite
    // coordinates sort exactly
    launch_sort_keys(d_coords, ntot, n_specs, w_x, w_y, win, loc, partials, st, &c->launches);
    check_launch();
    long long* mmf = ws<long long>(c, "minmax_frame", 4 * static_cast<size_t>(n_specs) * nf);
    launch_frame_minmax(win, ntot, n_specs, d_off, nf, mmf, st, &c->launches);
    std::vector<long long> hm(4 * static_cast<size_t>(n_specs) * nf);
    CUDA_OK(cudaMemcpyAsync(hm.data(), mmf, hm.size() * 8, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
    check_launch("window ranges");
    std::vector<SpecBins> sb(static_cast<size_t>(n_specs) * nf);
    double dense = 0.0;
    long long nbins = 0;
    for (int s = 0; s < n_specs; ++s)
        for (int f = 0; f < nf; ++f) {
            const long long* m = &hm[(static_cast<size_t>(s) * nf + f) * 4];
            SpecBins& b = sb[static_cast<size_t>(s) * nf + f];
            if (m[0] > m[1]) {  // empty frame (cannot happen: N >= G >= 1), no bins
                b = SpecBins{0, 0, 1, 0, nbins};
                continue;
            }
            const double rM = static_cast<double>(m[1]) - static_cast<double>(m[0]) + 1.0;
            const double rm = static_cast<double>(m[3]) - static_cast<double>(m[2]) + 1.0;
            dense += rM * rm;
            if (dense < 4.0e18) {
                b = SpecBins{m[0], m[2], static_cast<long long>(rm), static_cast<long long>(rM * rm), nbins};
                nbins += static_cast<long long>(rM * rm);
            }
        }
    const double dense_cap = std::max(static_cast<double>(1 << 22), 2.0 * static_cast<double>(total));
    uint32_t* bin_of = ws<uint32_t>(c, "bin_of", static_cast<size_t>(total));
    uint32_t* hist;
    if (dense <= dense_cap) {
        SpecBins* d_sb = ws<SpecBins>(c, "specbins_frame", sb.size());
        CUDA_OK(cudaMemcpyAsync(d_sb, sb.data(), sb.size() * sizeof(SpecBins), cudaMemcpyHostToDevice, st));
        hist = ws<uint32_t>(c, "hist", static_cast<size_t>(nbins));
        CUDA_OK(cudaMemsetAsync(hist, 0, static_cast<size_t>(nbins) * 4, st));
        launch_bins_hist(win, ntot, n_specs, d_off, nf, d_sb, bin_of, hist, nullptr, st, &c->launches, true);
        CUDA_OK(cudaStreamSynchronize(st));  // sb (host) is read by the copy above
    } else {
        const size_t tot = static_cast<size_t>(total);
        hist = ws<uint32_t>(c, "hist", tot);
        CUDA_OK(cudaMemsetAsync(hist, 0, tot * 4, st));
        const size_t tb = window_ranks_temp_bytes(total);
        uint32_t* d_count = ws<uint32_t>(c, "wr_count", 4);
        launch_window_ranks(win, ntot, n_specs, d_off, nf, ws<unsigned long long>(c, "wr_k64a", tot),
                            ws<unsigned long long>(c, "wr_k64b", tot), ws<uint32_t>(c, "wr_va", tot),
                            ws<uint32_t>(c, "wr_vb", tot), ws<uint32_t>(c, "wr_flag", tot),
                            ws<uint32_t>(c, "wr_ex", tot), ws<uint32_t>(c, "scan_tmp", scan_tmp_words(total) + 8),
                            d_count, ws<uint8_t>(c, "wr_temp", tb), tb, bin_of, hist, st, &c->launches);
        uint32_t cnt = 0;
        CUDA_OK(cudaMemcpyAsync(&cnt, d_count, 4, cudaMemcpyDeviceToHost, st));
        CUDA_OK(cudaStreamSynchronize(st));
        check_launch("window ranks");
        nbins = cnt;
    }
    uint32_t* bin_start = ws<uint32_t>(c, "bin_start", static_cast<size_t>(nbins));
    uint32_t* scan_tmp = ws<uint32_t>(c, "scan_tmp", scan_tmp_words(std::max<int64_t>(nbins, total)) + 8);
    exclusive_scan_u32(hist, bin_start, nbins, scan_tmp, nullptr, st, &c->launches);
    uint32_t* cursor = ws<uint32_t>(c, "cursor", static_cast<size_t>(nbins));
    CUDA_OK(cudaMemcpyAsync(cursor, bin_start, static_cast<size_t>(nbins) * 4, cudaMemcpyDeviceToDevice, st));
    int32_t* pre = ws<int32_t>(c, "pre", static_cast<size_t>(total));
    double* pre_loc = ws<double>(c, "pre_loc", 2 * static_cast<size_t>(total));
    uint32_t* pre_bin = ws<uint32_t>(c, "pre_bin", static_cast<size_t>(total));
    launch_bin_scatter(bin_of, loc, ntot, n_specs, cursor, pre, pre_loc, nullptr, nullptr, pre_bin, st,
                       &c->launches);
    int32_t* sorted = ws<int32_t>(c, "sorted", static_cast<size_t>(total));
    int32_t* inv = ws<int32_t>(c, "sorted_inv", static_cast<size_t>(total));
    int32_t* scratch = ws<int32_t>(c, "sort_scratch", 2 * static_cast<size_t>(total));
    uint32_t* large = ws<uint32_t>(c, "large_bins", static_cast<size_t>(nbins) + 1);
    launch_bin_sort(bin_start, hist, static_cast<uint32_t>(nbins), pre, pre_loc, pre_bin, loc, ntot, n_specs,
                    sorted, inv, scratch, large, nullptr, nullptr, st, &c->launches);
    check_launch();
    return sorted;
}

std::vector<int64_t> frame_table(const Schedule& S) {
    std::vector<int64_t> tab;
    tab.insert(tab.end(), S.off.begin(), S.off.end());
    tab.insert(tab.end(), S.rows.begin(), S.rows.end());
    tab.insert(tab.end(), S.drop_off.begin(), S.drop_off.end() - 1);
    return tab;
}

const int64_t* upload_frame_table(fwa_b200_ctx* c, const Schedule& S) {
    cudaStream_t st = c->stream;
    const int nf = S.n_frames;
    int64_t* d_tab = ws<int64_t>(c, "frame_tab", 3 * static_cast<size_t>(nf) + 2);
    std::vector<int64_t> tab = frame_table(S);
    // pinned staging so the copy is truly asynchronous (ring: the previous call's copy
    // may still be pending)
    constexpr int kSlots = fwa_b200_ctx::kTabSlots;
    if (c->h_tab_cap < tab.size() * kSlots) {
        if (c->h_tab) cudaFreeHost(c->h_tab);
        c->h_tab = nullptr;
        c->h_tab_cap = std::max<size_t>(tab.size() * kSlots, 64 * kSlots);
        CUDA_OK(cudaMallocHost(&c->h_tab, c->h_tab_cap * 8));
        c->h_tab_slot = 0;
    }
    // pinned staging ring: the host only waits when it runs kSlots calls ahead of the copies
    // (no wait on the side stream: the PE of this call is ordered after every earlier use of
    // its buffer by the fork event below)
    c->h_tab_slot = (c->h_tab_slot + 1) % kSlots;
    int64_t* h = c->h_tab + c->h_tab_slot * (c->h_tab_cap / kSlots);
    CUDA_OK(cudaEventSynchronize(c->ev_tab[c->h_tab_slot]));
    std::copy(tab.begin(), tab.end(), h);
    CUDA_OK(cudaMemcpyAsync(d_tab, h, tab.size() * 8, cudaMemcpyHostToDevice, st));
    CUDA_OK(cudaEventRecord(c->ev_tab[c->h_tab_slot], st));
    return d_tab;
}

void build_schedule_body(fwa_b200_ctx* c, const double* d_coords, const fwa_config_t* cfg, Schedule& S,
                         const int64_t* d_off, const int64_t* d_rows, const int64_t* d_drop_off, double w_x,
                         double w_y, int64_t ntot, int n_specs, int nf) {
    cudaStream_t st = c->stream;

    const int64_t total = ntot * n_specs;
    {
        RecSpan t(c, FWA_STAGE_SORT);
        S.sorted = sort_specs(c, d_coords, ntot, n_specs, w_x, w_y, d_off, nf, c->exact_bins);
    }
    RecSpan t_group(c, FWA_STAGE_GROUP);
    S.sorted_inv = ws<int32_t>(c, "sorted_inv", static_cast<size_t>(total));
    uint32_t* scan_tmp = ws<uint32_t>(c, "scan_tmp", scan_tmp_words(total) + 8);

    // drops (block 0 = spec 0), kept set
    S.dropped_ids = ws<int32_t>(c, "dropped_ids", static_cast<size_t>(S.n_drop) + 1);
    S.kept_rank = ws<uint32_t>(c, "kept_rank", static_cast<size_t>(ntot));
    S.kept_ids = ws<int32_t>(c, "kept_ids", static_cast<size_t>(S.K));
    S.idx = ws<int32_t>(c, "idx", static_cast<size_t>(S.K) * n_specs);
    S.out_pos = ws<int32_t>(c, "out_pos", static_cast<size_t>(S.K));
    const int s_last = (cfg->n_blocks - 1) % 4;
    if (S.n_drop <= kMaxDropTable) {
        // few drops (<= G-1 per frame): the drop tables read the tails of spec 0's plan,
        // compaction is a binary search -- no flags, no grid-wide scans
        const int nd = static_cast<int>(S.n_drop);
        int32_t* drop_sorted = ws<int32_t>(c, "drop_sorted", static_cast<size_t>(nd) + 1);
        int32_t* drop_pos = ws<int32_t>(c, "drop_pos", static_cast<size_t>(nd + 1) * n_specs);
        // one frame with few drops: compaction builds the tables itself (one launch fewer)
        const bool fuse = nf == 1 && nd <= kFuseDrops;
        if (nd > 0 && !fuse)
            launch_drop_tables(S.sorted, nd, d_off, d_rows, d_drop_off, nf, S.sorted_inv, ntot, n_specs,
                               S.dropped_ids, drop_sorted, drop_pos, st, &c->launches);
        launch_compact_all(S.sorted, ntot, n_specs, d_off, d_drop_off, nf, drop_sorted, drop_pos, nd, S.K, s_last, S.idx,
                           S.kept_rank, S.kept_ids, S.out_pos, st, &c->launches, fuse ? S.sorted_inv : nullptr,
                           fuse ? S.dropped_ids : nullptr);
        check_launch();
        return;
    }
    S.dropped = ws<uint8_t>(c, "dropped", static_cast<size_t>(ntot));
    CUDA_OK(cudaMemsetAsync(S.dropped, 0, static_cast<size_t>(ntot), st));
    launch_drop_mark(S.sorted, ntot, d_off, d_rows, d_drop_off, nf, S.dropped, S.dropped_ids, st,
                     &c->launches);
    // many drops (huge group sizes x many frames): flag scans
    uint32_t* flags = ws<uint32_t>(c, "flags", static_cast<size_t>(std::max(total, ntot)));
    launch_keep_flags(S.dropped, ntot, flags, st, &c->launches);
    exclusive_scan_u32(flags, S.kept_rank, ntot, scan_tmp, nullptr, st, &c->launches);
    launch_kept_ids(S.kept_rank, S.dropped, ntot, S.kept_ids, st, &c->launches);
    launch_spec_keep_flags(S.sorted, total, S.dropped, flags, st, &c->launches);
    uint32_t* pos = ws<uint32_t>(c, "compact_pos", static_cast<size_t>(total));
    exclusive_scan_u32(flags, pos, total, scan_tmp, nullptr, st, &c->launches);
    launch_spec_compact(S.sorted, total, S.dropped, pos, S.idx, st, &c->launches);
    k_out_pos<<<static_cast<unsigned>((S.K + 255) / 256), 256, 0, st>>>(S.idx + S.K * s_last,
                                                                       S.kept_rank, S.K, S.out_pos);
    ++c->launches;
    check_launch();
}

void build_schedule(fwa_b200_ctx* c, const double* d_coords, const fwa_config_t* cfg, Schedule& S,
                    const int64_t* d_tab_fixed = nullptr) {
    cudaStream_t st = c->stream;
    const int64_t ntot = S.ntot;
    const int n_specs = std::min(cfg->n_blocks, 4);
    S.n_specs = n_specs;
    const double w_x = cfg->window_px * cfg->resolution;  // window_x_m(), backbone.hpp:32
    const double w_y = cfg->window_py * cfg->resolution;

    // frame tables
    const int nf = S.n_frames;
    const int64_t* d_tab = d_tab_fixed;
    if (!d_tab) d_tab = upload_frame_table(c, S);
    const int64_t* d_off = d_tab;
    const int64_t* d_rows = d_tab + nf + 1;
    const int64_t* d_drop_off = d_tab + 2 * nf + 1;
    (void)st;
    build_schedule_body(c, d_coords, cfg, S, d_off, d_rows, d_drop_off, w_x, w_y, ntot, n_specs, nf);
}

// Reference plan-cache rule (backbone.hpp:224-234, 285-316) for a frame of n
// pillars: block b drops n_active mod G; any drop clears the cache.
void cache_stats(int n_blocks, int64_t n, int G, int32_t* computed, int32_t* hits,
                 std::vector<int64_t>* drops) {
    bool have[4] = {false, false, false, false};
    int64_t have_n[4] = {0, 0, 0, 0};
    int comp = 0, hit = 0;
    int64_t act = n;
    for (int b = 0; b < n_blocks; ++b) {
        const int s = b % 4;
        if (have[s] && have_n[s] == act) ++hit;
        else {
            ++comp;
            have[s] = true;
            have_n[s] = act;
        }
        const int64_t d = act % G;
        if (drops) drops->push_back(d);
        if (d) {
            act -= d;
            for (auto& h : have) h = false;
        }
    }
    *computed = comp;
    *hits = hit;
}

// ------------------------------------------------------------------ block pipeline

struct Scratch {
    float *h, *qkv, *cat, *mid, *ln2, *act;  // fp32 path
    __nv_bfloat16 *qkv16, *cat16;             // bf16 path
};

// One FlatFormer block over `rows` grouped rows: input rows x_in[ridx[r]]
// (f32, or f64 when x_in64), positional rows pe[ridx[r]], output
// x_out[sidx[r]].  kernels.hpp:636-650 composed with backbone.hpp:245-283.
void run_block(fwa_b200_ctx* c, const BlockParams& p, const fwa_config_t* cfg, int64_t rows,
               const int32_t* ridx, const float* x_in, const double* x_in64, const float* pe,
               const __half* pe16, float* x_out, const int32_t* sidx, bool fast,
               float* const* d_peers = nullptr) {
    cudaStream_t st = c->stream;
    const int d = cfg->d_model, dff = cfg->d_ff, G = cfg->group_size;
    if (rows == 0) return;
    if (fast && c->precision == FWA_PREC_BF16 && block_fused_supported(G)) {
        static const bool trace_fused = [] {
            const char* v = std::getenv("FWA_B200_TRACE");
            return v && v[0] == '1';
        }();
        unsigned long long* tr = trace_fused && !x_in64 ? ws<unsigned long long>(c, "trace", 2 * 148 * 64) : nullptr;
        StageEv t(c, FWA_PROF_BLOCK);
        StageRec* r = c->rec;
        const bool whole = r && r->blocks_whole;
        const int slot = whole ? 0 : r && r->next_slot < r->n_slots ? r->next_slot++ : -1;
        std::optional<RecSpan> span;
        if (!whole) span.emplace(c, slot >= 0 ? -1 : FWA_STAGE_ATTENTION, slot);
        if (!launch_block_fused(x_in, x_in64, pe16, ridx, sidx, x_out, rows, G, p.tc, c->d_flag, st, &c->launches, tr,
                                slot >= 0 ? r->d_phase + 4 * slot : nullptr, d_peers, d_peers ? 8 : 0))
            throw FwaError{FWA_ERR_CUDA, "k_block_fused: cuTensorMapEncodeTiled (x-row tensor map) failed"};
        check_launch("k_block_fused");
        return;
    }
    if (d_peers) throw FwaError{FWA_ERR_CONTRACT, "peer-memory split: needs the fused bf16 block kernel"};
    if (fast) {
        __nv_bfloat16* qkv = ws<__nv_bfloat16>(c, "qkv16", static_cast<size_t>(rows) * 3 * d);
        // attention output as per-128-row-tile SW128 images (the out-proj A operand)
        __nv_bfloat16* cat = ws<__nv_bfloat16>(c, "cat16", static_cast<size_t>((rows + 127) / 128) * 128 * d);
        // FWA_B200_TRACE=1: phase clocks of the f32-input blocks' tcgen05 kernels (last call wins)
        static const bool trace_on = [] {
            const char* v = std::getenv("FWA_B200_TRACE");
            return v && v[0] == '1';
        }();
        unsigned long long* tr = trace_on && !x_in64 ? ws<unsigned long long>(c, "trace", 2 * 148 * 64) : nullptr;
        // the gathered residual rows, tile-transposed so the out-proj kernel reads them coalesced
        static const bool no_xq = [] {
            const char* v = std::getenv("FWA_B200_NO_XQ");
            return v && v[0] == '1';
        }();
        float* xq = no_xq ? nullptr : ws<float>(c, "xq", static_cast<size_t>((rows + 127) / 128) * 128 * 128);
        {
            StageEv t(c, FWA_PROF_LN_QKV);
            RecSpan span(c, FWA_STAGE_ATTENTION);  // gather + LN1 + QKV: one kernel
            launch_ln1_qkv_tc(x_in, x_in64, pe16, ridx, rows, p.tc, qkv, c->d_flag, xq, st, &c->launches, tr);
            check_launch("k_ln1_qkv_tc");
        }
        {
            StageEv t(c, FWA_PROF_ATTENTION);
            RecSpan span(c, FWA_STAGE_ATTENTION);
            launch_attention_mma(qkv, rows, G, cat, st, &c->launches);
            check_launch("k_attention_mma");
        }
        {
            StageEv t(c, FWA_PROF_OUTPROJ_FFN);
            RecSpan span(c, FWA_STAGE_FFN);  // out-proj + LN2 + FFN + scatter: one kernel
            launch_outproj_ffn_tc(cat, x_in, x_in64, ridx, rows, p.tc, x_out, sidx, xq, st, &c->launches,
                                  tr ? tr + 148 * 64 : nullptr);
            check_launch("k_outproj_ffn_tc");
        }
        check_launch();
        return;
    }
    float* h = ws<float>(c, "h32", static_cast<size_t>(rows) * d);
    float* qkv = ws<float>(c, "qkv32", static_cast<size_t>(rows) * 3 * d);
    float* cat = ws<float>(c, "cat32", static_cast<size_t>(rows) * d);
    float* mid = ws<float>(c, "mid32", static_cast<size_t>(rows) * d);
    float* ln2 = ws<float>(c, "ln2_32", static_cast<size_t>(rows) * d);
    float* act = ws<float>(c, "act32", static_cast<size_t>(rows) * dff);
    GemmArgs g{};
    {
        StageEv t(c, FWA_PROF_LN_QKV);
        RecSpan span(c, FWA_STAGE_GATHER);  // gather + LN1 + PE
        launch_ln_gather_f32(x_in, x_in64, pe, ridx, rows, d, p.ln1_g, p.ln1_b, h, c->d_flag, st,
                             &c->launches);
    }
    {
        StageEv t(c, FWA_PROF_ATTENTION);
        RecSpan span(c, FWA_STAGE_ATTENTION);
        g.A = h; g.M = rows; g.K = d; g.W = p.w_qkv; g.N = 3 * d; g.bias = p.b_qkv; g.C = qkv;
        launch_gemm_f32(g, EPI_BIAS, st, &c->launches);
        launch_attention_f32(qkv, rows, G, d, cfg->n_heads, cat, st, &c->launches);
    }
    StageEv t_ffn(c, FWA_PROF_OUTPROJ_FFN);
    {
        RecSpan span(c, FWA_STAGE_ATTENTION);  // out-proj + residual (kernels.hpp:550-560)
        g = GemmArgs{};
        g.A = cat; g.M = rows; g.K = d; g.W = p.w_out; g.N = d; g.bias = p.b_out; g.C = mid;
        g.R = x_in; g.R64 = x_in64; g.ridx = ridx;
        launch_gemm_f32(g, EPI_RESID_GATHER, st, &c->launches);
    }
    RecSpan span_ffn(c, FWA_STAGE_FFN);  // LN2 + FFN + residual + scatter
    launch_ln_rows_f32(mid, rows, d, p.ln2_g, p.ln2_b, ln2, st, &c->launches);
    g = GemmArgs{};
    g.A = ln2; g.M = rows; g.K = d; g.W = p.w1; g.N = dff; g.bias = p.b1; g.C = act;
    launch_gemm_f32(g, EPI_BIAS_GELU, st, &c->launches);
    g = GemmArgs{};
    g.A = act; g.M = rows; g.K = dff; g.W = p.w2; g.N = d; g.bias = p.b2;
    g.R = mid; g.D = x_out; g.sidx = sidx;
    launch_gemm_f32(g, EPI_RESID_SCATTER, st, &c->launches);
    check_launch();
}

// Size every per-block workspace for `rows` rows up front (the split API keeps raw
// pointers into the workspace between calls).
void reserve_block_ws(fwa_b200_ctx* c, const fwa_config_t* cfg, int64_t rows, bool fast) {
    const size_t d = static_cast<size_t>(cfg->d_model), r = static_cast<size_t>(rows);
    if (fast) {
        ws<float>(c, "xq", static_cast<size_t>((rows + 127) / 128) * 128 * 128);
        ws<__nv_bfloat16>(c, "qkv16", r * 3 * d);
        ws<__nv_bfloat16>(c, "cat16", static_cast<size_t>((rows + 127) / 128) * 128 * d);
    } else {
        ws<float>(c, "h32", r * d);
        ws<float>(c, "qkv32", r * 3 * d);
        ws<float>(c, "cat32", r * d);
        ws<float>(c, "mid32", r * d);
        ws<float>(c, "ln2_32", r * d);
        ws<float>(c, "act32", r * static_cast<size_t>(cfg->d_ff));
    }
}

void require_params(fwa_b200_ctx* c, const fwa_config_t* cfg) {
    if (!c->have_params) throw FwaError{FWA_ERR_CONTRACT, "no parameters loaded (fwa_b200_load_params)"};
    if (static_cast<int>(c->blocks.size()) != cfg->n_blocks)
        throw FwaError{FWA_ERR_CONFIG, "backbone: params.blocks length must equal n_blocks"};
    if (c->pcfg.d_model != cfg->d_model || c->pcfg.n_heads != cfg->n_heads || c->pcfg.d_ff != cfg->d_ff)
        throw FwaError{FWA_ERR_CONFIG, "backbone: block params disagree with config"};
}

// BackboneParams::input_proj on the device (backbone.hpp:179-190): N x f_in (f64 or f32)
// -> N x d_model f32 in `dst`, enqueued on stream `st`
void project_input(fwa_b200_ctx* c, const void* x, bool f64, int64_t n, int d, float* dst, cudaStream_t st) {
    if (c->proj_in <= 0) throw FwaError{FWA_ERR_INTERNAL, "no input projection loaded"};
    if (d != static_cast<int>(c->proj_w.cap / (sizeof(float) * c->proj_in)))
        throw FwaError{FWA_ERR_SHAPE, "backbone: input projection width mismatch"};
    launch_input_proj(x, f64, n, c->proj_in, static_cast<const float*>(c->proj_w.p),
                      c->proj_bias ? static_cast<const float*>(c->proj_b.p) : nullptr, d, dst, st, &c->launches);
    check_launch("k_input_proj");
}

// Device-resident forward over S (already host-framed).  Writes d_out
// (K x d, active order) and, optionally, d_kept.
void forward_device(fwa_b200_ctx* c, const double* d_coords, const float* d_feats,
                    const double* d_feats64, const fwa_config_t* cfg, Schedule& S, float* d_out,
                    int32_t* d_kept, const int64_t* d_tab_fixed = nullptr,
                    cudaEvent_t feats_ready = nullptr, bool project_feats = false) {
    cudaStream_t st = c->stream;
    const int d = cfg->d_model;
    if (project_feats && c->proj_in > 0) {  // device API: d_feats holds N x f_in f32 rows
        float* pr = ws<float>(c, "proj_dev", static_cast<size_t>(S.ntot) * d);
        project_input(c, d_feats, false, S.ntot, d, pr, st);
        d_feats = pr;
    }
    CUDA_OK(cudaMemsetAsync(c->d_flag, 0, 2 * sizeof(int), st));
    const bool fast = fast_path_ok(c, d, cfg->n_heads, cfg->d_ff, cfg->group_size);
    // fast path: fp16 PE rows (|PE| <= 1, abs err <= 2^-12, below the bf16 rounding of
    // LN1 + PE that follows); check mode: fp32 rows.  PE depends only on coordinates:
    // it runs on a side stream, overlapping the schedule (and its host round trip).
    float* pe = fast ? nullptr : ws<float>(c, "pe", static_cast<size_t>(S.ntot) * d);
    __half* pe16 = fast ? ws<__half>(c, "pe16", static_cast<size_t>(S.ntot) * d) : nullptr;
    const double* freq = pe_freq(c, d);
    CUDA_OK(cudaEventRecord(c->ev_fork, st));
    CUDA_OK(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
    launch_positional_embedding(d_coords, S.ntot, d, freq, pe, pe16, c->side, &c->launches);
    // block 0's input rows into L2 while the schedule runs (the host API's copy stream
    // lands them later; then they are already in L2)
    if (!feats_ready)
        launch_prefetch_l2(d_feats ? static_cast<const void*>(d_feats) : static_cast<const void*>(d_feats64),
                           S.ntot * d * (d_feats ? 4 : 8), c->side, &c->launches);
    CUDA_OK(cudaEventRecord(c->ev_join, c->side));
    {
        StageEv t(c, FWA_PROF_SCHEDULE);
        build_schedule(c, d_coords, cfg, S, d_tab_fixed);
    }
    CUDA_OK(cudaStreamWaitEvent(st, c->ev_join, 0));
    if (feats_ready) CUDA_OK(cudaStreamWaitEvent(st, feats_ready, 0));  // block 0 reads them
    float* X = ws<float>(c, "X", static_cast<size_t>(S.ntot) * d);
    static const bool skip_blocks = std::getenv("FWA_B200_DEBUG_SCHEDULE_ONLY") != nullptr;  // timing probe
    // StageTimes of the fused blocks: one span around all of them, apportioned by their
    // summed phase counters (slot 0)
    std::optional<RecSpan> blocks_span;
    if (c->rec && fast && c->precision == FWA_PREC_BF16 && block_fused_supported(cfg->group_size) &&
        c->rec->n_slots > 0) {
        c->rec->blocks_whole = true;
        blocks_span.emplace(c, -1, 0);
    }
    for (int b = 0; b < (skip_blocks ? 0 : cfg->n_blocks); ++b) {
        const int s = b % 4;
        const int32_t* idx = S.idx + S.K * s;
        const bool last = b == cfg->n_blocks - 1;
        const float* xin = b == 0 ? d_feats : X;
        const double* xin64 = b == 0 ? d_feats64 : nullptr;
        run_block(c, c->blocks[static_cast<size_t>(b)], cfg, S.K, idx, xin, xin64, pe, pe16,
                  last ? d_out : X, last ? S.out_pos : idx, fast);
    }
    blocks_span.reset();
    if (c->rec) c->rec->blocks_whole = false;
    if (d_kept)
        CUDA_OK(cudaMemcpyAsync(d_kept, S.kept_ids, static_cast<size_t>(S.K) * 4,
                                cudaMemcpyDeviceToDevice, st));
}

int fail(fwa_b200_ctx* c, const FwaError& e) {
    if (c) c->err = e.msg;
    return e.code;
}

template <class Fn>
int guarded(fwa_b200_ctx* c, Fn&& fn) {
    try {
        if (c) {
            cudaSetDevice(c->device);
            c->err.clear();
        }
        fn();
        return FWA_OK;
    } catch (const FwaError& e) {
        return fail(c, e);
    } catch (const std::exception& e) {
        return fail(c, FwaError{FWA_ERR_INTERNAL, e.what()});
    }
}

// Host-buffer forward shared by the single-frame and batch entry points.
void forward_host(fwa_b200_ctx* c, const double* coords, const void* feats, int f64,
                  const int64_t* off, int n_frames, const fwa_config_t* cfg, fwa_output_t* out,
                  fwa_frame_stats_t* per_frame) {
    validate_cfg(cfg);
    require_params(c, cfg);
    Schedule S;
    host_frames(off, n_frames, cfg->group_size, S);  // N < G: numeric_error before any buffer check
    if (!coords || !feats || !out || !out->features) throw FwaError{FWA_ERR_SHAPE, "null buffer"};
    cudaStream_t st = c->stream;
    const int d = cfg->d_model;
    const int fin = c->proj_in > 0 ? c->proj_in : d;  // input width (BackboneParams::input_proj)
    c->st_used = 0;
    StageRec rec;
    StageScope scope(c, rec, ws<unsigned long long>(c, "phase_acc", 4 * static_cast<size_t>(cfg->n_blocks)),
                     cfg->n_blocks);
    double* d_coords = ws<double>(c, "in_coords", 2 * static_cast<size_t>(S.ntot));
    const float* d_f32 = nullptr;
    const double* d_f64 = nullptr;
    StageEv* h2d = new StageEv(c, FWA_PROF_H2D);
    CUDA_OK(cudaMemcpyAsync(d_coords, coords, static_cast<size_t>(S.ntot) * 16, cudaMemcpyHostToDevice, st));
    delete h2d;
    // the features (the bulk of the input) cross PCIe on a copy stream while the schedule
    // and the PE run (they need only the coordinates); block 0 waits for them (and for the
    // input projection, which runs on the copy stream right behind its input)
    CUDA_OK(cudaEventRecord(c->ev_copy, st));  // previous users of the buffer are done
    CUDA_OK(cudaStreamWaitEvent(c->copy, c->ev_copy, 0));
    const size_t esz = f64 ? 8 : 4;
    void* p = ws<uint8_t>(c, f64 ? "in_feats64" : "in_feats32", static_cast<size_t>(S.ntot) * fin * esz);
    CUDA_OK(cudaMemcpyAsync(p, feats, static_cast<size_t>(S.ntot) * fin * esz, cudaMemcpyHostToDevice, c->copy));
    if (c->proj_in > 0) {
        float* pr = ws<float>(c, "proj_out", static_cast<size_t>(S.ntot) * d);
        project_input(c, p, f64 != 0, S.ntot, d, pr, c->copy);
        d_f32 = pr;
    } else if (f64) {
        d_f64 = static_cast<const double*>(p);
    } else {
        d_f32 = static_cast<const float*>(p);
    }
    CUDA_OK(cudaEventRecord(c->ev_feats, c->copy));
    float* d_out = ws<float>(c, "out_feats", static_cast<size_t>(S.ntot) * d);
    forward_device(c, d_coords, d_f32, d_f64, cfg, S, d_out, nullptr, nullptr, c->ev_feats);
    StageEv* d2h = new StageEv(c, FWA_PROF_D2H);
    CUDA_OK(cudaMemcpyAsync(out->features, d_out, static_cast<size_t>(S.K) * d * 4, cudaMemcpyDeviceToHost, st));
    if (out->kept_indices)
        CUDA_OK(cudaMemcpyAsync(out->kept_indices, S.kept_ids, static_cast<size_t>(S.K) * 4,
                                cudaMemcpyDeviceToHost, st));
    if (out->dropped_ids && S.n_drop)
        CUDA_OK(cudaMemcpyAsync(out->dropped_ids, S.dropped_ids, static_cast<size_t>(S.n_drop) * 4,
                                cudaMemcpyDeviceToHost, st));
    std::vector<int32_t> h_sorted, h_rank, h_idx;
    const bool perms = out->block_perms && n_frames == 1;
    if (perms) {
        h_sorted.resize(static_cast<size_t>(S.ntot) * S.n_specs);
        h_idx.resize(static_cast<size_t>(S.K) * S.n_specs);
        h_rank.resize(static_cast<size_t>(S.ntot));
        CUDA_OK(cudaMemcpyAsync(h_sorted.data(), S.sorted, h_sorted.size() * 4, cudaMemcpyDeviceToHost, st));
        CUDA_OK(cudaMemcpyAsync(h_idx.data(), S.idx, h_idx.size() * 4, cudaMemcpyDeviceToHost, st));
        CUDA_OK(cudaMemcpyAsync(h_rank.data(), S.kept_rank, h_rank.size() * 4, cudaMemcpyDeviceToHost, st));
    }
    rec.h_phase.assign(4 * static_cast<size_t>(rec.n_slots), 0ull);
    CUDA_OK(cudaMemcpyAsync(rec.h_phase.data(), rec.d_phase, rec.h_phase.size() * 8, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaMemcpyAsync(c->h_flag, c->d_flag, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
    delete d2h;
    CUDA_OK(cudaStreamSynchronize(st));
    if (c->h_flag[1]) {  // window-bin capacity overflow: redo with host-sized bins
        c->exact_bins = true;
        struct Reset {
            fwa_b200_ctx* c;
            ~Reset() { c->exact_bins = false; }
        } reset{c};
        c->rec = nullptr;
        forward_host(c, coords, feats, f64, off, n_frames, cfg, out, per_frame);
        return;
    }
    if (c->h_flag[0]) throw FwaError{FWA_ERR_NUMERIC, "group_attention: non-finite input"};
    stage_finish(rec, out->stage_ms);
    out->n_kept = S.K;
    // sort-cache statistics: the reference rule per frame (each frame is its own run)
    for (int f = 0; f < n_frames; ++f) {
        int32_t comp = 0, hits = 0;
        cache_stats(cfg->n_blocks, S.off[f + 1] - S.off[f], cfg->group_size, &comp, &hits, nullptr);
        if (f == 0) {
            out->cache_computed = comp;
            out->cache_hits = hits;
        }
        if (per_frame) per_frame[f] = fwa_frame_stats_t{S.rows[f], static_cast<int32_t>(S.drop[f]), comp, hits};
    }
    if (out->dropped_per_block)
        for (int b = 0; b < cfg->n_blocks; ++b) {
            int64_t tot = 0;  // summed over frames (each frame drops only in block 0)
            for (int f = 0; f < n_frames; ++f) tot += b == 0 ? S.drop[f] : 0;
            out->dropped_per_block[b] = static_cast<int32_t>(tot);
        }
    if (perms) {
        const int64_t n = S.ntot;
        for (int b = 0; b < cfg->n_blocks; ++b) {
            const int s = b % 4;
            int32_t* row = out->block_perms + static_cast<int64_t>(b) * n;
            if (b == 0 || S.n_drop == 0) {
                std::memcpy(row, h_sorted.data() + static_cast<int64_t>(s) * n, static_cast<size_t>(n) * 4);
            } else {
                const int32_t* ix = h_idx.data() + static_cast<int64_t>(s) * S.K;
                for (int64_t r = 0; r < S.K; ++r) row[r] = static_cast<int32_t>(h_rank[static_cast<size_t>(ix[r])]);
            }
        }
    }
}

// Pipelined host-buffer forward over independent frames, each exactly one run_backbone
// (backbone.hpp:159-325, called once per frame of a sequence): while frame f
// computes on the context stream, frame f+1's inputs cross PCIe on the copy stream and
// frame f-1's outputs come back on the d2h stream (two slots of device buffers).  Device-
// side conditions are collected per frame and raised after the pipeline drains; a frame
// whose window range overflowed the sync-free bin histogram is re-run alone.
void forward_frames(fwa_b200_ctx* c, int F, const double* const* coords, const void* const* feats, int f64,
                    const int64_t* n, const fwa_config_t* cfg, fwa_output_t* outs) {
    validate_cfg(cfg);
    require_params(c, cfg);
    if (F < 1 || !coords || !feats || !n || !outs) throw FwaError{FWA_ERR_SHAPE, "need >= 1 frame"};
    const int d = cfg->d_model, G = cfg->group_size;
    const int fin = c->proj_in > 0 ? c->proj_in : d;  // input width (BackboneParams::input_proj)
    int64_t nmax = 0;
    for (int f = 0; f < F; ++f) {
        if (n[f] < G)  // backbone.hpp:218-222, before anything is enqueued
            throw FwaError{FWA_ERR_NUMERIC, "backbone: block 0 has " + std::to_string(n[f]) +
                                                " pillars, fewer than group size " + std::to_string(G) +
                                                "; refusing to emit empty output"};
        if (!coords[f] || !feats[f] || !outs[f].features) throw FwaError{FWA_ERR_SHAPE, "null buffer"};
        if (outs[f].block_perms) throw FwaError{FWA_ERR_CONTRACT, "block_perms: use fwa_b200_backbone_forward"};
        nmax = std::max(nmax, n[f]);
    }
    const size_t esz = f64 ? 8 : 4, nm = static_cast<size_t>(nmax);
    // every slot buffer sized up front: a workspace move frees memory copies are using
    double* in_c[2];
    void* in_f[2];
    float* in_p[2] = {nullptr, nullptr};
    float* o_f[2];
    int32_t* o_ids[2];  // [kept (K) | dropped (< G)]
    static const char* kNames[2][5] = {{"fr_c0", "fr_f0", "fr_o0", "fr_i0", "fr_p0"},
                                       {"fr_c1", "fr_f1", "fr_o1", "fr_i1", "fr_p1"}};
    for (int s = 0; s < 2; ++s) {
        in_c[s] = ws<double>(c, kNames[s][0], 2 * nm);
        in_f[s] = ws<uint8_t>(c, kNames[s][1], nm * fin * esz);
        if (c->proj_in > 0) in_p[s] = ws<float>(c, kNames[s][4], nm * d);
        o_f[s] = ws<float>(c, kNames[s][2], nm * d);
        o_ids[s] = ws<int32_t>(c, kNames[s][3], nm + G);
    }
    ws<float>(c, "X", nm * d);
    unsigned long long* d_phase = ws<unsigned long long>(c, "phase_acc", 4 * static_cast<size_t>(F) * cfg->n_blocks);
    if (!c->d2h) CUDA_OK(cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
    for (auto* e : {&c->fr_ev[0], &c->fr_ev[1], &c->fr_ev[2], &c->fr_ev[3], &c->fr_ev[4], &c->fr_ev[5],
                    &c->fr_ev[6], &c->fr_ev[7], &c->fr_ev[8], &c->fr_ev[9]})
        if (!*e) CUDA_OK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    cudaEvent_t* ev_inc = c->fr_ev;      // [2] coordinates landed
    cudaEvent_t* ev_inf = c->fr_ev + 2;  // [2] features landed
    cudaEvent_t* ev_done = c->fr_ev + 4; // [2] frame computed (inputs free, outputs ready)
    cudaEvent_t* ev_out = c->fr_ev + 6;  // [2] outputs copied back (slot free)
    cudaEvent_t* ev_in_free = c->fr_ev + 8;  // [2] the frame's kernels enqueued past their inputs
    if (c->h_fr_cap < static_cast<size_t>(F)) {
        if (c->h_fr_flags) CUDA_OK(cudaFreeHost(c->h_fr_flags));
        c->h_fr_flags = nullptr;
        CUDA_OK(cudaMallocHost(&c->h_fr_flags, 2 * sizeof(int) * static_cast<size_t>(F)));
        c->h_fr_cap = static_cast<size_t>(F);
    }
    cudaStream_t st = c->stream;
    CUDA_OK(cudaEventRecord(c->ev_copy, st));  // earlier users of the slot buffers are done
    CUDA_OK(cudaStreamWaitEvent(c->copy, c->ev_copy, 0));
    CUDA_OK(cudaStreamWaitEvent(c->d2h, c->ev_copy, 0));
    CUDA_OK(cudaMemsetAsync(d_phase, 0, 4 * static_cast<size_t>(F) * cfg->n_blocks * 8, st));
    std::vector<int64_t> K(static_cast<size_t>(F)), nd(static_cast<size_t>(F));
    std::vector<StageRec> recs(static_cast<size_t>(F));
    c->st_used = 0;
    struct Detach {
        fwa_b200_ctx* c;
        ~Detach() { c->rec = nullptr; }
    } detach{c};
    for (int f = 0; f < F; ++f) {
        const int s = f & 1;
        const size_t nf = static_cast<size_t>(n[f]);
        // the slot's inputs are free once the frame's kernels are done with them -- not after
        // its small device-to-host copies, which queue behind the previous frame's output copy
        if (f >= 2) CUDA_OK(cudaStreamWaitEvent(c->copy, ev_in_free[s], 0));
        CUDA_OK(cudaMemcpyAsync(in_c[s], coords[f], nf * 16, cudaMemcpyHostToDevice, c->copy));
        CUDA_OK(cudaEventRecord(ev_inc[s], c->copy));
        CUDA_OK(cudaMemcpyAsync(in_f[s], feats[f], nf * fin * esz, cudaMemcpyHostToDevice, c->copy));
        if (c->proj_in > 0) project_input(c, in_f[s], f64 != 0, n[f], d, in_p[s], c->copy);
        CUDA_OK(cudaEventRecord(ev_inf[s], c->copy));
        CUDA_OK(cudaStreamWaitEvent(st, ev_inc[s], 0));
        if (f >= 2) CUDA_OK(cudaStreamWaitEvent(st, ev_out[s], 0));
        Schedule S;
        const int64_t off[2] = {0, n[f]};
        host_frames(off, 1, G, S);
        StageRec& rec = recs[static_cast<size_t>(f)];
        rec.d_phase = d_phase + 4 * static_cast<size_t>(f) * cfg->n_blocks;
        rec.n_slots = cfg->n_blocks;
        c->rec = &rec;
        const float* x32 = c->proj_in > 0 ? in_p[s] : (f64 ? nullptr : static_cast<const float*>(in_f[s]));
        const double* x64 = c->proj_in > 0 || !f64 ? nullptr : static_cast<const double*>(in_f[s]);
        forward_device(c, in_c[s], x32, x64, cfg, S, o_f[s], nullptr, nullptr, ev_inf[s]);
        CUDA_OK(cudaEventRecord(ev_in_free[s], st));
        c->rec = nullptr;
        K[f] = S.K;
        nd[f] = S.n_drop;
        CUDA_OK(cudaMemcpyAsync(o_ids[s], S.kept_ids, static_cast<size_t>(S.K) * 4, cudaMemcpyDeviceToDevice, st));
        if (S.n_drop)
            CUDA_OK(cudaMemcpyAsync(o_ids[s] + S.K, S.dropped_ids, static_cast<size_t>(S.n_drop) * 4,
                                    cudaMemcpyDeviceToDevice, st));
        CUDA_OK(cudaMemcpyAsync(c->h_fr_flags + 2 * f, c->d_flag, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
        CUDA_OK(cudaEventRecord(ev_done[s], st));
        CUDA_OK(cudaStreamWaitEvent(c->d2h, ev_done[s], 0));
        fwa_output_t& o = outs[f];
        CUDA_OK(cudaMemcpyAsync(o.features, o_f[s], static_cast<size_t>(S.K) * d * 4, cudaMemcpyDeviceToHost,
                                c->d2h));
        if (o.kept_indices)
            CUDA_OK(cudaMemcpyAsync(o.kept_indices, o_ids[s], static_cast<size_t>(S.K) * 4, cudaMemcpyDeviceToHost,
                                    c->d2h));
        if (o.dropped_ids && S.n_drop)
            CUDA_OK(cudaMemcpyAsync(o.dropped_ids, o_ids[s] + S.K, static_cast<size_t>(S.n_drop) * 4,
                                    cudaMemcpyDeviceToHost, c->d2h));
        CUDA_OK(cudaEventRecord(ev_out[s], c->d2h));
    }
    CUDA_OK(cudaEventRecord(c->ev_copy, c->d2h));
    CUDA_OK(cudaStreamWaitEvent(st, c->ev_copy, 0));  // later work on the context stream follows
    std::vector<unsigned long long> h_phase(4 * static_cast<size_t>(F) * cfg->n_blocks);
    CUDA_OK(cudaMemcpyAsync(h_phase.data(), d_phase, h_phase.size() * 8, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(c->d2h));
    CUDA_OK(cudaStreamSynchronize(st));
    // stage times first (the per-frame event spans live in the context's pool, which a
    // re-run below reuses), then the deferred device conditions in frame order
    for (int f = 0; f < F; ++f) {
        StageRec& rec = recs[static_cast<size_t>(f)];
        rec.h_phase.assign(h_phase.begin() + 4 * static_cast<size_t>(f) * cfg->n_blocks,
                           h_phase.begin() + 4 * static_cast<size_t>(f + 1) * cfg->n_blocks);
        stage_finish(rec, outs[f].stage_ms);
    }
    for (int f = 0; f < F; ++f) {
        if (c->h_fr_flags[2 * f + 1]) {  // window-bin capacity overflow: this frame alone, exact bins
            const int64_t off[2] = {0, n[f]};
            forward_host(c, coords[f], feats[f], f64, off, 1, cfg, &outs[f], nullptr);
            continue;
        }
        if (c->h_fr_flags[2 * f]) throw FwaError{FWA_ERR_NUMERIC, "group_attention: non-finite input"};
        fwa_output_t& o = outs[f];
        o.n_kept = K[static_cast<size_t>(f)];
        cache_stats(cfg->n_blocks, n[f], G, &o.cache_computed, &o.cache_hits, nullptr);
        if (o.dropped_per_block)
            for (int b = 0; b < cfg->n_blocks; ++b)
                o.dropped_per_block[b] = static_cast<int32_t>(b == 0 ? nd[static_cast<size_t>(f)] : 0);
    }
}

} // namespace

extern "C" {

int fwa_b200_ctx_create(int device, void* stream, fwa_b200_ctx** out) {
    if (!out) return FWA_ERR_CONFIG;
    *out = nullptr;
    auto* c = new fwa_b200_ctx;
    c->device = device;
    const int rc = guarded(c, [&] {
        int n = 0;
        CUDA_OK(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n) throw FwaError{FWA_ERR_CUDA, "no such CUDA device"};
        CUDA_OK(cudaSetDevice(device));
        if (stream) {
            c->stream = static_cast<cudaStream_t>(stream);
        } else {
            CUDA_OK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
            c->own_stream = true;
        }
        CUDA_OK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
        CUDA_OK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
        CUDA_OK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
        CUDA_OK(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
        CUDA_OK(cudaEventCreateWithFlags(&c->ev_copy, cudaEventDisableTiming));
        CUDA_OK(cudaEventCreateWithFlags(&c->ev_feats, cudaEventDisableTiming));
        for (auto& e : c->ev_tab) CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CUDA_OK(cudaMalloc(&c->d_flag, 2 * sizeof(int)));
        CUDA_OK(cudaMallocHost(&c->h_flag, 2 * sizeof(int)));
        CUDA_OK(cudaMallocHost(&c->h_minmax, 16 * sizeof(long long)));
    });
    if (rc != FWA_OK) {
        static std::string last;
        last = c->err;
        delete c;
        return rc;
    }
    *out = c;
    return FWA_OK;
}

int fwa_b200_current_device(void) {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) {
        cudaGetLastError();
        d = 0;
    }
    return d;
}

void fwa_b200_ctx_destroy(fwa_b200_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (auto& kv : c->ws)
        if (kv.second.p) cudaFree(kv.second.p);
    if (c->params_f32.p) cudaFree(c->params_f32.p);
    if (c->params_bf16.p) cudaFree(c->params_bf16.p);
    if (c->freq.p) cudaFree(c->freq.p);
    if (c->proj_w.p) cudaFree(c->proj_w.p);
    if (c->proj_b.p) cudaFree(c->proj_b.p);
    for (auto e : c->st_pool) cudaEventDestroy(e);
    if (c->d_flag) cudaFree(c->d_flag);
    if (c->h_flag) cudaFreeHost(c->h_flag);
    if (c->h_minmax) cudaFreeHost(c->h_minmax);
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    for (auto& g : c->graphs) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        if (g.tab) cudaFree(g.tab);
    }
    if (c->side) {
        cudaStreamSynchronize(c->side);
        cudaStreamDestroy(c->side);
    }
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    for (auto e : c->ev_tab)
        if (e) cudaEventDestroy(e);
    if (c->h_tab) cudaFreeHost(c->h_tab);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->copy) {
        cudaStreamSynchronize(c->copy);
        cudaStreamDestroy(c->copy);
    }
    if (c->ev_copy) cudaEventDestroy(c->ev_copy);
    if (c->d2h) {
        cudaStreamSynchronize(c->d2h);
        cudaStreamDestroy(c->d2h);
    }
    for (auto e : c->fr_ev)
        if (e) cudaEventDestroy(e);
    if (c->h_fr_flags) cudaFreeHost(c->h_fr_flags);
    if (c->ev_feats) cudaEventDestroy(c->ev_feats);
    if (c->own_stream) cudaStreamDestroy(c->stream);
    delete c;
}

const char* fwa_b200_last_error(const fwa_b200_ctx* c) { return c ? c->err.c_str() : "null context"; }

int fwa_b200_set_precision(fwa_b200_ctx* c, int precision) {
    if (!c) return FWA_ERR_CONFIG;
    if (precision != FWA_PREC_BF16 && precision != FWA_PREC_FP32 && precision != FWA_PREC_BF16_3K) {
        c->err = "unknown precision";
        return FWA_ERR_CONFIG;
    }
    c->precision = precision;
    return FWA_OK;
}

int64_t fwa_b200_kernel_launches(const fwa_b200_ctx* c) { return c ? c->launches : 0; }

// Debug: copy the phase-trace buffer (2 x 148 x 64 u64 clocks) to the host.
int fwa_b200_debug_trace(fwa_b200_ctx* c, unsigned long long* out) {
    return guarded(c, [&] {
        auto it = c->ws.find("trace");
        if (it == c->ws.end() || !it->second.p) throw FwaError{FWA_ERR_CONTRACT, "no trace (FWA_B200_TRACE=1)"};
        CUDA_OK(cudaStreamSynchronize(c->stream));
        CUDA_OK(cudaMemcpy(out, it->second.p, 2 * 148 * 64 * 8, cudaMemcpyDeviceToHost));
    });
}

int fwa_b200_sync_check(fwa_b200_ctx* c) {
    return guarded(c, [&] {
        CUDA_OK(cudaMemcpyAsync(c->h_flag, c->d_flag, 2 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        CUDA_OK(cudaStreamSynchronize(c->stream));
        if (c->h_flag[1])
            throw FwaError{FWA_ERR_INTERNAL, "window-bin capacity exceeded: re-run through the host API"};
        if (c->h_flag[0]) throw FwaError{FWA_ERR_NUMERIC, "group_attention: non-finite input"};
    });
}

int fwa_b200_set_profiling(fwa_b200_ctx* c, int enable) {
    if (!c) return FWA_ERR_CONFIG;
    return guarded(c, [&] {
        prof_collect(c);
        c->profiling = enable != 0;
        for (int i = 0; i < FWA_PROF_SLOTS; ++i) {
            c->prof_ms[i] = 0.0;
            c->prof_n[i] = 0;
        }
    });
}

int fwa_b200_get_profile(fwa_b200_ctx* c, double* ms, int64_t* counts) {
    if (!c) return FWA_ERR_CONFIG;
    return guarded(c, [&] {
        prof_collect(c);
        for (int i = 0; i < FWA_PROF_SLOTS; ++i) {
            if (ms) ms[i] = c->prof_ms[i];
            if (counts) counts[i] = c->prof_n[i];
        }
    });
}

int fwa_b200_fast_path(const fwa_b200_ctx* c, const fwa_config_t* cfg) {
    return (c && cfg && fast_path_ok(c, cfg->d_model, cfg->n_heads, cfg->d_ff, cfg->group_size)) ? 1 : 0;
}

int fwa_b200_load_params(fwa_b200_ctx* c, const fwa_config_t* cfg, const void* blob, size_t len) {
    return guarded(c, [&] {
        validate_cfg(cfg);
        if (!blob) throw FwaError{FWA_ERR_PARSE, "null FWAP blob"};
        std::vector<std::vector<float>> keep;
        const auto recs = parse_fwap(blob, len, keep);
        if (static_cast<int>(recs.size()) != cfg->n_blocks)
            throw FwaError{FWA_ERR_CONFIG, "backbone: params.blocks length must equal n_blocks"};
        for (const auto& r : recs)
            if (r.d != cfg->d_model || r.h != cfg->n_heads || r.dff != cfg->d_ff)
                throw FwaError{FWA_ERR_CONFIG, "backbone: block params disagree with config"};
        c->blocks = upload_block_params(recs, c->params_f32, c->params_bf16, c->stream);
        ++c->params_version;
        c->pcfg = *cfg;
        c->have_params = true;
    });
}

int fwa_b200_load_input_proj(fwa_b200_ctx* c, int32_t d_model, int32_t f_in, const float* weight,
                             const float* bias) {
    return guarded(c, [&] {
        if (f_in == 0) {  // remove
            c->proj_in = 0;
            ++c->params_version;
            return;
        }
        if (f_in < 0 || d_model < 1) throw FwaError{FWA_ERR_SHAPE, "input projection: bad shape"};
        if (!weight) throw FwaError{FWA_ERR_SHAPE, "input projection: null weight"};
        const size_t wb = static_cast<size_t>(d_model) * f_in * sizeof(float);
        if (c->proj_w.p) cudaFree(c->proj_w.p);
        c->proj_w.p = nullptr;
        CUDA_OK(cudaMalloc(&c->proj_w.p, wb));
        c->proj_w.cap = wb;  // d_model x f_in floats exactly (project_input reads d_model from it)
        CUDA_OK(cudaMemcpy(c->proj_w.p, weight, wb, cudaMemcpyHostToDevice));
        c->proj_bias = bias != nullptr;
        if (bias) {
            if (c->proj_b.p) cudaFree(c->proj_b.p);
            c->proj_b.p = nullptr;
            CUDA_OK(cudaMalloc(&c->proj_b.p, static_cast<size_t>(d_model) * sizeof(float)));
            c->proj_b.cap = static_cast<size_t>(d_model) * sizeof(float);
            CUDA_OK(cudaMemcpy(c->proj_b.p, bias, c->proj_b.cap, cudaMemcpyHostToDevice));
        }
        c->proj_in = f_in;
        ++c->params_version;
    });
}

int fwa_b200_backbone_forward(fwa_b200_ctx* c, const double* coords, const void* feats, int f64,
                              int64_t n, const fwa_config_t* cfg, fwa_output_t* out) {
    return guarded(c, [&] {
        const int64_t off[2] = {0, n};
        forward_host(c, coords, feats, f64, off, 1, cfg, out, nullptr);
    });
}

int fwa_b200_backbone_forward_batch(fwa_b200_ctx* c, const double* coords, const void* feats,
                                    int f64, const int64_t* frame_offsets, int n_frames,
                                    const fwa_config_t* cfg, fwa_output_t* out,
                                    fwa_frame_stats_t* per_frame) {
    return guarded(c, [&] {
        if (!frame_offsets || n_frames < 1) throw FwaError{FWA_ERR_SHAPE, "need >= 1 frame"};
        if (frame_offsets[0] != 0) throw FwaError{FWA_ERR_SHAPE, "frame_offsets[0] must be 0"};
        forward_host(c, coords, feats, f64, frame_offsets, n_frames, cfg, out, per_frame);
    });
}

int fwa_b200_backbone_forward_frames(fwa_b200_ctx* c, int n_frames, const double* const* coords,
                                     const void* const* feats, int f64, const int64_t* n,
                                     const fwa_config_t* cfg, fwa_output_t* outs) {
    return guarded(c, [&] { forward_frames(c, n_frames, coords, feats, f64, n, cfg, outs); });
}

int fwa_b200_backbone_forward_device(fwa_b200_ctx* c, const double* d_coords, const float* d_feats,
                                     const int64_t* frame_offsets, int n_frames,
                                     const fwa_config_t* cfg, float* d_out, int32_t* d_kept,
                                     int64_t* n_kept_out) {
    return guarded(c, [&] {
        validate_cfg(cfg);
        require_params(c, cfg);
        if (!d_coords || !d_feats || !d_out) throw FwaError{FWA_ERR_SHAPE, "null buffer"};
        if (!frame_offsets || n_frames < 1) throw FwaError{FWA_ERR_SHAPE, "need frame offsets"};
        Schedule S;
        host_frames(frame_offsets, n_frames, cfg->group_size, S);
        if (n_kept_out) *n_kept_out = S.K;
        // CUDA graph: a repeated call (same buffers, frames, config, params, workspace)
        // replays the captured launch sequence — no per-kernel host launch cost.
        static const bool no_graph = [] {
            const char* v = std::getenv("FWA_B200_NO_GRAPH");
            return v && v[0] == '1';
        }();
        fwa_b200_ctx::GraphKey key;
        key.coords = d_coords;
        key.feats = d_feats;
        key.out = d_out;
        key.kept = d_kept;
        key.off.assign(frame_offsets, frame_offsets + n_frames + 1);
        key.cfg = *cfg;
        key.precision = c->precision;
        key.params_version = c->params_version;
        key.ws_epoch = c->ws_epoch;
        if (no_graph || c->g_disabled || c->profiling || c->exact_bins) {
            forward_device(c, d_coords, d_feats, nullptr, cfg, S, d_out, d_kept, nullptr, nullptr, true);
            return;
        }
        ++c->g_clock;
        for (auto& g : c->graphs)
            if (g.key == key) {
                CUDA_OK(cudaGraphLaunch(g.exec, c->stream));
                c->launches += g.launches;
                g.used = c->g_clock;
                return;
            }
        auto seen = std::find(c->g_seen.begin(), c->g_seen.end(), key);
        if (seen == c->g_seen.end()) {  // first sighting: run eagerly (sizes the workspace)
            forward_device(c, d_coords, d_feats, nullptr, cfg, S, d_out, d_kept, nullptr, nullptr, true);
            key.ws_epoch = c->ws_epoch;
            c->g_seen.push_back(key);
            if (static_cast<int>(c->g_seen.size()) > fwa_b200_ctx::kGraphs) c->g_seen.erase(c->g_seen.begin());
            return;
        }
        c->g_seen.erase(seen);
        // second sighting: capture into a free or the least recently used slot
        fwa_b200_ctx::GraphEntry* e = nullptr;
        if (static_cast<int>(c->graphs.size()) < fwa_b200_ctx::kGraphs) {
            c->graphs.emplace_back();
            e = &c->graphs.back();
        } else {
            e = &*std::min_element(c->graphs.begin(), c->graphs.end(),
                                   [](const auto& x, const auto& y) { return x.used < y.used; });
            if (e->exec) cudaGraphExecDestroy(e->exec);
            e->exec = nullptr;
        }
        const std::vector<int64_t> tab = frame_table(S);
        if (e->tab) cudaFree(e->tab);
        e->tab = nullptr;
        CUDA_OK(cudaMalloc(&e->tab, tab.size() * 8));
        CUDA_OK(cudaMemcpy(e->tab, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice));
        CUDA_OK(cudaStreamSynchronize(c->stream));
        const int64_t l0 = c->launches;
        cudaGraph_t graph = nullptr;
        auto drop_entry = [&] {
            if (e->tab) cudaFree(e->tab);
            c->graphs.erase(c->graphs.begin() + (e - c->graphs.data()));
        };
        CUDA_OK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        try {
            forward_device(c, d_coords, d_feats, nullptr, cfg, S, d_out, d_kept, e->tab, nullptr, true);
        } catch (...) {
            cudaStreamEndCapture(c->stream, &graph);
            if (graph) cudaGraphDestroy(graph);
            cudaGetLastError();
            drop_entry();
            c->g_disabled = true;
            throw;
        }
        const cudaError_t ec = cudaStreamEndCapture(c->stream, &graph);
        cudaGraphExec_t exec = nullptr;
        if (ec != cudaSuccess || !graph || cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
            if (graph) cudaGraphDestroy(graph);
            cudaGetLastError();
            drop_entry();
            c->g_disabled = true;  // not capturable here: stay eager
            forward_device(c, d_coords, d_feats, nullptr, cfg, S, d_out, d_kept, nullptr, nullptr, true);
            return;
        }
        cudaGraphDestroy(graph);
        e->exec = exec;
        e->launches = c->launches - l0;
        e->key = key;
        e->key.ws_epoch = c->ws_epoch;
        e->used = c->g_clock;
        CUDA_OK(cudaGraphLaunch(e->exec, c->stream));
    });
}

// ---- group-range split (BASELINE config 4): every rank builds the identical schedule
// from replicated coordinates, computes a contiguous range of groups of each block, and
// the ranks exchange the block's sorted-order output rows (NCCL all-gather, done by the
// caller) before scattering them back to pillar-id order for the next block.
int fwa_b200_split_begin(fwa_b200_ctx* c, const double* d_coords, int64_t n, const fwa_config_t* cfg,
                         int64_t* k_out) {
    return guarded(c, [&] {
        validate_cfg(cfg);
        require_params(c, cfg);
        if (c->proj_in > 0)
            throw FwaError{FWA_ERR_CONTRACT, "split: project the input rows first (no input projection here)"};
        Schedule S;
        const int64_t off[2] = {0, n};
        host_frames(off, 1, cfg->group_size, S);
        cudaStream_t st = c->stream;
        const int d = cfg->d_model;
        CUDA_OK(cudaMemsetAsync(c->d_flag, 0, 2 * sizeof(int), st));
        const bool fast = fast_path_ok(c, d, cfg->n_heads, cfg->d_ff, cfg->group_size);
        float* pe = fast ? nullptr : ws<float>(c, "pe", static_cast<size_t>(n) * d);
        __half* pe16 = fast ? ws<__half>(c, "pe16", static_cast<size_t>(n) * d) : nullptr;
        launch_positional_embedding(d_coords, n, d, pe_freq(c, d), pe, pe16, st, &c->launches);
        c->exact_bins = true;  // host-sized bins: one-time cost per scene
        struct Reset {
            fwa_b200_ctx* c;
            ~Reset() { c->exact_bins = false; }
        } reset{c};
        build_schedule(c, d_coords, cfg, S);
        check_launch();
        reserve_block_ws(c, cfg, S.K, fast);
        c->split.ready = true;
        c->split.cfg = *cfg;
        c->split.ntot = n;
        c->split.K = S.K;
        c->split.idx = S.idx;
        c->split.out_pos = S.out_pos;
        c->split.pe = pe;
        c->split.pe16 = pe16;
        c->split.fast = fast;
        c->split.ws_epoch = c->ws_epoch;
        if (k_out) *k_out = S.K;
    });
}

int fwa_b200_split_block(fwa_b200_ctx* c, int block, int64_t group_begin, int64_t group_end,
                         const float* d_x, float* d_y) {
    return guarded(c, [&] {
        auto& sp = c->split;
        if (!sp.ready) throw FwaError{FWA_ERR_CONTRACT, "fwa_b200_split_begin first"};
        const int G = sp.cfg.group_size;
        if (block < 0 || block >= sp.cfg.n_blocks || group_begin < 0 || group_end < group_begin ||
            group_end * G > sp.K)
            throw FwaError{FWA_ERR_SHAPE, "split: block / group range out of bounds"};
        const int64_t r0 = group_begin * G, rows = (group_end - group_begin) * G;
        const int32_t* idx = sp.idx + sp.K * (block % 4) + r0;
        if (sp.ws_epoch != c->ws_epoch)
            throw FwaError{FWA_ERR_CONTRACT, "split: workspace moved since split_begin (call it again)"};
        run_block(c, c->blocks[static_cast<size_t>(block)], &sp.cfg, rows, idx, d_x, nullptr, sp.pe, sp.pe16,
                  d_y, nullptr, sp.fast);
    });
}

int fwa_b200_split_plan(fwa_b200_ctx* c, int block, int32_t* ids_out) {
    return guarded(c, [&] {
        auto& sp = c->split;
        if (!sp.ready) throw FwaError{FWA_ERR_CONTRACT, "fwa_b200_split_begin first"};
        if (block < 0 || block >= sp.cfg.n_blocks || !ids_out) throw FwaError{FWA_ERR_SHAPE, "split: bad block"};
        CUDA_OK(cudaMemcpyAsync(ids_out, sp.idx + sp.K * (block % 4), static_cast<size_t>(sp.K) * 4,
                                cudaMemcpyDeviceToHost, c->stream));
        CUDA_OK(cudaStreamSynchronize(c->stream));
    });
}

int fwa_b200_split_plan_device(fwa_b200_ctx* c, int block, int32_t* d_ids_out) {
    return guarded(c, [&] {
        auto& sp = c->split;
        if (!sp.ready) throw FwaError{FWA_ERR_CONTRACT, "fwa_b200_split_begin first"};
        if (block < 0 || block >= sp.cfg.n_blocks || !d_ids_out) throw FwaError{FWA_ERR_SHAPE, "split: bad block"};
        CUDA_OK(cudaMemcpyAsync(d_ids_out, sp.idx + sp.K * (block % 4), static_cast<size_t>(sp.K) * 4,
                                cudaMemcpyDeviceToDevice, c->stream));
    });
}

int fwa_b200_split_scatter(fwa_b200_ctx* c, int block, const float* d_y, float* d_dst) {
    return guarded(c, [&] {
        auto& sp = c->split;
        if (!sp.ready) throw FwaError{FWA_ERR_CONTRACT, "fwa_b200_split_begin first"};
        if (block < 0 || block >= sp.cfg.n_blocks) throw FwaError{FWA_ERR_SHAPE, "split: bad block"};
        if (sp.ws_epoch != c->ws_epoch)
            throw FwaError{FWA_ERR_CONTRACT, "split: workspace moved since split_begin (call it again)"};
        const bool last = block == sp.cfg.n_blocks - 1;
        const int32_t* pos = last ? sp.out_pos : sp.idx + sp.K * (block % 4);
        launch_scatter_sorted(d_y, pos, sp.K, sp.cfg.d_model, d_dst, c->stream, &c->launches);
        check_launch();
    });
}

int fwa_b200_split_p2p_setup(fwa_b200_ctx* c, int world, int rank, float* const* x_peers, float* const* out_peers) {
    return guarded(c, [&] {
        auto& sp = c->split;
        if (!sp.ready) throw FwaError{FWA_ERR_CONTRACT, "fwa_b200_split_begin first"};
        if (sp.ws_epoch != c->ws_epoch)
            throw FwaError{FWA_ERR_CONTRACT, "split: workspace moved since split_begin (call it again)"};
        if (world < 1 || world > 8 || rank < 0 || rank >= world || !x_peers || !out_peers)
            throw FwaError{FWA_ERR_SHAPE, "split p2p: 1 <= world <= 8, 0 <= rank < world, peer pointers"};
        if (!sp.fast || c->precision != FWA_PREC_BF16 || !block_fused_supported(sp.cfg.group_size))
            throw FwaError{FWA_ERR_CONTRACT, "peer-memory split: needs the fused bf16 block kernel"};
        if (sp.ntot >= (int64_t{1} << 28)) throw FwaError{FWA_ERR_SHAPE, "peer-memory split: >= 2^28 pillars"};
        cudaStream_t st = c->stream;
        const int G = sp.cfg.group_size, nb = sp.cfg.n_blocks;
        const int64_t n_groups = sp.K / G;
        const int64_t per = std::max<int64_t>(1, (n_groups + world - 1) / world);  // split.py partition_groups
        sp.world = world;
        sp.rank = rank;
        sp.g0 = std::min(rank * per, n_groups);
        sp.g1 = std::min((rank + 1) * per, n_groups);
        const int64_t rows = (sp.g1 - sp.g0) * G, r0 = sp.g0 * G, chunk = per * G;
        const int n_specs = std::min(nb, 4);
        int32_t* inv = ws<int32_t>(c, "p2p_inv", static_cast<size_t>(n_specs) * sp.ntot);
        for (int s = 0; s < n_specs; ++s) {
            k_plan_inverse<<<static_cast<unsigned>((sp.K + 255) / 256), 256, 0, st>>>(sp.idx + sp.K * s, sp.K,
                                                                                       inv + sp.ntot * s);
            ++c->launches;
        }
        sp.p2p_sidx = ws<int32_t>(c, "p2p_sidx", static_cast<size_t>(nb) * std::max<int64_t>(rows, 1));
        for (int b = 0; b < nb; ++b) {
            const bool last = b == nb - 1;
            if (rows > 0) {
                k_p2p_rows<<<static_cast<unsigned>((rows + 255) / 256), 256, 0, st>>>(
                    sp.idx + sp.K * (b % 4), last ? nullptr : inv + sp.ntot * ((b + 1) % 4), sp.out_pos, r0, rows,
                    chunk, last ? 1 : 0, sp.p2p_sidx + static_cast<int64_t>(b) * rows);
                ++c->launches;
            }
        }
        float* hp[16];
        for (int k = 0; k < 8; ++k) {
            hp[k] = x_peers[k < world ? k : 0];
            hp[8 + k] = out_peers[k < world ? k : 0];
        }
        float** dp = ws<float*>(c, "p2p_peers", 16);
        CUDA_OK(cudaMemcpyAsync(dp, hp, sizeof(hp), cudaMemcpyHostToDevice, st));
        CUDA_OK(cudaStreamSynchronize(st));  // hp (host) is read by the copy
        check_launch("split p2p tables");
        sp.p2p_x = dp;
        sp.p2p_out = dp + 8;
        // the new table buffers bumped the workspace epoch; the schedule's own buffers (plans,
        // output rows, PE) did not move -- re-arm the staleness check at the current epoch
        if (c->ws["idx"].p != static_cast<void*>(sp.idx) || c->ws["out_pos"].p != static_cast<void*>(sp.out_pos)) {
            sp.ready = false;
            throw FwaError{FWA_ERR_CONTRACT, "split: workspace moved; call split_begin and p2p_setup again"};
        }
        sp.ws_epoch = c->ws_epoch;
    });
}

int fwa_b200_split_block_p2p(fwa_b200_ctx* c, int block, const float* d_x) {
    return guarded(c, [&] {
        auto& sp = c->split;
        if (!sp.ready || !sp.p2p_sidx) throw FwaError{FWA_ERR_CONTRACT, "fwa_b200_split_p2p_setup first"};
        if (block < 0 || block >= sp.cfg.n_blocks || !d_x) throw FwaError{FWA_ERR_SHAPE, "split: bad block"};
        if (sp.ws_epoch != c->ws_epoch)
            throw FwaError{FWA_ERR_CONTRACT, "split: workspace moved since split_begin (call it again)"};
        const int G = sp.cfg.group_size;
        const int64_t rows = (sp.g1 - sp.g0) * G;
        if (rows == 0) return;
        const bool last = block == sp.cfg.n_blocks - 1;
        const int32_t* idx = sp.idx + sp.K * (block % 4) + sp.g0 * G;
        run_block(c, c->blocks[static_cast<size_t>(block)], &sp.cfg, rows, idx, d_x, nullptr, sp.pe, sp.pe16,
                  nullptr, sp.p2p_sidx + static_cast<int64_t>(block) * rows, sp.fast, last ? sp.p2p_out : sp.p2p_x);
    });
}

void* fwa_b200_alloc(fwa_b200_ctx* c, size_t bytes) {
    void* p = nullptr;
    const int rc = guarded(c, [&] { CUDA_OK(cudaMalloc(&p, bytes ? bytes : 1)); });
    return rc == FWA_OK ? p : nullptr;
}

void fwa_b200_free(fwa_b200_ctx* c, void* d_ptr) {
    if (c) cudaSetDevice(c->device);
    if (d_ptr) cudaFree(d_ptr);
}

int fwa_b200_ipc_handle(fwa_b200_ctx* c, void* d_ptr, void* handle_out) {
    return guarded(c, [&] {
        if (!d_ptr || !handle_out) throw FwaError{FWA_ERR_SHAPE, "ipc: null pointer"};
        cudaIpcMemHandle_t h;
        CUDA_OK(cudaIpcGetMemHandle(&h, d_ptr));
        static_assert(sizeof(h) == FWA_IPC_HANDLE_BYTES, "cudaIpcMemHandle_t size");
        std::memcpy(handle_out, &h, sizeof(h));
    });
}

int fwa_b200_ipc_open(fwa_b200_ctx* c, const void* handle, void** d_ptr_out) {
    return guarded(c, [&] {
        if (!handle || !d_ptr_out) throw FwaError{FWA_ERR_SHAPE, "ipc: null pointer"};
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof(h));
        CUDA_OK(cudaIpcOpenMemHandle(d_ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
    });
}

int fwa_b200_ipc_close(fwa_b200_ctx* c, void* d_ptr) {
    return guarded(c, [&] { CUDA_OK(cudaIpcCloseMemHandle(d_ptr)); });
}

int fwa_b200_sort_plan(fwa_b200_ctx* c, const double* coords, int64_t n, double w_x, double w_y,
                       int shift, int major_axis_y, int32_t* perm_out) {
    return guarded(c, [&] {
        if (!(w_x > 0.0) || !(w_y > 0.0)) throw FwaError{FWA_ERR_CONFIG, "window dims must be positive"};
        if (n == 0) return;
        if (!coords || !perm_out) throw FwaError{FWA_ERR_SHAPE, "null buffer"};
        // one frame; specs 0..spec are keyed, only `spec` is read back
        cudaStream_t st = c->stream;
        const int64_t off[2] = {0, n};
        double* d_coords = ws<double>(c, "in_coords", 2 * static_cast<size_t>(n));
        CUDA_OK(cudaMemcpyAsync(d_coords, coords, static_cast<size_t>(n) * 16, cudaMemcpyHostToDevice, st));
        int64_t* d_off = ws<int64_t>(c, "frame_tab", 4);
        CUDA_OK(cudaMemcpyAsync(d_off, off, 16, cudaMemcpyHostToDevice, st));
        const int spec = 2 * (major_axis_y ? 1 : 0) + (shift ? 1 : 0);
        const int64_t ntot = n;
        const int32_t* sorted = sort_specs(c, d_coords, ntot, spec + 1, w_x, w_y, d_off, 1);
        CUDA_OK(cudaMemcpyAsync(perm_out, sorted + static_cast<int64_t>(spec) * ntot,
                                static_cast<size_t>(n) * 4, cudaMemcpyDeviceToHost, st));
        CUDA_OK(cudaStreamSynchronize(st));
    });
}

int fwa_b200_block_forward(fwa_b200_ctx* c, const float* f, const float* pe, int64_t rows,
                           int32_t n_groups, const void* record, size_t record_len, float* out) {
    return guarded(c, [&] {
        std::vector<std::vector<float>> keep;
        const auto recs = parse_fwap(record, record_len, keep);
        if (recs.size() != 1) throw FwaError{FWA_ERR_CONFIG, "expected exactly one FWAP record"};
        const Record& r = recs[0];
        const int d = r.d;
        if (n_groups == 0 && rows == 0) return;  // kernels.hpp:454
        if (n_groups < 1 || rows % n_groups != 0)
            throw FwaError{FWA_ERR_SHAPE, "group_attention: rows not divisible by n_groups"};
        fwa_config_t cfg{};
        cfg.resolution = 0.32;
        cfg.window_px = cfg.window_py = 9;
        cfg.group_size = static_cast<int32_t>(rows / n_groups);
        cfg.n_blocks = 1;
        cfg.d_model = d;
        cfg.n_heads = r.h;
        cfg.d_ff = r.dff;
        // parameters for this call only (the loaded backbone params are kept)
        const std::vector<BlockParams> bp =
            upload_block_params(recs, c->ws["blk_params_f32"], c->ws["blk_params_bf16"], c->stream);
        cudaStream_t st = c->stream;
        float* df = ws<float>(c, "bf_f", static_cast<size_t>(rows) * d);
        float* dpe = ws<float>(c, "bf_pe", static_cast<size_t>(rows) * d);
        float* dout = ws<float>(c, "bf_out", static_cast<size_t>(rows) * d);
        CUDA_OK(cudaMemcpyAsync(df, f, static_cast<size_t>(rows) * d * 4, cudaMemcpyHostToDevice, st));
        CUDA_OK(cudaMemcpyAsync(dpe, pe, static_cast<size_t>(rows) * d * 4, cudaMemcpyHostToDevice, st));
        CUDA_OK(cudaMemsetAsync(c->d_flag, 0, 2 * sizeof(int), st));
        const bool fast = fast_path_ok(c, d, r.h, r.dff, cfg.group_size);
        __half* dpe16 = nullptr;
        if (fast) {
            dpe16 = ws<__half>(c, "bf_pe16", static_cast<size_t>(rows) * d);
            launch_f32_to_f16(dpe, rows * d, dpe16, st, &c->launches);
        }
        run_block(c, bp[0], &cfg, rows, nullptr, df, nullptr, dpe, dpe16, dout, nullptr, fast);
        CUDA_OK(cudaMemcpyAsync(out, dout, static_cast<size_t>(rows) * d * 4, cudaMemcpyDeviceToHost, st));
        CUDA_OK(cudaMemcpyAsync(c->h_flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, st));
        CUDA_OK(cudaStreamSynchronize(st));
        if (*c->h_flag) throw FwaError{FWA_ERR_NUMERIC, "group_attention: non-finite input"};
    });
}

int fwa_b200_positional_embedding(fwa_b200_ctx* c, const double* coords, int64_t n, int32_t d,
                                  float* out) {
    return guarded(c, [&] {
        if (d < 4 || d % 4 != 0)
            throw FwaError{FWA_ERR_CONFIG, "positional_embedding: d_model must be divisible by 4"};
        if (n == 0) return;
        cudaStream_t st = c->stream;
        double* dc = ws<double>(c, "pe_coords", 2 * static_cast<size_t>(n));
        float* dp = ws<float>(c, "pe_out", static_cast<size_t>(n) * d);
        CUDA_OK(cudaMemcpyAsync(dc, coords, static_cast<size_t>(n) * 16, cudaMemcpyHostToDevice, st));
        launch_positional_embedding(dc, n, d, pe_freq(c, d), dp, nullptr, st, &c->launches);
        check_launch();
        CUDA_OK(cudaMemcpyAsync(out, dp, static_cast<size_t>(n) * d * 4, cudaMemcpyDeviceToHost, st));
        CUDA_OK(cudaStreamSynchronize(st));
    });
}

// geometry::pillarize (geometry.hpp:246-300) on the device; returns the pillar count P
// (one host round trip for the cell range, one for P).  coords_out == nullptr: count only.
static int64_t pillarize_device(fwa_b200_ctx* c, const double* d_xy, const double* d_feats, int64_t n, int32_t f_in,
                                double res, const double* d_w, const double* d_b, int32_t d_out, double* d_coords,
                                double* d_out_feats, int64_t cap) {
    if (!(res > 0.0)) throw FwaError{FWA_ERR_CONFIG, "pillarize: resolution must be > 0"};
    if (d_out < 1) throw FwaError{FWA_ERR_CONFIG, "pillarize: d_out must be >= 1"};
    if (f_in < 0 || n < 0) throw FwaError{FWA_ERR_SHAPE, "pillarize: negative size"};
    if (n == 0) return 0;
    cudaStream_t st = c->stream;
    long long* cell = ws<long long>(c, "pz_cell", 2 * static_cast<size_t>(n));
    long long* mm = ws<long long>(c, "pz_mm", 4);
    launch_cell_keys(d_xy, n, res, cell, mm, st, &c->launches);
    check_launch("k_cell_keys");
    CUDA_OK(cudaMemcpyAsync(c->h_minmax, mm, 4 * 8, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
    const long long min_x = c->h_minmax[0], min_y = c->h_minmax[2];
    const long long rx = c->h_minmax[1] - min_x + 1, ry = c->h_minmax[3] - min_y + 1;
    if (rx <= 0 || ry <= 0 || static_cast<double>(rx) * static_cast<double>(ry) > 2.0e9)
        throw FwaError{FWA_ERR_CONFIG, "pillarize: cell index range too large for the dense cell grid"};
    const int64_t ncell = rx * ry;
    uint32_t* hist = ws<uint32_t>(c, "pz_hist", static_cast<size_t>(ncell));
    uint32_t* cell_id = ws<uint32_t>(c, "pz_cellid", static_cast<size_t>(n));
    CUDA_OK(cudaMemsetAsync(hist, 0, static_cast<size_t>(ncell) * 4, st));
    launch_cell_hist(cell, n, min_x, min_y, ry, cell_id, hist, st, &c->launches);
    uint32_t* start = ws<uint32_t>(c, "pz_start", static_cast<size_t>(ncell));
    uint32_t* flag = ws<uint32_t>(c, "pz_flag", static_cast<size_t>(ncell));
    uint32_t* prow = ws<uint32_t>(c, "pz_prow", static_cast<size_t>(ncell));
    uint32_t* tmp = ws<uint32_t>(c, "pz_scan_tmp", scan_tmp_words(ncell) + 8);
    uint32_t* d_total = ws<uint32_t>(c, "pz_total", 4);
    exclusive_scan_u32(hist, start, ncell, tmp, nullptr, st, &c->launches);
    launch_nonempty(hist, ncell, flag, st, &c->launches);
    exclusive_scan_u32(flag, prow, ncell, tmp, d_total, st, &c->launches);
    CUDA_OK(cudaMemcpyAsync(c->h_flag, d_total, 4, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
    check_launch("pillarize cells");
    const int64_t np = static_cast<uint32_t>(*c->h_flag);
    if (!d_coords) return np;
    if (np > cap) throw FwaError{FWA_ERR_SHAPE, "pillarize: output capacity smaller than the pillar count"};
    uint32_t* pcell = ws<uint32_t>(c, "pz_pcell", static_cast<size_t>(np));
    launch_pillar_cells(hist, prow, ncell, min_x, min_y, ry, res, pcell, d_coords, st, &c->launches);
    uint32_t* cursor = ws<uint32_t>(c, "pz_cursor", static_cast<size_t>(ncell));
    CUDA_OK(cudaMemcpyAsync(cursor, start, static_cast<size_t>(ncell) * 4, cudaMemcpyDeviceToDevice, st));
    int32_t* slot = ws<int32_t>(c, "pz_slot", static_cast<size_t>(n));
    const size_t fi = static_cast<size_t>(f_in > 0 ? f_in : 1);
    double* fs = ws<double>(c, "pz_fs", static_cast<size_t>(n) * fi);
    launch_cell_members(cell_id, n, cursor, slot, start, hist, d_feats, f_in, fs, st, &c->launches);
    double* pooled = ws<double>(c, "pz_pooled", static_cast<size_t>(np) * fi);
    launch_pillar_features(pcell, start, hist, np, f_in, fs, pooled, d_w, d_b, d_out, d_out_feats, st,
                           &c->launches);
    check_launch("pillarize features");
    return np;
}

int fwa_b200_positional_embedding_f16(fwa_b200_ctx* c, const double* coords, int64_t n, int32_t d,
                                      uint16_t* out) {
    return guarded(c, [&] {
        if (d < 4 || d % 4 != 0)
            throw FwaError{FWA_ERR_CONFIG, "positional_embedding: d_model must be divisible by 4"};
        if (n == 0) return;
        cudaStream_t st = c->stream;
        double* dc = ws<double>(c, "pe_coords", 2 * static_cast<size_t>(n));
        __half* dp = ws<__half>(c, "pe_out16", static_cast<size_t>(n) * d);
        CUDA_OK(cudaMemcpyAsync(dc, coords, static_cast<size_t>(n) * 16, cudaMemcpyHostToDevice, st));
        launch_positional_embedding(dc, n, d, pe_freq(c, d), nullptr, dp, st, &c->launches);
        check_launch();
        CUDA_OK(cudaMemcpyAsync(out, dp, static_cast<size_t>(n) * d * 2, cudaMemcpyDeviceToHost, st));
        CUDA_OK(cudaStreamSynchronize(st));
    });
}


int fwa_b200_pillarize_device(fwa_b200_ctx* c, const double* d_xy, const double* d_feats, int64_t n, int32_t f_in,
                              double resolution, const double* d_weight, const double* d_bias, int32_t d_out,
                              double* d_coords_out, double* d_feats_out, int64_t capacity, int64_t* n_pillars) {
    return guarded(c, [&] {
        if (!n_pillars) throw FwaError{FWA_ERR_SHAPE, "null n_pillars"};
        *n_pillars = pillarize_device(c, d_xy, d_feats, n, f_in, resolution, d_weight, d_bias, d_out, d_coords_out,
                                      d_feats_out, capacity);
    });
}

int fwa_b200_pillarize(fwa_b200_ctx* c, const double* xy, const double* feats, int64_t n, int32_t f_in,
                       double resolution, const double* weight, const double* bias, int32_t d_out,
                       double* coords_out, double* feats_out, int64_t* n_pillars) {
    return guarded(c, [&] {
        if (!n_pillars || (n > 0 && !xy) || (n > 0 && f_in > 0 && (!feats || !weight)))
            throw FwaError{FWA_ERR_SHAPE, "null buffer"};
        cudaStream_t st = c->stream;
        const size_t un = static_cast<size_t>(n > 0 ? n : 1), fi = static_cast<size_t>(f_in > 0 ? f_in : 1);
        double* dxy = ws<double>(c, "pzh_xy", 2 * un);
        double* df = ws<double>(c, "pzh_f", un * fi);
        double* dw = ws<double>(c, "pzh_w", static_cast<size_t>(d_out > 0 ? d_out : 1) * fi);
        double* db = bias ? ws<double>(c, "pzh_b", static_cast<size_t>(d_out > 0 ? d_out : 1)) : nullptr;
        if (n > 0) {
            CUDA_OK(cudaMemcpyAsync(dxy, xy, static_cast<size_t>(n) * 16, cudaMemcpyHostToDevice, st));
            if (f_in > 0) {
                CUDA_OK(cudaMemcpyAsync(df, feats, static_cast<size_t>(n) * fi * 8, cudaMemcpyHostToDevice, st));
                CUDA_OK(cudaMemcpyAsync(dw, weight, static_cast<size_t>(d_out) * fi * 8, cudaMemcpyHostToDevice, st));
            }
            if (bias) CUDA_OK(cudaMemcpyAsync(db, bias, static_cast<size_t>(d_out) * 8, cudaMemcpyHostToDevice, st));
        }
        double* dco = coords_out ? ws<double>(c, "pzh_co", 2 * un) : nullptr;
        double* dfo = coords_out ? ws<double>(c, "pzh_fo", un * static_cast<size_t>(d_out > 0 ? d_out : 1)) : nullptr;
        const int64_t np = pillarize_device(c, dxy, df, n, f_in, resolution, dw, db, d_out, dco, dfo, n);
        *n_pillars = np;
        if (coords_out && np > 0) {
            CUDA_OK(cudaMemcpyAsync(coords_out, dco, static_cast<size_t>(np) * 16, cudaMemcpyDeviceToHost, st));
            CUDA_OK(cudaMemcpyAsync(feats_out, dfo, static_cast<size_t>(np) * d_out * 8, cudaMemcpyDeviceToHost, st));
        }
        CUDA_OK(cudaStreamSynchronize(st));
    });
}

int fwa_b200_row_checksums(fwa_b200_ctx* c, const float* d_features, int64_t n, int32_t d, double* d_out) {
    return guarded(c, [&] {
        if (n < 0 || d < 1) throw FwaError{FWA_ERR_SHAPE, "row_checksums: bad shape"};
        launch_row_checksums(d_features, n, d, d_out, c->stream, &c->launches);
        check_launch("k_row_checksums");
    });
}


int fwa_b200_equal_window_forward(fwa_b200_ctx* c, const double* d_coords, const float* d_feats, int64_t n,
                                  const fwa_config_t* cfg, const int32_t* edges, int32_t n_edges, float* d_out,
                                  fwa_ew_report_t* rep) {
    return guarded(c, [&] {
        validate_cfg(cfg);
        require_params(c, cfg);
        if (n <= 0) throw FwaError{FWA_ERR_CONFIG, "bench: empty input"};
        if (!edges || n_edges < 1 || n_edges > 8) throw FwaError{FWA_ERR_CONFIG, "padding_cost: no bucket edges"};
        for (int i = 1; i < n_edges; ++i)
            if (edges[i] <= edges[i - 1])
                throw FwaError{FWA_ERR_CONFIG, "padding_cost: bucket edges must be strictly increasing"};
        cudaStream_t st = c->stream;
        const int d = cfg->d_model;
        // ---- partition: the window sort of spec 0 (X axis, no shift), windows in lexicographic order
        int64_t off_h[2] = {0, n};
        int64_t* d_off = ws<int64_t>(c, "ew_off", 2);
        CUDA_OK(cudaMemcpyAsync(d_off, off_h, sizeof(off_h), cudaMemcpyHostToDevice, st));
        const double w_x = cfg->window_px * cfg->resolution, w_y = cfg->window_py * cfg->resolution;
        int32_t* sorted = sort_specs(c, d_coords, n, 1, w_x, w_y, d_off, 1, true);
        const uint32_t* bin_of = ws<uint32_t>(c, "bin_of", static_cast<size_t>(n));
        uint32_t* flag = ws<uint32_t>(c, "ew_flag", static_cast<size_t>(n));
        uint32_t* ex = ws<uint32_t>(c, "ew_ex", static_cast<size_t>(n));
        uint32_t* tmp = ws<uint32_t>(c, "ew_scan_tmp", scan_tmp_words(n) + 8);
        uint32_t* d_cnt = ws<uint32_t>(c, "ew_cnt", 4);
        launch_ew_runs(sorted, bin_of, n, flag, st, &c->launches);
        exclusive_scan_u32(flag, ex, n, tmp, d_cnt, st, &c->launches);
        uint32_t W32 = 0;
        CUDA_OK(cudaMemcpyAsync(&W32, d_cnt, 4, cudaMemcpyDeviceToHost, st));
        CUDA_OK(cudaStreamSynchronize(st));
        const int64_t W = W32;
        uint32_t* wstart = ws<uint32_t>(c, "ew_wstart", static_cast<size_t>(W));
        launch_ew_starts(flag, ex, n, wstart, st, &c->launches);
        int32_t* d_edges = ws<int32_t>(c, "ew_edges", 8);
        CUDA_OK(cudaMemcpyAsync(d_edges, edges, static_cast<size_t>(n_edges) * 4, cudaMemcpyHostToDevice, st));
        uint32_t* wocc = ws<uint32_t>(c, "ew_wocc", static_cast<size_t>(W));
        int32_t* wbucket = ws<int32_t>(c, "ew_wbucket", static_cast<size_t>(W));
        uint32_t* bstat = ws<uint32_t>(c, "ew_bstat", 18);  // bmax[8] | bcnt[8] | overflow
        CUDA_OK(cudaMemsetAsync(bstat, 0, 18 * 4, st));
        launch_ew_bucket(wstart, W, n, d_edges, n_edges, wocc, wbucket, bstat, bstat + 8,
                         reinterpret_cast<int*>(bstat + 16), st, &c->launches);
        uint32_t hb[18];
        std::vector<uint32_t> hocc(static_cast<size_t>(W));
        CUDA_OK(cudaMemcpyAsync(hb, bstat, sizeof(hb), cudaMemcpyDeviceToHost, st));
        CUDA_OK(cudaMemcpyAsync(hocc.data(), wocc, static_cast<size_t>(W) * 4, cudaMemcpyDeviceToHost, st));
        CUDA_OK(cudaStreamSynchronize(st));
        check_launch("equal-window partition");
        if (hb[16]) throw FwaError{FWA_ERR_CONFIG, "bench: occupancy exceeds final bucket edge"};
        // ---- extended inputs: row n = zeros (padding gathers it), row n + 1 = sink for padding outputs
        float* xe = ws<float>(c, "ew_x", static_cast<size_t>(n + 2) * d);
        CUDA_OK(cudaMemcpyAsync(xe, d_feats, static_cast<size_t>(n) * d * 4, cudaMemcpyDeviceToDevice, st));
        CUDA_OK(cudaMemsetAsync(xe + static_cast<size_t>(n) * d, 0, 2 * static_cast<size_t>(d) * 4, st));
        bool any_fast = false, any_slow = false;
        for (int b = 0; b < n_edges; ++b)
            if (hb[8 + b]) {
                const bool f = fast_path_ok(c, d, cfg->n_heads, cfg->d_ff, static_cast<int>(hb[b]));
                any_fast |= f;
                any_slow |= !f;
            }
        __half* pe16 = any_fast ? ws<__half>(c, "ew_pe16", static_cast<size_t>(n + 2) * d) : nullptr;
        float* pe32 = any_slow ? ws<float>(c, "ew_pe32", static_cast<size_t>(n + 2) * d) : nullptr;
        if (pe16) {
            launch_positional_embedding(d_coords, n, d, pe_freq(c, d), nullptr, pe16, st, &c->launches);
            CUDA_OK(cudaMemsetAsync(pe16 + static_cast<size_t>(n) * d, 0, 2 * static_cast<size_t>(d) * 2, st));
        }
        if (pe32) {
            launch_positional_embedding(d_coords, n, d, pe_freq(c, d), pe32, nullptr, st, &c->launches);
            CUDA_OK(cudaMemsetAsync(pe32 + static_cast<size_t>(n) * d, 0, 2 * static_cast<size_t>(d) * 4, st));
        }
        float* oe = ws<float>(c, "ew_out", static_cast<size_t>(n + 2) * d);
        uint32_t* wrank = ws<uint32_t>(c, "ew_wrank", static_cast<size_t>(W));
        CUDA_OK(cudaMemsetAsync(c->d_flag, 0, 2 * sizeof(int), st));
        int64_t rows_padded = 0;
        for (int b = 0; b < n_edges; ++b) {
            const int64_t cnt = hb[8 + b];
            if (!cnt) continue;
            const int pad = static_cast<int>(hb[b]);
            const int64_t rows = cnt * pad;
            rows_padded += rows;
            launch_ew_bflag(wbucket, W, b, flag, st, &c->launches);
            exclusive_scan_u32(flag, wrank, W, tmp, nullptr, st, &c->launches);
            int32_t* ridx = ws<int32_t>(c, "ew_ridx", static_cast<size_t>(rows));
            int32_t* sidx = ws<int32_t>(c, "ew_sidx", static_cast<size_t>(rows));
            launch_ew_fill(wstart, wocc, wbucket, wrank, W, b, pad, sorted, n, ridx, sidx, st, &c->launches);
            fwa_config_t cb = *cfg;
            cb.group_size = pad;
            run_block(c, c->blocks[0], &cb, rows, ridx, xe, nullptr, pe32, pe16, oe, sidx,
                      fast_path_ok(c, d, cfg->n_heads, cfg->d_ff, pad));
        }
        CUDA_OK(cudaMemcpyAsync(d_out, oe, static_cast<size_t>(n) * d * 4, cudaMemcpyDeviceToDevice, st));
        CUDA_OK(cudaMemcpyAsync(c->h_flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, st));
        CUDA_OK(cudaStreamSynchronize(st));
        check_launch("equal-window blocks");
        if (*c->h_flag) throw FwaError{FWA_ERR_NUMERIC, "group_attention: non-finite input"};
        if (rep) {
            // WorkloadReport (workload.hpp:92-142): MACs 2 L^2 D + 4 L D^2 per window
            auto macs = [&](double l) { return 2.0 * l * l * d + 4.0 * l * d * static_cast<double>(d); };
            double act = 0, padded = 0;
            int mx = 0, mn = 1 << 30;
            for (int64_t w = 0; w < W; ++w) {
                const int o = static_cast<int>(hocc[static_cast<size_t>(w)]);
                int b = 0;
                while (b < n_edges && o > edges[b]) ++b;
                act += macs(o);
                padded += macs(hb[b]);
                mx = std::max(mx, o);
                mn = std::min(mn, o);
            }
            *rep = fwa_ew_report_t{};
            rep->n_windows = W;
            rep->max_occ = mx;
            rep->min_nonzero_occ = mn;
            rep->padding_factor = padded / act;
            rep->rows_padded = rows_padded;
            rep->n_buckets = n_edges;
            for (int b = 0; b < n_edges; ++b) {
                rep->bucket_edge[b] = edges[b];
                rep->bucket_pad[b] = static_cast<int32_t>(hb[b]);
                rep->bucket_windows[b] = hb[8 + b];
            }
        }
    });
}


int fwa_b200_block_backward(fwa_b200_ctx* c, const float* f, const float* pe, int64_t rows, int32_t n_groups,
                            const void* record, size_t record_len, const float* grad_out, float* grad_f,
                            void* grad_record) {
    return guarded(c, [&] {
        std::vector<std::vector<float>> keep;
        const auto recs = parse_fwap(record, record_len, keep);
        if (recs.size() != 1) throw FwaError{FWA_ERR_CONFIG, "expected exactly one FWAP record"};
        const Record& r = recs[0];
        const int d = r.d, h = r.h, dff = r.dff;
        if (n_groups < 1 || rows < 1 || rows % n_groups != 0)
            throw FwaError{FWA_ERR_SHAPE, "group_attention: rows not divisible by n_groups"};
        const int G = static_cast<int>(rows / n_groups);
        const std::vector<BlockParams> bp =
            upload_block_params(recs, c->ws["bw_params_f32"], c->ws["bw_params_bf16"], c->stream);
        const BlockParams& P = bp[0];
        cudaStream_t st = c->stream;
        const size_t R = static_cast<size_t>(rows), D = static_cast<size_t>(d), F = static_cast<size_t>(dff);
        auto buf = [&](const char* name, size_t n) { return ws<float>(c, name, n); };
        // inputs
        float* df = buf("bw_f", R * D);
        float* dpe = buf("bw_pe", R * D);
        float* dgo = buf("bw_go", R * D);
        CUDA_OK(cudaMemcpyAsync(df, f, R * D * 4, cudaMemcpyHostToDevice, st));
        CUDA_OK(cudaMemcpyAsync(dpe, pe, R * D * 4, cudaMemcpyHostToDevice, st));
        CUDA_OK(cudaMemcpyAsync(dgo, grad_out, R * D * 4, cudaMemcpyHostToDevice, st));
        // transposed weights for the input gradients (dX = dY W = dY (W^T)^T)
        std::vector<float> tr;
        auto transpose_up = [&](const char* name, const float* hw, int J, int K) {
            tr.assign(static_cast<size_t>(J) * K, 0.f);
            for (int j = 0; j < J; ++j)
                for (int k = 0; k < K; ++k) tr[static_cast<size_t>(k) * J + j] = hw[static_cast<size_t>(j) * K + k];
            float* dw = buf(name, tr.size());
            CUDA_OK(cudaMemcpyAsync(dw, tr.data(), tr.size() * 4, cudaMemcpyHostToDevice, st));
            CUDA_OK(cudaStreamSynchronize(st));  // tr is reused
            return dw;
        };
        const float* hw = r.t;
        const float* h_wqkv = hw;
        const float* h_wout = hw + 3 * D * D + 3 * D;
        const float* h_w1 = h_wout + D * D + D + 4 * D;
        const float* h_w2 = h_w1 + F * D + F;
        float* wqkvT = transpose_up("bw_wqkvT", h_wqkv, 3 * d, d);
        float* woutT = transpose_up("bw_woutT", h_wout, d, d);
        float* w1T = transpose_up("bw_w1T", h_w1, dff, d);
        float* w2T = transpose_up("bw_w2T", h_w2, d, dff);
        // ---- forward with caches (kernels.hpp:447-633)
        float* hb = buf("bw_h", R * D);
        float* xhat1 = buf("bw_xhat1", R * D);
        float* inv1 = buf("bw_inv1", R);
        float* qkv = buf("bw_qkv", R * 3 * D);
        float* probs = buf("bw_probs", static_cast<size_t>(n_groups) * h * G * G);
        float* cat = buf("bw_cat", R * D);
        float* mid = buf("bw_mid", R * D);
        float* ln2 = buf("bw_ln2", R * D);
        float* xhat2 = buf("bw_xhat2", R * D);
        float* inv2 = buf("bw_inv2", R);
        float* u = buf("bw_u", R * F);
        float* a = buf("bw_a", R * F);
        launch_ln_fwd_cache(df, dpe, rows, d, P.ln1_g, P.ln1_b, hb, xhat1, inv1, st, &c->launches);
        GemmArgs g{};
        g.A = hb; g.M = rows; g.K = d; g.W = P.w_qkv; g.N = 3 * d; g.bias = P.b_qkv; g.C = qkv;
        launch_gemm_f32(g, EPI_BIAS, st, &c->launches);
        launch_attn_probs(qkv, n_groups, G, d, h, probs, cat, st, &c->launches);
        g = GemmArgs{};
        g.A = cat; g.M = rows; g.K = d; g.W = P.w_out; g.N = d; g.bias = P.b_out; g.C = mid; g.R = df;
        launch_gemm_f32(g, EPI_RESID_GATHER, st, &c->launches);
        launch_ln_fwd_cache(mid, nullptr, rows, d, P.ln2_g, P.ln2_b, ln2, xhat2, inv2, st, &c->launches);
        g = GemmArgs{};
        g.A = ln2; g.M = rows; g.K = d; g.W = P.w1; g.N = dff; g.bias = P.b1; g.C = u;
        launch_gemm_f32(g, EPI_BIAS, st, &c->launches);
        launch_gelu_fwd(u, static_cast<int64_t>(R * F), a, st, &c->launches);
        // ---- backward (kernels.hpp:681-764)
        const int nc = reduce_chunks(rows);
        float* part = buf("bw_part", static_cast<size_t>(nc) * static_cast<size_t>(std::max(3 * d * d, dff * d)));
        const size_t rec_f = record_floats(d, dff);
        float* gp = buf("bw_gparams", rec_f);  // FWAP field order
        float* g_wqkv = gp;
        float* g_bqkv = g_wqkv + 3 * D * D;
        float* g_wout = g_bqkv + 3 * D;
        float* g_bout = g_wout + D * D;
        float* g_ln1g = g_bout + D;
        float* g_ln1b = g_ln1g + D;
        float* g_ln2g = g_ln1b + D;
        float* g_ln2b = g_ln2g + D;
        float* g_w1 = g_ln2b + D;
        float* g_b1 = g_w1 + F * D;
        float* g_w2 = g_b1 + F;
        float* g_b2 = g_w2 + D * F;
        float* ga = buf("bw_ga", R * F);
        float* gu = buf("bw_gu", R * F);
        float* gln2 = buf("bw_gln2", R * D);
        float* gfp = buf("bw_gfp", R * D);
        float* tmp = buf("bw_tmp", R * D);
        float* gcat = buf("bw_gcat", R * D);
        float* gqkv = buf("bw_gqkv", R * 3 * D);
        float* gh = buf("bw_gh", R * D);
        float* gfo = buf("bw_gfo", R * D);
        // FFN sublayer
        launch_colsum(dgo, rows, d, part, g_b2, st, &c->launches);
        launch_wgrad(dgo, a, rows, d, dff, part, g_w2, st, &c->launches);
        g = GemmArgs{};
        g.A = dgo; g.M = rows; g.K = d; g.W = w2T; g.N = dff; g.C = ga;  // g_a = dY W2
        launch_gemm_f32(g, EPI_BIAS, st, &c->launches);
        launch_gelu_back(ga, u, static_cast<int64_t>(R * F), gu, st, &c->launches);
        launch_colsum(gu, rows, dff, part, g_b1, st, &c->launches);
        launch_wgrad(gu, ln2, rows, dff, d, part, g_w1, st, &c->launches);
        g = GemmArgs{};
        g.A = gu; g.M = rows; g.K = dff; g.W = w1T; g.N = d; g.C = gln2;  // g_ln2 = g_u W1
        launch_gemm_f32(g, EPI_BIAS, st, &c->launches);
        launch_ln_back(gln2, xhat2, inv2, P.ln2_g, rows, d, dgo, gfp, tmp, st, &c->launches);  // + residual
        launch_colsum(tmp, rows, d, part, g_ln2g, st, &c->launches);
        launch_colsum(gln2, rows, d, part, g_ln2b, st, &c->launches);
        // attention sublayer
        launch_colsum(gfp, rows, d, part, g_bout, st, &c->launches);
        launch_wgrad(gfp, cat, rows, d, d, part, g_wout, st, &c->launches);
        g = GemmArgs{};
        g.A = gfp; g.M = rows; g.K = d; g.W = woutT; g.N = d; g.C = gcat;
        launch_gemm_f32(g, EPI_BIAS, st, &c->launches);
        if (!launch_attn_back(qkv, probs, gcat, n_groups, G, d, h, gqkv, st, &c->launches))
            throw FwaError{FWA_ERR_CONFIG, "block_backward: group size too large"};
        launch_colsum(gqkv, rows, 3 * d, part, g_bqkv, st, &c->launches);
        launch_wgrad(gqkv, hb, rows, 3 * d, d, part, g_wqkv, st, &c->launches);
        g = GemmArgs{};
        g.A = gqkv; g.M = rows; g.K = 3 * d; g.W = wqkvT; g.N = d; g.C = gh;
        launch_gemm_f32(g, EPI_BIAS, st, &c->launches);
        launch_ln_back(gh, xhat1, inv1, P.ln1_g, rows, d, gfp, gfo, tmp, st, &c->launches);  // grad_f
        launch_colsum(tmp, rows, d, part, g_ln1g, st, &c->launches);
        launch_colsum(gh, rows, d, part, g_ln1b, st, &c->launches);
        check_launch("block_backward");
        CUDA_OK(cudaMemcpyAsync(grad_f, gfo, R * D * 4, cudaMemcpyDeviceToHost, st));
        if (grad_record) {
            std::memcpy(grad_record, record, 16);  // FWAP magic + dims
            CUDA_OK(cudaMemcpyAsync(static_cast<uint8_t*>(grad_record) + 16, gp, rec_f * 4, cudaMemcpyDeviceToHost,
                                    st));
        }
        CUDA_OK(cudaStreamSynchronize(st));
    });
}

} // extern "C"
