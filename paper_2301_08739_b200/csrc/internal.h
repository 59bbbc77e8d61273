// Internal launcher declarations shared by the driver (fwa_b200.cu) and the
// kernel translation units.  Not part of the C ABI.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace fwa_b200 {

struct LaunchCounter {
    int64_t* n;
    void operator++() const { ++*n; }
};

// ------------------------------------------------------------------ scan
// Exclusive prefix sum of n uint32 values (in -> out, may alias), total
// written to *d_total if non-null.  tmp must hold scan_tmp_words(n) words.
size_t scan_tmp_words(int64_t n);
void exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* tmp,
                        uint32_t* d_total, cudaStream_t s, int64_t* launches);

// ------------------------------------------------------------------ sort (flatten.hpp:49-120)
// Spec s in [0,4): axis Y iff s >= 2, shift iff s odd (block_schedule,
// flatten.hpp:150-161: block b uses spec b % 4).
struct SpecBins {
    long long min_major, min_minor;
    long long range_minor;      // max_minor - min_minor + 1
    long long bins_per_frame;   // range_major * range_minor
    long long base;             // first global bin id of this spec
};

// writes per-CTA window min/max partials ([spec][sort_keys_partials(ntot)][4]); with
// BinsFuse::ticket set, the last CTA also does launch_bins_setup's work
int64_t sort_keys_partials(int64_t ntot);
struct BinsFuse {
    unsigned* ticket = nullptr;  // zero-initialised once; reset by the kernel
    int nf = 1;
    long long cap = 0;
    long long* mm = nullptr;
    SpecBins* specs = nullptr;
    uint32_t* d_nbins = nullptr;
    int* overflow = nullptr;
    uint32_t* large = nullptr;   // reset to 0 (launch_bin_sort's queue counter)
};
void launch_sort_keys(const double* coords, int64_t ntot, int n_specs, double w_x, double w_y,
                      long long* win, double* loc, long long* partials, cudaStream_t s,
                      int64_t* launches, const BinsFuse& fz = BinsFuse{});
// d_nbins (may be null): device-side bin count of the sync-free path; 0 disables
void launch_bins_hist(const long long* win, int64_t ntot, int n_specs, const int64_t* d_frame_off,
                      int n_frames, const SpecBins* d_specs, uint32_t* bin_of, uint32_t* hist,
                      const uint32_t* d_nbins, cudaStream_t s, int64_t* launches, bool per_frame = false);
// exact path: window min/max per (spec, frame) -> mm[(s * nf + f) * 4 + {min_M, max_M, min_m, max_m}]
void launch_frame_minmax(const long long* win, int64_t ntot, int n_specs, const int64_t* d_frame_off, int n_frames,
                         long long* mm, cudaStream_t s, int64_t* launches);
// exact path, window ranges too wide for dense bins: bin_of[e] = dense rank of e's window
// (spec, frame, win_major, win_minor) by a stable 3-pass radix sort; *d_count = windows;
// hist (zeroed, capacity total) receives the per-window counts
size_t window_ranks_temp_bytes(int64_t total);
void launch_window_ranks(const long long* win, int64_t ntot, int n_specs, const int64_t* d_frame_off, int n_frames,
                         unsigned long long* k64a, unsigned long long* k64b, uint32_t* va, uint32_t* vb,
                         uint32_t* flag, uint32_t* ex, uint32_t* scan_tmp, uint32_t* d_count, void* temp,
                         size_t temp_bytes, uint32_t* bin_of, uint32_t* hist, cudaStream_t s, int64_t* launches);
// reduces the key partials -> mm[4*n_specs] (min/max per spec), bin specs, *d_nbins
// (0 + *overflow = 1 when the dense range exceeds cap)
void launch_bins_setup(const long long* partials, int64_t n_part, int n_specs, int nf, long long cap,
                       long long* mm, SpecBins* specs, uint32_t* d_nbins, int* overflow, cudaStream_t s,
                       int64_t* launches);
void launch_zero_bins(uint32_t* hist, const uint32_t* d_nbins, cudaStream_t s, int64_t* launches);
// per-frame dense bins of a frame batch from launch_frame_minmax's (spec, frame) ranges
void launch_bins_setup_frames(const long long* mm, int n_specs, int nf, long long cap, SpecBins* specs,
                              uint32_t* d_nbins, int* overflow, cudaStream_t s, int64_t* launches);
// tile-local exclusive scan; tile_sums becomes the per-4096-bin tile offsets the
// consumers add (tile_off below); ticket: zero-initialised, self-resetting
void launch_scan_bins_dev(const uint32_t* hist, uint32_t* bin_start, uint32_t* cursor, const uint32_t* d_nbins,
                          long long cap, uint32_t* tile_sums, unsigned* ticket, cudaStream_t s,
                          int64_t* launches);
// pre[pos] = id, pre_loc[pos] = (integer key images of loc_major, loc_minor) as 2 x u64,
// pre_bin[pos] = window bin, pos = the element's slot in its bin
void launch_bin_scatter(const uint32_t* bin_of, const double* loc, int64_t ntot, int n_specs,
                        uint32_t* cursor, int32_t* pre, double* pre_loc, const uint32_t* d_nbins,
                        const uint32_t* tile_off, uint32_t* pre_bin, cudaStream_t s, int64_t* launches);
// also writes the inverse permutation inv[s*ntot + id] = position in sorted
// zeroes hist[] as it consumes it (the sync-free path relies on a clean histogram)
void launch_bin_sort(const uint32_t* bin_start, uint32_t* hist, uint32_t n_bins,
                     const int32_t* pre, const double* pre_loc, const uint32_t* pre_bin, const double* loc,
                     int64_t ntot, int n_specs, int32_t* sorted, int32_t* inv, int32_t* scratch,
                     uint32_t* large /* 1 + n_bins words */, const uint32_t* d_nbins,
                     const uint32_t* tile_off, cudaStream_t s, int64_t* launches);
constexpr int kMaxDropTable = 8192;
void launch_drop_tables(const int32_t* sorted0, int n, const int64_t* frame_off, const int64_t* rows,
                        const int64_t* drop_off, int n_frames, const int32_t* inv, int64_t ntot, int n_specs,
                        int32_t* dropped_ids, int32_t* drop_sorted, int32_t* drop_pos, cudaStream_t s,
                        int64_t* launches);
void launch_compact_all(const int32_t* sorted, int64_t ntot, int n_specs, const int64_t* frame_off,
                        const int64_t* drop_off, int n_frames, const int32_t* drop_sorted,
                        const int32_t* drop_pos, int n_drop, int64_t K, int s_last, int32_t* idx,
                        uint32_t* kept_rank, int32_t* kept_ids, int32_t* out_pos, cudaStream_t s,
                        int64_t* launches, const int32_t* fuse_inv = nullptr, int32_t* fuse_dropped_ids = nullptr);
constexpr int kFuseDrops = 256;  // one frame with at most this many drops: the drop tables inside compaction

// ------------------------------------------------------------------ schedule (backbone.hpp:236-316)
void launch_drop_mark(const int32_t* sorted0, int64_t ntot, const int64_t* d_frame_off,
                      const int64_t* d_rows, const int64_t* d_drop_off, int n_frames,
                      uint8_t* dropped, int32_t* dropped_ids, cudaStream_t s, int64_t* launches);
void launch_keep_flags(const uint8_t* dropped, int64_t ntot, uint32_t* flags, cudaStream_t s,
                       int64_t* launches);
void launch_kept_ids(const uint32_t* kept_rank, const uint8_t* dropped, int64_t ntot,
                     int32_t* kept_ids, cudaStream_t s, int64_t* launches);
void launch_spec_keep_flags(const int32_t* sorted, int64_t total, const uint8_t* dropped,
                            uint32_t* flags, cudaStream_t s, int64_t* launches);
void launch_spec_compact(const int32_t* sorted, int64_t total, const uint8_t* dropped,
                         const uint32_t* pos, int32_t* idx, cudaStream_t s, int64_t* launches);

// ------------------------------------------------------------------ fp32 SIMT path (check mode)
// f32 PE (pe != nullptr) and/or fp16 PE rows (pe16 != nullptr, the bf16 fast path's copy)
void launch_positional_embedding(const double* coords, int64_t n, int d, const double* d_freq,
                                 float* pe, __half* pe16, cudaStream_t s, int64_t* launches);
void launch_prefetch_l2(const void* p, int64_t bytes, cudaStream_t s, int64_t* launches);
void launch_row_checksums(const float* f, int64_t n, int d, double* out, cudaStream_t s, int64_t* launches);
void launch_f32_to_f16(const float* in, int64_t n, __half* out, cudaStream_t s, int64_t* launches);
// h[r] = LN1(x[idx[r]]) * g + b + pe[idx[r]]  (x f32, or f64 when x64 != nullptr)
void launch_ln_gather_f32(const float* x, const double* x64, const float* pe, const int32_t* idx,
                          int64_t rows, int d, const float* gamma, const float* beta,
                          float* h, int* d_nonfinite, cudaStream_t s, int64_t* launches);
void launch_ln_rows_f32(const float* x, int64_t rows, int d, const float* gamma,
                        const float* beta, float* out, cudaStream_t s, int64_t* launches);

enum GemmEpi {
    EPI_BIAS = 0,          // C = A W^T + b
    EPI_BIAS_GELU = 1,     // C = gelu(A W^T + b)
    EPI_RESID_GATHER = 2,  // C[r] = (R[ridx[r]] + A W^T) + b   (kernels.hpp:559 order)
    EPI_RESID_SCATTER = 3  // D[sidx[r]] = R[r] + (A W^T + b)    (kernels.hpp:612-614)
};
struct GemmArgs {
    const float* A; int64_t M; int K;
    const float* W; int N;         // W: N x K row-major (out x in)
    const float* bias;
    float* C;                      // M x N (EPI_BIAS/GELU/RESID_GATHER)
    const float* R; const double* R64; const int32_t* ridx;  // residual (gather) source
    float* D; const int32_t* sidx;                           // scatter destination
};
void launch_gemm_f32(const GemmArgs& a, GemmEpi epi, cudaStream_t s, int64_t* launches);
void launch_attention_f32(const float* qkv, int64_t rows, int G, int d, int heads, float* cat,
                          cudaStream_t s, int64_t* launches);

// ------------------------------------------------------------------ bf16 tensor-core path
// Fast path: d_model 128, d_ff 256, head dim 16, group_size <= 128.
struct TcBlockWeights {
    const __nv_bfloat16* w_qkv; // 384 x 128, pre-swizzled UMMA K-major SW128 image
    const __nv_bfloat16* w_out; // 128 x 128, swizzled
    const __nv_bfloat16* w1;    // 256 x 128, swizzled, LN2 gamma folded in (W1 diag(g2))
    const __nv_bfloat16* w2;    // 128 x 256, swizzled
    const float* vec;           // [b_qkv 384 | b_out 128 | b2 128 | b1 + W1 b2ln 256]
    const float *ln1_g, *ln1_b;
    // CTA-pair images for the fused block kernel: [rank 0 | rank 1], 128 KB each; rank v
    // holds output-feature rows [64v, 64v+64) of every 128-row weight chunk:
    // W_qkv chunks q,k,v (3 x 16 KB) | W_out (16 KB) | W1' halves (2 x 16 KB) | W2 (32 KB)
    const uint8_t* w_pair;
    // the fused kernel's vectors: [b_qkv' 384 | b_out 128 | b2 128 | b1' 256 | ln1_g 128 | 0 128]
    // with LN1's beta folded into b_qkv' (+ W_qkv beta1) and the Q rows (W_q in w_pair, b_q')
    // pre-scaled by log2(e) / sqrt(16) -- the attention's base-2 exponent
    const float* vec_pair;
};
// Host-side: write the UMMA SW128 K-major smem image of a row-major f32
// [rows x k] weight as bf16 (rows multiple of 8, k multiple of 64).
void swizzle_weight_bf16(const float* w, int rows, int k, uint16_t* out);

void launch_ln1_qkv_tc(const float* x, const double* x64, const __half* pe16, const int32_t* idx,
                       int64_t rows, const TcBlockWeights& w, __nv_bfloat16* qkv,
                       int* d_nonfinite, float* xq /* optional tile-transposed x copy */, cudaStream_t s,
                       int64_t* launches, unsigned long long* trace = nullptr);
void launch_attention_mma(const __nv_bfloat16* qkv, int64_t rows, int G, __nv_bfloat16* cat,
                          cudaStream_t s, int64_t* launches);
// x_out[sidx[r]] = FFN-block(x_in[ridx[r]] + cat[r] Wout^T + b_out)
void launch_outproj_ffn_tc(const __nv_bfloat16* cat, const float* x_in, const double* x_in64,
                           const int32_t* ridx, int64_t rows, const TcBlockWeights& w,
                           float* x_out, const int32_t* sidx, const float* xq, cudaStream_t s,
                           int64_t* launches, unsigned long long* trace = nullptr);

// One whole block (gather .. scatter) in one persistent kernel on CTA pairs
// (block_fused.cu); supported group sizes: see block_fused_supported.
bool block_fused_supported(int G);
// false: the x-row tensor map could not be encoded (nothing launched)
bool launch_block_fused(const float* x, const double* x64, const __half* pe16, const int32_t* ridx,
                        const int32_t* sidx, float* x_out, int64_t rows, int G, const TcBlockWeights& w,
                        int* d_nonfinite, cudaStream_t s, int64_t* launches,
                        unsigned long long* trace = nullptr, unsigned long long* phase = nullptr,
                        float* const* peers = nullptr, int n_peers = 0);  // peers: DEVICE array of 8 pointers
// BackboneParams::input_proj (backbone.hpp:179-190), bit-exact: out[r][j] = bias[j] +
// sum_c w[j][c] * (float)x[r][c], fp32, c in order, no FMA contraction
void launch_input_proj(const void* x, bool x_f64, int64_t n, int f_in, const float* w, const float* b,
                       int d, float* out, cudaStream_t s, int64_t* launches);
// host: the per-rank pair images (2 x 128 KB) of one block's weights (W1 LN2-folded)
void build_pair_images(const float* w_qkv, const float* w_out, const float* w1f, const float* w2,
                       uint16_t* out /* 2 * 65536 bf16 */);

// ------------------------------------------------------------------ pillarization (pillarize.cu)
void launch_cell_keys(const double* xy, int64_t n, double res, long long* cell, long long* mm, cudaStream_t s,
                      int64_t* launches);
void launch_cell_hist(const long long* cell, int64_t n, long long min_x, long long min_y, long long range_y,
                      uint32_t* cell_id, uint32_t* hist, cudaStream_t s, int64_t* launches);
void launch_nonempty(const uint32_t* hist, int64_t ncell, uint32_t* flag, cudaStream_t s, int64_t* launches);
void launch_pillar_cells(const uint32_t* hist, const uint32_t* prow, int64_t ncell, long long min_x, long long min_y,
                         long long range_y, double res, uint32_t* pcell, double* coords, cudaStream_t s,
                         int64_t* launches);
void launch_cell_members(const uint32_t* cell_id, int64_t n, uint32_t* cursor, int32_t* slot_pt,
                         const uint32_t* start, const uint32_t* hist, const double* feats, int f_in, double* fs,
                         cudaStream_t s, int64_t* launches);
void launch_pillar_features(const uint32_t* pcell, const uint32_t* start, const uint32_t* hist, int64_t np,
                            int f_in, const double* fs, double* pooled, const double* w, const double* bias,
                            int d_out, double* out, cudaStream_t s, int64_t* launches);

// ------------------------------------------------------------------ equal-window baseline (equal_window.cu)
void launch_ew_runs(const int32_t* sorted, const uint32_t* bin_of, int64_t n, uint32_t* flag, cudaStream_t s,
                    int64_t* launches);
void launch_ew_starts(const uint32_t* flag, const uint32_t* ex, int64_t n, uint32_t* wstart, cudaStream_t s,
                      int64_t* launches);
void launch_ew_bucket(const uint32_t* wstart, int64_t W, int64_t n, const int32_t* edges, int n_edges, uint32_t* wocc,
                      int32_t* wbucket, uint32_t* bmax, uint32_t* bcnt, int* overflow, cudaStream_t s,
                      int64_t* launches);
void launch_ew_bflag(const int32_t* wbucket, int64_t W, int b, uint32_t* flag, cudaStream_t s, int64_t* launches);
void launch_ew_fill(const uint32_t* wstart, const uint32_t* wocc, const int32_t* wbucket, const uint32_t* wrank,
                    int64_t W, int b, int pad, const int32_t* sorted, int64_t n, int32_t* ridx, int32_t* sidx,
                    cudaStream_t s, int64_t* launches);

// ------------------------------------------------------------------ block backward (backward.cu)
void launch_ln_fwd_cache(const float* x, const float* pe, int64_t rows, int d, const float* g, const float* b,
                         float* y, float* xhat, float* inv_std, cudaStream_t s, int64_t* launches);
void launch_attn_probs(const float* qkv, int64_t n_groups, int G, int d, int heads, float* probs, float* cat,
                       cudaStream_t s, int64_t* launches);
void launch_gelu_fwd(const float* u, int64_t n, float* a, cudaStream_t s, int64_t* launches);
void launch_gelu_back(const float* ga, const float* u, int64_t n, float* gu, cudaStream_t s, int64_t* launches);
void launch_ln_back(const float* gy, const float* xhat, const float* inv_std, const float* gamma, int64_t rows,
                    int d, const float* add, float* gx, float* gy_xhat, cudaStream_t s, int64_t* launches);
bool launch_attn_back(const float* qkv, const float* probs, const float* gcat, int64_t n_groups, int G, int d,
                      int heads, float* gqkv, cudaStream_t s, int64_t* launches);
int reduce_chunks(int64_t rows);
void launch_wgrad(const float* dy, const float* x, int64_t rows, int J, int K, float* part, float* dw, cudaStream_t s,
                  int64_t* launches);
void launch_colsum(const float* y, int64_t rows, int J, float* part, float* out, cudaStream_t s, int64_t* launches);
void launch_mul(const float* a, const float* b, int64_t n, float* out, cudaStream_t s, int64_t* launches);

// ------------------------------------------------------------------ misc
void launch_scatter_rows(const float* src, const int32_t* ids, const uint32_t* rank, int64_t n,
                         int d, float* dst, cudaStream_t s, int64_t* launches);
// dst[pos[r]] = src[r] for r < n (d % 4 == 0)
void launch_scatter_sorted(const float* src, const int32_t* pos, int64_t n, int d, float* dst, cudaStream_t s,
                           int64_t* launches);

} // namespace fwa_b200
