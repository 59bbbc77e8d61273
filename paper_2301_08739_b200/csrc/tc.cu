// tcgen05/TMEM kernels of the bf16 fast path (d_model 128, d_ff 256, head dim 16).
//
//   k_ln1_qkv_tc:      gather rows by the block's window-sort permutation +
//                      LN1 + affine + PE (kernels.hpp:472-485) -> bf16 A tile in
//                      SW128 shared memory -> packed QKV GEMM (kernels.hpp:488-500)
//                      on the 5th-gen tensor cores, fp32 accumulate in TMEM ->
//                      +bias -> bf16 q|k|v rows.
//   k_outproj_ffn_tc:  out-proj + b_out + gathered fp32 residual (kernels.hpp:550-560)
//                      -> LN2 (575-600) -> W1 + b1 -> exact-erf GELU -> W2 + b2 ->
//                      + residual (601-614) -> scatter to the pillar-id row
//                      (backbone.hpp:276-283).  Three chained tcgen05 GEMMs per
//                      128-row tile, all weights resident in shared memory
//                      (TMA bulk-loaded once per persistent CTA), the post-attention
//                      residual held in registers between them.
//
// Persistent CTAs (one per SM, 128-row tiles), one elected thread issues the
// MMAs, completion via tcgen05.commit -> mbarrier.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include <cstring>

#include "common.cuh"
#include "internal.h"
#include "tcgen05.cuh"

namespace fwa_b200 {

using namespace tc;

// ------------------------------------------------------------------ host: weight images

static uint16_t f32_to_bf16_rn(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return static_cast<uint16_t>((u >> 16) | 0x40);  // NaN
    const uint32_t lsb = (u >> 16) & 1u;
    u += 0x7fffu + lsb;
    return static_cast<uint16_t>(u >> 16);
}

void swizzle_weight_bf16(const float* w, int rows, int k, uint16_t* out) {
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < k; ++c)
            out[sw128_offset(r, c, rows) / 2] = f32_to_bf16_rn(w[static_cast<size_t>(r) * k + c]);
}

static uint16_t f32_to_f16_rn(float f) {
    const __half h = __float2half_rn(f);
    return *reinterpret_cast<const uint16_t*>(&h);
}
static void swizzle_weight_f16(const float* w, int rows, int k, uint16_t* out) {
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < k; ++c)
            out[sw128_offset(r, c, rows) / 2] = f32_to_f16_rn(w[static_cast<size_t>(r) * k + c]);
}

void build_pair_images(const float* w_qkv, const float* w_out, const float* w1f, const float* w2,
                       uint16_t* out) {
    // the fused kernel's GELU omits its factor 1/2 (x (1 + tanh g) instead of x/2 (1 + tanh g)):
    // W2 carries it (exact: a power of two)
    std::vector<float> w2h(w2, w2 + 128 * 256);
    for (float& v : w2h) v *= 0.5f;
    w2 = w2h.data();
    for (int v = 0; v < 2; ++v) {
        uint16_t* o = out + v * 65536;  // 128 KB per rank
        for (int c = 0; c < 3; ++c) swizzle_weight_bf16(w_qkv + (128 * c + 64 * v) * 128, 64, 128, o + c * 8192);
        swizzle_weight_bf16(w_out + 64 * v * 128, 64, 128, o + 24576);
        for (int h = 0; h < 2; ++h) swizzle_weight_bf16(w1f + (128 * h + 64 * v) * 128, 64, 128, o + 32768 + h * 8192);
        swizzle_weight_f16(w2 + 64 * v * 256, 64, 256, o + 49152);  // fp16: the GELU activations are fp16
    }
}

// Phase tracing (FWA_B200_TRACE=1): SM clock at phase boundaries, 64 slots per CTA.
#define FWA_TR(k)                                                                         \
    do {                                                                                  \
        if (trace) trace[blockIdx.x * 64 + (k)] = static_cast<unsigned long long>(clock64()); \
    } while (0)

// pointer arithmetic on the extern __shared__ array keeps the shared address space
// visible to the compiler (STS/LDS instead of generic ST/LD)
FWA_DEVINL uint8_t* align1024(uint8_t* p) { return p + ((1024u - (smem_u32(p) & 1023u)) & 1023u); }

// ------------------------------------------------------------------ K_a: gather + LN1 + PE + QKV
//
// Warp-specialised persistent kernel, 16 warps:
//   warps 0-11  producers: a 128-row tile is 32 passes of 4 rows (8 lanes per row, each
//              lane 16 channels 32i + 4*sub + e, so every load instruction reads whole
//              128 B lines: 64 B of fp32 x, 32 B of fp16 PE per lane), passes w, w+12,
//              w+24 per warp software-pipelined (pass k+1 in flight while pass k is
//              reduced), pillar ids of the NEXT tile prefetched; LN1 + affine + PE in
//              fp32 -> bf16 SW128 A tile; the gathered fp32 row also goes to the
//              tile-transposed residual copy xq.  A is double-buffered.
//   warps 12-15 MMA issue (one elected thread) + epilogue (TMEM lane quarter each):
//              TMEM -> +bias -> bf16 rows staged in shared memory -> one bulk TMA store
//              per (tile, column chunk): the chunk-major q|k|v layout (12 chunks of
//              [rows x 32]) makes each such block 8 KB contiguous, and the attention
//              kernel reads each group's rows as contiguous runs.
// mbarriers: full[s] (12 producer warps), empty[s] (tcgen05.commit), done (commit).

constexpr int kQkvW = 384 * 128 * 2;   // 98304 B weight image
constexpr int kTileA = 128 * 128 * 2;  // 32768 B per A stage
constexpr int kQkvThreads = 512;
constexpr int kQkvProd = 12;  // producer warps; the remaining 4 drain TMEM (MMA issue: the first of them)
constexpr int kQkvStage = 2 * 16384;  // 2 x (2 chunks x 128 rows x 64 B) qkv store staging
constexpr int kQkvSmem = kQkvW + 2 * kTileA + kQkvStage + (384 + 256) * 4 /*bias, ln1 g|b*/ + 128 /*bars*/ + 1024;

// One lane's 16 channels of a row: channels 32i + 4*sub + e (i, e < 4), so each load
// instruction of the 8 lanes sharing a row reads one contiguous 128 B line of the fp32
// row (64 B of the fp16 PE row).
template <bool kF64>
FWA_DEVINL void load_row_quads(const float* x, const double* x64, const __half* pe16, int64_t id,
                               int sub, bool valid, float (&v)[16], uint2 (&ph)[4]) {
    if (!valid) {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i) ph[i] = make_uint2(0u, 0u);
        return;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (kF64) {
            const double2* p = reinterpret_cast<const double2*>(x64 + id * 128 + 32 * i + 4 * sub);
            const double2 d0 = __ldg(p), d1 = __ldg(p + 1);
            v[4 * i] = static_cast<float>(d0.x); v[4 * i + 1] = static_cast<float>(d0.y);
            v[4 * i + 2] = static_cast<float>(d1.x); v[4 * i + 3] = static_cast<float>(d1.y);
        } else {
            const float4 f4 = __ldg(reinterpret_cast<const float4*>(x + id * 128 + 32 * i + 4 * sub));
            v[4 * i] = f4.x; v[4 * i + 1] = f4.y; v[4 * i + 2] = f4.z; v[4 * i + 3] = f4.w;
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) ph[i] = __ldg(reinterpret_cast<const uint2*>(pe16 + id * 128 + 32 * i + 4 * sub));
}

// LN1 (two-pass, 8 lanes per row) + affine + PE -> 4 x 8 B of the bf16 SW128 A image.
FWA_DEVINL void ln1_row_to_tile(const float (&v)[16], const uint2 (&ph)[4], bool valid, int r, int sub,
                                const float* sG, const float* sB, uint8_t* A, bool& bad) {
    float sm = 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) sm += v[j];
    sm += __shfl_xor_sync(0xffffffffu, sm, 1);
    sm += __shfl_xor_sync(0xffffffffu, sm, 2);
    sm += __shfl_xor_sync(0xffffffffu, sm, 4);
    const float mean = sm * (1.0f / 128.0f);
    float sq = 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        bad |= !isfinite(v[j]);
        sq += (v[j] - mean) * (v[j] - mean);
    }
    sq += __shfl_xor_sync(0xffffffffu, sq, 1);
    sq += __shfl_xor_sync(0xffffffffu, sq, 2);
    sq += __shfl_xor_sync(0xffffffffu, sq, 4);
    const float inv = 1.0f / sqrtf(sq * (1.0f / 128.0f) + 1e-5f);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int c = 32 * i + 4 * sub;
        const float4 g = *reinterpret_cast<const float4*>(sG + c);
        const float4 b = *reinterpret_cast<const float4*>(sB + c);
        const float2 p0 = __half22float2(*reinterpret_cast<const __half2*>(&ph[i].x));
        const float2 p1 = __half22float2(*reinterpret_cast<const __half2*>(&ph[i].y));
        bad |= !(isfinite(p0.x) && isfinite(p0.y) && isfinite(p1.x) && isfinite(p1.y));
        uint32_t o0 = pack_bf16x2(g.x * ((v[4 * i] - mean) * inv) + b.x + p0.x,
                                  g.y * ((v[4 * i + 1] - mean) * inv) + b.y + p0.y);
        uint32_t o1 = pack_bf16x2(g.z * ((v[4 * i + 2] - mean) * inv) + b.z + p1.x,
                                  g.w * ((v[4 * i + 3] - mean) * inv) + b.w + p1.y);
        if (!valid) o0 = o1 = 0u;
        *reinterpret_cast<uint2*>(A + sw128_offset(r, c, 128)) = make_uint2(o0, o1);
    }
}

FWA_DEVINL uint4 pick4(const uint4 (&P)[4], int j) {
    const uint4 a = (j & 1) ? P[1] : P[0];
    const uint4 b = (j & 1) ? P[3] : P[2];
    return (j & 2) ? b : a;
}

template <bool kF64>
__global__ void __launch_bounds__(kQkvThreads, 1)
    k_ln1_qkv_tc(const float* __restrict__ x, const double* __restrict__ x64,
                 const __half* __restrict__ pe16, const int32_t* __restrict__ idx, int64_t rows,
                 TcBlockWeights w, __nv_bfloat16* __restrict__ qkv, int* __restrict__ nonfinite,
                 float* __restrict__ xq, unsigned long long* __restrict__ trace) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    uint8_t* sW = smem;
    uint8_t* sA = smem + kQkvW;                                        // 2 stages
    uint8_t* sStage = sA + 2 * kTileA;                                 // 2 staging buffers
    float* sBias = reinterpret_cast<float*>(sStage + kQkvStage);       // 384
    float* sG = sBias + 384;                                           // 128
    float* sB = sG + 128;                                              // 128
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + 128);            // wbar, full[2], empty[2], done
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 6);
    uint64_t* wbar = bars;
    uint64_t* full = bars + 1;
    uint64_t* empty = bars + 3;
    uint64_t* done = bars + 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    griddep_launch_dependents();
    if (threadIdx.x == 0) {
        mbar_init(wbar, 1);
        mbar_init(&full[0], kQkvProd);
        mbar_init(&full[1], kQkvProd);
        mbar_init(&empty[0], 1);
        mbar_init(&empty[1], 1);
        mbar_init(done, 1);
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < 384; i += blockDim.x) sBias[i] = w.vec[i];
    for (int i = threadIdx.x; i < 128; i += blockDim.x) {
        sG[i] = w.ln1_g[i];
        sB[i] = w.ln1_b[i];
    }
    if (warp == kQkvProd) {
        __syncwarp();
        tmem_alloc(tmem_slot, 512);
    }
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tmem = *tmem_slot;
    const int64_t ntiles = (rows + 127) / 128;

    if (warp < kQkvProd) {
        // ------------------------------------------------ producers
        if (threadIdx.x == 0) {
            mbar_arrive_expect_tx(wbar, kQkvW);
#pragma unroll
            for (int c = 0; c < 3; ++c)
                bulk_g2s(sW + c * 32768, reinterpret_cast<const uint8_t*>(w.w_qkv) + c * 32768, 32768, wbar);
        }
        bool bad = false;
        if (threadIdx.x == 0) FWA_TR(0);
        griddep_wait();  // x / PE / ids come from earlier kernels
        const int sub = lane & 7, rl = lane >> 3;  // 8 lanes per row, 4 rows per pass
        // 32 passes of 4 rows per tile over kQkvProd warps: warp w owns passes w, w+P, w+2P
        constexpr int kMaxPass = (32 + kQkvProd - 1) / kQkvProd;
        const int n_my = (32 - warp + kQkvProd - 1) / kQkvProd;
        auto pass_id = [&](int64_t tile, int p) {
            const int64_t g = tile * 128 + p * 4 + rl;
            return (tile < ntiles && p < 32 && g < rows) ? (idx ? idx[g] : static_cast<int>(g)) : 0;
        };
        int ids[kMaxPass];
#pragma unroll
        for (int k = 0; k < kMaxPass; ++k) ids[k] = pass_id(blockIdx.x, warp + k * kQkvProd);
        int it = 0;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const int s = it & 1;
            float v[2][16];
            uint2 ph[2][4];
            int64_t id[kMaxPass];
            bool ok[kMaxPass];
#pragma unroll
            for (int k = 0; k < kMaxPass; ++k) {
                id[k] = ids[k];
                ok[k] = k < n_my && tile * 128 + (warp + k * kQkvProd) * 4 + rl < rows;
            }
#pragma unroll
            for (int k = 0; k < kMaxPass; ++k) ids[k] = pass_id(tile + gridDim.x, warp + k * kQkvProd);  // prefetch
            load_row_quads<kF64>(x, x64, pe16, id[0], sub, ok[0], v[0], ph[0]);
            if (threadIdx.x == 0 && it < 6) FWA_TR(1 + 4 * it);
            if (it >= 2) mbar_wait(&empty[s], ((it >> 1) - 1) & 1);
            if (threadIdx.x == 0 && it < 6) FWA_TR(2 + 4 * it);
            uint8_t* A = sA + s * kTileA;
#pragma unroll
            for (int k = 0; k < kMaxPass; ++k) {  // pass k+1's rows in flight while pass k is reduced
                if (k >= n_my) break;
                if (k + 1 < n_my)
                    load_row_quads<kF64>(x, x64, pe16, id[k + 1], sub, ok[k + 1], v[(k + 1) & 1], ph[(k + 1) & 1]);
                const int r = (warp + k * kQkvProd) * 4 + rl;
                ln1_row_to_tile(v[k & 1], ph[k & 1], ok[k], r, sub, sG, sB, A, bad);
                if (xq && ok[k]) {
                    // the gathered fp32 row, tile-transposed for the out-proj kernel's residual:
                    // float4 ((tile*4 + cq)*8 + j)*128 + row  (cq = channel/32, j = channel%32/4)
                    float4* q = reinterpret_cast<float4*>(xq) + (tile * 32 + sub) * 128 + r;
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        q[i * 1024] = make_float4(v[k & 1][4 * i], v[k & 1][4 * i + 1], v[k & 1][4 * i + 2],
                                                  v[k & 1][4 * i + 3]);
                }
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[s]);
            if (threadIdx.x == 0 && it < 6) FWA_TR(3 + 4 * it);
        }
        if (__any_sync(0xffffffffu, bad) && lane == 0) atomicExch(nonfinite, 1);
    } else {
        // ------------------------------------------------ MMA issue + epilogue (warps kQkvProd..15)
        const int q = warp - kQkvProd;  // TMEM lane quarter = tile rows 32q..32q+31
        const bool issuer = warp == kQkvProd && lane == 0;
        const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
        const int erow = q * 32 + lane, rot = (lane >> 1) & 3;
        constexpr uint32_t idesc = idesc_bf16_f32(128, 128);
        int it = 0, sit = 0;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const int s = it & 1;
            if (issuer) {
                if (it == 0) mbar_wait(wbar, 0);
                mbar_wait(&full[s], (it >> 1) & 1);
                fence_after_sync();
                const uint32_t a0 = smem_u32(sA + s * kTileA), b0 = smem_u32(sW);
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) {
                    const uint64_t ad = sdesc_sw128(a0 + (ks >> 2) * 16384 + (ks & 3) * 32);
#pragma unroll
                    for (int n = 0; n < 3; ++n) {
                        const uint64_t bd = sdesc_sw128(b0 + (ks >> 2) * (384 * 128) + n * (128 * 128) + (ks & 3) * 32);
                        mma_bf16(tmem + n * 128, ad, bd, idesc, ks > 0 ? 1u : 0u);
                    }
                }
                mma_commit(&empty[s]);
                mma_commit(done);
                if (it < 6) FWA_TR(30 + 4 * it);
            }
            __syncwarp();
            mbar_wait(done, it & 1);
            fence_after_sync();
            if (issuer && it < 6) FWA_TR(31 + 4 * it);
            const int64_t vrows = rows - tile * 128 < 128 ? rows - tile * 128 : 128;
            // TMEM -> +bias -> bf16 rows staged in shared memory (the 64 B row pieces written
            // in a lane-rotated order: conflict-free), then each chunk's [rows x 32] block --
            // contiguous in the chunk-major qkv layout -- leaves by one bulk TMA store.
#pragma unroll 1
            for (int ch = 0; ch < 12; ch += 2, ++sit) {
                uint32_t v[32], u[32];
                tmem_ld32(tmem + lane_off + ch * 32, v);
                tmem_ld32(tmem + lane_off + ch * 32 + 32, u);
                tmem_ld_wait();
                uint8_t* stg = sStage + (sit & 1) * 16384;
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const uint32_t* src = hh ? u : v;
                    const float* bias = sBias + (ch + hh) * 32;
                    uint4 P[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const float4 b0 = *reinterpret_cast<const float4*>(bias + 8 * j);
                        const float4 b1 = *reinterpret_cast<const float4*>(bias + 8 * j + 4);
                        P[j] = make_uint4(pack_bf16x2(__uint_as_float(src[8 * j]) + b0.x, __uint_as_float(src[8 * j + 1]) + b0.y),
                                          pack_bf16x2(__uint_as_float(src[8 * j + 2]) + b0.z, __uint_as_float(src[8 * j + 3]) + b0.w),
                                          pack_bf16x2(__uint_as_float(src[8 * j + 4]) + b1.x, __uint_as_float(src[8 * j + 5]) + b1.y),
                                          pack_bf16x2(__uint_as_float(src[8 * j + 6]) + b1.z, __uint_as_float(src[8 * j + 7]) + b1.w));
                    }
                    uint8_t* rowp = stg + hh * 8192 + erow * 64;
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) {
                        const int j = (jj + rot) & 3;
                        *reinterpret_cast<uint4*>(rowp + j * 16) = pick4(P, j);
                    }
                }
                fence_proxy_async_smem();
                fence_before_sync();  // on the last pair: TMEM drained before the next tile's MMA
                if (issuer) bulk_wait_read_all();  // the other buffer's store has left shared memory
                asm volatile("bar.sync 1, %0;" ::"n"((16 - kQkvProd) * 32) : "memory");
                if (issuer) {
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh)
                        bulk_s2g(qkv + (static_cast<int64_t>(ch + hh) * rows + tile * 128) * 32, stg + hh * 8192,
                                 static_cast<uint32_t>(vrows * 64));
                    bulk_commit();
                }
            }
            if (issuer && it < 6) FWA_TR(32 + 4 * it);
        }
        if (issuer) bulk_wait_all();
        if (warp == kQkvProd && lane == 0) FWA_TR(60);
    }
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    if (warp == kQkvProd) tmem_dealloc(tmem, 512);
}

void launch_ln1_qkv_tc(const float* x, const double* x64, const __half* pe, const int32_t* idx,
                       int64_t rows, const TcBlockWeights& w, __nv_bfloat16* qkv, int* d_nonfinite,
                       float* xq, cudaStream_t s, int64_t* launches, unsigned long long* trace) {
    static bool init = false;
    if (!init) {
        cudaFuncSetAttribute(k_ln1_qkv_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kQkvSmem);
        cudaFuncSetAttribute(k_ln1_qkv_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kQkvSmem);
        init = true;
    }
    const int64_t ntiles = (rows + 127) / 128;
    const unsigned grid = static_cast<unsigned>(ntiles < kNumSMs ? ntiles : kNumSMs);
    if (x64)
        launch_pdl(k_ln1_qkv_tc<true>, grid, kQkvThreads, kQkvSmem, s, x, x64, pe, idx, rows, w, qkv,
                   d_nonfinite, xq, trace);
    else
        launch_pdl(k_ln1_qkv_tc<false>, grid, kQkvThreads, kQkvSmem, s, x, x64, pe, idx, rows, w, qkv,
                   d_nonfinite, xq, trace);
    ++*launches;
}

// ------------------------------------------------------------------ K_c: out-proj + LN2 + FFN + scatter
//
// Per 128-row tile (persistent, 1 CTA/SM, 16 warps: warp w owns TMEM lanes
// 32*(w%4).. (= tile rows) and the column quarter w/4; thread 0 issues MMAs):
//   1. the attention output tile arrives by ONE TMA bulk copy (it is written as a
//      SW128 image by the attention kernel) -> R0;  P = A Wout^T -> TMEM[0,128)
//   2. residual x[ridx[r]] (fp32, this thread's 32 channels = one 128 B line) is
//      loaded into registers while MMA1 runs; x1 = (x + P) + b_out stays in registers
//   3. LN2: the 4 column quarters of a row exchange partial sums through TMEM
//      columns [384,392) (no shared memory left) -> bf16 SW128 image R1
//   4. U_a = LN2 W1[0:128]^T, U_b = LN2 W1[128:256]^T issued back to back;
//      GELU(U_a) -> act_a (R0) runs while U_b is computed, then O = act_a W2_a^T
//      runs while GELU(U_b) -> act_b (R1), then O += act_b W2_b^T  (O reuses P's columns)
//   5. out = x1 + (O + b2) -> swizzled f32 rows in R -> coalesced 512 B row stores
//      to x_out[sidx[r]] (the scatter, backbone.hpp:278-283); R0 then receives the
//      next tile's A by TMA.

constexpr int kWout = 128 * 128 * 2;  // 32768
constexpr int kW1 = 256 * 128 * 2;    // 65536
constexpr int kW2 = 128 * 256 * 2;    // 65536
constexpr int kRegion = 65536;        // R0 | R1
constexpr int kFfnThreads = 512;
constexpr int kFfnVec = 512;           // b_out 128 | b2 128 | b1 (LN2-folded) 256, fp32
constexpr int kFfnSmemUsed = kWout + kW1 + kW2 + kRegion + kFfnVec * 4 + 64 /*bars*/;
constexpr int kFfnSmem = 232448;       // the sm_100 per-block maximum; slack absorbs base alignment

// f32 row staging in R: row r (512 B) chunk c (16 B) at r*512 + ((c ^ (r & 7)) * 16)
FWA_DEVINL uint32_t stage_off(int r, int c) { return static_cast<uint32_t>(r * 512 + ((c ^ (r & 7)) << 4)); }

// The reference's exact-erf GELU (dense.hpp:67-72), x * Phi(x), evaluated as
// x * 0.5 * (1 + tanh(g(x))) with g an odd degree-7 polynomial fitted to
// atanh(erf(x / sqrt 2)) on |x| <= 3.2 (|x| clamped to 6, where Phi is 1 to 1e-9) and
// the hardware tanh.approx.f32 (rel 2^-11): |dGELU| <= 3.2e-5 from the fit plus
// <= 2.5e-4 |x| from tanh.approx -- below the bf16 rounding (2^-9 rel) of the
// activation it feeds.  9 FMA-pipe ops + 1 MUFU instead of ~20 + 2 for erff.
FWA_DEVINL float tanh_approx(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
FWA_DEVINL float gelu_fast(float x) {
    const float xc = fminf(fmaxf(x, -6.0f), 6.0f);
    const float x2 = xc * xc;
    const float p = fmaf(fmaf(fmaf(-4.71338576e-06f, x2, -3.19044083e-04f), x2, 3.69914203e-02f), x2,
                         7.97462955e-01f);
    const float t = tanh_approx(xc * p);
    const float hx = 0.5f * x;
    return fmaf(hx, t, hx);
}

FWA_DEVINL void tmem_st1(uint32_t taddr, float v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(__float_as_uint(v))
                 : "memory");
}
FWA_DEVINL void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
FWA_DEVINL float4 tmem_ld4(uint32_t taddr) {
    uint32_t a, b, c, d;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    return make_float4(__uint_as_float(a), __uint_as_float(b), __uint_as_float(c), __uint_as_float(d));
}
FWA_DEVINL void cta_sync_tc() {
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
}

template <bool kF64>
FWA_DEVINL void load_residual(const float* x_in, const double* x_in64, const int32_t* ridx, int64_t rows,
                              int64_t grow, int c0, float (&x1)[32], const float* xq) {
    if (xq) {  // tile-transposed copy written by the QKV kernel: lanes = consecutive rows
        if (grow < rows) {
            const float4* q = reinterpret_cast<const float4*>(xq) + ((grow >> 7) * 4 + (c0 >> 5)) * 8 * 128 +
                              (grow & 127);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float4 f4 = __ldg(q + j * 128);
                x1[4 * j] = f4.x; x1[4 * j + 1] = f4.y; x1[4 * j + 2] = f4.z; x1[4 * j + 3] = f4.w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) x1[j] = 0.f;
        }
        return;
    }
    if (grow < rows) {
        const int64_t src = ridx ? ridx[grow] : grow;
        if (kF64) {
            const double2* p = reinterpret_cast<const double2*>(x_in64 + src * 128 + c0);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const double2 d2 = __ldg(p + j);
                x1[2 * j] = static_cast<float>(d2.x);
                x1[2 * j + 1] = static_cast<float>(d2.y);
            }
        } else {
            const float4* p = reinterpret_cast<const float4*>(x_in + src * 128 + c0);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float4 f4 = __ldg(p + j);
                x1[4 * j] = f4.x; x1[4 * j + 1] = f4.y; x1[4 * j + 2] = f4.z; x1[4 * j + 3] = f4.w;
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) x1[j] = 0.f;
    }
}

template <bool kF64>
__global__ void __launch_bounds__(kFfnThreads, 1)
    k_outproj_ffn_tc(const uint8_t* __restrict__ cat_img, const float* __restrict__ x_in,
                     const double* __restrict__ x_in64, const int32_t* __restrict__ ridx,
                     int64_t rows, TcBlockWeights w, float* __restrict__ x_out,
                     const int32_t* __restrict__ sidx, const float* __restrict__ xq,
                     unsigned long long* __restrict__ trace) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    uint8_t* sWo = smem;
    if (threadIdx.x == 0) FWA_TR(0);
    uint8_t* sW1 = sWo + kWout;
    uint8_t* sW2 = sW1 + kW1;
    uint8_t* sR = sW2 + kW2;
    uint8_t* sR1 = sR + 32768;
    float* sVec = reinterpret_cast<float*>(sR + kRegion);        // b_out | b2 | b1'
    uint64_t* bars = reinterpret_cast<uint64_t*>(sVec + kFfnVec);  // w, a, p, ua, ub, o
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 6);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = warp & 3, cq = warp >> 2;
    const int row = q * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;

    if (smem - smem_raw > kFfnSmem - kFfnSmemUsed) __trap();  // dynamic smem base misaligned
    griddep_launch_dependents();
    if (threadIdx.x == 0) {
        for (int i = 0; i < 6; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < kFfnVec; i += blockDim.x) sVec[i] = w.vec[384 + i];
    if (warp == 0) {
        __syncwarp();
        tmem_alloc(tmem_slot, 512);
    }
    cta_sync_tc();
    const uint32_t tmem = *tmem_slot;
    const int64_t ntiles = (rows + 127) / 128;
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bars[0], kWout + kW1 + kW2);
        bulk_g2s(sWo, w.w_out, kWout, &bars[0]);
        bulk_g2s(sW1, w.w1, 32768, &bars[0]);
        bulk_g2s(sW1 + 32768, reinterpret_cast<const uint8_t*>(w.w1) + 32768, 32768, &bars[0]);
        bulk_g2s(sW2, w.w2, 32768, &bars[0]);
        bulk_g2s(sW2 + 32768, reinterpret_cast<const uint8_t*>(w.w2) + 32768, 32768, &bars[0]);
    }
    griddep_wait();  // attention rows + residual come from earlier kernels
    if (threadIdx.x == 0 && blockIdx.x < ntiles) {
        mbar_arrive_expect_tx(&bars[1], 32768);
        bulk_g2s(sR, cat_img + static_cast<int64_t>(blockIdx.x) * 32768, 32768, &bars[1]);
    }
    constexpr uint32_t id128 = idesc_bf16_f32(128, 128);
    const uint32_t TP = tmem, TUa = tmem + 128, TUb = tmem + 256, TS = tmem + 384;
    const int c0 = cq * 32;  // this thread's 32 channels / hidden units
    // x1 holds the residual row of the CURRENT tile on loop entry (prefetched while the
    // previous tile's output was being stored)
    float x1[32];
    load_residual<kF64>(x_in, x_in64, ridx, rows, static_cast<int64_t>(blockIdx.x) * 128 + row, c0, x1, xq);
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const uint32_t ph = it & 1;
        const int64_t grow = tile * 128 + row;
        const bool valid = grow < rows;
        (void)valid;
        // ---- 1. P = A Wout^T
        if (threadIdx.x == 0) {
            if (it == 0) mbar_wait(&bars[0], 0);
            if (it < 4) FWA_TR(1 + 12 * it);
            mbar_wait(&bars[1], ph);
            if (it < 4) FWA_TR(2 + 12 * it);
            fence_after_sync();
            const uint32_t a0 = smem_u32(sR), b0 = smem_u32(sWo);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
                mma_bf16(TP, sdesc_sw128(a0 + (ks >> 2) * 16384 + (ks & 3) * 32),
                         sdesc_sw128(b0 + (ks >> 2) * 16384 + (ks & 3) * 32), id128, ks > 0);
            mma_commit(&bars[2]);
        }
        mbar_wait(&bars[2], ph);
        if (threadIdx.x == 0 && it < 4) FWA_TR(3 + 12 * it);
        fence_after_sync();
        {
            uint32_t v[32];
            tmem_ld32(TP + lane_off + c0, v);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
                const float4 bo = *reinterpret_cast<const float4*>(sVec + c0 + j);
                x1[j + 0] = (x1[j + 0] + __uint_as_float(v[j + 0])) + bo.x;
                x1[j + 1] = (x1[j + 1] + __uint_as_float(v[j + 1])) + bo.y;
                x1[j + 2] = (x1[j + 2] + __uint_as_float(v[j + 2])) + bo.z;
                x1[j + 3] = (x1[j + 3] + __uint_as_float(v[j + 3])) + bo.w;
            }
        }
        // ---- 3. LN2 (row statistics over the 4 column quarters via TMEM)
        float s = 0.f;
#pragma unroll
        for (int j = 0; j < 32; ++j) s += x1[j];
        tmem_st1(TS + lane_off + cq, s);
        tmem_st_wait();
        cta_sync_tc();
        float4 ps = tmem_ld4(TS + lane_off);
        const float mean = ((ps.x + ps.y) + (ps.z + ps.w)) * (1.0f / 128.0f);
        float v2 = 0.f;
#pragma unroll
        for (int j = 0; j < 32; ++j) v2 += (x1[j] - mean) * (x1[j] - mean);
        tmem_st1(TS + lane_off + 4 + cq, v2);
        tmem_st_wait();
        cta_sync_tc();
        ps = tmem_ld4(TS + lane_off + 4);
        const float inv = 1.0f / sqrtf(((ps.x + ps.y) + (ps.z + ps.w)) * (1.0f / 128.0f) + 1e-5f);
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
            uint32_t o[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int j = ch * 8 + 2 * e, col = c0 + j;
                (void)col;  // LN2 affine folded into W1 / b1 on the host
                o[e] = pack_bf16x2((x1[j] - mean) * inv, (x1[j + 1] - mean) * inv);
            }
            *reinterpret_cast<uint4*>(sR1 + sw128_offset(row, c0 + ch * 8, 128)) = make_uint4(o[0], o[1], o[2], o[3]);
        }
        fence_proxy_async_smem();
        cta_sync_tc();
        if (threadIdx.x == 0 && it < 4) FWA_TR(4 + 12 * it);
        // ---- 4. U_a, U_b = LN2 W1^T halves (N = 128 each)
        if (threadIdx.x == 0) {
            const uint32_t a0 = smem_u32(sR1), b0 = smem_u32(sW1);
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
                for (int ks = 0; ks < 8; ++ks)
                    mma_bf16(hh ? TUb : TUa, sdesc_sw128(a0 + (ks >> 2) * 16384 + (ks & 3) * 32),
                             sdesc_sw128(b0 + (ks >> 2) * 32768 + hh * 16384 + (ks & 3) * 32), id128, ks > 0);
                mma_commit(&bars[3 + hh]);
            }
        }
#pragma unroll 1
        for (int hh = 0; hh < 2; ++hh) {
            mbar_wait(&bars[3 + hh], ph);
            if (threadIdx.x == 0 && it < 4) FWA_TR(5 + 2 * hh + 12 * it);
            fence_after_sync();
            uint8_t* act = hh ? sR1 : sR;  // [128 x 128] SW128 image (K-blocks 2hh, 2hh+1 of act)
            uint32_t v[32];
            tmem_ld32((hh ? TUb : TUa) + lane_off + c0, v);
            tmem_ld_wait();
            const float* b1 = sVec + 256 + hh * 128 + c0;
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
                uint32_t o[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int j = ch * 8 + 2 * e;
                    o[e] = pack_bf16x2(gelu_fast(__uint_as_float(v[j]) + b1[j]),
                                       gelu_fast(__uint_as_float(v[j + 1]) + b1[j + 1]));
                }
                *reinterpret_cast<uint4*>(act + sw128_offset(row, c0 + ch * 8, 128)) = make_uint4(o[0], o[1], o[2], o[3]);
            }
            fence_proxy_async_smem();
            cta_sync_tc();
            if (threadIdx.x == 0 && it < 4) FWA_TR(6 + 2 * hh + 12 * it);
            // ---- O (+)= act_hh W2[:, 128hh : 128hh+128]^T  (O reuses P's columns)
            if (threadIdx.x == 0) {
                const uint32_t a0 = smem_u32(act), b0 = smem_u32(sW2) + hh * 2 * 16384;
#pragma unroll
                for (int ks = 0; ks < 8; ++ks)
                    mma_bf16(TP, sdesc_sw128(a0 + (ks >> 2) * 16384 + (ks & 3) * 32),
                             sdesc_sw128(b0 + (ks >> 2) * 16384 + (ks & 3) * 32), id128, (hh | ks) > 0);
                if (hh) mma_commit(&bars[5]);
            }
        }
        // ---- 5. out = x1 + (O + b2) -> coalesced scatter through R1 in two 64-row halves;
        //         R0 (act_a, consumed) immediately receives the next tile's A by TMA, and each
        //         thread prefetches its next residual row right after staging its output
        mbar_wait(&bars[5], ph);
        if (threadIdx.x == 0 && it < 4) FWA_TR(9 + 12 * it);
        fence_after_sync();
        const int64_t next = tile + gridDim.x;
        if (threadIdx.x == 0 && next < ntiles) {
            mbar_arrive_expect_tx(&bars[1], 32768);
            bulk_g2s(sR, cat_img + next * 32768, 32768, &bars[1]);
        }
        {
            uint32_t v[32];
            tmem_ld32(TP + lane_off + c0, v);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
                const float4 b2 = *reinterpret_cast<const float4*>(sVec + 128 + c0 + j);
                x1[j + 0] = x1[j + 0] + (__uint_as_float(v[j + 0]) + b2.x);
                x1[j + 1] = x1[j + 1] + (__uint_as_float(v[j + 1]) + b2.y);
                x1[j + 2] = x1[j + 2] + (__uint_as_float(v[j + 2]) + b2.z);
                x1[j + 3] = x1[j + 3] + (__uint_as_float(v[j + 3]) + b2.w);
            }
        }
#pragma unroll 1
        for (int hf = 0; hf < 2; ++hf) {
            if ((row >> 6) == hf) {  // my row is in this half: stage it, then prefetch
                const int rr = row & 63;
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                    *reinterpret_cast<float4*>(sR1 + stage_off(rr, (c0 + j) >> 2)) =
                        make_float4(x1[j], x1[j + 1], x1[j + 2], x1[j + 3]);
                if (next < ntiles) load_residual<kF64>(x_in, x_in64, ridx, rows, next * 128 + row, c0, x1, xq);
            }
            __syncthreads();
            {
                const int rbase = warp * 4;  // 16 warps x 4 rows = 64 rows of this half
                int myid = 0;
                const int64_t gl = tile * 128 + hf * 64 + rbase + (lane & 3);
                if (lane < 4 && gl < rows) myid = sidx ? sidx[gl] : static_cast<int>(gl);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int64_t id = __shfl_sync(0xffffffffu, myid, i);
                    const float4 o = *reinterpret_cast<const float4*>(sR1 + stage_off(rbase + i, lane));
                    if (tile * 128 + hf * 64 + rbase + i < rows) reinterpret_cast<float4*>(x_out + id * 128)[lane] = o;
                }
            }
            __syncthreads();
        }
        if (threadIdx.x == 0 && it < 4) FWA_TR(10 + 12 * it);
    }
    if (threadIdx.x == 0 && blockIdx.x >= ntiles) mbar_wait(&bars[0], 0);
    cta_sync_tc();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

void launch_outproj_ffn_tc(const __nv_bfloat16* cat, const float* x_in, const double* x_in64,
                           const int32_t* ridx, int64_t rows, const TcBlockWeights& w, float* x_out,
                           const int32_t* sidx, const float* xq, cudaStream_t s, int64_t* launches,
                           unsigned long long* trace) {
    static bool init = false;
    if (!init) {
        cudaFuncSetAttribute(k_outproj_ffn_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFfnSmem);
        cudaFuncSetAttribute(k_outproj_ffn_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFfnSmem);
        init = true;
    }
    const int64_t ntiles = (rows + 127) / 128;
    const unsigned grid = static_cast<unsigned>(ntiles < kNumSMs ? ntiles : kNumSMs);
    const uint8_t* img = reinterpret_cast<const uint8_t*>(cat);
    if (x_in64)
        launch_pdl(k_outproj_ffn_tc<true>, grid, kFfnThreads, kFfnSmem, s, img, x_in, x_in64, ridx, rows, w,
                   x_out, sidx, xq, trace);
    else
        launch_pdl(k_outproj_ffn_tc<false>, grid, kFfnThreads, kFfnSmem, s, img, x_in, x_in64, ridx, rows, w,
                   x_out, sidx, xq, trace);
    ++*launches;
}

} // namespace fwa_b200
