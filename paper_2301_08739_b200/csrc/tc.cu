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
#include <cuda_runtime.h>
#include <stdint.h>

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

FWA_DEVINL uint8_t* align1024(uint8_t* p) {
    return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// ------------------------------------------------------------------ K_a: gather + LN1 + PE + QKV

constexpr int kQkvW = 384 * 128 * 2;   // 98304 B
constexpr int kTileA = 128 * 128 * 2;  // 32768 B
constexpr int kQkvSmem = kQkvW + kTileA + 64 + 1024;

template <bool kF64>
__global__ void __launch_bounds__(256, 1)
    k_ln1_qkv_tc(const float* __restrict__ x, const double* __restrict__ x64,
                 const float* __restrict__ pe, const int32_t* __restrict__ idx, int64_t rows,
                 TcBlockWeights w, __nv_bfloat16* __restrict__ qkv, int* __restrict__ nonfinite) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    uint8_t* sW = smem;
    uint8_t* sA = smem + kQkvW;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sA + kTileA);  // [0] weights, [1] mma
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc(tmem_slot, 512);
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bars[0], kQkvW);
#pragma unroll
        for (int c = 0; c < 3; ++c)
            bulk_g2s(sW + c * 32768, reinterpret_cast<const uint8_t*>(w.w_qkv) + c * 32768, 32768, &bars[0]);
    }
    constexpr uint32_t idesc = idesc_bf16_f32(128, 128);
    uint32_t phase = 0;
    bool w_ready = false;
    bool bad = false;
    const int64_t ntiles = (rows + 127) / 128;
    const float4 g4 = reinterpret_cast<const float4*>(w.ln1_g)[lane];
    const float4 b4 = reinterpret_cast<const float4*>(w.ln1_b)[lane];
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        // ---- gather + LN1 + PE -> bf16 SW128 A tile (one warp per row, 4 channels per lane)
        for (int rr = 0; rr < 16; ++rr) {
            const int r = warp * 16 + rr;
            const int64_t grow = tile * 128 + r;
            uint2 packed = make_uint2(0u, 0u);
            if (grow < rows) {
                const int64_t id = idx ? idx[grow] : grow;
                float4 xv;
                if (kF64) {
                    const double2* p = reinterpret_cast<const double2*>(x64 + id * 128 + lane * 4);
                    const double2 a = p[0], b = p[1];
                    xv = make_float4(static_cast<float>(a.x), static_cast<float>(a.y),
                                     static_cast<float>(b.x), static_cast<float>(b.y));
                } else {
                    xv = reinterpret_cast<const float4*>(x + id * 128)[lane];
                }
                const float4 pv = reinterpret_cast<const float4*>(pe + id * 128)[lane];
                bad |= !(isfinite(xv.x) && isfinite(xv.y) && isfinite(xv.z) && isfinite(xv.w) &&
                         isfinite(pv.x) && isfinite(pv.y) && isfinite(pv.z) && isfinite(pv.w));
                const float mean = warp_sum(xv.x + xv.y + xv.z + xv.w) * (1.0f / 128.0f);
                const float dx = xv.x - mean, dy = xv.y - mean, dz = xv.z - mean, dw = xv.w - mean;
                const float var = warp_sum(dx * dx + dy * dy + dz * dz + dw * dw) * (1.0f / 128.0f);
                const float inv = 1.0f / sqrtf(var + 1e-5f);
                const float h0 = g4.x * (dx * inv) + b4.x + pv.x;
                const float h1 = g4.y * (dy * inv) + b4.y + pv.y;
                const float h2 = g4.z * (dz * inv) + b4.z + pv.z;
                const float h3 = g4.w * (dw * inv) + b4.w + pv.w;
                packed = make_uint2(pack_bf16x2(h0, h1), pack_bf16x2(h2, h3));
            }
            *reinterpret_cast<uint2*>(sA + sw128_offset(r, lane * 4, 128)) = packed;
        }
        fence_proxy_async_smem();
        fence_before_sync();
        __syncthreads();
        // ---- packed QKV GEMM: [128 x 128] x [384 x 128]^T -> TMEM cols [0, 384)
        if (threadIdx.x == 0) {
            if (!w_ready) {
                mbar_wait(&bars[0], 0);
                w_ready = true;
            }
            fence_after_sync();
            const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sW);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const uint64_t ad = sdesc_sw128(a0 + (ks >> 2) * 16384 + (ks & 3) * 32);
#pragma unroll
                for (int n = 0; n < 3; ++n) {
                    const uint64_t bd = sdesc_sw128(b0 + (ks >> 2) * (384 * 128) + n * (128 * 128) + (ks & 3) * 32);
                    mma_bf16(tmem + n * 128, ad, bd, idesc, ks > 0 ? 1u : 0u);
                }
            }
            mma_commit(&bars[1]);
        }
        mbar_wait(&bars[1], phase);
        phase ^= 1;
        fence_after_sync();
        // ---- epilogue: TMEM -> +bias -> bf16 rows of q|k|v
        {
            const int q = warp & 3, half = warp >> 2;
            const int row = q * 32 + lane;
            const int64_t grow = tile * 128 + row;
#pragma unroll 1
            for (int ch = 0; ch < 6; ++ch) {
                const int col0 = half * 192 + ch * 32;
                uint32_t v[32];
                tmem_ld32(tmem + (static_cast<uint32_t>(q * 32) << 16) + col0, v);
                tmem_ld_wait();
                if (grow < rows) {
                    uint32_t o[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        o[j] = pack_bf16x2(__uint_as_float(v[2 * j]) + w.b_qkv[col0 + 2 * j],
                                           __uint_as_float(v[2 * j + 1]) + w.b_qkv[col0 + 2 * j + 1]);
                    uint4* dst = reinterpret_cast<uint4*>(qkv + grow * 384 + col0);
#pragma unroll
                    for (int j = 0; j < 4; ++j) dst[j] = make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
                }
            }
        }
        fence_before_sync();
        __syncthreads();
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicExch(nonfinite, 1);
    // drain the weight barrier if this CTA had no tile (bulk copy must land before exit)
    if (threadIdx.x == 0 && !w_ready) mbar_wait(&bars[0], 0);
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

void launch_ln1_qkv_tc(const float* x, const double* x64, const float* pe, const int32_t* idx,
                       int64_t rows, const TcBlockWeights& w, __nv_bfloat16* qkv, int* d_nonfinite,
                       cudaStream_t s, int64_t* launches) {
    static bool init = false;
    if (!init) {
        cudaFuncSetAttribute(k_ln1_qkv_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kQkvSmem);
        cudaFuncSetAttribute(k_ln1_qkv_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kQkvSmem);
        init = true;
    }
    const int64_t ntiles = (rows + 127) / 128;
    const unsigned grid = static_cast<unsigned>(ntiles < kNumSMs ? ntiles : kNumSMs);
    if (x64)
        k_ln1_qkv_tc<true><<<grid, 256, kQkvSmem, s>>>(x, x64, pe, idx, rows, w, qkv, d_nonfinite);
    else
        k_ln1_qkv_tc<false><<<grid, 256, kQkvSmem, s>>>(x, x64, pe, idx, rows, w, qkv, d_nonfinite);
    ++*launches;
}

// ------------------------------------------------------------------ K_c: out-proj + LN2 + FFN + scatter

constexpr int kWout = 128 * 128 * 2;  // 32768
constexpr int kW1 = 256 * 128 * 2;    // 65536
constexpr int kW2 = 128 * 256 * 2;    // 65536
constexpr int kRegion = 65536;        // A tile | LN2 tile, later the 128 x 256 GELU tile
constexpr int kFfnSmem = kWout + kW1 + kW2 + kRegion + 1024 /*red*/ + 64 /*bars*/ + 1024 /*align*/;

template <bool kF64>
__global__ void __launch_bounds__(256, 1)
    k_outproj_ffn_tc(const __nv_bfloat16* __restrict__ cat, const float* __restrict__ x_in,
                     const double* __restrict__ x_in64, const int32_t* __restrict__ ridx,
                     int64_t rows, TcBlockWeights w, float* __restrict__ x_out,
                     const int32_t* __restrict__ sidx) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    uint8_t* sWo = smem;
    uint8_t* sW1 = sWo + kWout;
    uint8_t* sW2 = sW1 + kW1;
    uint8_t* sR = sW2 + kW2;        // R0 = sR (A tile), R1 = sR + 32768 (LN2 tile)
    float* red = reinterpret_cast<float*>(sR + kRegion);  // [128][2]
    uint64_t* bars = reinterpret_cast<uint64_t*>(red + 256);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = warp & 3, half = warp >> 2;
    const int row = q * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;

    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc(tmem_slot, 512);
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bars[0], kWout + kW1 + kW2);
        bulk_g2s(sWo, w.w_out, kWout, &bars[0]);
        bulk_g2s(sW1, w.w1, 32768, &bars[0]);
        bulk_g2s(sW1 + 32768, reinterpret_cast<const uint8_t*>(w.w1) + 32768, 32768, &bars[0]);
        bulk_g2s(sW2, w.w2, 32768, &bars[0]);
        bulk_g2s(sW2 + 32768, reinterpret_cast<const uint8_t*>(w.w2) + 32768, 32768, &bars[0]);
    }
    constexpr uint32_t id128 = idesc_bf16_f32(128, 128);
    constexpr uint32_t id256 = idesc_bf16_f32(128, 256);
    const uint32_t TP = tmem, TU = tmem + 128, TO = tmem + 384;
    uint32_t phase = 0;
    bool w_ready = false;
    const int64_t ntiles = (rows + 127) / 128;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t grow = tile * 128 + row;
        const bool valid = grow < rows;
        // ---- 1. attention rows (bf16, 256 B each) -> SW128 A tile in R0
        for (int t = threadIdx.x; t < 128 * 16; t += 256) {
            const int r = t >> 4, c16 = t & 15;
            const int64_t g = tile * 128 + r;
            uint4 v = make_uint4(0u, 0u, 0u, 0u);
            if (g < rows) v = reinterpret_cast<const uint4*>(cat + g * 128)[c16];
            *reinterpret_cast<uint4*>(sR + sw128_offset(r, c16 * 8, 128)) = v;
        }
        fence_proxy_async_smem();
        fence_before_sync();
        __syncthreads();
        // ---- 2. P = A Wout^T
        if (threadIdx.x == 0) {
            if (!w_ready) {
                mbar_wait(&bars[0], 0);
                w_ready = true;
            }
            fence_after_sync();
            const uint32_t a0 = smem_u32(sR), b0 = smem_u32(sWo);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
                mma_bf16(TP, sdesc_sw128(a0 + (ks >> 2) * 16384 + (ks & 3) * 32),
                         sdesc_sw128(b0 + (ks >> 2) * 16384 + (ks & 3) * 32), id128, ks > 0);
            mma_commit(&bars[1]);
        }
        mbar_wait(&bars[1], phase);
        phase ^= 1;
        fence_after_sync();
        // ---- 3. x1 = (x + P) + b_out in registers; LN2 -> bf16 R1 (K-block `half`)
        float x1[64];
        {
            const int64_t src = valid ? (ridx ? ridx[grow] : grow) : 0;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                uint32_t v[32];
                tmem_ld32(TP + lane_off + half * 64 + c * 32, v);
                tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 32; j += 4) {
                    const int col = half * 64 + c * 32 + j;
                    float4 xr = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (valid) {
                        if (kF64) {
                            const double2* p = reinterpret_cast<const double2*>(x_in64 + src * 128 + col);
                            const double2 a = p[0], b = p[1];
                            xr = make_float4(static_cast<float>(a.x), static_cast<float>(a.y),
                                             static_cast<float>(b.x), static_cast<float>(b.y));
                        } else {
                            xr = *reinterpret_cast<const float4*>(x_in + src * 128 + col);
                        }
                    }
                    const float4 bo = *reinterpret_cast<const float4*>(w.b_out + col);
                    x1[c * 32 + j + 0] = (xr.x + __uint_as_float(v[j + 0])) + bo.x;
                    x1[c * 32 + j + 1] = (xr.y + __uint_as_float(v[j + 1])) + bo.y;
                    x1[c * 32 + j + 2] = (xr.z + __uint_as_float(v[j + 2])) + bo.z;
                    x1[c * 32 + j + 3] = (xr.w + __uint_as_float(v[j + 3])) + bo.w;
                }
            }
        }
        float s = 0.f;
#pragma unroll
        for (int j = 0; j < 64; ++j) s += x1[j];
        red[row * 2 + half] = s;
        __syncthreads();
        const float mean = (red[row * 2] + red[row * 2 + 1]) * (1.0f / 128.0f);
        __syncthreads();
        float v2 = 0.f;
#pragma unroll
        for (int j = 0; j < 64; ++j) v2 += (x1[j] - mean) * (x1[j] - mean);
        red[row * 2 + half] = v2;
        __syncthreads();
        const float inv = 1.0f / sqrtf((red[row * 2] + red[row * 2 + 1]) * (1.0f / 128.0f) + 1e-5f);
        {
            uint8_t* r1 = sR + 32768;
#pragma unroll
            for (int ch = 0; ch < 8; ++ch) {
                uint32_t o[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int j = ch * 8 + 2 * e, col = half * 64 + j;
                    const float l0 = w.ln2_g[col] * ((x1[j] - mean) * inv) + w.ln2_b[col];
                    const float l1 = w.ln2_g[col + 1] * ((x1[j + 1] - mean) * inv) + w.ln2_b[col + 1];
                    o[e] = pack_bf16x2(l0, l1);
                }
                // K-block 0 of R1 holds cols 0..63; the LN2 tile is its own 2-K-block image
                *reinterpret_cast<uint4*>(r1 + sw128_offset(row, half * 64 + ch * 8, 128)) =
                    make_uint4(o[0], o[1], o[2], o[3]);
            }
        }
        fence_proxy_async_smem();
        fence_before_sync();
        __syncthreads();
        // ---- 4. U = LN2 W1^T  (N = 256)
        if (threadIdx.x == 0) {
            fence_after_sync();
            const uint32_t a0 = smem_u32(sR + 32768), b0 = smem_u32(sW1);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
                mma_bf16(TU, sdesc_sw128(a0 + (ks >> 2) * 16384 + (ks & 3) * 32),
                         sdesc_sw128(b0 + (ks >> 2) * 32768 + (ks & 3) * 32), id256, ks > 0);
            mma_commit(&bars[1]);
        }
        mbar_wait(&bars[1], phase);
        phase ^= 1;
        fence_after_sync();
        // ---- 5. act = gelu(U + b1) -> bf16 128 x 256 SW128 image over R (4 K-blocks)
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
            const int h0 = half * 128 + c * 32;
            uint32_t v[32];
            tmem_ld32(TU + lane_off + h0, v);
            tmem_ld_wait();
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
                uint32_t o[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int j = ch * 8 + 2 * e;
                    const float a0 = gelu_erf(__uint_as_float(v[j]) + w.b1[h0 + j]);
                    const float a1 = gelu_erf(__uint_as_float(v[j + 1]) + w.b1[h0 + j + 1]);
                    o[e] = pack_bf16x2(a0, a1);
                }
                *reinterpret_cast<uint4*>(sR + sw128_offset(row, h0 + ch * 8, 128)) =
                    make_uint4(o[0], o[1], o[2], o[3]);
            }
        }
        fence_proxy_async_smem();
        fence_before_sync();
        __syncthreads();
        // ---- 6. O = act W2^T  (K = 256)
        if (threadIdx.x == 0) {
            fence_after_sync();
            const uint32_t a0 = smem_u32(sR), b0 = smem_u32(sW2);
#pragma unroll
            for (int ks = 0; ks < 16; ++ks)
                mma_bf16(TO, sdesc_sw128(a0 + (ks >> 2) * 16384 + (ks & 3) * 32),
                         sdesc_sw128(b0 + (ks >> 2) * 16384 + (ks & 3) * 32), id128, ks > 0);
            mma_commit(&bars[1]);
        }
        mbar_wait(&bars[1], phase);
        phase ^= 1;
        fence_after_sync();
        // ---- 7. out = x1 + (O + b2) -> pillar-id row
        {
            const int64_t dst = valid ? (sidx ? sidx[grow] : grow) : 0;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                uint32_t v[32];
                tmem_ld32(TO + lane_off + half * 64 + c * 32, v);
                tmem_ld_wait();
                if (valid) {
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        const int col = half * 64 + c * 32 + j;
                        const float4 b2 = *reinterpret_cast<const float4*>(w.b2 + col);
                        float4 o;
                        o.x = x1[c * 32 + j + 0] + (__uint_as_float(v[j + 0]) + b2.x);
                        o.y = x1[c * 32 + j + 1] + (__uint_as_float(v[j + 1]) + b2.y);
                        o.z = x1[c * 32 + j + 2] + (__uint_as_float(v[j + 2]) + b2.z);
                        o.w = x1[c * 32 + j + 3] + (__uint_as_float(v[j + 3]) + b2.w);
                        *reinterpret_cast<float4*>(x_out + dst * 128 + col) = o;
                    }
                }
            }
        }
        fence_before_sync();
        __syncthreads();
    }
    if (threadIdx.x == 0 && !w_ready) mbar_wait(&bars[0], 0);
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

void launch_outproj_ffn_tc(const __nv_bfloat16* cat, const float* x_in, const double* x_in64,
                           const int32_t* ridx, int64_t rows, const TcBlockWeights& w, float* x_out,
                           const int32_t* sidx, cudaStream_t s, int64_t* launches) {
    static bool init = false;
    if (!init) {
        cudaFuncSetAttribute(k_outproj_ffn_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFfnSmem);
        cudaFuncSetAttribute(k_outproj_ffn_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFfnSmem);
        init = true;
    }
    const int64_t ntiles = (rows + 127) / 128;
    const unsigned grid = static_cast<unsigned>(ntiles < kNumSMs ? ntiles : kNumSMs);
    if (x_in64)
        k_outproj_ffn_tc<true><<<grid, 256, kFfnSmem, s>>>(cat, x_in, x_in64, ridx, rows, w, x_out, sidx);
    else
        k_outproj_ffn_tc<false><<<grid, 256, kFfnSmem, s>>>(cat, x_in, x_in64, ridx, rows, w, x_out, sidx);
    ++*launches;
}

} // namespace fwa_b200
