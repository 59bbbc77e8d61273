// fp32 CUDA-core kernels: the FWA_PREC_FP32 check mode (tolerance 1e-4) and
// the path for configurations outside the tensor-core fast path's shapes.
// All run on the GPU; there is no CPU fallback.
//
//   positional_embedding   /root/reference/proj/include/fwa/kernels.hpp:364-393
//   LN1 + affine + PE      kernels.hpp:235-249, 472-485
//   packed QKV / out-proj  kernels.hpp:488-500, 550-560 (matmul_nt dense.hpp:50-64)
//   group attention        kernels.hpp:512-548 (softmax_row 251-262)
//   FFN (LN2, W1, GELU, W2, residual)  kernels.hpp:575-633
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "internal.h"

namespace fwa_b200 {

// ------------------------------------------------------------------ PE

// pe[i] = [sin/cos(2*pi*freq_k*x) pairs | sin/cos(2*pi*freq_k*y) pairs] in fp64,
// rounded to f32.  freq_k comes from the host (glibc pow, as the reference).
__global__ void k_positional_embedding(const double* __restrict__ coords, int64_t n, int d,
                                       const double* __restrict__ freq, float* __restrict__ pe,
                                       __half* __restrict__ pe16) {
    const int nf = d / 4;
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t i = t / (2 * nf);
    if (i >= n) return;
    const int r = static_cast<int>(t % (2 * nf));
    const int axis = r / nf, k = r % nf;
    const double c = coords[2 * i + axis];
    const double phase = __dmul_rn(__dmul_rn(6.283185307179586, freq[k]), c);
    double sv, cv;
    sincos(phase, &sv, &cv);
    const float2 o = make_float2(static_cast<float>(sv), static_cast<float>(cv));
    if (pe) reinterpret_cast<float2*>(pe + i * d + axis * (d / 2))[k] = o;
    if (pe16) reinterpret_cast<__half2*>(pe16 + i * d + axis * (d / 2))[k] = __floats2half2_rn(o.x, o.y);
}

// fp16 fast path (PE rows feed the bf16 LN1 + PE sum): one thread per (pillar, axis), all
// d/4 frequencies.  sin(2 pi f c) = sin(pi t), t = 2 f c: with 2f = Fh + Fl and
// c = ch + cl as float pairs, t = p + e where p = Fh ch (e = its exact FMA residual plus
// the cross terms); p is reduced EXACTLY mod 2 in fp32 (|p| < 2^22), then the SFU's
// sin / cos of pi r.  |err| < 1e-6, far below the fp16 rounding (2^-12) of the stored value.
template <int GR>
__global__ void k_pe_fp16(const double* __restrict__ coords, int64_t n, int nf, const float2* __restrict__ F,
                          __half* __restrict__ pe16) {
    // one thread per (row, axis, 4 frequencies): consecutive threads write consecutive 16 B
    // of the fp16 PE rows (every store instruction fills whole 128 B lines).  GR: the
    // frequency groups per axis at compile time (8 for D = 128: the index split is a shift;
    // a runtime 64-bit division would cost more than the row's arithmetic)
    const int groups = GR > 0 ? GR : nf >> 2;  // nf % 4 == 0
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t ra = GR > 0 ? t / GR : t / groups;  // row * 2 + axis
    const int k0 = static_cast<int>(t - ra * groups) * 4;
    const int64_t i = ra >> 1;
    const int axis = static_cast<int>(ra & 1);
    if (i >= n) return;
    const double c = __ldg(coords + 2 * i + axis);
    const float ch = static_cast<float>(c);
    const float cl = static_cast<float>(c - static_cast<double>(ch));
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const float2 f = __ldg(F + k0 + j);
        const float p = f.x * ch;
        const float e = fmaf(f.x, ch, -p) + fmaf(f.x, cl, f.y * ch);
        const float r = fmaf(-2.0f, rintf(0.5f * p), p) + e;
        // |pi r| <= pi (+ tiny): the SFU sin/cos (abs err <= 2^-21.4 on [-pi, pi]; fp32 pi and
        // the product add < 1e-6) -- 2 MUFU ops instead of the software sincospi
        float sv, cv;
        __sincosf(r * 3.14159265358979f, &sv, &cv);
        const __half2 h = __floats2half2_rn(sv, cv);
        w[j] = *reinterpret_cast<const uint32_t*>(&h);
    }
    reinterpret_cast<uint4*>(pe16 + i * (4 * nf) + axis * (2 * nf))[k0 >> 2] = make_uint4(w[0], w[1], w[2], w[3]);
}

// `fwa attend` row checksums (tools/fwa_cli.cpp:214-218): sum = 0.0; sum += (double)f[c]
// for c = 0..d-1, in that order -- one thread per row, bit-exact
__global__ void k_row_checksums(const float* __restrict__ f, int64_t n, int d, double* __restrict__ out) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const float* row = f + r * d;
    double s = 0.0;
    for (int c = 0; c < d; ++c) s = __dadd_rn(s, static_cast<double>(row[c]));
    out[r] = s;
}

void launch_row_checksums(const float* f, int64_t n, int d, double* out, cudaStream_t s, int64_t* launches) {
    if (n <= 0) return;
    k_row_checksums<<<static_cast<unsigned>((n + 127) / 128), 128, 0, s>>>(f, n, d, out);
    ++*launches;
}

// Pull a buffer into L2 (TMA bulk prefetch, 16 KB per request): block 0's row gather then
// hits L2 instead of HBM.  Issued on the side stream while the schedule runs.
__global__ void k_prefetch_l2(const uint8_t* __restrict__ p, int64_t bytes) {
    const int64_t chunk = 16384;
    for (int64_t o = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * chunk; o < bytes;
         o += static_cast<int64_t>(gridDim.x) * blockDim.x * chunk) {
        const int64_t len = bytes - o < chunk ? bytes - o : chunk;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p + o), "r"(static_cast<uint32_t>(len & ~15LL))
                     : "memory");
    }
}

void launch_prefetch_l2(const void* p, int64_t bytes, cudaStream_t s, int64_t* launches) {
    // only while the rows fit L2 with room for the schedule's buffers (a batch of frames
    // larger than that would only evict its own rows)
    if (!p || bytes < 16 || bytes > (48ll << 20)) return;
    k_prefetch_l2<<<kNumSMs, 128, 0, s>>>(static_cast<const uint8_t*>(p), bytes);
    ++*launches;
}

void launch_positional_embedding(const double* coords, int64_t n, int d, const double* d_freq,
                                 float* pe, __half* pe16, cudaStream_t s, int64_t* launches) {
    if (!pe && pe16 && (d / 4) % 4 == 0) {  // d_freq holds [nf doubles | nf float2 (2f hi, lo)]
        const int nf = d / 4;
        if (nf == 32)
            k_pe_fp16<8><<<static_cast<unsigned>((2 * n * (nf / 4) + 255) / 256), 256, 0, s>>>(
            coords, n, nf, reinterpret_cast<const float2*>(d_freq + nf), pe16);
        else
            k_pe_fp16<0><<<static_cast<unsigned>((2 * n * (nf / 4) + 255) / 256), 256, 0, s>>>(
            coords, n, nf, reinterpret_cast<const float2*>(d_freq + nf), pe16);
        ++*launches;
        return;
    }
    const int64_t total = n * (d / 2);
    k_positional_embedding<<<static_cast<unsigned>((total + 255) / 256), 256, 0, s>>>(
        coords, n, d, d_freq, pe, pe16);
    ++*launches;
}

// ------------------------------------------------------------------ LN (one warp per row)

template <bool kF64>
__global__ void __launch_bounds__(256) k_ln_gather_f32(const float* __restrict__ x,
                                                       const double* __restrict__ x64,
                                                       const float* __restrict__ pe,
                                                       const int32_t* __restrict__ idx,
                                                       int64_t rows, int d,
                                                       const float* __restrict__ g,
                                                       const float* __restrict__ b,
                                                       float* __restrict__ h,
                                                       int* __restrict__ nonfinite) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    const int64_t id = idx ? idx[r] : r;
    float sum = 0.f;
    bool bad = false;
    for (int c = lane; c < d; c += 32) {
        const float v = kF64 ? static_cast<float>(x64[id * d + c]) : x[id * d + c];
        const float p = pe[id * d + c];
        bad |= !isfinite(v) || !isfinite(p);
        sum += v;
    }
    const float mean = warp_sum(sum) / static_cast<float>(d);
    float var = 0.f;
    for (int c = lane; c < d; c += 32) {
        const float v = kF64 ? static_cast<float>(x64[id * d + c]) : x[id * d + c];
        var += (v - mean) * (v - mean);
    }
    var = warp_sum(var) / static_cast<float>(d);
    const float inv = 1.0f / sqrtf(var + 1e-5f);
    for (int c = lane; c < d; c += 32) {
        const float v = kF64 ? static_cast<float>(x64[id * d + c]) : x[id * d + c];
        h[r * d + c] = g[c] * ((v - mean) * inv) + b[c] + pe[id * d + c];
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicExch(nonfinite, 1);
}

void launch_ln_gather_f32(const float* x, const double* x64, const float* pe, const int32_t* idx,
                          int64_t rows, int d, const float* gamma, const float* beta, float* h,
                          int* d_nonfinite, cudaStream_t s, int64_t* launches) {
    const unsigned grid = static_cast<unsigned>((rows + 7) / 8);
    if (x64)
        k_ln_gather_f32<true><<<grid, 256, 0, s>>>(x, x64, pe, idx, rows, d, gamma, beta, h,
                                                   d_nonfinite);
    else
        k_ln_gather_f32<false><<<grid, 256, 0, s>>>(x, x64, pe, idx, rows, d, gamma, beta, h,
                                                    d_nonfinite);
    ++*launches;
}

__global__ void __launch_bounds__(256) k_ln_rows_f32(const float* __restrict__ x, int64_t rows,
                                                     int d, const float* __restrict__ g,
                                                     const float* __restrict__ b,
                                                     float* __restrict__ out) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    float sum = 0.f;
    for (int c = lane; c < d; c += 32) sum += x[r * d + c];
    const float mean = warp_sum(sum) / static_cast<float>(d);
    float var = 0.f;
    for (int c = lane; c < d; c += 32) {
        const float v = x[r * d + c] - mean;
        var += v * v;
    }
    var = warp_sum(var) / static_cast<float>(d);
    const float inv = 1.0f / sqrtf(var + 1e-5f);
    for (int c = lane; c < d; c += 32) out[r * d + c] = g[c] * ((x[r * d + c] - mean) * inv) + b[c];
}

void launch_ln_rows_f32(const float* x, int64_t rows, int d, const float* gamma,
                        const float* beta, float* out, cudaStream_t s, int64_t* launches) {
    k_ln_rows_f32<<<static_cast<unsigned>((rows + 7) / 8), 256, 0, s>>>(x, rows, d, gamma, beta,
                                                                       out);
    ++*launches;
}

// ------------------------------------------------------------------ SIMT GEMM, C = A W^T (+epilogue)

constexpr int kTM = 64, kTN = 64, kTK = 16;

template <int kEpi>
__global__ void __launch_bounds__(256) k_gemm_f32(GemmArgs a) {
    __shared__ float As[kTK][kTM + 4];
    __shared__ float Ws[kTK][kTN + 4];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int64_t m0 = static_cast<int64_t>(blockIdx.y) * kTM;
    const int n0 = blockIdx.x * kTN;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < a.K; k0 += kTK) {
        for (int t = threadIdx.x; t < kTM * kTK; t += 256) {
            const int mm = t / kTK, kk = t % kTK;
            const int64_t gm = m0 + mm;
            const int gk = k0 + kk;
            As[kk][mm] = (gm < a.M && gk < a.K) ? a.A[gm * a.K + gk] : 0.f;
            const int gn = n0 + mm;
            Ws[kk][mm] = (gn < a.N && gk < a.K) ? a.W[static_cast<int64_t>(gn) * a.K + gk] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < kTK; ++kk) {
            float av[4], wv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) wv[j] = Ws[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], wv[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t m = m0 + ty * 4 + i;
        if (m >= a.M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = n0 + tx * 4 + j;
            if (n >= a.N) continue;
            const float bias = a.bias ? a.bias[n] : 0.f;
            if (kEpi == EPI_BIAS) {
                a.C[m * a.N + n] = acc[i][j] + bias;
            } else if (kEpi == EPI_BIAS_GELU) {
                a.C[m * a.N + n] = gelu_erf(acc[i][j] + bias);
            } else if (kEpi == EPI_RESID_GATHER) {
                const int64_t src = a.ridx ? a.ridx[m] : m;
                const float res = a.R64 ? static_cast<float>(a.R64[src * a.N + n]) : a.R[src * a.N + n];
                a.C[m * a.N + n] = (res + acc[i][j]) + bias;
            } else {
                const int64_t dst = a.sidx ? a.sidx[m] : m;
                a.D[dst * a.N + n] = a.R[m * a.N + n] + (acc[i][j] + bias);
            }
        }
    }
}

void launch_gemm_f32(const GemmArgs& a, GemmEpi epi, cudaStream_t s, int64_t* launches) {
    dim3 grid(static_cast<unsigned>((a.N + kTN - 1) / kTN), static_cast<unsigned>((a.M + kTM - 1) / kTM));
    switch (epi) {
        case EPI_BIAS: k_gemm_f32<EPI_BIAS><<<grid, 256, 0, s>>>(a); break;
        case EPI_BIAS_GELU: k_gemm_f32<EPI_BIAS_GELU><<<grid, 256, 0, s>>>(a); break;
        case EPI_RESID_GATHER: k_gemm_f32<EPI_RESID_GATHER><<<grid, 256, 0, s>>>(a); break;
        case EPI_RESID_SCATTER: k_gemm_f32<EPI_RESID_SCATTER><<<grid, 256, 0, s>>>(a); break;
    }
    ++*launches;
}

// ------------------------------------------------------------------ attention fp32
// One CTA per (group, head); K/V of the head staged in shared memory when they fit, one
// thread per query row with its query and output row in registers (HD = head dim as a
// template; any other width takes the generic body with the rows in memory); the logits
// are recomputed in a second pass instead of materialising the G x G matrix (the
// reference's O(G) cache-free path, kernels.hpp:512-548: max-subtracted softmax, the same
// fp32 operation order).

template <int HD>
__global__ void __launch_bounds__(128) k_attention_f32(const float* __restrict__ qkv, int G, int d,
                                                       int heads, float* __restrict__ cat,
                                                       bool stage) {
    extern __shared__ float sm[];
    const int grp = blockIdx.x, head = blockIdx.y;
    const int hd = HD > 0 ? HD : d / heads;
    const int64_t base = static_cast<int64_t>(grp) * G;
    const int off = head * hd;
    const float scale = 1.0f / sqrtf(static_cast<float>(hd));
    float* Ks = sm;
    float* Vs = sm + static_cast<size_t>(G) * hd;
    if (stage) {
        for (int t = threadIdx.x; t < G * hd; t += blockDim.x) {
            const int j = t / hd, c = t % hd;
            Ks[t] = qkv[(base + j) * 3 * d + d + off + c];
            Vs[t] = qkv[(base + j) * 3 * d + 2 * d + off + c];
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < G; i += blockDim.x) {
        const float* qg = qkv + (base + i) * 3 * d + off;
        float* og = cat + (base + i) * d + off;
        if constexpr (HD > 0) {
            float q[HD], o[HD];
#pragma unroll
            for (int c = 0; c < HD; ++c) {
                q[c] = qg[c];
                o[c] = 0.f;
            }
            float mx = -INFINITY;
            for (int j = 0; j < G; ++j) {
                const float* kj = stage ? Ks + j * HD : qkv + (base + j) * 3 * d + d + off;
                float acc = 0.f;
#pragma unroll
                for (int c = 0; c < HD; ++c) acc = fmaf(q[c], kj[c], acc);
                mx = fmaxf(mx, acc * scale);
            }
            float sum = 0.f;
            for (int j = 0; j < G; ++j) {
                const float* kj = stage ? Ks + j * HD : qkv + (base + j) * 3 * d + d + off;
                const float* vj = stage ? Vs + j * HD : qkv + (base + j) * 3 * d + 2 * d + off;
                float acc = 0.f;
#pragma unroll
                for (int c = 0; c < HD; ++c) acc = fmaf(q[c], kj[c], acc);
                const float p = expf(acc * scale - mx);
                sum += p;
#pragma unroll
                for (int c = 0; c < HD; ++c) o[c] = fmaf(p, vj[c], o[c]);
            }
            const float inv = 1.0f / sum;
#pragma unroll
            for (int c = 0; c < HD; ++c) og[c] = o[c] * inv;
        } else {
            float mx = -INFINITY;
            for (int j = 0; j < G; ++j) {
                const float* kj = stage ? Ks + j * hd : qkv + (base + j) * 3 * d + d + off;
                float acc = 0.f;
                for (int c = 0; c < hd; ++c) acc = fmaf(qg[c], kj[c], acc);
                mx = fmaxf(mx, acc * scale);
            }
            float sum = 0.f;
            for (int c = 0; c < hd; ++c) og[c] = 0.f;
            for (int j = 0; j < G; ++j) {
                const float* kj = stage ? Ks + j * hd : qkv + (base + j) * 3 * d + d + off;
                const float* vj = stage ? Vs + j * hd : qkv + (base + j) * 3 * d + 2 * d + off;
                float acc = 0.f;
                for (int c = 0; c < hd; ++c) acc = fmaf(qg[c], kj[c], acc);
                const float p = expf(acc * scale - mx);
                sum += p;
                for (int c = 0; c < hd; ++c) og[c] = fmaf(p, vj[c], og[c]);
            }
            const float inv = 1.0f / sum;
            for (int c = 0; c < hd; ++c) og[c] *= inv;
        }
    }
}

void launch_attention_f32(const float* qkv, int64_t rows, int G, int d, int heads, float* cat,
                          cudaStream_t s, int64_t* launches) {
    const int64_t n_groups = rows / G;
    if (n_groups == 0) return;
    const int hd = d / heads;
    const size_t smem = 2ull * G * hd * sizeof(float);
    const bool stage = smem <= 48 * 1024;
    dim3 grid(static_cast<unsigned>(n_groups), static_cast<unsigned>(heads));
    const size_t sb = stage ? smem : 0;
    switch (hd) {
        case 4: k_attention_f32<4><<<grid, 128, sb, s>>>(qkv, G, d, heads, cat, stage); break;
        case 8: k_attention_f32<8><<<grid, 128, sb, s>>>(qkv, G, d, heads, cat, stage); break;
        case 16: k_attention_f32<16><<<grid, 128, sb, s>>>(qkv, G, d, heads, cat, stage); break;
        case 32: k_attention_f32<32><<<grid, 128, sb, s>>>(qkv, G, d, heads, cat, stage); break;
        default: k_attention_f32<0><<<grid, 128, sb, s>>>(qkv, G, d, heads, cat, stage); break;
    }
    ++*launches;
}

// ------------------------------------------------------------------ row scatter to active order

__global__ void k_scatter_rows(const float* __restrict__ src, const int32_t* __restrict__ ids,
                               const uint32_t* __restrict__ rank, int64_t n, int d,
                               float* __restrict__ dst) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (r >= n) return;
    const int64_t id = ids ? ids[r] : r;
    const int64_t o = rank ? rank[id] : r;
    for (int c = threadIdx.x & 31; c < d; c += 32) dst[o * d + c] = src[id * d + c];
}

__global__ void k_f32_to_f16(const float* __restrict__ in, int64_t n, __half* __restrict__ out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = __float2half_rn(in[i]);
}

void launch_f32_to_f16(const float* in, int64_t n, __half* out, cudaStream_t s, int64_t* launches) {
    k_f32_to_f16<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(in, n, out);
    ++*launches;
}

void launch_scatter_rows(const float* src, const int32_t* ids, const uint32_t* rank, int64_t n,
                         int d, float* dst, cudaStream_t s, int64_t* launches) {
    k_scatter_rows<<<static_cast<unsigned>((n + 7) / 8), 256, 0, s>>>(src, ids, rank, n, d, dst);
    ++*launches;
}

// dst[pos[r]] = src[r] (pos = the block's sorted pillar ids, or their output rows):
// the inverse of the block's gather, one warp per 512 B row
__global__ void k_scatter_sorted(const float* __restrict__ src, const int32_t* __restrict__ pos, int64_t n,
                                 int d, float* __restrict__ dst) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (r >= n) return;
    const int64_t o = pos[r];
    for (int c = (threadIdx.x & 31) * 4; c < d; c += 128)
        *reinterpret_cast<float4*>(dst + o * d + c) = *reinterpret_cast<const float4*>(src + r * d + c);
}

void launch_scatter_sorted(const float* src, const int32_t* pos, int64_t n, int d, float* dst, cudaStream_t s,
                           int64_t* launches) {
    k_scatter_sorted<<<static_cast<unsigned>((n + 7) / 8), 256, 0, s>>>(src, pos, n, d, dst);
    ++*launches;
}

// BackboneParams::input_proj (backbone.hpp:179-190): one thread per output element,
// the reference's fp32 loop op by op (acc = bias[j]; acc += w[j][c] * (float)x[c], c in
// order; -ffp-contract=off there, explicit round-to-nearest mul/add here) -- bit-exact.
template <typename T>
__global__ void k_input_proj(const T* __restrict__ x, int64_t n, int f_in, const float* __restrict__ w,
                             const float* __restrict__ b, int d, float* __restrict__ out) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= n * d) return;
    const int64_t r = e / d;
    const int j = static_cast<int>(e - r * d);
    const T* xr = x + r * f_in;
    const float* wj = w + static_cast<int64_t>(j) * f_in;
    float acc = b ? b[j] : 0.0f;
    for (int c = 0; c < f_in; ++c) acc = __fadd_rn(acc, __fmul_rn(__ldg(wj + c), static_cast<float>(__ldg(xr + c))));
    out[e] = acc;
}

void launch_input_proj(const void* x, bool x_f64, int64_t n, int f_in, const float* w, const float* b, int d,
                       float* out, cudaStream_t s, int64_t* launches) {
    if (n <= 0) return;
    const unsigned grid = static_cast<unsigned>((n * d + 255) / 256);
    if (x_f64) k_input_proj<double><<<grid, 256, 0, s>>>(static_cast<const double*>(x), n, f_in, w, b, d, out);
    else k_input_proj<float><<<grid, 256, 0, s>>>(static_cast<const float*>(x), n, f_in, w, b, d, out);
    ++*launches;
}

} // namespace fwa_b200
