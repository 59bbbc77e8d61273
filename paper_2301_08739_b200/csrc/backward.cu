// Block backward on the GPU: fwa_block_backward
// (include/fwa/kernels.hpp:660-765) with its cached forward (kernels.hpp:447-633).
// fp32 SIMT, deterministic (no floating-point atomics: every reduction over rows is a
// fixed-order split into partial sums followed by a fixed-order reduction).  The GEMM-
// shaped pieces (projections, input gradients) use the fp32 tiled GEMM of simt.cu.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "common.cuh"
#include "internal.h"

namespace fwa_b200 {

// ---------------------------------------------------------------- forward pieces with caches

// LayerNorm over d columns, one warp per row (normalize_row, kernels.hpp:235-249):
// xhat = (x - mean) * inv, inv = 1 / sqrt(var + 1e-5); y = g * xhat + b (+ pe)
__global__ void k_ln_fwd_cache(const float* __restrict__ x, const float* __restrict__ pe, int64_t rows, int d,
                               const float* __restrict__ g, const float* __restrict__ b, float* __restrict__ y,
                               float* __restrict__ xhat, float* __restrict__ inv_std) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    const float* xr = x + r * d;
    float s = 0.f;
    for (int c = lane; c < d; c += 32) s += xr[c];
    const float mean = warp_sum(s) / static_cast<float>(d);
    float v = 0.f;
    for (int c = lane; c < d; c += 32) v += (xr[c] - mean) * (xr[c] - mean);
    const float inv = 1.0f / sqrtf(warp_sum(v) / static_cast<float>(d) + 1e-5f);
    for (int c = lane; c < d; c += 32) {
        const float xh = (xr[c] - mean) * inv;
        xhat[r * d + c] = xh;
        y[r * d + c] = g[c] * xh + b[c] + (pe ? pe[r * d + c] : 0.f);
    }
    if (lane == 0) inv_std[r] = inv;
}

// per (group, head): probabilities (max-subtracted softmax, kernels.hpp:512-548) and the
// head outputs; thread per query row
__global__ void k_attn_probs(const float* __restrict__ qkv, int G, int d, int heads, float* __restrict__ probs,
                             float* __restrict__ cat) {
    const int grp = blockIdx.x / heads, head = blockIdx.x % heads;
    const int hd = d / heads;
    const float scale = 1.0f / sqrtf(static_cast<float>(hd));
    const int64_t base = static_cast<int64_t>(grp) * G;
    float* P = probs + (static_cast<int64_t>(grp) * heads + head) * G * G;
    for (int i = threadIdx.x; i < G; i += blockDim.x) {
        const float* qi = qkv + (base + i) * 3 * d + head * hd;
        float m = -INFINITY;
        for (int j = 0; j < G; ++j) {
            const float* kj = qkv + (base + j) * 3 * d + d + head * hd;
            float acc = 0.f;
            for (int c = 0; c < hd; ++c) acc += qi[c] * kj[c];
            acc *= scale;
            P[i * G + j] = acc;
            m = fmaxf(m, acc);
        }
        float sum = 0.f;
        for (int j = 0; j < G; ++j) {
            const float e = expf(P[i * G + j] - m);
            P[i * G + j] = e;
            sum += e;
        }
        const float inv = 1.0f / sum;
        for (int j = 0; j < G; ++j) P[i * G + j] *= inv;
        float* out = cat + (base + i) * d + head * hd;
        for (int c = 0; c < hd; ++c) {
            float acc = 0.f;
            for (int j = 0; j < G; ++j) acc += P[i * G + j] * qkv[(base + j) * 3 * d + 2 * d + head * hd + c];
            out[c] = acc;
        }
    }
}

__global__ void k_gelu_fwd(const float* __restrict__ u, int64_t n, float* __restrict__ a) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) a[i] = gelu_erf(u[i]);
}

// ---------------------------------------------------------------- backward pieces

// g_u = g_a * gelu_grad(u), gelu_grad in fp64 as dense.hpp:74-80
__global__ void k_gelu_back(const float* __restrict__ ga, const float* __restrict__ u, int64_t n,
                            float* __restrict__ gu) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double x = static_cast<double>(u[i]);
    const double cdf = 0.5 * (1.0 + erf(x / 1.4142135623730951));
    const double pdf = exp(-0.5 * x * x) / 2.5066282746310002;
    gu[i] = ga[i] * static_cast<float>(cdf + x * pdf);
}

// layer_norm_backward (kernels.hpp:303-330) per row: g_x = inv (g_xh - m1 - xhat m2),
// g_xh = g_y gamma; also writes g_y * xhat (for d gamma); optional + add[r]
__global__ void k_ln_back(const float* __restrict__ gy, const float* __restrict__ xhat,
                          const float* __restrict__ inv_std, const float* __restrict__ gamma, int64_t rows, int d,
                          const float* __restrict__ add, float* __restrict__ gx, float* __restrict__ gy_xhat) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    float m1 = 0.f, m2 = 0.f;
    for (int c = lane; c < d; c += 32) {
        const float gxh = gy[r * d + c] * gamma[c];
        m1 += gxh;
        m2 += gxh * xhat[r * d + c];
        gy_xhat[r * d + c] = gy[r * d + c] * xhat[r * d + c];
    }
    m1 = warp_sum(m1) / static_cast<float>(d);
    m2 = warp_sum(m2) / static_cast<float>(d);
    const float inv = inv_std[r];
    for (int c = lane; c < d; c += 32) {
        const float gxh = gy[r * d + c] * gamma[c];
        float v = inv * (gxh - m1 - xhat[r * d + c] * m2);
        if (add) v += add[r * d + c];
        gx[r * d + c] = v;
    }
}

// per (group, head): g_q, g_k, g_v (kernels.hpp:708-744) into the packed g_qkv rows
__global__ void k_attn_back(const float* __restrict__ qkv, const float* __restrict__ probs,
                            const float* __restrict__ gcat, int G, int d, int heads, float* __restrict__ gqkv) {
    extern __shared__ float gs[];  // G x G softmax-input gradients (already x scale)
    const int grp = blockIdx.x / heads, head = blockIdx.x % heads;
    const int hd = d / heads;
    const float scale = 1.0f / sqrtf(static_cast<float>(hd));
    const int64_t base = static_cast<int64_t>(grp) * G;
    const float* P = probs + (static_cast<int64_t>(grp) * heads + head) * G * G;
    auto Q = [&](int r, int c) { return qkv[(base + r) * 3 * d + head * hd + c]; };
    auto K = [&](int r, int c) { return qkv[(base + r) * 3 * d + d + head * hd + c]; };
    auto V = [&](int r, int c) { return qkv[(base + r) * 3 * d + 2 * d + head * hd + c]; };
    auto GO = [&](int r, int c) { return gcat[(base + r) * d + head * hd + c]; };
    for (int i = threadIdx.x; i < G; i += blockDim.x) {
        float dot = 0.f;
        for (int j = 0; j < G; ++j) {
            float gp = 0.f;
            for (int c = 0; c < hd; ++c) gp += GO(i, c) * V(j, c);
            gs[i * G + j] = gp;
            dot += gp * P[i * G + j];
        }
        for (int j = 0; j < G; ++j) gs[i * G + j] = P[i * G + j] * (gs[i * G + j] - dot) * scale;
    }
    __syncthreads();
    for (int r = threadIdx.x; r < G; r += blockDim.x) {
        float* gq = gqkv + (base + r) * 3 * d + head * hd;
        float* gk = gq + d;
        float* gv = gq + 2 * d;
        for (int c = 0; c < hd; ++c) {
            float aq = 0.f, ak = 0.f, av = 0.f;
            for (int j = 0; j < G; ++j) {
                aq += gs[r * G + j] * K(j, c);
                ak += gs[j * G + r] * Q(j, c);
                av += P[j * G + r] * GO(j, c);
            }
            gq[c] = aq;
            gk[c] = ak;
            gv[c] = av;
        }
    }
}

// Deterministic reductions over rows.  kChunk rows per partial; partials reduced in chunk
// order.  (1) weight gradient dW[j][k] = sum_r dY[r][j] X[r][k]; (2) column sums.
constexpr int kChunk = 2048;

__global__ void k_wgrad_partial(const float* __restrict__ dy, const float* __restrict__ x, int64_t rows, int J,
                                int K, float* __restrict__ part) {
    __shared__ float sdy[32][33], sx[32][33];
    const int j0 = blockIdx.x * 32, k0 = blockIdx.y * 32, chunk = blockIdx.z;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 256 threads: ty 0..7
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    const int64_t r_begin = static_cast<int64_t>(chunk) * kChunk;
    const int64_t r_end = r_begin + kChunk < rows ? r_begin + kChunk : rows;
    for (int64_t r0 = r_begin; r0 < r_end; r0 += 32) {
        for (int q = 0; q < 4; ++q) {
            const int rr = ty + 8 * q;
            const int64_t r = r0 + rr;
            sdy[rr][tx] = (r < r_end && j0 + tx < J) ? dy[r * J + j0 + tx] : 0.f;
            sx[rr][tx] = (r < r_end && k0 + tx < K) ? x[r * K + k0 + tx] : 0.f;
        }
        __syncthreads();
        for (int rr = 0; rr < 32; ++rr) {
            const float xv = sx[rr][tx];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] += sdy[rr][ty + 8 * q] * xv;
        }
        __syncthreads();
    }
    for (int q = 0; q < 4; ++q) {
        const int j = j0 + ty + 8 * q, k = k0 + tx;
        if (j < J && k < K) part[(static_cast<int64_t>(chunk) * J + j) * K + k] = acc[q];
    }
}

__global__ void k_colsum_partial(const float* __restrict__ y, int64_t rows, int J, float* __restrict__ part) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x, chunk = blockIdx.y;
    if (j >= J) return;
    const int64_t r_begin = static_cast<int64_t>(chunk) * kChunk;
    const int64_t r_end = r_begin + kChunk < rows ? r_begin + kChunk : rows;
    float acc = 0.f;
    for (int64_t r = r_begin; r < r_end; ++r) acc += y[r * J + j];
    part[static_cast<int64_t>(chunk) * J + j] = acc;
}

__global__ void k_reduce_partials(const float* __restrict__ part, int n_chunks, int64_t m, float* __restrict__ out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= m) return;
    float acc = 0.f;
    for (int c = 0; c < n_chunks; ++c) acc += part[c * m + i];
    out[i] = acc;
}

__global__ void k_mul(const float* __restrict__ a, const float* __restrict__ b, int64_t n, float* __restrict__ out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = a[i] * b[i];
}

// ---------------------------------------------------------------- launchers

static unsigned nb(int64_t n, int t = 256) { return static_cast<unsigned>((n + t - 1) / t); }

void launch_ln_fwd_cache(const float* x, const float* pe, int64_t rows, int d, const float* g, const float* b,
                         float* y, float* xhat, float* inv_std, cudaStream_t s, int64_t* launches) {
    k_ln_fwd_cache<<<nb(rows, 8), 256, 0, s>>>(x, pe, rows, d, g, b, y, xhat, inv_std);
    ++*launches;
}

void launch_attn_probs(const float* qkv, int64_t n_groups, int G, int d, int heads, float* probs, float* cat,
                       cudaStream_t s, int64_t* launches) {
    k_attn_probs<<<static_cast<unsigned>(n_groups * heads), 128, 0, s>>>(qkv, G, d, heads, probs, cat);
    ++*launches;
}

void launch_gelu_fwd(const float* u, int64_t n, float* a, cudaStream_t s, int64_t* launches) {
    k_gelu_fwd<<<nb(n), 256, 0, s>>>(u, n, a);
    ++*launches;
}

void launch_gelu_back(const float* ga, const float* u, int64_t n, float* gu, cudaStream_t s, int64_t* launches) {
    k_gelu_back<<<nb(n), 256, 0, s>>>(ga, u, n, gu);
    ++*launches;
}

void launch_ln_back(const float* gy, const float* xhat, const float* inv_std, const float* gamma, int64_t rows,
                    int d, const float* add, float* gx, float* gy_xhat, cudaStream_t s, int64_t* launches) {
    k_ln_back<<<nb(rows, 8), 256, 0, s>>>(gy, xhat, inv_std, gamma, rows, d, add, gx, gy_xhat);
    ++*launches;
}

bool launch_attn_back(const float* qkv, const float* probs, const float* gcat, int64_t n_groups, int G, int d,
                      int heads, float* gqkv, cudaStream_t s, int64_t* launches) {
    const size_t smem = static_cast<size_t>(G) * G * 4;
    if (smem > 200 * 1024) return false;
    static size_t attr = 0;
    if (smem > 48 * 1024 && smem > attr) {
        cudaFuncSetAttribute(k_attn_back, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        attr = smem;
    }
    k_attn_back<<<static_cast<unsigned>(n_groups * heads), 128, smem, s>>>(qkv, probs, gcat, G, d, heads, gqkv);
    ++*launches;
    return true;
}

int reduce_chunks(int64_t rows) { return static_cast<int>((rows + kChunk - 1) / kChunk); }

void launch_wgrad(const float* dy, const float* x, int64_t rows, int J, int K, float* part, float* dw, cudaStream_t s,
                  int64_t* launches) {
    const int nc = reduce_chunks(rows);
    dim3 grid(static_cast<unsigned>((J + 31) / 32), static_cast<unsigned>((K + 31) / 32), static_cast<unsigned>(nc));
    k_wgrad_partial<<<grid, 256, 0, s>>>(dy, x, rows, J, K, part);
    k_reduce_partials<<<nb(static_cast<int64_t>(J) * K), 256, 0, s>>>(part, nc, static_cast<int64_t>(J) * K, dw);
    *launches += 2;
}

void launch_colsum(const float* y, int64_t rows, int J, float* part, float* out, cudaStream_t s, int64_t* launches) {
    const int nc = reduce_chunks(rows);
    k_colsum_partial<<<dim3(static_cast<unsigned>((J + 127) / 128), static_cast<unsigned>(nc)), 128, 0, s>>>(
        y, rows, J, part);
    k_reduce_partials<<<nb(J), 256, 0, s>>>(part, nc, J, out);
    *launches += 2;
}

void launch_mul(const float* a, const float* b, int64_t n, float* out, cudaStream_t s, int64_t* launches) {
    k_mul<<<nb(n), 256, 0, s>>>(a, b, n, out);
    ++*launches;
}

}  // namespace fwa_b200
