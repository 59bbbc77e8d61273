// GPU pillarization: fwa::geometry::pillarize (include/fwa/geometry.hpp:246-300), the
// stage right before the backbone boundary.
//
//   cell   = (floor(x / res), floor(y / res))            fp64 RN, op by op (geometry.hpp:266-271)
//   pillars = the non-empty cells in ascending lexicographic (x-cell, y-cell) order
//             (std::map order), members in ingestion order
//   pooled[c] = pairwise_sum(member features of channel c) / m   (dense.hpp:84-94)
//   feature[o] = gelu(bias[o] + sum_c w[o][c] pooled[c])         (geometry.hpp:287-292, dense.hpp:67-72)
//   coord   = ((cell + 0.5) * res)                               (geometry.hpp:293-294)
//
// Dense cell grid over the cloud's cell range: histogram -> exclusive scan (cell order IS
// the lexicographic order) -> non-empty flag scan (pillar rows) -> atomic scatter of point
// ids into their cell's slots -> rank of each id among its cell's ids (ingestion order)
// -> the features gathered into pillar order -> pooling and the linear + GELU per
// (pillar, output).  Integer structure (cells, order, coords) is bit-exact; the features
// use the same fp64 operation order as the reference (no FMA contraction: RN intrinsics),
// with CUDA's erf (<= 2 ulp) for libm's.
#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>

#include "common.cuh"
#include "internal.h"

namespace fwa_b200 {

__global__ void k_cell_keys(const double* __restrict__ xy, int64_t n, double res, long long* __restrict__ cell,
                            long long* __restrict__ mm) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    long long a0 = LLONG_MAX, a1 = LLONG_MIN, b0 = LLONG_MAX, b1 = LLONG_MIN;
    if (i < n) {
        const double2 p = reinterpret_cast<const double2*>(xy)[i];
        const long long cx = static_cast<long long>(floor(__ddiv_rn(p.x, res)));
        const long long cy = static_cast<long long>(floor(__ddiv_rn(p.y, res)));
        reinterpret_cast<longlong2*>(cell)[i] = make_longlong2(cx, cy);
        a0 = a1 = cx;
        b0 = b1 = cy;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a0 = min(a0, __shfl_xor_sync(0xffffffffu, a0, o));
        a1 = max(a1, __shfl_xor_sync(0xffffffffu, a1, o));
        b0 = min(b0, __shfl_xor_sync(0xffffffffu, b0, o));
        b1 = max(b1, __shfl_xor_sync(0xffffffffu, b1, o));
    }
    if ((threadIdx.x & 31) == 0 && a0 != LLONG_MAX) {
        atomicMin(mm + 0, a0);
        atomicMax(mm + 1, a1);
        atomicMin(mm + 2, b0);
        atomicMax(mm + 3, b1);
    }
}

__global__ void k_init_cell_mm(long long* mm) {
    mm[0] = LLONG_MAX;
    mm[1] = LLONG_MIN;
    mm[2] = LLONG_MAX;
    mm[3] = LLONG_MIN;
}

// dense cell id (lexicographic in (cx, cy)) + histogram
__global__ void k_cell_hist(const long long* __restrict__ cell, int64_t n, long long min_x, long long min_y,
                            long long range_y, uint32_t* __restrict__ cell_id, uint32_t* __restrict__ hist) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const longlong2 c = reinterpret_cast<const longlong2*>(cell)[i];
    const uint32_t id = static_cast<uint32_t>((c.x - min_x) * range_y + (c.y - min_y));
    cell_id[i] = id;
    atomicAdd(hist + id, 1u);
}

__global__ void k_nonempty(const uint32_t* __restrict__ hist, int64_t ncell, uint32_t* __restrict__ flag) {
    const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c < ncell) flag[c] = hist[c] ? 1u : 0u;
}

// pillar row p -> its cell, coordinates ((cell + 0.5) * res)
__global__ void k_pillar_cells(const uint32_t* __restrict__ hist, const uint32_t* __restrict__ prow, int64_t ncell,
                               long long min_x, long long min_y, long long range_y, double res,
                               uint32_t* __restrict__ pcell, double* __restrict__ coords) {
    const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= ncell || hist[c] == 0u) return;
    const uint32_t p = prow[c];
    pcell[p] = static_cast<uint32_t>(c);
    const long long cx = min_x + c / range_y, cy = min_y + c % range_y;
    reinterpret_cast<double2*>(coords)[p] =
        make_double2(__dmul_rn(__dadd_rn(static_cast<double>(cx), 0.5), res),
                     __dmul_rn(__dadd_rn(static_cast<double>(cy), 0.5), res));
}

__global__ void k_cell_scatter(const uint32_t* __restrict__ cell_id, int64_t n, uint32_t* __restrict__ cursor,
                               int32_t* __restrict__ slot_pt) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    slot_pt[atomicAdd(cursor + cell_id[i], 1u)] = static_cast<int32_t>(i);
}

// each point's rank among its cell's points (= ingestion order), its features copied to
// the member-ordered array fs[(start + rank) * f_in + c]
__global__ void k_member_order(const uint32_t* __restrict__ cell_id, const uint32_t* __restrict__ start,
                               const uint32_t* __restrict__ hist, const int32_t* __restrict__ slot_pt, int64_t n,
                               const double* __restrict__ feats, int f_in, double* __restrict__ fs) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t c = cell_id[i];
    const uint32_t s0 = start[c], m = hist[c];
    uint32_t rank = 0;
    for (uint32_t k = 0; k < m; ++k) rank += slot_pt[s0 + k] < i ? 1u : 0u;
    for (int ch = 0; ch < f_in; ++ch)
        fs[(static_cast<int64_t>(s0) + rank) * f_in + ch] = feats[i * f_in + ch];
}

// pairwise_sum (dense.hpp:84-94): <= 8 summed left to right from 0.0, else the two halves
__device__ double pw_sum(const double* v, int stride, uint32_t n) {
    if (n <= 8u) {
        double s = 0.0;
        for (uint32_t k = 0; k < n; ++k) s = __dadd_rn(s, v[static_cast<int64_t>(k) * stride]);
        return s;
    }
    const uint32_t h = n / 2;
    return __dadd_rn(pw_sum(v, stride, h), pw_sum(v + static_cast<int64_t>(h) * stride, stride, n - h));
}

// one thread per (pillar, channel): the pooled (mean) feature
__global__ void k_pool(const uint32_t* __restrict__ pcell, const uint32_t* __restrict__ start,
                       const uint32_t* __restrict__ hist, int64_t np, int f_in, const double* __restrict__ fs,
                       double* __restrict__ pooled) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= np * f_in) return;
    const int64_t p = t / f_in;
    const int ch = static_cast<int>(t % f_in);
    const uint32_t c = pcell[p], m = hist[c];
    pooled[t] = __ddiv_rn(pw_sum(fs + static_cast<int64_t>(start[c]) * f_in + ch, f_in, m), static_cast<double>(m));
}

// one thread per (pillar, output): gelu(bias[o] + sum_c w[o][c] pooled[c]) in fp64
__global__ void k_pillar_linear_gelu(const double* __restrict__ pooled, int64_t np, int f_in,
                                     const double* __restrict__ w, const double* __restrict__ bias, int d_out,
                                     double* __restrict__ out) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= np * d_out) return;
    const int64_t p = t / d_out;
    const int o = static_cast<int>(t % d_out);
    double acc = bias ? bias[o] : 0.0;
    for (int c = 0; c < f_in; ++c)
        acc = __dadd_rn(acc, __dmul_rn(w[static_cast<int64_t>(o) * f_in + c], pooled[p * f_in + c]));
    // T(0.5) * x * (T(1) + erf(x / sqrt 2))
    out[t] = __dmul_rn(__dmul_rn(0.5, acc), __dadd_rn(1.0, erf(__ddiv_rn(acc, 1.4142135623730951))));
}

// ------------------------------------------------------------------ launchers

static unsigned blocks(int64_t n, int t = 256) { return static_cast<unsigned>((n + t - 1) / t); }

void launch_cell_keys(const double* xy, int64_t n, double res, long long* cell, long long* mm, cudaStream_t s,
                      int64_t* launches) {
    k_init_cell_mm<<<1, 1, 0, s>>>(mm);
    if (n > 0) k_cell_keys<<<blocks(n), 256, 0, s>>>(xy, n, res, cell, mm);
    *launches += 2;
}

void launch_cell_hist(const long long* cell, int64_t n, long long min_x, long long min_y, long long range_y,
                      uint32_t* cell_id, uint32_t* hist, cudaStream_t s, int64_t* launches) {
    k_cell_hist<<<blocks(n), 256, 0, s>>>(cell, n, min_x, min_y, range_y, cell_id, hist);
    ++*launches;
}

void launch_nonempty(const uint32_t* hist, int64_t ncell, uint32_t* flag, cudaStream_t s, int64_t* launches) {
    k_nonempty<<<blocks(ncell), 256, 0, s>>>(hist, ncell, flag);
    ++*launches;
}

void launch_pillar_cells(const uint32_t* hist, const uint32_t* prow, int64_t ncell, long long min_x, long long min_y,
                         long long range_y, double res, uint32_t* pcell, double* coords, cudaStream_t s,
                         int64_t* launches) {
    k_pillar_cells<<<blocks(ncell), 256, 0, s>>>(hist, prow, ncell, min_x, min_y, range_y, res, pcell, coords);
    ++*launches;
}

void launch_cell_members(const uint32_t* cell_id, int64_t n, uint32_t* cursor, int32_t* slot_pt,
                         const uint32_t* start, const uint32_t* hist, const double* feats, int f_in, double* fs,
                         cudaStream_t s, int64_t* launches) {
    k_cell_scatter<<<blocks(n), 256, 0, s>>>(cell_id, n, cursor, slot_pt);
    k_member_order<<<blocks(n), 256, 0, s>>>(cell_id, start, hist, slot_pt, n, feats, f_in, fs);
    *launches += 2;
}

void launch_pillar_features(const uint32_t* pcell, const uint32_t* start, const uint32_t* hist, int64_t np,
                            int f_in, const double* fs, double* pooled, const double* w, const double* bias,
                            int d_out, double* out, cudaStream_t s, int64_t* launches) {
    if (f_in > 0) k_pool<<<blocks(np * f_in), 256, 0, s>>>(pcell, start, hist, np, f_in, fs, pooled);
    k_pillar_linear_gelu<<<blocks(np * d_out), 256, 0, s>>>(pooled, np, f_in, w, bias, d_out, out);
    *launches += 2;
}

}  // namespace fwa_b200
