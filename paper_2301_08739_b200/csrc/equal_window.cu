// Equal-window (SST-style) padded baseline on the GPU, the
// comparison the reference's `fwa bench --mode equal-window` makes
// (include/fwa/bench.hpp:266-326, include/fwa/workload.hpp:44-142):
//   partition the pillars by window (X axis, no shift), bucket the windows by occupancy
//   (edges 16/32/64/128/256), pad every window to its bucket's largest occupancy with
//   zero rows, then run the SAME block kernel per bucket with G = that pad.
// The window partition reuses the window sort (windows in lexicographic order; members
// inside a window in window-local coordinate order -- attention is permutation-
// equivariant inside a window, so outputs match the reference's ingestion order up to
// rounding).  Padding rows gather a zero row (index n) and scatter to a sink row (n + 1).
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "internal.h"

namespace fwa_b200 {

__global__ void k_ew_flags(const int32_t* __restrict__ sorted, const uint32_t* __restrict__ bin_of, int64_t n,
                           uint32_t* __restrict__ flag) {
    const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= n) return;
    flag[p] = (p == 0 || bin_of[sorted[p]] != bin_of[sorted[p - 1]]) ? 1u : 0u;
}

// window starts (in sorted order) from the run flags and their exclusive scan
__global__ void k_ew_starts(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ ex, int64_t n,
                            uint32_t* __restrict__ wstart) {
    const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p < n && flag[p]) wstart[ex[p]] = static_cast<uint32_t>(p);
}

// occupancy and bucket of every window; per-bucket window count and largest occupancy
__global__ void k_ew_bucket(const uint32_t* __restrict__ wstart, int64_t W, int64_t n, const int32_t* __restrict__ edges,
                            int n_edges, uint32_t* __restrict__ wocc, int32_t* __restrict__ wbucket,
                            uint32_t* __restrict__ bmax, uint32_t* __restrict__ bcnt, int* __restrict__ overflow) {
    const int64_t w = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (w >= W) return;
    const uint32_t occ = (w + 1 < W ? wstart[w + 1] : static_cast<uint32_t>(n)) - wstart[w];
    int b = 0;
    while (b < n_edges && static_cast<int>(occ) > edges[b]) ++b;
    wocc[w] = occ;
    if (b == n_edges) {  // bench.hpp:288 "occupancy exceeds final bucket edge"
        *overflow = 1;
        b = n_edges - 1;
    }
    wbucket[w] = b;
    atomicMax(bmax + b, occ);
    atomicAdd(bcnt + b, 1u);
}

__global__ void k_ew_bflag(const int32_t* __restrict__ wbucket, int64_t W, int b, uint32_t* __restrict__ flag) {
    const int64_t w = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (w < W) flag[w] = wbucket[w] == b ? 1u : 0u;
}

// rows of bucket b: window w (bucket rank r) occupies rows [r*pad, (r+1)*pad): its members,
// then zero rows (gather index n, scatter index n + 1)
__global__ void k_ew_fill(const uint32_t* __restrict__ wstart, const uint32_t* __restrict__ wocc,
                          const int32_t* __restrict__ wbucket, const uint32_t* __restrict__ wrank, int64_t W, int b,
                          int pad, const int32_t* __restrict__ sorted, int64_t n, int32_t* __restrict__ ridx,
                          int32_t* __restrict__ sidx) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= W * pad) return;
    const int64_t w = t / pad;
    const int k = static_cast<int>(t % pad);
    if (wbucket[w] != b) return;
    const int64_t row = static_cast<int64_t>(wrank[w]) * pad + k;
    if (k < static_cast<int>(wocc[w])) {
        const int32_t id = sorted[wstart[w] + k];
        ridx[row] = id;
        sidx[row] = id;
    } else {
        ridx[row] = static_cast<int32_t>(n);
        sidx[row] = static_cast<int32_t>(n + 1);
    }
}

static unsigned nblk(int64_t n) { return static_cast<unsigned>((n + 255) / 256); }

void launch_ew_runs(const int32_t* sorted, const uint32_t* bin_of, int64_t n, uint32_t* flag, cudaStream_t s,
                    int64_t* launches) {
    k_ew_flags<<<nblk(n), 256, 0, s>>>(sorted, bin_of, n, flag);
    ++*launches;
}

void launch_ew_starts(const uint32_t* flag, const uint32_t* ex, int64_t n, uint32_t* wstart, cudaStream_t s,
                      int64_t* launches) {
    k_ew_starts<<<nblk(n), 256, 0, s>>>(flag, ex, n, wstart);
    ++*launches;
}

void launch_ew_bucket(const uint32_t* wstart, int64_t W, int64_t n, const int32_t* edges, int n_edges, uint32_t* wocc,
                      int32_t* wbucket, uint32_t* bmax, uint32_t* bcnt, int* overflow, cudaStream_t s,
                      int64_t* launches) {
    k_ew_bucket<<<nblk(W), 256, 0, s>>>(wstart, W, n, edges, n_edges, wocc, wbucket, bmax, bcnt, overflow);
    ++*launches;
}

void launch_ew_bflag(const int32_t* wbucket, int64_t W, int b, uint32_t* flag, cudaStream_t s, int64_t* launches) {
    k_ew_bflag<<<nblk(W), 256, 0, s>>>(wbucket, W, b, flag);
    ++*launches;
}

void launch_ew_fill(const uint32_t* wstart, const uint32_t* wocc, const int32_t* wbucket, const uint32_t* wrank,
                    int64_t W, int b, int pad, const int32_t* sorted, int64_t n, int32_t* ridx, int32_t* sidx,
                    cudaStream_t s, int64_t* launches) {
    k_ew_fill<<<nblk(W * pad), 256, 0, s>>>(wstart, wocc, wbucket, wrank, W, b, pad, sorted, n, ridx, sidx);
    ++*launches;
}

}  // namespace fwa_b200
