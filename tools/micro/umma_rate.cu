// Pair-MMA (tcgen05.mma.cta_group::2, kind::f16, A and B from shared memory, SW128 K-major)
// issue-to-completion time in isolation: 74 CTA pairs, the leader issues NM MMAs of
// M = 256, N = {128, 256}, K = 16 (cycling over the 8 K-steps of a 128-wide K) and waits for
// the commit.  Compare with the tensor floor max(M,128)*N/(256*2) cycles per MMA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2301_08739_b200/csrc tools/micro/umma_rate.cu -o /tmp/umma_rate
#include <cstdio>
#include <cstdint>
#include "common.cuh"
#include "tcgen05.cuh"
using namespace fwa_b200;
using namespace fwa_b200::tc;

__device__ __forceinline__ uint32_t crank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void csync() { asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit2(uint64_t* bar) {
    const uint16_t mask = 3;
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(bar)), "h"(mask) : "memory");
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
template <int N, int NM, bool TS = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k(long long* out, int reps) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 131072);
    uint32_t* slot = reinterpret_cast<uint32_t*>(sm + 131072 + 64);
    for (int i = threadIdx.x; i < 131072 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x3c003c00u, 0, 0x3c00u, 0);
    const uint32_t rank = crank();
    if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    fence_before_sync();
    __syncthreads();
    csync();
    fence_after_sync();
    const uint32_t tmem = *slot;
    const uint32_t sA = smem_u32(sm), sB = sA + 32768;
    constexpr uint32_t id = idesc_bf16_f32(256, N);
    long long best = 1LL << 60, tot = 0;
    for (int r = 0; r < reps; ++r) {
        if (rank == 0 && threadIdx.x == 0) {
            const long long t0 = clock64();
#pragma unroll 1
            for (int m = 0; m < NM; ++m) {
                const int ks = m & 7;
                if (TS) mma2_ts(tmem, tmem + 384 + 8 * ks, sdesc_sw128(sB + (ks >> 2) * (N / 2) * 128 + (ks & 3) * 32), id, m ? 1u : 0u);
                else mma2(tmem, sdesc_sw128(sA + (ks >> 2) * 16384 + (ks & 3) * 32), sdesc_sw128(sB + (ks >> 2) * (N / 2) * 128 + (ks & 3) * 32), id, m ? 1u : 0u);
            }
            commit2(bar);
            mbar_wait(bar, r & 1);
            const long long dt = clock64() - t0;
            best = dt < best ? dt : best;
            tot += dt;
        } else if (threadIdx.x == 0) {
            mbar_wait(bar, r & 1);
        }
        fence_after_sync();
        __syncthreads();
        csync();
    }
    if (rank == 0 && threadIdx.x == 0) { out[blockIdx.x] = best; out[gridDim.x + blockIdx.x] = tot / reps; }
    fence_before_sync();
    __syncthreads();
    csync();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}
template <int N, int NM, bool TS = false> void run() {
    long long* d; cudaMalloc(&d, 2 * 148 * 8);
    cudaFuncSetAttribute(k<N, NM, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072 + 2048);
    k<N, NM, TS><<<148, 128, 131072 + 2048>>>(d, 20);
    k<N, NM, TS><<<148, 128, 131072 + 2048>>>(d, 20);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[296]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const double floor_ = 256.0 * N / 512.0;
    printf("%s N=%3d x %3d MMAs: best %6lld clk (%.1f per MMA), mean %6lld; floor %.0f per MMA  [%s]\n", TS ? "A:tmem" : "A:smem", N, NM, h[0], (double)h[0] / NM, h[148], floor_, cudaGetErrorString(e));
    cudaFree(d);
}
int main() {
    run<128, 8>(); run<128, 24>(); run<128, 64>();
    run<256, 8>(); run<256, 24>(); run<256, 64>();
    run<128, 8, true>(); run<128, 24, true>(); run<128, 64, true>();
    return 0;
}
