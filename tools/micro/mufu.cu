// MUFU throughput probe: warp-instructions per SM clock for ex2.f32, ex2.f16x2,
// ex2.bf16x2, tanh.f32, tanh.f16x2, rcp.f32 (8 independent chains per thread).
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
template <int OP>
__global__ void k(float* out, long long* clk, int iters) {
    float v[8];
    uint32_t h[8];
    for (int i = 0; i < 8; ++i) { v[i] = -0.001f * (threadIdx.x + i); h[i] = 0x3c00bc00u ^ (threadIdx.x + i); }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
            if (OP == 1) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h[i]));
            if (OP == 2) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h[i]));
            if (OP == 3) asm volatile("tanh.approx.f32 %0, %0;" : "+f"(v[i]));
            if (OP == 4) asm volatile("tanh.approx.f16x2 %0, %0;" : "+r"(h[i]));
            if (OP == 5) asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
            if (OP == 6) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(v[i]));
            if (OP == 7) asm volatile("tanh.approx.bf16x2 %0, %0;" : "+r"(h[i]));
            if (OP == 8) asm volatile("cvt.rn.f16x2.f32 %0, %1, %1;" : "+r"(h[i]) : "f"(__uint_as_float(h[i])));
            if (OP == 9) asm volatile("fma.rn.f16x2 %0, %0, %0, %0;" : "+r"(h[i]));
        }
    }
    __syncthreads();
    long long t1 = clock64();
    float s = 0; for (int i = 0; i < 8; ++i) s += v[i] + __uint_as_float(h[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
template <int OP> void run(const char* name) {
    float* o; long long* c; cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 148 * 8);
    const int iters = 4096;
    k<OP><<<148, 1024>>>(o, c, iters); cudaDeviceSynchronize();
    k<OP><<<148, 1024>>>(o, c, iters); cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    double warp_instr = 32.0 * iters * 8;  // per SM: 32 warps x iters x 8
    printf("%-12s %.3f warp-instr/clk/SM  (%.1f lanes/clk/SM)\n", name, warp_instr / h[0], 32 * warp_instr / h[0]);
    cudaFree(o); cudaFree(c);
}
int main() {
    run<0>("ex2.f32"); run<1>("ex2.f16x2"); run<2>("ex2.bf16x2"); run<3>("tanh.f32"); run<4>("tanh.f16x2");
    run<5>("rcp.f32"); run<6>("ffma"); run<7>("tanh.bf16x2"); run<8>("cvt.f16x2.f32"); run<9>("hfma2");
}
