// Do legacy HMMA (mma.sync m16n8k16) and MUFU ex2 overlap?  16 warps per SM (one 512-thread
// CTA per SM), each warp runs independent chains: MODE 0 = 8 HMMA f16-accum chains, 1 = 8
// HMMA f32-accum chains, 2 = 8 MUFU.EX2.F16x2 chains, 3 = HMMA(f16) + MUFU chains
// interleaved (8 + 8), 4 = 8 LDSM.x4, 5 = 8 LDSM.x4 + 8 MUFU, 6 = 8 MUFU.EX2 f32,
// 7 = 8 LDSM.x4 + 8 MUFU f32, 8 = 8 LDS.128, 9 = 8 LDS.128 + 8 MUFU.F16x2.  Prints SM clocks per loop iteration (per SM sub-partition: 4 warps).
#include <cstdio>
#include <cstdint>
template <int MODE>
__global__ void __launch_bounds__(512, 1) k(uint32_t* out, long long* clk, int iters) {
    uint32_t a0 = threadIdx.x * 0x00010001u, a1 = a0 ^ 0x3c003c00u, a2 = a0 + 7, a3 = a1 + 9, b0 = a0 ^ 5, b1 = a1 ^ 3;
    uint32_t c[8][2];
    float f[8][4];
    uint32_t m[8];
    for (int i = 0; i < 8; ++i) { c[i][0] = c[i][1] = i; m[i] = 0x3c00bc00u ^ (threadIdx.x + i); for (int j = 0; j < 4; ++j) f[i][j] = 0.f; }
    __shared__ uint4 sm[3072];
    for (int i = threadIdx.x; i < 3072; i += blockDim.x) sm[i] = make_uint4(i, i, i, i);
    uint32_t ld[8][4];
    float mf[8];
    for (int i = 0; i < 8; ++i) { mf[i] = -0.001f * i; for (int j = 0; j < 4; ++j) ld[i][j] = 0; }
    const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(sm)) + (threadIdx.x & 31) * 16 + (threadIdx.x >> 5) * 1024;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0 || MODE == 3)
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f16.f16.f16.f16 {%0,%1}, {%2,%3,%4,%5}, {%6,%7}, {%0,%1};"
                             : "+r"(c[i][0]), "+r"(c[i][1]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
            if (MODE == 1)
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+f"(f[i][0]), "+f"(f[i][1]), "+f"(f[i][2]), "+f"(f[i][3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
            if (MODE == 2 || MODE == 3 || MODE == 5 || MODE == 9) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(m[i]));
            if (MODE == 6 || MODE == 7) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(mf[i]));
            if (MODE == 4 || MODE == 5 || MODE == 7) {
                uint32_t r0, r1, r2, r3;
                asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];" : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(sbase + ((it * 8 + i) & 1) * 16384));
                ld[i][0] ^= r0; ld[i][1] ^= r1; ld[i][2] ^= r2; ld[i][3] ^= r3;
            }
            if (MODE == 8 || MODE == 9) {
                uint32_t r0, r1, r2, r3;
                asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(sbase + ((it * 8 + i) & 1) * 16384));
                ld[i][0] ^= r0; ld[i][1] ^= r1; ld[i][2] ^= r2; ld[i][3] ^= r3;
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    uint32_t s = 0;
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + m[i] + __float_as_uint(f[i][0]) + ld[i][0] + ld[i][3] + __float_as_uint(mf[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
template <int MODE> void run(const char* name) {
    uint32_t* o; long long* c; cudaMalloc(&o, 148 * 512 * 4); cudaMalloc(&c, 148 * 8);
    const int iters = 2048;
    k<MODE><<<148, 512>>>(o, c, iters); cudaDeviceSynchronize();
    k<MODE><<<148, 512>>>(o, c, iters); cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-28s %.2f clk per iteration (8 ops per warp, 4 warps per SMSP)\n", name, (double)h[0] / iters);
    cudaFree(o); cudaFree(c);
}
int main() {
    run<0>("HMMA f16 acc x8"); run<1>("HMMA f32 acc x8"); run<2>("MUFU ex2.f16x2 x8"); run<3>("HMMA f16 + MUFU x8 each");
    run<4>("LDSM.x4 x8"); run<5>("LDSM.x4 + MUFU.F16x2 x8 each"); run<6>("MUFU f32 x8"); run<7>("LDSM.x4 + MUFU f32 x8 each");
    run<8>("LDS.128 x8"); run<9>("LDS.128 + MUFU.F16x2 x8 each");
}
