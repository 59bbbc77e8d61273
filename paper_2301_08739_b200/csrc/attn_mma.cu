// Fused per-group multi-head self-attention on the tensor cores (bf16 fast
// path, head dim 16).  Reference: group_attention_forward's per-group/per-head
// loop, /root/reference/proj/include/fwa/kernels.hpp:512-548 (+ softmax_row 251-262):
//   S = q_i . k_j / sqrt(16);  P = softmax_j(S) (max-subtracted);  O = P V.
//
// One CTA per group, one warp per head.  The group's q|k|v rows (G x 384 bf16,
// contiguous in HBM because rows are in window-sort order) are staged in
// shared memory with a 784 B row pitch (conflict-free ldmatrix), padded to a
// multiple of 16 rows with zeros.  Per 16-query tile: QK^T with
// mma.sync.m16n8k16 (fp32 accumulate) into registers, key columns >= G masked
// to -inf, warp-quad softmax in fp32 (exp2 with pre-scaled log2e), P re-used
// straight from the accumulator registers as the bf16 A operand of PV.
// G <= 128 (8 n-tile pairs); no padding to spatial windows.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "internal.h"

namespace fwa_b200 {

constexpr int kPitch = 768 + 16;  // bytes per staged row

// element (row, col) of a 128-row K-major SW128 bf16 image (see tcgen05.cuh sw128_offset)
FWA_DEVINL uint32_t tc_sw128_offset(int row, int col) {
    return static_cast<uint32_t>((col >> 6) * 16384 + row * 128 + ((((col & 63) >> 3) ^ (row & 7)) << 4) +
                                 (col & 7) * 2);
}

// 2^x on the SFU (rel err 2^-22), -inf -> +0
FWA_DEVINL float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

FWA_DEVINL void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
FWA_DEVINL void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
FWA_DEVINL void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// NT = padded group / 8 (even); MT = NT / 2 query tiles; KT = NT / 2 key tiles.
// GC > 0: the group size is a compile-time constant (the default config's 69) so the key
// masking and the skipped all-padding tiles are resolved at compile time.
template <int NT, int GC>
__global__ void __launch_bounds__(256, 3) k_attention_mma(const __nv_bfloat16* __restrict__ qkv,
                                                          int64_t rows, int G_rt,
                                                          uint8_t* __restrict__ cat) {
    const int G = GC > 0 ? GC : G_rt;
    extern __shared__ __align__(16) uint8_t sm[];
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");  // q|k|v come from the previous kernel
    constexpr int Gp = NT * 8;
    const int64_t base = static_cast<int64_t>(blockIdx.x) * G;
    // ---- stage q|k|v rows: the QKV kernel writes 12 column chunks of [rows x 32]
    // bf16, so each chunk of this group is one contiguous 64*G-byte run; cp.async
    // (16 B, L1-bypassing) into a 784 B row pitch; padding rows zeroed.
    const uint32_t s_base = smem_u32(sm);
#pragma unroll 4
    for (int t = threadIdx.x; t < 12 * Gp * 4; t += 256) {
        const int c = t / (Gp * 4), rem = t - c * (Gp * 4), r = rem >> 2, pp = rem & 3;  // Gp constexpr
        const uint32_t dst = s_base + r * kPitch + c * 64 + pp * 16;
        if (r < G) {
            const __nv_bfloat16* src = qkv + (static_cast<int64_t>(c) * rows + base + r) * 32 + pp * 8;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
        } else {
            asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(dst), "r"(0u) : "memory");
        }
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    const int head = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t4 = lane & 3;
    const uint32_t s0 = smem_u32(sm);
    const uint32_t qcol = head * 32, kcol = 256 + head * 32, vcol = 512 + head * 32;  // bytes
    constexpr float kScaleLog2 = 0.25f * 1.4426950408889634f;  // (1/sqrt(16)) * log2(e)

    // K fragments for all key tiles are reused by every query tile: keep in registers.
    uint32_t kb[NT][2];
#pragma unroll
    for (int np = 0; np < NT; np += 2) {
        const int krow = (np + (lane >> 4)) * 8 + (lane & 7);
        const uint32_t addr = s0 + krow * kPitch + kcol + ((lane >> 3) & 1) * 16;
        ldsm_x4(addr, kb[np][0], kb[np][1], kb[np + 1][0], kb[np + 1][1]);
    }
    uint32_t vb[NT / 2][4];
#pragma unroll
    for (int kt = 0; kt < NT / 2; ++kt) {
        const int vrow = kt * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const uint32_t addr = s0 + vrow * kPitch + vcol + (lane >> 4) * 16;
        ldsm_x4_t(addr, vb[kt][0], vb[kt][1], vb[kt][2], vb[kt][3]);
    }

#pragma unroll 1
    for (int mt = 0; mt < NT / 2; ++mt) {
        uint32_t a0, a1, a2, a3;
        {
            const int qrow = mt * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
            ldsm_x4(s0 + qrow * kPitch + qcol + (lane >> 4) * 16, a0, a1, a2, a3);
        }
        // key tiles entirely beyond G carry P = 0: skip their QK^T, exp and PV work;
        // only the boundary tile needs a mask (G is uniform across the CTA)
        const int nt_live = (G + 7) >> 3;
        float s[NT][4];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
            if (nt < nt_live) mma16816(s[nt], a0, a1, a2, a3, kb[nt][0], kb[nt][1]);
        }
        float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            if (nt >= nt_live) continue;
            if (nt * 8 + 8 > G) {
                const int col = nt * 8 + 2 * t4;
                if (col >= G) { s[nt][0] = -INFINITY; s[nt][2] = -INFINITY; }
                if (col + 1 >= G) { s[nt][1] = -INFINITY; s[nt][3] = -INFINITY; }
            }
            m0 = fmaxf(m0, fmaxf(s[nt][0], s[nt][1]));
            m1 = fmaxf(m1, fmaxf(s[nt][2], s[nt][3]));
        }
        m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 1));
        m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 2));
        m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 1));
        m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 2));
        const float mb0 = m0 * kScaleLog2, mb1 = m1 * kScaleLog2;
        float l0 = 0.f, l1 = 0.f;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            if (nt >= nt_live) continue;
            s[nt][0] = ex2_approx(fmaf(s[nt][0], kScaleLog2, -mb0));
            s[nt][1] = ex2_approx(fmaf(s[nt][1], kScaleLog2, -mb0));
            s[nt][2] = ex2_approx(fmaf(s[nt][2], kScaleLog2, -mb1));
            s[nt][3] = ex2_approx(fmaf(s[nt][3], kScaleLog2, -mb1));
            l0 += s[nt][0] + s[nt][1];
            l1 += s[nt][2] + s[nt][3];
        }
        l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
        l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
        l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
        l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
        // O = P V  (P from the accumulator registers, bf16)
        float o[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
        for (int kt = 0; kt < NT / 2; ++kt) {
            if (2 * kt >= nt_live) continue;
            const uint32_t p0 = pack_bf16x2(s[2 * kt][0], s[2 * kt][1]);
            const uint32_t p1 = pack_bf16x2(s[2 * kt][2], s[2 * kt][3]);
            const uint32_t p2 = pack_bf16x2(s[2 * kt + 1][0], s[2 * kt + 1][1]);
            const uint32_t p3 = pack_bf16x2(s[2 * kt + 1][2], s[2 * kt + 1][3]);
            mma16816(o[0], p0, p1, p2, p3, vb[kt][0], vb[kt][1]);
            mma16816(o[1], p0, p1, p2, p3, vb[kt][2], vb[kt][3]);
        }
        const float i0 = 1.0f / l0, i1 = 1.0f / l1;
        const int r0 = mt * 16 + g, r1 = r0 + 8;
        // output rows go straight into the out-proj kernel's A-operand images: per
        // 128-row tile, a K-major SW128 [128 x 128] bf16 image (one TMA bulk load there)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
            const int col = head * 16 + nt * 8 + 2 * t4;
            if (r0 < G) {
                const int64_t gr = base + r0;
                *reinterpret_cast<uint32_t*>(cat + (gr >> 7) * 32768 + tc_sw128_offset(static_cast<int>(gr & 127), col)) =
                    pack_bf16x2(o[nt][0] * i0, o[nt][1] * i0);
            }
            if (r1 < G) {
                const int64_t gr = base + r1;
                *reinterpret_cast<uint32_t*>(cat + (gr >> 7) * 32768 + tc_sw128_offset(static_cast<int>(gr & 127), col)) =
                    pack_bf16x2(o[nt][2] * i1, o[nt][3] * i1);
            }
        }
    }
}

template <int NT, int GC = 0>
static void launch_nt(const __nv_bfloat16* qkv, int64_t rows, int64_t n_groups, int G, uint8_t* cat,
                      cudaStream_t s) {
    const int smem = NT * 8 * kPitch;
    static bool init = false;
    if (!init) {
        cudaFuncSetAttribute(k_attention_mma<NT, GC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_attention_mma<NT, GC>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        init = true;
    }
    launch_pdl(k_attention_mma<NT, GC>, dim3(static_cast<unsigned>(n_groups)), dim3(256), smem, s, qkv, rows, G,
               cat);
}

void launch_attention_mma(const __nv_bfloat16* qkv, int64_t rows, int G, __nv_bfloat16* cat_img,
                          cudaStream_t s, int64_t* launches) {
    uint8_t* cat = reinterpret_cast<uint8_t*>(cat_img);
    const int64_t n_groups = rows / G;
    if (n_groups == 0) return;
    const int nt = ((G + 15) / 16) * 2;
    if (G == 69) {  // FwaConfig default group size (backbone.hpp:26)
        launch_nt<10, 69>(qkv, rows, n_groups, G, cat, s);
        ++*launches;
        return;
    }
    switch (nt) {
        case 2: launch_nt<2>(qkv, rows, n_groups, G, cat, s); break;
        case 4: launch_nt<4>(qkv, rows, n_groups, G, cat, s); break;
        case 6: launch_nt<6>(qkv, rows, n_groups, G, cat, s); break;
        case 8: launch_nt<8>(qkv, rows, n_groups, G, cat, s); break;
        case 10: launch_nt<10>(qkv, rows, n_groups, G, cat, s); break;
        case 12: launch_nt<12>(qkv, rows, n_groups, G, cat, s); break;
        case 14: launch_nt<14>(qkv, rows, n_groups, G, cat, s); break;
        default: launch_nt<16>(qkv, rows, n_groups, G, cat, s); break;
    }
    ++*launches;
}

} // namespace fwa_b200
