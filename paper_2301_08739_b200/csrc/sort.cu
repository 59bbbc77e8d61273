// Window sort (Eq. 1 of FlatFormer), equal-size grouping and drop schedule on
// the device, bit-exact with the reference:
//
//   make_sort_key   /root/reference/proj/include/fwa/flatten.hpp:49-69
//   key_less        flatten.hpp:41-47
//   sort            flatten.hpp:97-120
//   group           flatten.hpp:134-146
//   drop/compaction /root/reference/proj/include/fwa/backbone.hpp:285-316
//
// Design: all four (axis, shift) specs of one or many
// frames are sorted in ONE batched pass.
//   K1 keys:   fp64 shift/div/floor/mul/sub with explicit round-to-nearest
//              intrinsics (no FMA contraction can change a key bit), + window
//              min/max per spec.
//   K2 bins:   dense window-bin id (spec, frame, win_major, win_minor) — the
//              lexicographic order of (win_major, win_minor) IS the bin order —
//              and an HBM histogram (1-digit counting sort on the window id).
//   K3 scan + scatter into bins (order inside a bin is irrelevant: K4 totally
//              orders it).
//   K4 per-bin exact comparator sort on (loc_major, loc_minor, orig index):
//              a warp rank-sort in shared memory for bins <= 128 points (pillar
//              windows hold <= (9+1)^2), a CTA rank-sort for <= 4096, and a
//              CTA bitonic network in global scratch beyond that, so any input
//              is ordered exactly as std::sort(key_less) orders it.
#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>

#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"
#include "internal.h"

namespace fwa_b200 {


// ------------------------------------------------------------------ scan

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(const uint32_t* in, uint32_t* out,
                                                              int64_t n, uint32_t* tile_sums) {
    __shared__ uint32_t warp_tot[32];
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
    uint32_t v[kScanItems];
    uint32_t run = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const int64_t i = base + k;
        v[k] = i < n ? in[i] : 0u;
        const uint32_t t = v[k];
        v[k] = run;
        run += t;
    }
    // warp-inclusive scan of per-thread totals
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
        uint32_t w = warp_tot[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        warp_tot[lane] = w;
    }
    __syncthreads();
    const uint32_t excl = x - run + (wid ? warp_tot[wid - 1] : 0u);
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const int64_t i = base + k;
        if (i < n) out[i] = v[k] + excl;
    }
    if (threadIdx.x == kScanThreads - 1 && tile_sums) tile_sums[blockIdx.x] = excl + run;
}

__global__ void k_scan_add(uint32_t* out, int64_t n, const uint32_t* tile_off) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * kScanTile + threadIdx.x;
    const uint32_t add = tile_off[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const int64_t j = i + static_cast<int64_t>(k) * kScanThreads;
        if (j < n) out[j] += add;
    }
}

size_t scan_tmp_words(int64_t n) {
    size_t words = 0;
    int64_t m = n;
    while (m > kScanTile) {
        m = (m + kScanTile - 1) / kScanTile;
        words += static_cast<size_t>(m);
    }
    return words + 1;
}

void exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* tmp,
                        uint32_t* d_total, cudaStream_t s, int64_t* launches) {
    if (n <= 0) return;
    // in-place safe: every element is read and rewritten by the same thread
    const int64_t tiles = (n + kScanTile - 1) / kScanTile;
    if (tiles == 1) {
        k_scan_tiles<<<1, kScanThreads, 0, s>>>(in, out, n, d_total);
        ++*launches;
        return;
    }
    uint32_t* sums = tmp;
    k_scan_tiles<<<static_cast<unsigned>(tiles), kScanThreads, 0, s>>>(in, out, n, sums);
    ++*launches;
    exclusive_scan_u32(sums, sums, tiles, tmp + tiles, d_total, s, launches);
    k_scan_add<<<static_cast<unsigned>(tiles), kScanThreads, 0, s>>>(out, n, sums);
    ++*launches;
}

// ------------------------------------------------------------------ K1 keys

__global__ void k_init_minmax(long long* mm, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) mm[i] = (i & 1) ? LLONG_MIN : LLONG_MAX;  // [min_M, max_M, min_m, max_m] per spec
}

FWA_DEVINL long long wmin(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const long long y = __shfl_xor_sync(0xffffffffu, v, o);
        v = y < v ? y : v;
    }
    return v;
}
FWA_DEVINL long long wmax(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const long long y = __shfl_xor_sync(0xffffffffu, v, o);
        v = y > v ? y : v;
    }
    return v;
}

__device__ void bins_setup_cta(const long long* __restrict__ partials, int64_t n_part, int n_specs, int nf,
                               long long cap, long long* __restrict__ mm, SpecBins* __restrict__ specs,
                               uint32_t* __restrict__ d_nbins, int* __restrict__ overflow);
__device__ void bins_from_minmax(const long long (*fin)[4], int n_specs, int nf, long long cap,
                                 SpecBins* __restrict__ specs, uint32_t* __restrict__ d_nbins,
                                 int* __restrict__ overflow);

// One thread per (spec, point).  flatten.hpp:49-69, op by op, round-to-nearest.
// With `fz`, the last CTA to finish (atomic ticket) also reduces the min/max partials
// into the bin layout (bins_setup_cta) -- no separate launch.
__global__ void __launch_bounds__(256) k_sort_keys(const double* __restrict__ coords, int64_t ntot,
                                                   int n_specs, double w_x, double w_y,
                                                   long long* __restrict__ win,
                                                   double* __restrict__ loc,
                                                   long long* __restrict__ minmax, BinsFuse fz) {
    const int s = blockIdx.y;
    const bool axis_y = s >= 2, shift = (s & 1) != 0;
    long long wM = LLONG_MAX, wm = LLONG_MAX, xM = LLONG_MIN, xm = LLONG_MIN;
    // grid-stride: few CTAs per spec -> few partials and few last-CTA tickets; the
    // coordinates of 4 strides are loaded up front (independent loads in flight)
    const int64_t gs = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i0 < ntot; i0 += 4 * gs) {
      double2 cc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
          cc[u] = i0 + u * gs < ntot ? __ldg(reinterpret_cast<const double2*>(coords) + i0 + u * gs)
                                     : make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = i0 + u * gs;
        if (i >= ntot) break;
        const double2 c = cc[u];
        double cx = c.x, cy = c.y;
        if (shift) {
            cx = __dadd_rn(cx, __ddiv_rn(w_x, 2.0));
            cy = __dadd_rn(cy, __ddiv_rn(w_y, 2.0));
        }
        const double cm = axis_y ? cy : cx, cn = axis_y ? cx : cy;
        const double wmj = axis_y ? w_y : w_x, wmn = axis_y ? w_x : w_y;
        const long long a = static_cast<long long>(floor(__ddiv_rn(cm, wmj)));
        const long long b = static_cast<long long>(floor(__ddiv_rn(cn, wmn)));
        const double la = __dsub_rn(cm, __dmul_rn(static_cast<double>(a), wmj));
        const double lb = __dsub_rn(cn, __dmul_rn(static_cast<double>(b), wmn));
        const int64_t e = static_cast<int64_t>(s) * ntot + i;
        reinterpret_cast<longlong2*>(win)[e] = make_longlong2(a, b);
        reinterpret_cast<double2*>(loc)[e] = make_double2(la, lb);
        wM = a < wM ? a : wM;
        xM = a > xM ? a : xM;
        wm = b < wm ? b : wm;
        xm = b > xm ? b : xm;
      }
    }
    wM = wmin(wM);
    xM = wmax(xM);
    wm = wmin(wm);
    xm = wmax(xm);
    __shared__ long long red[4][8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        red[0][wid] = wM;
        red[1][wid] = xM;
        red[2][wid] = wm;
        red[3][wid] = xm;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        const int q = threadIdx.x;
        long long v = red[q][0];
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
            v = (q & 1) ? (red[q][w] > v ? red[q][w] : v) : (red[q][w] < v ? red[q][w] : v);
        // per-CTA partial [spec][cta][4], reduced by the last CTA or k_bins_setup (64-bit
        // atomics into 16 shared addresses instead serialise ~4k CTAs at L2: +3.7 us)
        minmax[(static_cast<int64_t>(s) * gridDim.x + blockIdx.x) * 4 + q] = v;
    }
    if (fz.ticket) {
        __shared__ bool last;
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) last = atomicAdd(fz.ticket, 1u) == gridDim.x * gridDim.y - 1;
        __syncthreads();
        if (last) {
            __threadfence();
            bins_setup_cta(minmax, gridDim.x, n_specs, fz.nf, fz.cap, fz.mm, fz.specs, fz.d_nbins, fz.overflow);
            if (threadIdx.x == 0) {
                *fz.ticket = 0u;               // self-resetting for the next call
                if (fz.large) *fz.large = 0u;  // the bin sort's oversize-bin queue
            }
        }
    }
}

// CTAs (= min/max partials) per spec: each thread's elements are serial fp64 division chains,
// so more threads shorten the kernel until the last CTA's partial reduction grows; measured
// (F60, in the graph): 74 CTAs 67.5 us schedule, 110 57.1, 148 58.4, 180 59.0, 296 61.0
int64_t sort_keys_partials(int64_t ntot) {
    const int64_t n = (ntot + 255) / 256;
    return n < 110 ? n : 110;
}

void launch_sort_keys(const double* coords, int64_t ntot, int n_specs, double w_x, double w_y,
                      long long* win, double* loc, long long* partials, cudaStream_t s,
                      int64_t* launches, const BinsFuse& fz) {
    dim3 grid(static_cast<unsigned>(sort_keys_partials(ntot)), static_cast<unsigned>(n_specs));
    k_sort_keys<<<grid, 256, 0, s>>>(coords, ntot, n_specs, w_x, w_y, win, loc, partials, fz);
    *launches += 1;
}

// ------------------------------------------------------------------ K2 bins + histogram

FWA_DEVINL int frame_of(const int64_t* off, int n_frames, int64_t i) {
    int lo = 0, hi = n_frames - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (off[mid] <= i) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// specs: one SpecBins per spec (union window range of all frames, bins_per_frame apart),
// or with per_frame one per (spec, frame) (each frame's own range; base = its first bin)
__global__ void __launch_bounds__(256) k_bins_hist(const long long* __restrict__ win, int64_t ntot,
                                                   const int64_t* __restrict__ frame_off,
                                                   int n_frames, const SpecBins* __restrict__ specs,
                                                   uint32_t* __restrict__ bin_of,
                                                   uint32_t* __restrict__ hist,
                                                   const uint32_t* __restrict__ d_nbins, int per_frame) {
    const int s = blockIdx.y;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= ntot) return;
    if (d_nbins && *d_nbins == 0u) return;  // bin capacity overflow: host falls back
    const int64_t e = static_cast<int64_t>(s) * ntot + i;
    const longlong2 w = reinterpret_cast<const longlong2*>(win)[e];
    const int f = n_frames > 1 ? frame_of(frame_off, n_frames, i) : 0;
    const SpecBins sb = specs[per_frame ? s * n_frames + f : s];
    const long long bin = sb.base + (per_frame ? 0LL : static_cast<long long>(f) * sb.bins_per_frame) +
                          (w.x - sb.min_major) * sb.range_minor + (w.y - sb.min_minor);
    bin_of[e] = static_cast<uint32_t>(bin);
    // warp-aggregated: consecutive pillar ids mostly share a window
    const unsigned grp = __match_any_sync(__activemask(), static_cast<uint32_t>(bin));
    if ((threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(hist + bin, static_cast<uint32_t>(__popc(grp)));
}

void launch_bins_hist(const long long* win, int64_t ntot, int n_specs, const int64_t* d_frame_off,
                      int n_frames, const SpecBins* d_specs, uint32_t* bin_of, uint32_t* hist,
                      const uint32_t* d_nbins, cudaStream_t s, int64_t* launches, bool per_frame) {
    dim3 grid(static_cast<unsigned>((ntot + 255) / 256), static_cast<unsigned>(n_specs));
    k_bins_hist<<<grid, 256, 0, s>>>(win, ntot, d_frame_off, n_frames, d_specs, bin_of, hist, d_nbins,
                                     per_frame ? 1 : 0);
    ++*launches;
}

// ---- exact (host-sized) path helpers

// window min/max per (spec, frame): mm[((s * nf) + f) * 4 + {min_M, max_M, min_m, max_m}]
// (initialised to LLONG_MAX / LLONG_MIN).  A CTA's 256 consecutive pillars span few frames:
// shared-memory atomics for the first 8 frames from the CTA's first one, then one global
// atomic per touched slot (the rare farther frame goes straight to global)
__global__ void __launch_bounds__(256) k_frame_minmax(const long long* __restrict__ win, int64_t ntot,
                                                      const int64_t* __restrict__ frame_off, int n_frames,
                                                      long long* __restrict__ mm, int64_t chunk) {
    // each CTA reduces a contiguous chunk of pillars (few frames) into 8 shared-memory slots
    // (frames f0 .. f0 + 7 from its first), then one global atomic per touched slot value;
    // a warp whose lanes share a frame reduces by shuffles first
    const int s = blockIdx.y;
    __shared__ long long sm[8][4];
    __shared__ int f0;
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * chunk;
    const int64_t c1 = c0 + chunk < ntot ? c0 + chunk : ntot;
    if (threadIdx.x < 32) sm[threadIdx.x >> 2][threadIdx.x & 3] = (threadIdx.x & 1) ? LLONG_MIN : LLONG_MAX;
    if (threadIdx.x == 0) f0 = n_frames > 1 && c0 < ntot ? frame_of(frame_off, n_frames, c0) : 0;
    __syncthreads();
    // per-thread running extremes of the current frame in registers (a CTA's chunk spans one
    // or two frames at batch scale), flushed into the slots only when the frame changes;
    // four rows' loads in flight per thread
    int f = f0;
    int64_t next_b = f + 1 < n_frames ? frame_off[f + 1] : INT64_MAX;
    int fc = -1;
    long long a0 = LLONG_MAX, a1 = LLONG_MIN, a2 = LLONG_MAX, a3 = LLONG_MIN;
    auto flush = [&]() {
        if (fc < 0) return;
        const int k = fc - f0;
        long long* m = k < 8 ? sm[k] : mm + (static_cast<int64_t>(s) * n_frames + fc) * 4;
        atomicMin(m, a0);
        atomicMax(m + 1, a1);
        atomicMin(m + 2, a2);
        atomicMax(m + 3, a3);
        a0 = LLONG_MAX, a1 = LLONG_MIN, a2 = LLONG_MAX, a3 = LLONG_MIN;
    };
    const longlong2* ws = reinterpret_cast<const longlong2*>(win) + static_cast<int64_t>(s) * ntot;
    for (int64_t t0 = c0 + threadIdx.x; t0 < c1; t0 += 4 * blockDim.x) {
        longlong2 w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = t0 + u * blockDim.x;
            w[u] = i < c1 ? ws[i] : make_longlong2(0, 0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = t0 + u * blockDim.x;
            if (i >= c1) break;
            while (next_b <= i) {
                ++f;
                next_b = f + 1 < n_frames ? frame_off[f + 1] : INT64_MAX;
            }
            if (f != fc) {
                flush();
                fc = f;
            }
            a0 = w[u].x < a0 ? w[u].x : a0;
            a1 = w[u].x > a1 ? w[u].x : a1;
            a2 = w[u].y < a2 ? w[u].y : a2;
            a3 = w[u].y > a3 ? w[u].y : a3;
        }
    }
    flush();
    __syncthreads();
    if (threadIdx.x < 32) {
        const int k = threadIdx.x >> 2, q = threadIdx.x & 3;
        const long long v = sm[k][q];
        if (v != ((q & 1) ? LLONG_MIN : LLONG_MAX) && f0 + k < n_frames) {
            long long* m = mm + (static_cast<int64_t>(s) * n_frames + f0 + k) * 4 + q;
            if (q & 1) atomicMax(m, v);
            else atomicMin(m, v);
        }
    }
}

void launch_frame_minmax(const long long* win, int64_t ntot, int n_specs, const int64_t* d_frame_off, int n_frames,
                         long long* mm, cudaStream_t s, int64_t* launches) {
    k_init_minmax<<<(4 * n_specs * n_frames + 255) / 256, 256, 0, s>>>(mm, 4 * n_specs * n_frames);
    const int64_t tiles = (ntot + 255) / 256;
    const int64_t ctas = tiles < 2 * kNumSMs ? tiles : 2 * kNumSMs;  // per spec
    const int64_t chunk = ((ntot + ctas - 1) / ctas + 255) / 256 * 256;
    dim3 grid(static_cast<unsigned>((ntot + chunk - 1) / chunk), static_cast<unsigned>(n_specs));
    k_frame_minmax<<<grid, 256, 0, s>>>(win, ntot, d_frame_off, n_frames, mm, chunk);
    *launches += 2;
}

// ---- window-rank compression: the exact path's fallback for window ranges too wide for a
// dense bin per window (a far outlier, frames kilometres apart).  A stable LSD radix sort of
// the elements by (spec * nf + frame, win_major, win_minor) -- three CUB passes, least
// significant key first -- then a new-window flag + scan: bin_of[e] = the dense rank of e's
// window in lexicographic window order, exactly the bin order of the dense layout.
FWA_DEVINL unsigned long long flip64(long long v) {
    return static_cast<unsigned long long>(v) ^ 0x8000000000000000ULL;
}

__global__ void k_wr_minor(const long long* __restrict__ win, int64_t total, unsigned long long* __restrict__ key,
                           uint32_t* __restrict__ val) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= total) return;
    key[e] = flip64(reinterpret_cast<const longlong2*>(win)[e].y);
    val[e] = static_cast<uint32_t>(e);
}

__global__ void k_wr_major(const long long* __restrict__ win, int64_t total, const uint32_t* __restrict__ val,
                           unsigned long long* __restrict__ key) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= total) return;
    key[k] = flip64(reinterpret_cast<const longlong2*>(win)[val[k]].x);
}

__global__ void k_wr_frame(int64_t total, int64_t ntot, const int64_t* __restrict__ frame_off, int n_frames,
                           const uint32_t* __restrict__ val, uint32_t* __restrict__ key) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= total) return;
    const int64_t e = val[k];
    const int64_t i = e % ntot;
    key[k] = static_cast<uint32_t>((e / ntot) * n_frames + (n_frames > 1 ? frame_of(frame_off, n_frames, i) : 0));
}

__global__ void k_wr_flags(const long long* __restrict__ win, int64_t total, int64_t ntot,
                           const int64_t* __restrict__ frame_off, int n_frames, const uint32_t* __restrict__ val,
                           uint32_t* __restrict__ flag) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= total) return;
    uint32_t f = 1u;
    if (k > 0) {
        const int64_t a = val[k], b = val[k - 1];
        const longlong2 wa = reinterpret_cast<const longlong2*>(win)[a];
        const longlong2 wb = reinterpret_cast<const longlong2*>(win)[b];
        const int64_t sa = a / ntot, sb = b / ntot;
        const int fa = n_frames > 1 ? frame_of(frame_off, n_frames, a % ntot) : 0;
        const int fb = n_frames > 1 ? frame_of(frame_off, n_frames, b % ntot) : 0;
        f = (sa != sb || fa != fb || wa.x != wb.x || wa.y != wb.y) ? 1u : 0u;
    }
    flag[k] = f;
}

__global__ void k_wr_assign(int64_t total, const uint32_t* __restrict__ val, const uint32_t* __restrict__ flag,
                            const uint32_t* __restrict__ ex, uint32_t* __restrict__ bin_of,
                            uint32_t* __restrict__ hist) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= total) return;
    const uint32_t b = ex[k] + flag[k] - 1u;
    bin_of[val[k]] = b;
    atomicAdd(hist + b, 1u);
}

size_t window_ranks_temp_bytes(int64_t total) {
    size_t a = 0, b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, static_cast<const unsigned long long*>(nullptr),
                                    static_cast<unsigned long long*>(nullptr), static_cast<const uint32_t*>(nullptr),
                                    static_cast<uint32_t*>(nullptr), static_cast<int>(total));
    cub::DeviceRadixSort::SortPairs(nullptr, b, static_cast<const uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                    static_cast<const uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                    static_cast<int>(total));
    return a > b ? a : b;
}

void launch_window_ranks(const long long* win, int64_t ntot, int n_specs, const int64_t* d_frame_off, int n_frames,
                         unsigned long long* k64a, unsigned long long* k64b, uint32_t* va, uint32_t* vb,
                         uint32_t* flag, uint32_t* ex, uint32_t* scan_tmp, uint32_t* d_count, void* temp,
                         size_t temp_bytes, uint32_t* bin_of, uint32_t* hist, cudaStream_t s, int64_t* launches) {
    const int64_t total = ntot * n_specs;
    const unsigned g = static_cast<unsigned>((total + 255) / 256);
    const int nt = static_cast<int>(total);
    k_wr_minor<<<g, 256, 0, s>>>(win, total, k64a, va);
    size_t tb = temp_bytes;
    cub::DeviceRadixSort::SortPairs(temp, tb, k64a, k64b, va, vb, nt, 0, 64, s);
    k_wr_major<<<g, 256, 0, s>>>(win, total, vb, k64a);
    tb = temp_bytes;
    cub::DeviceRadixSort::SortPairs(temp, tb, k64a, k64b, vb, va, nt, 0, 64, s);
    uint32_t* k32a = reinterpret_cast<uint32_t*>(k64a);
    uint32_t* k32b = reinterpret_cast<uint32_t*>(k64b);
    k_wr_frame<<<g, 256, 0, s>>>(total, ntot, d_frame_off, n_frames, va, k32a);
    tb = temp_bytes;
    cub::DeviceRadixSort::SortPairs(temp, tb, k32a, k32b, va, vb, nt, 0, 32, s);
    k_wr_flags<<<g, 256, 0, s>>>(win, total, ntot, d_frame_off, n_frames, vb, flag);
    exclusive_scan_u32(flag, ex, total, scan_tmp, d_count, s, launches);
    k_wr_assign<<<g, 256, 0, s>>>(total, vb, flag, ex, bin_of, hist);
    *launches += 8;
}

// Order-preserving integer image of a window-local coordinate: unsigned compare of the
// images == the reference's double compare (key_less, flatten.hpp:41-47), with -0.0 and
// +0.0 equal (both map to the +0.0 image).  Coordinates are finite.
FWA_DEVINL unsigned long long ord_key(double d) {
    const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(d == 0.0 ? 0.0 : d));
    return (u >> 63) ? ~u : (u | 0x8000000000000000ULL);
}

// ------------------------------------------------------------------ K3 scatter into bins

__global__ void __launch_bounds__(256) k_bin_scatter(const uint32_t* __restrict__ bin_of,
                                                     const double* __restrict__ loc, int64_t total,
                                                     int64_t ntot, uint32_t* __restrict__ cursor,
                                                     int32_t* __restrict__ pre,
                                                     double* __restrict__ pre_loc,
                                                     const uint32_t* __restrict__ d_nbins,
                                                     const uint32_t* __restrict__ tile_off,
                                                     uint32_t* __restrict__ pre_bin) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= total) return;
    if (d_nbins && *d_nbins == 0u) return;
    const uint32_t b = bin_of[e];
    // warp-aggregated slot claims (the order inside a bin is irrelevant: the rank sort
    // orders by (key, key, id))
    const unsigned grp = __match_any_sync(__activemask(), b);
    const int lane = threadIdx.x & 31, leader = __ffs(grp) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(cursor + b, static_cast<uint32_t>(__popc(grp)));
    base = __shfl_sync(grp, base, leader);
    const uint32_t pos = base + static_cast<uint32_t>(__popc(grp & ((1u << lane) - 1u))) +
                         (tile_off ? tile_off[b / kScanTile] : 0u);
    pre[pos] = static_cast<int32_t>(e % ntot);
    pre_bin[pos] = b;
    // the window-local keys travel with the id as order-preserving integer images: the
    // per-bin rank kernel reads them contiguously and compares integers
    const double2 l = reinterpret_cast<const double2*>(loc)[e];
    reinterpret_cast<ulonglong2*>(pre_loc)[pos] = make_ulonglong2(ord_key(l.x), ord_key(l.y));
}

void launch_bin_scatter(const uint32_t* bin_of, const double* loc, int64_t ntot, int n_specs,
                        uint32_t* cursor, int32_t* pre, double* pre_loc, const uint32_t* d_nbins,
                        const uint32_t* tile_off, uint32_t* pre_bin, cudaStream_t s, int64_t* launches) {
    const int64_t total = ntot * n_specs;
    k_bin_scatter<<<static_cast<unsigned>((total + 255) / 256), 256, 0, s>>>(bin_of, loc, total, ntot,
                                                                           cursor, pre, pre_loc, d_nbins,
                                                                           tile_off, pre_bin);
    ++*launches;
}

// ------------------------------------------------------------------ K4 per-bin exact sort

// key_less restricted to one window: (loc_major, loc_minor, orig index).
FWA_DEVINL bool loc_less(double a0, double a1, int ai, double b0, double b1, int bi) {
    if (a0 != b0) return a0 < b0;
    if (a1 != b1) return a1 < b1;
    return ai < bi;
}

constexpr int kWarpBin = 128;   // bins up to this size: one warp, shared memory
constexpr int kCtaBin = 4096;   // up to this: one CTA, shared-memory rank sort
constexpr int kBinWarps = 8;

// One thread per binned element: its rank among the elements of its window bin (integer
// key images, then the original index -- key_less, flatten.hpp:41-47) by one pass over
// the bin (n <= kWarpBin; the bin's elements are contiguous and staged in shared memory
// per CTA, so the loads of a warp are broadcasts).  Bigger bins are queued for
// k_bin_sort_large by their first element.  Writes sorted[] and the inverse inv[].
__global__ void __launch_bounds__(256) k_bin_rank(const uint32_t* __restrict__ bin_start,
                                                  uint32_t* __restrict__ hist, uint32_t n_bins,
                                                  const int32_t* __restrict__ pre,
                                                  const ulonglong2* __restrict__ pkey,
                                                  const uint32_t* __restrict__ pre_bin, int64_t total,
                                                  int64_t ntot, int32_t* __restrict__ sorted,
                                                  int32_t* __restrict__ inv, uint32_t* __restrict__ large,
                                                  const uint32_t* __restrict__ d_nbins,
                                                  const uint32_t* __restrict__ tile_off) {
    const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (d_nbins) {
        n_bins = *d_nbins;
        if (n_bins == 0u) {
            // bin-capacity overflow (the host re-runs the frame set with exact bins): leave an
            // identity permutation so every consumer of the plans (drop tables, compaction,
            // the block kernels' gathers) stays in bounds on this discarded pass
            if (p < total) {
                const int64_t id = p % ntot;
                sorted[p] = static_cast<int32_t>(id);
                inv[p] = static_cast<int32_t>(p);
            }
            return;
        }
    }
    // every bin that holds one of this CTA's elements lies inside [c0, c0 + 512) (bins of
    // up to kWarpBin elements): its keys and ids are staged in shared memory once
    __shared__ ulonglong2 s_key[256 + 2 * kWarpBin];
    __shared__ int s_id[256 + 2 * kWarpBin];
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * blockDim.x - kWarpBin;
    for (int i = threadIdx.x; i < 256 + 2 * kWarpBin; i += blockDim.x) {
        const int64_t q = c0 + i;
        if (q >= 0 && q < total) {
            s_key[i] = pkey[q];
            s_id[i] = pre[q];
        }
    }
    __syncthreads();
    if (p >= total) return;
    const uint32_t b = pre_bin[p];
    const int64_t start = bin_start[b] + (tile_off ? tile_off[b / kScanTile] : 0u);
    const int64_t end = b + 1 < n_bins ? bin_start[b + 1] + (tile_off ? tile_off[(b + 1) / kScanTile] : 0u) : total;
    const int n = static_cast<int>(end - start);
    if (n > kWarpBin) {
        if (p == start) large[1 + atomicAdd(large, 1u)] = b;  // k_bin_sort_large zeroes hist[b]
        return;
    }
    if (p == start) hist[b] = 0u;  // leave the histogram zeroed for the next call
    const ulonglong2 me = pkey[p];
    const int my = pre[p];
    int rank = 0;
    const int nn = n;
    const uint32_t mxh = static_cast<uint32_t>(me.x >> 32), mxl = static_cast<uint32_t>(me.x);
    const uint32_t myh = static_cast<uint32_t>(me.y >> 32), myl = static_cast<uint32_t>(me.y);
#pragma unroll 8
    for (int j = 0; j < nn; ++j) {
        const ulonglong2 o = s_key[start + j - c0];
        const int oid = s_id[start + j - c0];
        // (o.x, o.y, oid) < (me.x, me.y, my) lexicographically == the borrow of the 160-bit
        // subtraction o - me (every field unsigned, fixed width): one carry chain
        uint32_t b;
        asm("{\n\t.reg .u32 t;\n\t"
            "sub.cc.u32 t, %1, %2;\n\t"
            "subc.cc.u32 t, %3, %4;\n\t"
            "subc.cc.u32 t, %5, %6;\n\t"
            "subc.cc.u32 t, %7, %8;\n\t"
            "subc.cc.u32 t, %9, %10;\n\t"
            "subc.u32 %0, 0, 0;\n\t}"
            : "=r"(b)
            : "r"(static_cast<uint32_t>(oid)), "r"(static_cast<uint32_t>(my)),
              "r"(static_cast<uint32_t>(o.y)), "r"(myl), "r"(static_cast<uint32_t>(o.y >> 32)), "r"(myh),
              "r"(static_cast<uint32_t>(o.x)), "r"(mxl), "r"(static_cast<uint32_t>(o.x >> 32)), "r"(mxh));
        rank -= static_cast<int>(b);  // b = 0xFFFFFFFF when o < me
    }
    const int64_t spec_base = (start / ntot) * ntot;
    sorted[start + rank] = my;
    inv[spec_base + my] = static_cast<int32_t>(start + rank);
}

__global__ void __launch_bounds__(512) k_bin_sort_large(
    const uint32_t* __restrict__ bin_start, uint32_t* __restrict__ hist,
    const uint32_t* __restrict__ large, const int32_t* __restrict__ pre,
    const double* __restrict__ loc, int64_t ntot, int32_t* __restrict__ sorted,
    int32_t* __restrict__ inv, int32_t* __restrict__ scratch, const uint32_t* __restrict__ tile_off) {
    extern __shared__ unsigned char smem_raw[];
    double* s_a = reinterpret_cast<double*>(smem_raw);
    double* s_b = s_a + kCtaBin;
    int* s_i = reinterpret_cast<int*>(s_b + kCtaBin);
    const uint32_t n_large = large[0];
    for (uint32_t li = blockIdx.x; li < n_large; li += gridDim.x) {
        const uint32_t bin = large[1 + li];
        const int n = static_cast<int>(hist[bin]);
        const uint32_t start = bin_start[bin] + (tile_off ? tile_off[bin / kScanTile] : 0u);
        const int64_t spec_base = (static_cast<int64_t>(start) / ntot) * ntot;
        const double2* L = reinterpret_cast<const double2*>(loc) + spec_base;
        if (n <= kCtaBin) {
            for (int k = threadIdx.x; k < n; k += blockDim.x) {
                const int id = pre[start + k];
                const double2 l = L[id];
                s_a[k] = l.x;
                s_b[k] = l.y;
                s_i[k] = id;
            }
            __syncthreads();
            for (int k = threadIdx.x; k < n; k += blockDim.x) {
                const double a = s_a[k], b = s_b[k];
                const int id = s_i[k];
                int rank = 0;
                for (int j = 0; j < n; ++j) rank += loc_less(s_a[j], s_b[j], s_i[j], a, b, id);
                sorted[start + rank] = id;
                inv[spec_base + id] = static_cast<int32_t>(start + rank);
            }
            __syncthreads();
        } else {
            // bitonic network over next_pow2(n) slots of global scratch
            // (slot range [2*start, 2*start + P) never overlaps another bin's).
            int P = 1;
            while (P < n) P <<= 1;
            int32_t* v = scratch + 2 * static_cast<int64_t>(start);
            for (int k = threadIdx.x; k < P; k += blockDim.x) v[k] = k < n ? pre[start + k] : -1;
            __syncthreads();
            for (int size = 2; size <= P; size <<= 1) {
                for (int stride = size >> 1; stride > 0; stride >>= 1) {
                    for (int t = threadIdx.x; t < P / 2; t += blockDim.x) {
                        const int lo = 2 * t - (t & (stride - 1));
                        const int hi = lo + stride;
                        const bool up = (lo & size) == 0;
                        const int a = v[lo], b = v[hi];
                        // -1 is +infinity
                        bool b_less_a;
                        if (a < 0) b_less_a = b >= 0;
                        else if (b < 0) b_less_a = false;
                        else {
                            const double2 la = L[a], lb = L[b];
                            b_less_a = loc_less(lb.x, lb.y, b, la.x, la.y, a);
                        }
                        if (b_less_a == up) {
                            v[lo] = b;
                            v[hi] = a;
                        }
                    }
                    __syncthreads();
                }
            }
            for (int k = threadIdx.x; k < n; k += blockDim.x) {
                sorted[start + k] = v[k];
                inv[spec_base + v[k]] = static_cast<int32_t>(start + k);
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) hist[bin] = 0u;  // zeroed for the next call
    }
}

void launch_bin_sort(const uint32_t* bin_start, uint32_t* hist, uint32_t n_bins,
                     const int32_t* pre, const double* pre_loc, const uint32_t* pre_bin, const double* loc,
                     int64_t ntot, int n_specs, int32_t* sorted, int32_t* inv, int32_t* scratch,
                     uint32_t* large, const uint32_t* d_nbins, const uint32_t* tile_off, cudaStream_t s,
                     int64_t* launches) {
    const int64_t total = ntot * n_specs;
    if (!d_nbins) cudaMemsetAsync(large, 0, sizeof(uint32_t), s);  // sync-free path: reset by the key kernel
    k_bin_rank<<<static_cast<unsigned>((total + 255) / 256), 256, 0, s>>>(
        bin_start, hist, n_bins, pre, reinterpret_cast<const ulonglong2*>(pre_loc), pre_bin, total, ntot, sorted,
        inv, large, d_nbins, tile_off);
    static bool attr_set = false;
    const int smem = kCtaBin * (8 + 8 + 4);
    if (!attr_set) {
        cudaFuncSetAttribute(k_bin_sort_large, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr_set = true;
    }
    k_bin_sort_large<<<kNumSMs, 512, smem, s>>>(bin_start, hist, large, pre, loc, ntot, sorted, inv,
                                                scratch, tile_off);
    *launches += 2;
}

// ------------------------------------------------------------------ schedule kernels

// Block 0 uses spec 0 (X, no shift).  Its per-frame tail beyond rows_f is the
// dropped residual (flatten.hpp:134-146); record ids in tail order
// (backbone.hpp:285-291) and flag them.
__global__ void k_drop_mark(const int32_t* __restrict__ sorted0, int64_t ntot,
                            const int64_t* __restrict__ frame_off, const int64_t* __restrict__ rows,
                            const int64_t* __restrict__ drop_off, int n_frames,
                            uint8_t* __restrict__ dropped, int32_t* __restrict__ dropped_ids) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= ntot) return;
    const int f = n_frames > 1 ? frame_of(frame_off, n_frames, j) : 0;
    const int64_t t = j - frame_off[f] - rows[f];
    if (t >= 0) {
        const int id = sorted0[j];
        dropped[id] = 1;
        if (dropped_ids) dropped_ids[drop_off[f] + t] = id;
    }
}

void launch_drop_mark(const int32_t* sorted0, int64_t ntot, const int64_t* d_frame_off,
                      const int64_t* d_rows, const int64_t* d_drop_off, int n_frames,
                      uint8_t* dropped, int32_t* dropped_ids, cudaStream_t s, int64_t* launches) {
    k_drop_mark<<<static_cast<unsigned>((ntot + 255) / 256), 256, 0, s>>>(
        sorted0, ntot, d_frame_off, d_rows, d_drop_off, n_frames, dropped, dropped_ids);
    ++*launches;
}

__global__ void k_keep_flags(const uint8_t* __restrict__ dropped, int64_t n, uint32_t* flags) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) flags[i] = dropped[i] ? 0u : 1u;
}

void launch_keep_flags(const uint8_t* dropped, int64_t ntot, uint32_t* flags, cudaStream_t s,
                       int64_t* launches) {
    k_keep_flags<<<static_cast<unsigned>((ntot + 255) / 256), 256, 0, s>>>(dropped, ntot, flags);
    ++*launches;
}

__global__ void k_kept_ids(const uint32_t* __restrict__ rank, const uint8_t* __restrict__ dropped,
                           int64_t n, int32_t* __restrict__ kept) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n && !dropped[i]) kept[rank[i]] = static_cast<int32_t>(i);
}

void launch_kept_ids(const uint32_t* kept_rank, const uint8_t* dropped, int64_t ntot,
                     int32_t* kept_ids, cudaStream_t s, int64_t* launches) {
    k_kept_ids<<<static_cast<unsigned>((ntot + 255) / 256), 256, 0, s>>>(kept_rank, dropped, ntot,
                                                                        kept_ids);
    ++*launches;
}

__global__ void k_spec_keep_flags(const int32_t* __restrict__ sorted, int64_t total,
                                  const uint8_t* __restrict__ dropped, uint32_t* flags) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j < total) flags[j] = dropped[sorted[j]] ? 0u : 1u;
}

void launch_spec_keep_flags(const int32_t* sorted, int64_t total, const uint8_t* dropped,
                            uint32_t* flags, cudaStream_t s, int64_t* launches) {
    k_spec_keep_flags<<<static_cast<unsigned>((total + 255) / 256), 256, 0, s>>>(sorted, total,
                                                                               dropped, flags);
    ++*launches;
}

// Restrict each spec's full-set plan to the kept set, preserving order: the
// result is bit-identical to re-sorting the compacted coordinates (the order
// is total on (key, original id) and compaction preserves relative order;
// SURVEY.md Appendix B.6, pinned by tests/test_gpu_parity.py).
__global__ void k_spec_compact(const int32_t* __restrict__ sorted, int64_t total,
                               const uint8_t* __restrict__ dropped,
                               const uint32_t* __restrict__ pos, int32_t* __restrict__ idx) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j < total) {
        const int id = sorted[j];
        if (!dropped[id]) idx[pos[j]] = id;
    }
}

void launch_spec_compact(const int32_t* sorted, int64_t total, const uint8_t* dropped,
                         const uint32_t* pos, int32_t* idx, cudaStream_t s, int64_t* launches) {
    k_spec_compact<<<static_cast<unsigned>((total + 255) / 256), 256, 0, s>>>(sorted, total,
                                                                            dropped, pos, idx);
    ++*launches;
}


// ------------------------------------------------------------------ small-drop schedule (no scans)
//
// Block 0 drops at most G-1 pillars per frame.  With the dropped ids sorted ascending
// and, per spec, their positions in that spec's full-set plan sorted ascending, every
// compaction index is a binary search instead of a grid-wide scan:
//   kept_rank(id)        = id - #{dropped ids < id}
//   compact position(j)  = j  - #{dropped positions < j}   (per spec)

constexpr int kSmemDrops = 1024;  // k_compact_all: drop tables staged in shared memory up to this
FWA_DEVINL int count_less(const int32_t* a, int n, int32_t v) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// the same by one warp: each round the 32 lanes probe 32 evenly spaced elements of the
// remaining range and narrow it to one slot (3 dependent loads for n <= 32^3)
FWA_DEVINL int warp_count_less(const int32_t* a, int n, int32_t v) {
    const int lane = threadIdx.x & 31;
    int lo = 0, hi = n;  // answer in [lo, hi]
    while (hi - lo > 32) {
        const int step = (hi - lo + 31) / 32;
        const int idx = lo + lane * step;
        const bool less = idx < hi && a[idx] < v;
        const unsigned m = __ballot_sync(0xffffffffu, less);
        const int k = 32 - __clz(m);  // probes 0..k-1 are < v (a is sorted)
        const int nlo = k ? lo + (k - 1) * step + 1 : lo;
        const int nhi = lo + k * step < hi ? lo + k * step : hi;
        lo = nlo;
        hi = nhi;
    }
    const int idx = lo + lane;
    const unsigned m = __ballot_sync(0xffffffffu, idx < hi && a[idx] < v);
    return lo + __popc(m);
}

// One CTA: sort the dropped ids, then (per spec) the positions of those ids in the
// spec's full-set plan (inv[s][id]).  Rank sort for n <= blockDim.x, else a bitonic sort
// in shared memory, n <= kMaxDrop.
constexpr int kMaxDrop = 8192;

__global__ void __launch_bounds__(1024) k_drop_tables(const int32_t* __restrict__ sorted0, int n,
                                                      const int64_t* __restrict__ frame_off,
                                                      const int64_t* __restrict__ rows,
                                                      const int64_t* __restrict__ drop_off, int n_frames,
                                                      const int32_t* __restrict__ inv, int64_t ntot,
                                                      int n_specs, int32_t* __restrict__ dropped_ids,
                                                      int32_t* __restrict__ drop_sorted,
                                                      int32_t* __restrict__ drop_pos) {
    __shared__ int32_t v[kMaxDrop];
    int P = 1;
    while (P < n) P <<= 1;
    // one CTA per table: blockIdx.x 0 = dropped ids, 1 + s = their positions in spec s.
    // Block 0 (spec 0) drops each frame's tail beyond rows_f (flatten.hpp:134-146).
    const int pass = static_cast<int>(blockIdx.x) - 1;
    for (int k = threadIdx.x; k < P; k += blockDim.x) {
        int32_t x = INT32_MAX;
        if (k < n) {
            int f = 0;
            while (f + 1 < n_frames && drop_off[f + 1] <= k) ++f;
            const int32_t id = sorted0[frame_off[f] + rows[f] + (k - drop_off[f])];
            if (pass < 0 && dropped_ids) dropped_ids[k] = id;  // tail order (backbone.hpp:285-291)
            x = pass < 0 ? id : inv[static_cast<int64_t>(pass) * ntot + id];
        }
        v[k] = x;
    }
    __syncthreads();
    int32_t* dst = pass < 0 ? drop_sorted : drop_pos + static_cast<int64_t>(pass) * (n > 0 ? n : 1);
    if (n <= static_cast<int>(blockDim.x)) {
        // the usual case (one frame drops at most G - 1): the values are distinct (pillar ids,
        // or their positions in one plan), so each one's rank is its count of smaller values
        if (static_cast<int>(threadIdx.x) < n) {
            const int32_t x = v[threadIdx.x];
            int r = 0;
            for (int j = 0; j < n; ++j) r += v[j] < x;
            dst[r] = x;
        }
        return;
    }
    for (int size = 2; size <= P; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < P / 2; t += blockDim.x) {
                const int lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const int32_t a = v[lo], b = v[hi];
                if ((b < a) == up) {
                    v[lo] = b;
                    v[hi] = a;
                }
            }
            __syncthreads();
        }
    for (int k = threadIdx.x; k < n; k += blockDim.x) dst[k] = v[k];
}

// Grid (pillar-index chunks of 256, n_specs + 1):
//   y = s < n_specs, plan entry (s, j): kept id -> idx[s][j - #drop_pos[s] < j]; for the last
//   block's spec also out_pos[that] = kept_rank(id)
//   y = n_specs, pillar id i: kept_rank[i] = i - #drop_sorted < i; kept_ids[kept_rank] = i
// Each CTA finds the first sorted drop value at or past its first index by one binary
// search; every thread walks on from there to its own index (a 256-index range holds few
// drops), so it has both its count and whether it is itself dropped -- no gathers.  The
// kept rank of a plan entry's id (out_pos) searches only the id's frame's drops (ids of a
// frame are contiguous, so are its entries of the sorted drop list).
__global__ void __launch_bounds__(256) k_compact_all(const int32_t* __restrict__ sorted, int64_t ntot, int n_specs,
                                                     const int64_t* __restrict__ frame_off,
                                                     const int64_t* __restrict__ drop_off, int n_frames,
                                                     const int32_t* __restrict__ drop_sorted,
                                                     const int32_t* __restrict__ drop_pos, int n_drop, int64_t K,
                                                     int s_last, int32_t* __restrict__ idx,
                                                     uint32_t* __restrict__ kept_rank,
                                                     int32_t* __restrict__ kept_ids, int32_t* __restrict__ out_pos,
                                                     const int32_t* __restrict__ fuse_inv,
                                                     int32_t* __restrict__ fuse_dropped_ids) {
    const int s = static_cast<int>(blockIdx.y);
    const bool plan = s < n_specs;
    const int64_t j0 = static_cast<int64_t>(blockIdx.x) * blockDim.x;
    const int64_t j = j0 + threadIdx.x;
    const int64_t base = plan ? static_cast<int64_t>(s) * ntot : 0;  // drop_pos holds stacked plan indices
    const int32_t* dl = plan ? drop_pos + static_cast<int64_t>(s) * (n_drop > 0 ? n_drop : 1) : drop_sorted;
    __shared__ int s_lo, s_f0;
    // up to kSmemDrops drops (single frames: < G): this table, and for out_pos the sorted drop
    // ids, are staged in shared memory and every thread binary-searches there (no dependent
    // L2 loads); larger tables (frame batches) use the warp search + walk in global memory
    __shared__ int32_t s_dl[kSmemDrops], s_ds[kSmemDrops];
    const bool staged = n_drop <= kSmemDrops;
    const bool need_out = plan && s == s_last;
    if (fuse_inv) {
        // one frame, n_drop <= kFuseDrops: this CTA builds its own tables (no k_drop_tables
        // launch) -- the dropped ids are spec 0's plan tail sorted[K, K + n_drop) (block 0
        // drops its tail, flatten.hpp:134-146), the table of plan s their positions in it
        // (inverse permutation), ranked by counting (distinct values)
        __shared__ int32_t s_v[kFuseDrops], s_id[kFuseDrops];
        int32_t v = 0, id = 0;
        if (static_cast<int>(threadIdx.x) < n_drop) {
            id = sorted[K + threadIdx.x];
            if (!plan && blockIdx.x == 0 && fuse_dropped_ids) fuse_dropped_ids[threadIdx.x] = id;  // tail order
            v = plan ? fuse_inv[static_cast<int64_t>(s) * ntot + id] : id;
            s_v[threadIdx.x] = v;
            s_id[threadIdx.x] = id;
        }
        __syncthreads();
        if (static_cast<int>(threadIdx.x) < n_drop) {
            int r = 0, ri = 0;
            for (int k = 0; k < n_drop; ++k) {
                r += s_v[k] < v;
                ri += s_id[k] < id;
            }
            s_dl[r] = v;
            if (need_out) s_ds[ri] = id;
        }
        if (threadIdx.x == 0) s_f0 = 0;
    } else if (staged) {
        for (int i = threadIdx.x; i < n_drop; i += blockDim.x) {
            s_dl[i] = dl[i];
            if (need_out) s_ds[i] = drop_sorted[i];
        }
        if (threadIdx.x == 0)
            s_f0 = need_out && n_frames > 1 ? frame_of(frame_off, n_frames, j0 < ntot ? j0 : ntot - 1) : 0;
    } else if (threadIdx.x < 32) {  // warp 0: 32-way searches (a few dependent loads, not log2 n)
        const int lo = warp_count_less(dl, n_drop, static_cast<int32_t>(base + j0));
        if (threadIdx.x == 0) {
            s_lo = lo;
            s_f0 = need_out && n_frames > 1 ? frame_of(frame_off, n_frames, j0 < ntot ? j0 : ntot - 1) : 0;
        }
    }
    __syncthreads();
    if (j >= ntot) return;
    int lb;
    if (staged) {
        lb = count_less(s_dl, n_drop, static_cast<int32_t>(base + j));
        if (lb < n_drop && s_dl[lb] == base + j) return;  // dropped (block 0's tail of its frame)
    } else {
        lb = s_lo;
        while (lb < n_drop && dl[lb] < base + j) ++lb;
        if (lb < n_drop && dl[lb] == base + j) return;
    }
    const int64_t c = j - lb;
    if (plan) {
        const int32_t id = sorted[base + j];
        idx[static_cast<int64_t>(s) * K + c] = id;
        if (need_out) {
            int f = s_f0;
            while (f + 1 < n_frames && frame_off[f + 1] <= j) ++f;
            const int d0 = n_frames > 1 ? static_cast<int>(drop_off[f]) : 0;
            const int d1 = n_frames > 1 && f + 1 < n_frames ? static_cast<int>(drop_off[f + 1]) : n_drop;
            out_pos[c] = id - d0 - count_less((staged ? s_ds : drop_sorted) + d0, d1 - d0, id);
        }
    } else {
        kept_rank[j] = static_cast<uint32_t>(c);
        kept_ids[c] = static_cast<int32_t>(j);
    }
}

void launch_drop_tables(const int32_t* sorted0, int n, const int64_t* frame_off, const int64_t* rows,
                        const int64_t* drop_off, int n_frames, const int32_t* inv, int64_t ntot, int n_specs,
                        int32_t* dropped_ids, int32_t* drop_sorted, int32_t* drop_pos, cudaStream_t s,
                        int64_t* launches) {
    k_drop_tables<<<1 + n_specs, 1024, 0, s>>>(sorted0, n, frame_off, rows, drop_off, n_frames, inv, ntot,
                                               n_specs, dropped_ids, drop_sorted, drop_pos);
    ++*launches;
}

void launch_compact_all(const int32_t* sorted, int64_t ntot, int n_specs, const int64_t* frame_off,
                        const int64_t* drop_off, int n_frames, const int32_t* drop_sorted,
                        const int32_t* drop_pos, int n_drop, int64_t K, int s_last, int32_t* idx,
                        uint32_t* kept_rank, int32_t* kept_ids, int32_t* out_pos, cudaStream_t s,
                        int64_t* launches, const int32_t* fuse_inv, int32_t* fuse_dropped_ids) {
    static_assert(kFuseDrops <= 256 && kFuseDrops <= kSmemDrops, "one value per thread of a 256-thread CTA");
    if (fuse_inv && (n_frames != 1 || n_drop > kFuseDrops)) fuse_inv = nullptr;
    dim3 grid(static_cast<unsigned>((ntot + 255) / 256), static_cast<unsigned>(n_specs + 1));
    k_compact_all<<<grid, 256, 0, s>>>(sorted, ntot, n_specs, frame_off, drop_off, n_frames, drop_sorted, drop_pos,
                                       n_drop, K, s_last, idx, kept_rank, kept_ids, out_pos, fuse_inv,
                                       fuse_dropped_ids);
    ++*launches;
}


// ------------------------------------------------------------------ sync-free bin setup
//
// The window-bin ranges are computed on the device from the key kernel's min/max, so the
// whole schedule is enqueued without a host round trip.  The histogram has a fixed
// capacity; a frame set whose dense window range exceeds it raises *overflow (nbins = 0
// disables every bin kernel) and the host re-runs the exact-size path.

// One CTA (blockDim a multiple of 32, <= 1024) reduces the key kernel's per-CTA window
// min/max partials into the dense bin layout of every spec and the device-side bin count.
__device__ void bins_setup_cta(const long long* __restrict__ partials, int64_t n_part, int n_specs, int nf,
                               long long cap, long long* __restrict__ mm, SpecBins* __restrict__ specs,
                               uint32_t* __restrict__ d_nbins, int* __restrict__ overflow) {
    // one pass over all specs' partials (loads of every spec in flight together), then a
    // shared-memory reduction of the 4 x n_specs values
    __shared__ long long red[32][16];
    __shared__ long long fin[4][4];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    long long v[4][4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        v[s][0] = LLONG_MAX; v[s][1] = LLONG_MIN; v[s][2] = LLONG_MAX; v[s][3] = LLONG_MIN;
    }
    for (int64_t i = threadIdx.x; i < n_part; i += blockDim.x) {
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            if (s >= n_specs) break;
            const longlong2* p = reinterpret_cast<const longlong2*>(partials + (static_cast<int64_t>(s) * n_part + i) * 4);
            const longlong2 a = __ldcg(p), b = __ldcg(p + 1);
            v[s][0] = a.x < v[s][0] ? a.x : v[s][0];
            v[s][1] = a.y > v[s][1] ? a.y : v[s][1];
            v[s][2] = b.x < v[s][2] ? b.x : v[s][2];
            v[s][3] = b.y > v[s][3] ? b.y : v[s][3];
        }
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        v[s][0] = wmin(v[s][0]);
        v[s][1] = wmax(v[s][1]);
        v[s][2] = wmin(v[s][2]);
        v[s][3] = wmax(v[s][3]);
        if (lane == 0)
#pragma unroll
            for (int q = 0; q < 4; ++q) red[wid][4 * s + q] = v[s][q];
    }
    __syncthreads();
    if (threadIdx.x < 4 * n_specs) {
        const int s = threadIdx.x >> 2, q = threadIdx.x & 3;
        long long r = red[0][threadIdx.x];
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
            r = (q & 1) ? (red[w][threadIdx.x] > r ? red[w][threadIdx.x] : r)
                        : (red[w][threadIdx.x] < r ? red[w][threadIdx.x] : r);
        fin[s][q] = r;
        mm[4 * s + q] = r;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    bins_from_minmax(fin, n_specs, nf, cap, specs, d_nbins, overflow);
}

// one thread: window ranges -> dense bin layout of every spec + the device-side bin count
__device__ void bins_from_minmax(const long long (*fin)[4], int n_specs, int nf, long long cap,
                                 SpecBins* __restrict__ specs, uint32_t* __restrict__ d_nbins,
                                 int* __restrict__ overflow) {
    long long nbins = 0;
    bool bad = false;
    for (int s = 0; s < n_specs; ++s) {
        const long long rM = fin[s][1] - fin[s][0] + 1, rm = fin[s][3] - fin[s][2] + 1;
        if (rM <= 0 || rm <= 0 || rM > (1LL << 31) || rm > (1LL << 31) ||
            static_cast<double>(rM) * static_cast<double>(rm) * nf > 1.5e9) {
            bad = true;
            break;
        }
        specs[s] = SpecBins{fin[s][0], fin[s][2], rm, rM * rm, nbins};
        nbins += rM * rm * nf;
    }
    if (bad || nbins > cap) {
        *d_nbins = 0u;
        if (overflow) *overflow = 1;
    } else {
        *d_nbins = static_cast<uint32_t>(nbins);
    }
}

__global__ void __launch_bounds__(1024) k_bins_setup(const long long* __restrict__ partials, int64_t n_part,
                                                      int n_specs, int nf, long long cap,
                                                      long long* __restrict__ mm,
                                                      SpecBins* __restrict__ specs,
                                                      uint32_t* __restrict__ d_nbins,
                                                      int* __restrict__ overflow) {
    bins_setup_cta(partials, n_part, n_specs, nf, cap, mm, specs, d_nbins, overflow);
}

__global__ void k_zero_bins(uint32_t* __restrict__ a, const uint32_t* __restrict__ d_n) {
    const uint32_t n = *d_n;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = 0u;
}

// exclusive scan of hist[0, *d_n) into bin_start and cursor (<= 1024 tiles of 4096)
// Tile-local exclusive scan into out[] and cursor[]; the last active tile (atomic ticket)
// turns tile_sums[] into the exclusive tile offsets.  Consumers add
// tile_off[bin / kScanTile] (one launch instead of three).
__global__ void __launch_bounds__(kScanThreads) k_scan_tiles_dev(const uint32_t* __restrict__ in,
                                                                   uint32_t* __restrict__ out,
                                                                   uint32_t* __restrict__ cursor,
                                                                   const uint32_t* __restrict__ d_n,
                                                                   uint32_t* __restrict__ tile_sums,
                                                                   unsigned* __restrict__ ticket) {
    const int64_t n = *d_n;
    __shared__ uint32_t warp_tot[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // persistent: CTA b scans tiles b, b + gridDim.x, ...
    for (int64_t tile = blockIdx.x; tile * kScanTile < n; tile += gridDim.x) {
        const int64_t base = tile * kScanTile + threadIdx.x * kScanItems;
        uint32_t v[kScanItems];
        uint32_t run = 0;
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            const int64_t i = base + k;
            const uint32_t t = i < n ? in[i] : 0u;
            v[k] = run;
            run += t;
        }
        uint32_t x = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_tot[wid] = x;
        __syncthreads();
        if (wid == 0) {
            uint32_t w = warp_tot[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            warp_tot[lane] = w;
        }
        __syncthreads();
        const uint32_t excl = x - run + (wid ? warp_tot[wid - 1] : 0u);
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            const int64_t i = base + k;
            if (i < n) {
                out[i] = v[k] + excl;
                cursor[i] = v[k] + excl;
            }
        }
        if (threadIdx.x == kScanThreads - 1) tile_sums[tile] = excl + run;
        __syncthreads();  // warp_tot reused by the next tile
    }
    const unsigned tiles = static_cast<unsigned>((n + kScanTile - 1) / kScanTile);
    if (tiles == 0) return;  // capacity overflow: nothing binned
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    const uint32_t t = threadIdx.x < tiles ? __ldcg(tile_sums + threadIdx.x) : 0u;
    uint32_t y = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t z = __shfl_up_sync(0xffffffffu, y, o);
        if (lane >= o) y += z;
    }
    __syncthreads();
    if (lane == 31) warp_tot[wid] = y;
    __syncthreads();
    if (wid == 0) {
        uint32_t w = warp_tot[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t z = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += z;
        }
        warp_tot[lane] = w;
    }
    __syncthreads();
    if (threadIdx.x < tiles) tile_sums[threadIdx.x] = y - t + (wid ? warp_tot[wid - 1] : 0u);
    if (threadIdx.x == 0) *ticket = 0u;
}

void launch_bins_setup(const long long* partials, int64_t n_part, int n_specs, int nf, long long cap,
                       long long* mm, SpecBins* specs, uint32_t* d_nbins, int* overflow, cudaStream_t s,
                       int64_t* launches) {
    k_bins_setup<<<1, 1024, 0, s>>>(partials, n_part, n_specs, nf, cap, mm, specs, d_nbins, overflow);
    ++*launches;
}

// Per-frame dense bin layout of a frame batch on the device (no host round trip): one CTA
// turns the (spec, frame) window min/max of k_frame_minmax into SpecBins[s * nf + f] (each
// frame's own window range, bases by an exclusive scan in (spec, frame) order -- the
// lexicographic window order of the union) and the device-side bin count; a total beyond
// the capacity raises *overflow (the host API then re-runs with exact bins), otherwise it
// clears it (a union range too wide for the fused setup is not an overflow here).
__global__ void __launch_bounds__(1024) k_bins_setup_frames(const long long* __restrict__ mm, int n_specs, int nf,
                                                            long long cap, SpecBins* __restrict__ specs,
                                                            uint32_t* __restrict__ d_nbins, int* __restrict__ overflow) {
    __shared__ long long carry;
    __shared__ long long wsum[32];
    __shared__ int bad;
    const int n = n_specs * nf;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        carry = 0;
        bad = 0;
    }
    __syncthreads();
    for (int i0 = 0; i0 < n; i0 += blockDim.x) {
        const int i = i0 + threadIdx.x;
        long long sz = 0;
        const long long* m = mm + static_cast<int64_t>(i) * 4;
        if (i < n) {
            const long long rM = m[1] - m[0] + 1, rm = m[3] - m[2] + 1;
            if (rM <= 0 || rm <= 0 || rM > (1LL << 31) || rm > (1LL << 31) ||
                static_cast<double>(rM) * static_cast<double>(rm) > static_cast<double>(cap))
                bad = 1;
            else
                sz = rM * rm;
        }
        long long x = sz;  // inclusive warp scan
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[wid] = x;
        __syncthreads();
        if (wid == 0) {
            long long w = lane < static_cast<int>(blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            wsum[lane] = w;
        }
        __syncthreads();
        const long long base = carry + x - sz + (wid ? wsum[wid - 1] : 0);
        if (i < n) specs[i] = SpecBins{m[0], m[2], m[3] - m[2] + 1, sz, base};
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = base + sz;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const bool over = bad || carry > cap;
        *d_nbins = over ? 0u : static_cast<uint32_t>(carry);
        if (overflow) *overflow = over ? 1 : 0;
    }
}

void launch_bins_setup_frames(const long long* mm, int n_specs, int nf, long long cap, SpecBins* specs,
                              uint32_t* d_nbins, int* overflow, cudaStream_t s, int64_t* launches) {
    k_bins_setup_frames<<<1, 1024, 0, s>>>(mm, n_specs, nf, cap, specs, d_nbins, overflow);
    ++*launches;
}

void launch_zero_bins(uint32_t* hist, const uint32_t* d_nbins, cudaStream_t s, int64_t* launches) {
    k_zero_bins<<<kNumSMs * 4, 256, 0, s>>>(hist, d_nbins);
    ++*launches;
}

void launch_scan_bins_dev(const uint32_t* hist, uint32_t* bin_start, uint32_t* cursor, const uint32_t* d_nbins,
                          long long cap, uint32_t* tile_sums, unsigned* ticket, cudaStream_t s,
                          int64_t* launches) {
    const unsigned tiles = static_cast<unsigned>((cap + kScanTile - 1) / kScanTile);
    const unsigned grid = tiles < static_cast<unsigned>(kNumSMs) ? tiles : static_cast<unsigned>(kNumSMs);
    k_scan_tiles_dev<<<grid, kScanThreads, 0, s>>>(hist, bin_start, cursor, d_nbins, tile_sums, ticket);
    *launches += 1;
}

} // namespace fwa_b200
