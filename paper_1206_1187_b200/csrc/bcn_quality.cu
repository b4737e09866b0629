// bcn_quality.cu — device statistical smoke suite, the
// B200 counterpart of the reference's quality.cpp:
//   chi_square_uniformity (quality.cpp:21-54)  -> k_chi_hist    (bin counts)
//   monobit_mantissa      (quality.cpp:56-90)  -> k_monobit     (per-bit one counts)
//   serial_correlation    (quality.cpp:92-118) -> k_lag_sums    (per-block partial sums)
// The kernels produce exact integer counts (chi-square, monobit) or per-block
// double partial sums reduced on the host in a fixed order (correlation), and
// the host applies the reference's formulas, so the chi-square and monobit
// statistics are bit-identical to the reference and the correlation is
// deterministic run to run.
#include <cuda_runtime.h>

#include <cstdint>

#include "bcn_kernels.cuh"

namespace bcn_b200 {

// Bin counts of u * bins (truncated, clamped to bins-1) exactly as
// quality.cpp:33-39; any sample outside (0,1) (or NaN) raises the error flag.
__global__ void __launch_bounds__(256) k_chi_hist(const double* u, uint64_t n, int bins,
                                                  unsigned long long* counts, int* error) {
    extern __shared__ unsigned int h[];
    const bool use_smem = bins <= kChiSmemBins;
    if (use_smem)
        for (int b = threadIdx.x; b < bins; b += blockDim.x) h[b] = 0;
    __syncthreads();
    const double fb = static_cast<double>(bins);
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double x = u[i];
        if (!(x > 0.0) || !(x < 1.0)) {
            *error = 1;
            continue;
        }
        uint64_t b = static_cast<uint64_t>(x * fb);
        if (b >= static_cast<uint64_t>(bins)) b = bins - 1;
        if (use_smem)
            atomicAdd(&h[b], 1u);
        else
            atomicAdd(&counts[b], 1ull);
    }
    __syncthreads();
    if (use_smem)
        for (int b = threadIdx.x; b < bins; b += blockDim.x)
            if (h[b]) atomicAdd(&counts[b], static_cast<unsigned long long>(h[b]));
}

// Lane-private variant for bins <= kChiLaneBins: counter (bin, lane) lives at
// h[bin * 32 + lane], so lane l only ever touches bank l and a warp's 32
// shared atomics never conflict, whatever bins its samples fall in. 16 loads
// per thread are in flight per pass.
constexpr int kChiLaneBins = 1600;  // 32 x 4 B x 1600 = 200 KiB of shared memory
constexpr int kChiLoads = 16;

constexpr int kChiThreads = 1024;

__global__ void __launch_bounds__(kChiThreads) k_chi_hist_lanes(const double* u, uint64_t n, int bins,
                                                        unsigned long long* counts, int* error) {
    extern __shared__ unsigned int hl[];
    const unsigned lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < bins * 32; i += blockDim.x) hl[i] = 0;
    __syncthreads();
    const double fb = static_cast<double>(bins);
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    bool bad = false;
    for (uint64_t i0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i0 < n;
         i0 += stride * kChiLoads) {
        double x[kChiLoads];
        if (i0 + (kChiLoads - 1) * stride < n) {  // whole pass: unguarded loads, all in flight
#pragma unroll
            for (int j = 0; j < kChiLoads; ++j) x[j] = u[i0 + j * stride];
        } else {
#pragma unroll
            for (int j = 0; j < kChiLoads; ++j) x[j] = i0 + j * stride < n ? u[i0 + j * stride] : 0.5;
        }
#pragma unroll
        for (int j = 0; j < kChiLoads; ++j) {
            if (!(x[j] > 0.0) || !(x[j] < 1.0)) {
                bad = true;
                continue;
            }
            unsigned b = static_cast<unsigned>(x[j] * fb);
            if (b >= static_cast<unsigned>(bins)) b = bins - 1;
            if (i0 + j * stride < n) atomicAdd(&hl[b * 32 + lane], 1u);
        }
    }
    if (bad) *error = 1;
    __syncthreads();
    for (int b = threadIdx.x; b < bins; b += blockDim.x) {
        unsigned long long c = 0;
#pragma unroll 8
        for (int l = 0; l < 32; ++l) c += hl[b * 32 + ((l + b) & 31)];  // rotated: conflict-free
        if (c) atomicAdd(&counts[b], c);
    }
}

// One counts of bits 5..52 of w = floor(z 2^53 / m) (quality.cpp:66-73).
// w is the modified-Barrett quotient q3, +1 when the step needed its
// correction; residues >= m raise the error flag (and count as w = 0). For
// v = 0 the formula is not used (w = 0).
// Branch-free: `bad` collects out-of-range residues (reported once per thread).
__device__ __forceinline__ uint64_t mantissa_w(uint64_t v, bool& bad) {
    const bool out = v >= kModulus;
    bad |= out;
    const uint64_t hi = __umul64hi(v, kMu), lo = v * kMu;
    uint64_t w = (hi << 11) | (lo >> 53);  // q3 in {Q-1, Q}
    const uint64_t r = 0x20000000000000ull - ((w * kModulus) & 0x1FFFFFFFFFFFFFull);
    w += (r >= kModulus) ? 1 : 0;          // the step's correction => q3 was Q-1
    return (v == 0 || out) ? 0 : w;
}

// Carry-save adder: (h, l) = the two-bit column sums of a + b + c.
__device__ __forceinline__ void csa(uint32_t& h, uint32_t& l, uint32_t a, uint32_t b, uint32_t c) {
    const uint32_t u = a ^ b;
    h = (a & b) | (u & c);
    l = u ^ c;
}

// Bit-sliced column counter of one 32-bit word stream: Harley-Seal
// compression of 16 words into a weight-16 word (15 CSAs), rippled into
// kPlanes counter planes (bit j of plane k = bit k of column j's count / 16).
constexpr int kPlanes = 8;  // up to 255 add16 calls between flushes
struct ColumnCounter {
    uint32_t ones = 0, twos = 0, fours = 0, eights = 0;
    uint32_t plane[kPlanes] = {};

    __device__ __forceinline__ void add16(const uint32_t (&d)[16]) {
        uint32_t twosA, twosB, foursA, foursB, eightsA, eightsB, sixteens;
        csa(twosA, ones, ones, d[0], d[1]);
        csa(twosB, ones, ones, d[2], d[3]);
        csa(foursA, twos, twos, twosA, twosB);
        csa(twosA, ones, ones, d[4], d[5]);
        csa(twosB, ones, ones, d[6], d[7]);
        csa(foursB, twos, twos, twosA, twosB);
        csa(eightsA, fours, fours, foursA, foursB);
        csa(twosA, ones, ones, d[8], d[9]);
        csa(twosB, ones, ones, d[10], d[11]);
        csa(foursA, twos, twos, twosA, twosB);
        csa(twosA, ones, ones, d[12], d[13]);
        csa(twosB, ones, ones, d[14], d[15]);
        csa(foursB, twos, twos, twosA, twosB);
        csa(eightsB, fours, fours, foursA, foursB);
        csa(sixteens, eights, eights, eightsA, eightsB);
        uint32_t carry = sixteens;
#pragma unroll
        for (int k = 0; k < kPlanes; ++k) {
            const uint32_t t = plane[k] & carry;
            plane[k] ^= carry;
            carry = t;
        }
    }
    // Count of column j.
    __device__ __forceinline__ uint32_t column(int j) const {
        uint32_t c = ((ones >> j) & 1) + 2 * ((twos >> j) & 1) + 4 * ((fours >> j) & 1) + 8 * ((eights >> j) & 1);
#pragma unroll
        for (int k = 0; k < kPlanes; ++k) c += ((plane[k] >> j) & 1) << (k + 4);
        return c;
    }
};

// Each thread takes 32 residues per group. The 48-bit windows x = w >> 5 are
// split into two word streams, counted column-wise by a ColumnCounter each:
// the low 32 bits of every residue (two add16 calls per group) and the high
// 16 bits of residue pairs packed into one word (one add16). Counts are flushed (warp-reduced, then shared and global atomics) at the
// end and every 127 groups, before the counter planes can overflow.
constexpr int kMonoGroup = 32;
constexpr uint32_t kMonoFlushGroups = 127;  // 2 add16 per group on the low stream

__device__ __forceinline__ void monobit_flush(ColumnCounter& lo, ColumnCounter& hi, unsigned long long* acc) {
    const unsigned lane = threadIdx.x & 31;
#pragma unroll 1
    for (int b = 5; b < 53; ++b) {
        uint32_t c = b < 37 ? lo.column(b - 5) : hi.column(b - 37) + hi.column(b - 37 + 16);
#pragma unroll
        for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0 && c) atomicAdd(&acc[b], static_cast<unsigned long long>(c));
    }
    lo = ColumnCounter{};
    hi = ColumnCounter{};
}

__device__ __forceinline__ void monobit_load(const uint64_t* z, uint64_t n, uint64_t base, uint64_t stride,
                                             uint64_t (&v)[kMonoGroup]) {
    if (base + (kMonoGroup - 1) * stride < n) {
#pragma unroll
        for (int j = 0; j < kMonoGroup; ++j) v[j] = z[base + j * stride];
    } else {
#pragma unroll
        for (int j = 0; j < kMonoGroup; ++j) v[j] = base + j * stride < n ? z[base + j * stride] : 0;
    }
}

__global__ void __launch_bounds__(256) k_monobit(const uint64_t* z, uint64_t n,
                                                 unsigned long long* ones, int* error) {
    __shared__ unsigned long long acc[53];
    for (int b = threadIdx.x; b < 53; b += blockDim.x) acc[b] = 0;
    __syncthreads();
    ColumnCounter lo, hi;
    bool bad = false;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t groups = (n + nthreads * kMonoGroup - 1) / (nthreads * kMonoGroup);
    // group g of this thread: elements (g * kMonoGroup + j) * nthreads + tid
    uint32_t since_flush = 0;
#pragma unroll 1
    for (uint64_t g = 0; g < groups; ++g) {
        uint64_t v[kMonoGroup];
        monobit_load(z, n, (g * kMonoGroup) * nthreads + tid, nthreads, v);
        uint32_t wl[kMonoGroup], wh[kMonoGroup / 2];
#pragma unroll
        for (int j = 0; j < kMonoGroup / 2; ++j) {
            const uint64_t xa = mantissa_w(v[2 * j], bad) >> 5;
            const uint64_t xb = mantissa_w(v[2 * j + 1], bad) >> 5;
            wl[2 * j] = static_cast<uint32_t>(xa);
            wl[2 * j + 1] = static_cast<uint32_t>(xb);
            wh[j] = static_cast<uint32_t>(xa >> 32) | (static_cast<uint32_t>(xb >> 32) << 16);
        }
        lo.add16(*reinterpret_cast<const uint32_t(*)[16]>(&wl[0]));
        lo.add16(*reinterpret_cast<const uint32_t(*)[16]>(&wl[16]));
        hi.add16(wh);
        if (++since_flush == kMonoFlushGroups) {
            monobit_flush(lo, hi, acc);
            since_flush = 0;
        }
    }
    monobit_flush(lo, hi, acc);
    if (bad) *error = 1;
    __syncthreads();
    for (int b = threadIdx.x; b < 53; b += blockDim.x)
        if (acc[b]) atomicAdd(&ones[b], acc[b]);
}

// Per-block partial sums sx, sy, sxx, syy, sxy over pairs (s[i], s[i+lag]),
// i < pairs (quality.cpp:98-108); out[block*5 + k]. Fixed grid => the host's
// fixed-order reduction makes the result deterministic.
__global__ void __launch_bounds__(256) k_lag_sums(const double* s, uint64_t pairs, uint64_t lag,
                                                  double* out) {
    constexpr int U = 8;  // loads of x (and of y) in flight per thread
    double a[5] = {0, 0, 0, 0, 0};
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i0 < pairs;
         i0 += stride * U) {
        double x[U], y[U];
        if (i0 + (U - 1) * stride < pairs) {  // whole pass: unguarded loads, all in flight
#pragma unroll
            for (int j = 0; j < U; ++j) {
                x[j] = s[i0 + j * stride];
                y[j] = s[i0 + j * stride + lag];
            }
        } else {
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const bool in = i0 + j * stride < pairs;
                x[j] = in ? s[i0 + j * stride] : 0.0;
                y[j] = in ? s[i0 + j * stride + lag] : 0.0;
            }
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            a[0] += x[j];
            a[1] += y[j];
            a[2] += x[j] * x[j];
            a[3] += y[j] * y[j];
            a[4] += x[j] * y[j];
        }
    }
    __shared__ double red[5][256];
#pragma unroll
    for (int k = 0; k < 5; ++k) red[k][threadIdx.x] = a[k];
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w)
#pragma unroll
            for (int k = 0; k < 5; ++k) red[k][threadIdx.x] += red[k][threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x < 5) out[blockIdx.x * 5 + threadIdx.x] = red[threadIdx.x][0];
}

cudaError_t launch_chi_hist(const double* u, uint64_t n, int bins, unsigned long long* counts, int* error,
                            int grid, cudaStream_t s) {
    if (bins <= kChiLaneBins) {
        const size_t smem = static_cast<size_t>(bins) * 32 * 4;
        cudaFuncSetAttribute(k_chi_hist_lanes, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        int dev = 0, sms = 148, per_sm = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_chi_hist_lanes, kChiThreads, smem);
        const uint64_t want = (n + kChiThreads * kChiLoads - 1) / (kChiThreads * kChiLoads);
        const uint64_t cap = static_cast<uint64_t>(sms) * (per_sm > 0 ? per_sm : 1);
        k_chi_hist_lanes<<<static_cast<unsigned>(want < cap ? want : cap), kChiThreads, smem, s>>>(u, n, bins, counts, error);
        return cudaGetLastError();
    }
    const size_t smem = bins <= kChiSmemBins ? static_cast<size_t>(bins) * 4 : 0;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_chi_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k_chi_hist<<<grid, 256, smem, s>>>(u, n, bins, counts, error);
    return cudaGetLastError();
}

cudaError_t launch_monobit(const uint64_t* z, uint64_t n, unsigned long long* ones, int* error, int grid,
                           cudaStream_t s) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_monobit, 256, 0);
    const int resident = sms * (per_sm > 0 ? per_sm : 1);  // one wave: every thread loops over groups
    if (grid > resident) grid = resident;
    k_monobit<<<grid, 256, 0, s>>>(z, n, ones, error);
    return cudaGetLastError();
}

cudaError_t launch_lag_sums(const double* x, uint64_t pairs, uint64_t lag, double* out, int grid,
                            cudaStream_t s) {
    k_lag_sums<<<grid, 256, 0, s>>>(x, pairs, lag, out);
    return cudaGetLastError();
}

}  // namespace bcn_b200
