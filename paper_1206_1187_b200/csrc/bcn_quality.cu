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

// One counts of bits 5..52 of w = floor(z 2^53 / m) (quality.cpp:66-73).
// w is the modified-Barrett quotient q3, +1 when the step needed its
// correction; residues >= m raise the error flag.
__global__ void __launch_bounds__(256) k_monobit(const uint64_t* z, uint64_t n,
                                                 unsigned long long* ones, int* error) {
    __shared__ unsigned long long acc[53];
    for (int b = threadIdx.x; b < 53; b += blockDim.x) acc[b] = 0;
    __syncthreads();
    unsigned int local[48];
#pragma unroll
    for (int b = 0; b < 48; ++b) local[b] = 0;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t v = z[i];
        if (v >= kModulus) {
            *error = 1;
            continue;
        }
        const uint64_t hi = __umul64hi(v, kMu), lo = v * kMu;
        uint64_t w = (hi << 11) | (lo >> 53);  // q3 in {Q-1, Q}
        const uint64_t r = 0x20000000000000ull - ((w * kModulus) & 0x1FFFFFFFFFFFFFull);
        if (v != 0 && r >= kModulus) ++w;      // the step's correction => q3 was Q-1
        if (v == 0) w = 0;
#pragma unroll
        for (int b = 0; b < 48; ++b) local[b] += static_cast<unsigned int>((w >> (b + 5)) & 1);
    }
#pragma unroll
    for (int b = 0; b < 48; ++b) {
        unsigned int c = local[b];
#pragma unroll
        for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if ((threadIdx.x & 31) == 0 && c) atomicAdd(&acc[b + 5], static_cast<unsigned long long>(c));
    }
    __syncthreads();
    for (int b = threadIdx.x; b < 53; b += blockDim.x)
        if (acc[b]) atomicAdd(&ones[b], acc[b]);
}

// Per-block partial sums sx, sy, sxx, syy, sxy over pairs (s[i], s[i+lag]),
// i < pairs (quality.cpp:98-108); out[block*5 + k]. Fixed grid => the host's
// fixed-order reduction makes the result deterministic.
__global__ void __launch_bounds__(256) k_lag_sums(const double* s, uint64_t pairs, uint64_t lag,
                                                  double* out) {
    double a[5] = {0, 0, 0, 0, 0};
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < pairs; i += stride) {
        const double x = s[i], y = s[i + lag];
        a[0] += x;
        a[1] += y;
        a[2] += x * x;
        a[3] += y * y;
        a[4] += x * y;
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
    const size_t smem = bins <= kChiSmemBins ? static_cast<size_t>(bins) * 4 : 0;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_chi_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k_chi_hist<<<grid, 256, smem, s>>>(u, n, bins, counts, error);
    return cudaGetLastError();
}

cudaError_t launch_monobit(const uint64_t* z, uint64_t n, unsigned long long* ones, int* error, int grid,
                           cudaStream_t s) {
    k_monobit<<<grid, 256, 0, s>>>(z, n, ones, error);
    return cudaGetLastError();
}

cudaError_t launch_lag_sums(const double* x, uint64_t pairs, uint64_t lag, double* out, int grid,
                            cudaStream_t s) {
    k_lag_sums<<<grid, 256, 0, s>>>(x, pairs, lag, out);
    return cudaGetLastError();
}

}  // namespace bcn_b200
