// Tests of the header-only device API (include/bcnrand_device.cuh): a user
// kernel that seeks with state_at and generates in registers must reproduce
// the library fill (bcn_fill) bit for bit. Run by tests/test_dropin.py.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <vector>

#include "bcnrand_b200.h"
#include "bcnrand_device.cuh"

namespace {

// Each thread regenerates a run of `per` consecutive variates of the fill that
// starts at logical offset `base` (element j = z_{base + j + 1}).
__global__ void k_consume(uint64_t a, uint64_t base, int per, double* out, unsigned long long* sum) {
    const uint64_t t = blockIdx.x * blockDim.x + threadIdx.x;
    bcn::dev::Stream s = bcn::dev::state_at(a, base + t * per);
    double acc = 0.0;
    for (int i = 0; i < per; ++i) {
        const double u = s.next_unit();
        out[t * per + i] = u;
        acc += u;
    }
    atomicAdd(sum, static_cast<unsigned long long>(acc * 1e6));
}

int failures = 0;
void check(bool ok, const char* what) {
    if (!ok) {
        ++failures;
        std::printf("FAILED: %s\n", what);
    }
}

}  // namespace

int main() {
    // Host-side goldens through the same header (host path of the API).
    check(bcn::dev::seed_from_index(bcn::dev::kMinSeedIndex).z == 4258649398211344ull, "z0(a0)");
    check(bcn::dev::state_at(bcn::dev::kMinSeedIndex, 1000).z == 5492007519572011ull, "z1000");
    check(bcn::dev::seed_from_index(bcn::dev::kMaxSeedIndex).z == 1895384862748766ull, "z0(2^53)");
    bcn::dev::Stream s = bcn::dev::seed_from_index(bcn::dev::kMinSeedIndex);
    check(s.next() == 2138759898642167ull, "z1");
    bcn::dev::Stream w = bcn::dev::state_at(bcn::dev::kMinSeedIndex, 7);
    w.skip(bcn::dev::kPeriod - 7);
    check(w.z == 4258649398211344ull, "skip wraps the period");

    const int threads = 1 << 16, per = 64;
    const uint64_t n = static_cast<uint64_t>(threads) * per;
    const uint64_t base = 123456789012ull;
    double *d_dev = nullptr, *d_lib = nullptr;
    unsigned long long* d_sum = nullptr;
    if (cudaMalloc(&d_dev, n * 8) != cudaSuccess || cudaMalloc(&d_lib, n * 8) != cudaSuccess ||
        cudaMalloc(&d_sum, 8) != cudaSuccess) {
        std::printf("FAILED: cudaMalloc\n");
        return 1;
    }
    cudaMemset(d_sum, 0, 8);
    k_consume<<<threads / 256, 256>>>(bcn::dev::kMinSeedIndex, base, per, d_dev, d_sum);
    check(cudaDeviceSynchronize() == cudaSuccess, "device kernel");
    check(bcn_fill(d_lib, n, n, BCN_FORMAT_F64, 1, BCN_LAYOUT_CONTIGUOUS, bcn::dev::kMinSeedIndex,
                   BCN_METHOD_BARRETT_MODIFIED, base, BCN_ENGINE_AUTO, 0, nullptr) == BCN_OK,
          "bcn_fill");
    std::vector<double> a(n), b(n);
    cudaMemcpy(a.data(), d_dev, n * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), d_lib, n * 8, cudaMemcpyDeviceToHost);
    check(std::memcmp(a.data(), b.data(), n * 8) == 0, "device API == library fill");
    std::printf("[device-api] %s (%llu variates compared)\n", failures ? "FAILED" : "ok",
                static_cast<unsigned long long>(n));
    return failures ? 1 : 0;
}
