// Generate-and-consume throughput of the header-only device API
// (include/bcnrand_device.cuh): each thread seeks with state_at and sums
// `per` consecutive variates in registers (nothing stored). Also times the
// seeding alone. Exploration / evidence tool:
//   make -C tools/c device_api_perf && tools/c/device_api_perf
#include <cuda_runtime.h>

#include <cstdio>

#include "bcnrand_device.cuh"

__global__ void k_consume(uint64_t a, uint64_t base, int per, double* sink) {
    const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    bcn::dev::Stream s = bcn::dev::state_at(a, base + t * per);
    double acc = 0.0;
    for (int i = 0; i < per; ++i) acc += s.next_unit();
    if (acc < 0) sink[t] = acc;  // never true; keeps the loop
}

__global__ void k_seed_only(uint64_t a, uint64_t base, uint64_t* sink) {
    const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const bcn::dev::Stream s = bcn::dev::state_at(a, base + t * 0x9E3779B97F4A7C15ull);
    if (s.z == 0) sink[t] = s.z;
}

int main() {
    const uint64_t a0 = bcn::dev::kMinSeedIndex;
    double* sink = nullptr;
    cudaMalloc(&sink, 8 << 20);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int threads = 148 * 2048;  // full occupancy on 148 SMs
    for (int per : {64, 1024, 16384}) {
        k_consume<<<threads / 256, 256>>>(a0, 0, per, sink);
        cudaEventRecord(e0);
        k_consume<<<threads / 256, 256>>>(a0, 0, per, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        std::printf("{\"path\": \"device_api_consume\", \"threads\": %d, \"per_thread\": %d, \"ms\": %.4f, "
                    "\"gvariates_s\": %.1f}\n", threads, per, ms, 1.0 * threads * per / ms * 1e-6);
    }
    k_seed_only<<<threads / 256, 256>>>(a0, 1, reinterpret_cast<uint64_t*>(sink));
    cudaEventRecord(e0);
    k_seed_only<<<threads / 256, 256>>>(a0, 1, reinterpret_cast<uint64_t*>(sink));
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::printf("{\"path\": \"device_api_state_at\", \"threads\": %d, \"ms\": %.4f, \"gseeks_s\": %.2f}\n",
                threads, ms, threads / ms * 1e-6);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
