// Pageable-output probe (exploration): cost of pinning a pageable buffer in
// place (cudaHostRegister) per 64 MiB chunk vs the staging-copy path.
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main() {
    const size_t total = 8ull << 30, chunk = 64ull << 20;
    char* host = static_cast<char*>(malloc(total));
    memset(host, 1, total);  // touched, like a std::vector
    void* dev;
    cudaMalloc(&dev, chunk * 2);
    cudaMemset(dev, 7, chunk * 2);
    cudaStream_t st[2];
    cudaStreamCreate(&st[0]); cudaStreamCreate(&st[1]);
    // (a) register + unregister only
    double t0 = now();
    for (size_t off = 0; off < total; off += chunk) {
        cudaHostRegister(host + off, chunk, cudaHostRegisterDefault);
        cudaHostUnregister(host + off);
    }
    double t1 = now();
    printf("register+unregister 64 MiB chunks: %.1f GB/s\n", total / (t1 - t0) / 1e9);
    // (b) register whole buffer once
    t0 = now();
    cudaHostRegister(host, total, cudaHostRegisterDefault);
    t1 = now();
    printf("register 8 GiB at once: %.3f s (%.1f GB/s)\n", t1 - t0, total / (t1 - t0) / 1e9);
    double t2 = now();
    for (size_t off = 0; off < total; off += chunk) cudaMemcpyAsync(host + off, dev, chunk, cudaMemcpyDeviceToHost, st[(off / chunk) & 1]);
    cudaDeviceSynchronize();
    double t3 = now();
    printf("D2H into the registered buffer: %.1f GB/s\n", total / (t3 - t2) / 1e9);
    t2 = now();
    cudaHostUnregister(host);
    t3 = now();
    printf("unregister 8 GiB: %.3f s\n", t3 - t2);
    // (c) pipelined: register chunk k+1 on a helper thread while chunk k copies
    t0 = now();
    const size_t n = total / chunk;
    std::vector<int> ready(n, 0);
    std::thread reg([&] {
        for (size_t k = 0; k < n; ++k) {
            cudaHostRegister(host + k * chunk, chunk, cudaHostRegisterDefault);
            __atomic_store_n(&ready[k], 1, __ATOMIC_RELEASE);
        }
    });
    for (size_t k = 0; k < n; ++k) {
        while (!__atomic_load_n(&ready[k], __ATOMIC_ACQUIRE)) {}
        cudaMemcpyAsync(host + k * chunk, dev, chunk, cudaMemcpyDeviceToHost, st[k & 1]);
        if (k >= 2) { cudaStreamSynchronize(st[k & 1 ^ 1]); }
    }
    cudaDeviceSynchronize();
    reg.join();
    t1 = now();
    for (size_t k = 0; k < n; ++k) cudaHostUnregister(host + k * chunk);
    double t4 = now();
    printf("pipelined register+D2H: %.1f GB/s (excluding unregister), %.1f GB/s with unregister\n",
           total / (t1 - t0) / 1e9, total / (t4 - t0) / 1e9);
    return 0;
}
