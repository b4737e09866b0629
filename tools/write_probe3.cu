// write_probe3.cu — can the copy engines write HBM faster than SM stores?
// cudaMemset (a copy-engine fill, no kernel) writes at ~7.39 TB/s while SM
// stores top out near 6.3-6.4 TB/s. Measures CE D2D copies from DRAM and from
// an L2-resident source (exploration tool).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                \
    do {                                                                     \
        cudaError_t e = (x);                                                 \
        if (e != cudaSuccess) {                                              \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
            exit(1);                                                         \
        }                                                                    \
    } while (0)

template <class F>
float time_ms(F f, int reps) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int i = 0; i < 2; ++i) f();
    CK(cudaDeviceSynchronize());
    std::vector<float> t;
    for (int i = 0; i < reps; ++i) {
        CK(cudaEventRecord(a));
        f();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        t.push_back(ms);
    }
    std::sort(t.begin(), t.end());
    return t[t.size() / 2];
}

int main() {
    const uint64_t bytes = 8ull << 30;
    char *dst, *src;
    CK(cudaMalloc(&dst, bytes));
    CK(cudaMalloc(&src, bytes / 2));
    CK(cudaMemset(src, 1, bytes / 2));
    auto rep = [](const char* name, uint64_t b, float ms) {
        printf("{\"op\":\"%s\",\"bytes\":%llu,\"ms\":%.4f,\"write_gbs\":%.1f}\n", name, (unsigned long long)b, ms,
               b / ms / 1e6);
    };
    rep("memset", bytes, time_ms([&] { CK(cudaMemsetAsync(dst, 0, bytes)); }, 10));
    rep("d2d_dram_4g", bytes / 2, time_ms([&] { CK(cudaMemcpyAsync(dst, src, bytes / 2, cudaMemcpyDeviceToDevice)); }, 10));
    for (uint64_t chunk : {8ull << 20, 32ull << 20, 64ull << 20}) {
        const uint64_t n = bytes / chunk;
        char name[64];
        snprintf(name, sizeof name, "d2d_l2src_%lluMB", (unsigned long long)(chunk >> 20));
        rep(name, bytes, time_ms([&] {
                for (uint64_t i = 0; i < n; ++i)
                    CK(cudaMemcpyAsync(dst + i * chunk, src, chunk, cudaMemcpyDeviceToDevice));
            }, 5));
    }
    // Several streams in parallel (more copy engines).
    cudaStream_t s[4];
    for (auto& x : s) CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
    cudaEvent_t ev;
    CK(cudaEventCreate(&ev));
    rep("d2d_l2src_32MB_4streams", bytes, time_ms([&] {
            const uint64_t chunk = 32ull << 20, n = bytes / chunk;
            CK(cudaEventRecord(ev, 0));
            for (auto& x : s) CK(cudaStreamWaitEvent(x, ev));
            for (uint64_t i = 0; i < n; ++i)
                CK(cudaMemcpyAsync(dst + i * chunk, src + (i % 4) * chunk, chunk, cudaMemcpyDeviceToDevice, s[i % 4]));
            for (auto& x : s) {
                CK(cudaEventRecord(ev, x));
                CK(cudaStreamWaitEvent(0, ev));
            }
        }, 5));
    rep("memset_4streams", bytes, time_ms([&] {
            const uint64_t q = bytes / 4;
            CK(cudaEventRecord(ev, 0));
            for (auto& x : s) CK(cudaStreamWaitEvent(x, ev));
            for (int i = 0; i < 4; ++i) CK(cudaMemsetAsync(dst + i * q, 0, q, s[i]));
            for (auto& x : s) {
                CK(cudaEventRecord(ev, x));
                CK(cudaStreamWaitEvent(0, ev));
            }
        }, 5));
    return 0;
}
