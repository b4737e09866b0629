// write_probe4.cu — does pacing SM stores raise HBM write bandwidth?
// The compute-heavy fill kernels (f32 FP64 engine: 6.52 TB/s, u64 Barrett:
// 6.40 TB/s) out-write the back-to-back Constant writer (~6.25 TB/s). Here a
// constant writer spins `delay` dependent FFMAs between 1 KiB warp stores, for
// several occupancies and both row orders (exploration tool).
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

template <bool STRIDE>
__global__ void k_paced(char* out, uint64_t rows, int delay, float seed) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const uint64_t w = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    uint64_t r, e, step;
    if (STRIDE) {
        r = w;
        e = rows;
        step = nw;
    } else {
        const uint64_t q = rows / nw, rem = rows % nw;
        r = w * q + (w < rem ? w : rem);
        e = r + q + (w < rem ? 1 : 0);
        step = 1;
    }
    float x = seed + lane;
    for (; r < e; r += step) {
        for (int i = 0; i < delay; ++i) x = fmaf(x, 1.0000001f, 1e-7f);
        const uint64_t v = 0x3FE0000000000000ull ^ (uint64_t)__float_as_uint(x) * (x == 12345.f);
        asm volatile("st.global.v4.b64 [%0], {%1, %1, %1, %1};" ::"l"(out + r * 1024 + lane * 32), "l"(v)
                     : "memory");
    }
}

template <class F>
float time_ms(F f, int reps) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int i = 0; i < 3; ++i) f();
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
    const uint64_t bytes = 8ull << 30, rows = bytes / 1024;
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    char* buf;
    CK(cudaMalloc(&buf, bytes));
    for (int cps : {1, 2, 4, 8}) {
        for (int delay : {0, 4, 8, 16, 32, 64, 128, 256}) {
            for (int stride = 0; stride < 2; ++stride) {
                const int grid = sms * cps;
                float ms = time_ms([&] {
                    if (stride)
                        k_paced<true><<<grid, 256>>>(buf, rows, delay, 1.f);
                    else
                        k_paced<false><<<grid, 256>>>(buf, rows, delay, 1.f);
                }, 9);
                printf("{\"ctas_per_sm\":%d,\"delay\":%d,\"order\":\"%s\",\"ms\":%.4f,\"gbs\":%.1f}\n", cps, delay,
                       stride ? "stride" : "rows", ms, bytes / ms / 1e6);
            }
        }
    }
    return 0;
}
