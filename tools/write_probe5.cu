// write_probe5.cu — offered-load sweep: each warp spaces its 1 KiB row stores
// by `gap` SM cycles (clock64 pacing with catch-up), for the Constant writer
// and the real generator loops, at several occupancies and both row orders.
// Finds the offered rate at which HBM write efficiency peaks (exploration tool).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1206_1187_b200/csrc/bcn_math.cuh"

using namespace bcn_b200;

#define CK(x)                                                                \
    do {                                                                     \
        cudaError_t e = (x);                                                 \
        if (e != cudaSuccess) {                                              \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
            exit(1);                                                         \
        }                                                                    \
    } while (0)

// KIND 0 constant, 1 u64 Barrett, 2 f64 FP64 engine, 3 f64 Barrett
template <int KIND>
__global__ void __launch_bounds__(256) k_paced(char* out, uint64_t rows, int stride, long long gap,
                                               Mult k1, Mult kS, uint64_t z0) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const uint64_t w = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    uint64_t r, e, step;
    if (stride) {
        r = w;
        e = rows;
        step = nw;
    } else {
        const uint64_t q = rows / nw, rem = rows % nw;
        r = w * q + (w < rem ? w : rem);
        e = r + q + (w < rem ? 1 : 0);
        step = 1;
    }
    const Mult k = stride ? kS : k1;
    uint64_t zi[4];
    double zd[4];
    uint64_t z = z0 + r * 977 + lane;
    for (int v = 0; v < 4; ++v) {
        zi[v] = z % kModulus;
        zd[v] = (double)(int64_t)(zi[v] > kModulus / 2 ? zi[v] - kModulus : zi[v]);
        z = step_modified_barrett(zi[v] | 1);
    }
    long long t = clock64();
    for (; r < e; r += step) {
        if (gap) {
            while (clock64() < t) {
            }
            t += gap;
        }
        uint64_t b[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            if (KIND == 0) {
                b[v] = 0x3FE0000000000000ull;
            } else if (KIND == 1) {
                b[v] = zi[v];
                zi[v] = mul_barrett(zi[v], k.c, k.shoup);
            } else if (KIND == 2) {
                b[v] = (uint64_t)__double_as_longlong(__dmul_rn(fp64_canonical(zd[v]), kInvModulus));
                zd[v] = mul_fp64(zd[v], k.cb, k.com);
            } else {
                b[v] = (uint64_t)__double_as_longlong(unit_from_u64(zi[v]));
                zi[v] = mul_barrett(zi[v], k.c, k.shoup);
            }
        }
        asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(out + r * 1024 + lane * 32), "l"(b[0]),
                     "l"(b[1]), "l"(b[2]), "l"(b[3])
                     : "memory");
    }
}

template <class F>
float time_ms(F f, int reps) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int i = 0; i < 2; ++i) f();
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
    int sms, clk_khz;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
    char* buf;
    CK(cudaMalloc(&buf, bytes));
    const Mult k1 = host_make_mult(host_jump(128));
    const char* names[4] = {"constant", "u64_barrett", "f64_fp64", "f64_barrett"};
    printf("{\"sm_clock_mhz_attr\":%d}\n", clk_khz / 1000);
    for (int kind = 0; kind < 4; ++kind) {
        for (int cps : {1, 2, 4}) {
            const int grid = sms * cps;
            const int wps = cps * 8;
            const Mult kS = host_make_mult(host_jump(128ull * grid * 8));
            for (int stride = 0; stride < 2; ++stride) {
                for (double tbs : {0.0, 6.4, 6.8, 7.0, 7.2, 7.4, 7.6, 8.0, 9.0}) {
                    // per-warp gap (cycles) for an offered rate `tbs` at 1.965 GHz
                    const long long gap = tbs == 0.0 ? 0
                                                     : (long long)(wps * 1024.0 * sms * 1.965e9 / (tbs * 1e12));
                    float ms = time_ms([&] {
                        switch (kind) {
                            case 0: k_paced<0><<<grid, 256>>>(buf, rows, stride, gap, k1, kS, 12345); break;
                            case 1: k_paced<1><<<grid, 256>>>(buf, rows, stride, gap, k1, kS, 12345); break;
                            case 2: k_paced<2><<<grid, 256>>>(buf, rows, stride, gap, k1, kS, 12345); break;
                            default: k_paced<3><<<grid, 256>>>(buf, rows, stride, gap, k1, kS, 12345); break;
                        }
                    }, 7);
                    printf("{\"kind\":\"%s\",\"ctas_per_sm\":%d,\"order\":\"%s\",\"offered_tbs\":%.1f,\"gap\":%lld,"
                           "\"ms\":%.4f,\"gbs\":%.1f}\n",
                           names[kind], cps, stride ? "stride" : "rows", tbs, gap, ms, bytes / ms / 1e6);
                    fflush(stdout);
                }
            }
        }
    }
    return 0;
}
