// write_probe6.cu — clock-independent pacing with %globaltimer (ns):
// (1) globaltimer resolution; (2) offered-load sweep (ns pacing, grid-strided
// rows) for the Constant writer and the production engines' loops
// (exploration tool).
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

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void k_res(uint64_t* out) {
    uint64_t prev = gtimer(), minstep = ~0ull, changes = 0, t0 = prev;
    for (int i = 0; i < 200000; ++i) {
        uint64_t t = gtimer();
        if (t != prev) {
            if (t - prev < minstep) minstep = t - prev;
            ++changes;
            prev = t;
        }
    }
    out[0] = minstep;
    out[1] = changes;
    out[2] = prev - t0;
}

// KIND 0 constant, 1 u64 Barrett, 2 f64 FP64, 3 f32 FP64 (8 chains), SLEEP: nanosleep in spin
template <int KIND, int SLEEP>
__global__ void __launch_bounds__(256) k_paced(char* out, uint64_t rows, uint64_t gap_ps, Mult kS, uint64_t z0) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
    uint64_t r = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    constexpr int V = KIND == 3 ? 8 : 4;
    uint64_t zi[V];
    double zd[V];
    uint64_t z = z0 + r * 977 + lane;
    for (int v = 0; v < V; ++v) {
        zi[v] = z % kModulus;
        zd[v] = (double)(int64_t)(zi[v] > kModulus / 2 ? zi[v] - kModulus : zi[v]);
        z = step_modified_barrett(zi[v] | 1);
    }
    // target time in picoseconds to keep fractional gaps exact
    uint64_t t_ps = gtimer() * 1000;
    for (; r < rows; r += nw) {
        if (gap_ps) {
            t_ps += gap_ps;
            const uint64_t t_ns = t_ps / 1000;
            while (gtimer() < t_ns) {
                if (SLEEP) __nanosleep(SLEEP);
            }
        }
        uint64_t b[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            if (KIND == 0) {
                b[v] = 0x3FE0000000000000ull;
            } else if (KIND == 1) {
                b[v] = zi[v];
                zi[v] = mul_barrett(zi[v], kS.c, kS.shoup);
            } else if (KIND == 2) {
                b[v] = (uint64_t)__double_as_longlong(__dmul_rn(fp64_canonical(zd[v]), kInvModulus));
                zd[v] = mul_fp64(zd[v], kS.cb, kS.com);
            } else {
                b[v] = __float_as_uint(f32_rz_from_unit(__dmul_rn(fp64_canonical(zd[v]), kInvModulus)));
                zd[v] = mul_fp64(zd[v], kS.cb, kS.com);
            }
        }
        uint64_t w[4];
        if (V == 4) {
            for (int i = 0; i < 4; ++i) w[i] = b[i];
        } else {
            for (int i = 0; i < 4; ++i) w[i] = b[2 * i] | (b[2 * i + 1] << 32);
        }
        asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(out + r * 1024 + lane * 32), "l"(w[0]),
                     "l"(w[1]), "l"(w[2]), "l"(w[3])
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
    uint64_t* d;
    CK(cudaMalloc(&d, 64));
    k_res<<<1, 1>>>(d);
    uint64_t h[3];
    CK(cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost));
    printf("{\"globaltimer_min_step_ns\":%llu,\"changes\":%llu,\"span_ns\":%llu}\n", (unsigned long long)h[0],
           (unsigned long long)h[1], (unsigned long long)h[2]);
    const uint64_t bytes = 8ull << 30, rows = bytes / 1024;
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    char* buf;
    CK(cudaMalloc(&buf, bytes));
    const char* names[4] = {"constant", "u64_barrett", "f64_fp64", "f32_fp64"};
    for (int kind = 0; kind < 4; ++kind) {
        for (int cps : {2, 4, 6}) {
            const int grid = sms * cps;
            const uint64_t nwarps = (uint64_t)grid * 8;
            const uint64_t step_elems = (kind == 3 ? 256ull : 128ull) * nwarps;
            const Mult kS = host_make_mult(host_jump(step_elems));
            for (int sleep = 0; sleep < 2; ++sleep) {
                for (double tbs : {0.0, 7.0, 7.2, 7.3, 7.4, 7.5, 7.6, 7.8}) {
                    // per-warp gap in ps: nwarps * 1 KiB / rate
                    const uint64_t gap_ps = tbs == 0.0 ? 0 : (uint64_t)(nwarps * 1024.0 / (tbs * 1e12) * 1e12);
                    float ms = time_ms([&] {
#define L(K)                                                                                  \
    if (sleep)                                                                                \
        k_paced<K, 32><<<grid, 256>>>(buf, rows, gap_ps, kS, 12345);                          \
    else                                                                                      \
        k_paced<K, 0><<<grid, 256>>>(buf, rows, gap_ps, kS, 12345);
                        switch (kind) {
                            case 0: L(0) break;
                            case 1: L(1) break;
                            case 2: L(2) break;
                            default: L(3) break;
                        }
                    }, 7);
                    printf("{\"kind\":\"%s\",\"ctas_per_sm\":%d,\"sleep\":%d,\"target_tbs\":%.1f,\"ms\":%.4f,\"gbs\":%.1f}\n",
                           names[kind], cps, sleep, tbs, ms, bytes / ms / 1e6);
                    fflush(stdout);
                }
            }
        }
    }
    return 0;
}
