// write_probe7.cu — production-shaped paced fill loops: grid-strided rows,
// clock64 pacing with __nanosleep back-off (no issue-slot burning), FP64 /
// Barrett engines, 4 or 8 chains per lane. Also reports the SM clock measured
// against %globaltimer during the run (exploration tool).
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

__device__ unsigned long long g_clk[2];

// KIND 1 u64 Barrett, 2 f64 FP64, 3 f32 FP64. ROWS rows per iteration (ILP).
template <int KIND, int ROWS>
__global__ void __launch_bounds__(256) k_fill(char* out, uint64_t rows, long long gap, int sleep_shift, Mult kS,
                                              uint64_t z0) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const uint64_t w = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    constexpr int V = KIND == 3 ? 8 : 4;
    uint64_t zi[ROWS][V];
    double zd[ROWS][V];
    for (int h = 0; h < ROWS; ++h) {
        uint64_t z = z0 + (w + h * nw) * 977 + lane;
        for (int v = 0; v < V; ++v) {
            zi[h][v] = z % kModulus;
            zd[h][v] = (double)(int64_t)(zi[h][v] > kModulus / 2 ? zi[h][v] - kModulus : zi[h][v]);
            z = step_modified_barrett(zi[h][v] | 1);
        }
    }
    const bool timer = blockIdx.x == 0 && threadIdx.x == 0;
    uint64_t g0 = 0;
    long long c0 = 0;
    if (timer) {
        g0 = gtimer();
        c0 = clock64();
    }
    long long t = clock64();
    for (uint64_t r = w; r < rows; r += ROWS * nw) {
#pragma unroll
        for (int h = 0; h < ROWS; ++h) {
            const uint64_t rr = r + h * nw;
            if (gap) {
                t += gap;
                long long now = clock64();
                while (now < t) {
                    if (sleep_shift >= 0) __nanosleep((unsigned)((t - now) >> sleep_shift));
                    now = clock64();
                }
            }
            uint64_t b[V];
#pragma unroll
            for (int v = 0; v < V; ++v) {
                if (KIND == 1) {
                    b[v] = zi[h][v];
                    zi[h][v] = mul_barrett(zi[h][v], kS.c, kS.shoup);
                } else if (KIND == 2) {
                    b[v] = (uint64_t)__double_as_longlong(__dmul_rn(fp64_canonical(zd[h][v]), kInvModulus));
                    zd[h][v] = mul_fp64(zd[h][v], kS.cb, kS.com);
                } else {
                    b[v] = __float_as_uint(f32_rz_from_unit(__dmul_rn(fp64_canonical(zd[h][v]), kInvModulus)));
                    zd[h][v] = mul_fp64(zd[h][v], kS.cb, kS.com);
                }
            }
            uint64_t q[4];
            if (V == 4) {
                for (int i = 0; i < 4; ++i) q[i] = b[i];
            } else {
                for (int i = 0; i < 4; ++i) q[i] = b[2 * i] | (b[2 * i + 1] << 32);
            }
            if (rr < rows)
                asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(out + rr * 1024 + lane * 32),
                             "l"(q[0]), "l"(q[1]), "l"(q[2]), "l"(q[3])
                             : "memory");
        }
    }
    if (timer) {
        g_clk[0] = gtimer() - g0;
        g_clk[1] = clock64() - c0;
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
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    char* buf;
    CK(cudaMalloc(&buf, bytes));
    const char* names[4] = {"", "u64_barrett", "f64_fp64", "f32_fp64"};
    for (int kind = 1; kind <= 3; ++kind) {
        for (int rows_per_it : {1, 2}) {
            for (int cps : {2, 3, 4}) {
                const int grid = sms * cps;
                const uint64_t nwarps = (uint64_t)grid * 8;
                const uint64_t step_elems = (kind == 3 ? 256ull : 128ull) * nwarps;
                const Mult kS = host_make_mult(host_jump(step_elems * rows_per_it));
                for (int sleep_shift : {-1, 2}) {
                    for (double tbs : {0.0, 7.0, 7.2, 7.4, 7.6, 7.8}) {
                        const long long gap =
                            tbs == 0.0 ? 0 : (long long)(nwarps * 1024.0 * 1.965e9 / (tbs * 1e12) / sms * sms);
                        float ms = time_ms([&] {
#define L(K)                                                                                                  \
    if (rows_per_it == 1)                                                                                     \
        k_fill<K, 1><<<grid, 256>>>(buf, rows, gap, sleep_shift, kS, 12345);                                  \
    else                                                                                                      \
        k_fill<K, 2><<<grid, 256>>>(buf, rows, gap, sleep_shift, kS, 12345);
                            switch (kind) {
                                case 1: L(1) break;
                                case 2: L(2) break;
                                default: L(3) break;
                            }
                        }, 7);
                        unsigned long long clk[2];
                        CK(cudaMemcpyFromSymbol(clk, g_clk, sizeof clk));
                        const double sm_mhz = clk[0] ? 1e3 * clk[1] / (double)clk[0] : 0;
                        const double nbytes = kind == 3 ? bytes : bytes;
                        printf("{\"kind\":\"%s\",\"rows_per_it\":%d,\"ctas_per_sm\":%d,\"sleep\":%d,\"target_tbs\":%.1f,"
                               "\"ms\":%.4f,\"gbs\":%.1f,\"sm_mhz\":%.0f}\n",
                               names[kind], rows_per_it, cps, sleep_shift, tbs, ms, nbytes / ms / 1e6, sm_mhz);
                        fflush(stdout);
                    }
                }
            }
        }
    }
    return 0;
}
