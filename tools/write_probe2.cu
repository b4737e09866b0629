// write_probe2.cu — what limits SM-issued HBM writes below cudaMemset's rate?
// (exploration tool; results summarised in profiles/ and DESIGN.md §5)
//
// Variants: grid size below the SM count, L2 cache-policy hints on the stores,
// TMA bulk stores of several sizes / depths, memset flavours.
#include <cuda.h>
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

__device__ __forceinline__ void split(uint64_t rows, uint64_t& b, uint64_t& e) {
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const uint64_t w = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint64_t q = rows / nw, r = rows % nw;
    b = w * q + (w < r ? w : r);
    e = b + q + (w < r ? 1 : 0);
}

// MODE 0 plain, 1 L2::evict_first policy, 2 L2::evict_last, 3 L1::no_allocate,
// 4 evict_unchanged, 5 grid-stride plain
template <int MODE>
__global__ void k_write(char* out, uint64_t rows, uint64_t v) {
    const unsigned lane = threadIdx.x & 31;
    uint64_t pol = 0;
    if (MODE == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    if (MODE == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    if (MODE == 4) asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(pol));
    uint64_t r, e;
    if (MODE == 5) {
        const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
        for (r = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += nw)
            asm volatile("st.global.v4.b64 [%0], {%1, %1, %1, %1};" ::"l"(out + r * 1024 + lane * 32), "l"(v) : "memory");
        return;
    }
    split(rows, r, e);
#pragma unroll 4
    for (; r < e; ++r) {
        char* p = out + r * 1024 + lane * 32;
        if (MODE == 0)
            asm volatile("st.global.v4.b64 [%0], {%1, %1, %1, %1};" ::"l"(p), "l"(v) : "memory");
        else if (MODE == 3)
            asm volatile("st.global.L1::no_allocate.v4.b64 [%0], {%1, %1, %1, %1};" ::"l"(p), "l"(v) : "memory");
        else
            asm volatile("st.global.L2::cache_hint.v4.b64 [%0], {%1, %1, %1, %1}, %2;" ::"l"(p), "l"(v), "l"(pol)
                         : "memory");
    }
}

template <uint32_t TB, int DEPTH>
__global__ void k_bulk(char* out, uint64_t tiles, uint64_t v) {
    extern __shared__ __align__(128) uint64_t sm[];
    for (uint32_t i = threadIdx.x; i < TB / 8; i += blockDim.x) sm[i] = v;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x != 0) return;
    const uint32_t src = (uint32_t)__cvta_generic_to_shared(sm);
    for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(DEPTH - 1) : "memory");
        asm volatile(
            "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n\t"
            "cp.async.bulk.commit_group;" ::"l"(out + t * TB),
            "r"(src), "n"(TB)
            : "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
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

int main(int argc, char** argv) {
    const int lg = argc > 1 ? atoi(argv[1]) : 33;
    const uint64_t bytes = 1ull << lg;
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    char* buf;
    CK(cudaMalloc(&buf, bytes));
    const uint64_t rows = bytes / 1024;
    const uint64_t v = 0x3FE0000000000000ull;
    auto rep = [&](const char* name, int grid, int block, float ms) {
        printf("{\"kernel\":\"%s\",\"grid\":%d,\"block\":%d,\"ms\":%.4f,\"gbs\":%.1f}\n", name, grid, block, ms,
               bytes / ms / 1e6);
    };
    // memset flavours (is it a kernel? ncu will tell)
    rep("memset_d8_0x3f", 0, 0, time_ms([&] { CK(cudaMemsetAsync(buf, 0x3f, bytes)); }, 20));
    rep("memset_d8_0", 0, 0, time_ms([&] { CK(cudaMemsetAsync(buf, 0, bytes)); }, 20));
    rep("memsetD32", 0, 0, time_ms([&] { cuMemsetD32Async((CUdeviceptr)buf, 0x3FE00000u, bytes / 4, 0); }, 20));
    // grid size sweep with 1024-thread CTAs, plain stores
    for (int g : {sms / 4, sms / 2, (3 * sms) / 4, sms, 2 * sms}) {
        rep("rows256_b1024", g, 1024, time_ms([&] { k_write<0><<<g, 1024>>>(buf, rows, v); }, 20));
    }
    for (int bs : {128, 256, 512}) {
        const int g = sms * (2048 / bs);
        rep("rows256", g, bs, time_ms([&] { k_write<0><<<g, bs>>>(buf, rows, v); }, 20));
    }
    const int g = sms * 4;
    rep("evict_first", g, 256, time_ms([&] { k_write<1><<<g, 256>>>(buf, rows, v); }, 20));
    rep("evict_last", g, 256, time_ms([&] { k_write<2><<<g, 256>>>(buf, rows, v); }, 20));
    rep("l1_no_allocate", g, 256, time_ms([&] { k_write<3><<<g, 256>>>(buf, rows, v); }, 20));
    rep("evict_unchanged", g, 256, time_ms([&] { k_write<4><<<g, 256>>>(buf, rows, v); }, 20));
    rep("stride256", g, 256, time_ms([&] { k_write<5><<<g, 256>>>(buf, rows, v); }, 20));
    rep("stride256_1cta", sms, 1024, time_ms([&] { k_write<5><<<sms, 1024>>>(buf, rows, v); }, 20));
#define BULK(TB, D, CPS)                                                                                   \
    {                                                                                                      \
        CK(cudaFuncSetAttribute(k_bulk<TB, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, TB));          \
        const int gg = sms * CPS;                                                                          \
        rep("bulk_" #TB "_d" #D, gg, 128, time_ms([&] { k_bulk<TB, D><<<gg, 128, TB>>>(buf, bytes / TB, v); }, 20)); \
    }
    BULK(16384, 4, 2) BULK(32768, 8, 2) BULK(65536, 4, 1) BULK(65536, 8, 2) BULK(131072, 4, 1)
    BULK(4096, 16, 4) BULK(8192, 16, 4)
    return 0;
}
