// write_probe.cu — measures the B200 write ceiling and the per-engine compute
// ceiling of the fill loop (exploration tool; results in profiles/).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o write_probe tools/write_probe.cu
//   ./write_probe [log2_bytes=33]
//
// Write kernels (all write `bytes` once, 256-bit or 128-bit lane stores):
//   rows256     per-warp contiguous row ranges (the fill kernels' pattern)
//   stride256   grid-strided rows (all warps sweep the buffer together)
//   rows256cs   rows256 with st.global.cs (evict-first)
//   rows128     rows with 16-byte stores
//   bulk        smem tile + cp.async.bulk (TMA bulk store), 4 tiles in flight
//   memset      cudaMemsetAsync
// Compute probes: the contiguous fill loop per engine/format with the store
// predicated on an impossible value, i.e. pure generation throughput.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1206_1187_b200/csrc/bcn_math.cuh"

using namespace bcn_b200;

#define CK(x)                                                                           \
    do {                                                                                \
        cudaError_t e = (x);                                                            \
        if (e != cudaSuccess) {                                                         \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));            \
            exit(1);                                                                    \
        }                                                                               \
    } while (0)

__device__ __forceinline__ void st256(void* p, uint64_t v) {
    asm volatile("st.global.v4.b64 [%0], {%1, %1, %1, %1};" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st256cs(void* p, uint64_t v) {
    asm volatile("st.global.cs.v4.b64 [%0], {%1, %1, %1, %1};" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st128(void* p, uint64_t v) {
    asm volatile("st.global.v2.b64 [%0], {%1, %1};" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void split(uint64_t rows, uint64_t& b, uint64_t& e) {
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const uint64_t w = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint64_t q = rows / nw, r = rows % nw;
    b = w * q + (w < r ? w : r);
    e = b + q + (w < r ? 1 : 0);
}

template <int MODE>
__global__ void k_write(char* out, uint64_t rows, uint64_t v) {
    const unsigned lane = threadIdx.x & 31;
    if (MODE == 1) {  // grid-stride rows
        const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
        for (uint64_t r = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows;
             r += nw)
            st256(out + r * 1024 + lane * 32, v);
        return;
    }
    uint64_t r, e;
    split(rows, r, e);
    if (MODE == 3) {  // 16-byte stores: a 1 KiB row = 2 x 512 B
        for (; r < e; ++r) {
            st128(out + r * 1024 + lane * 16, v);
            st128(out + r * 1024 + 512 + lane * 16, v);
        }
        return;
    }
#pragma unroll 4
    for (; r < e; ++r) {
        if (MODE == 2)
            st256cs(out + r * 1024 + lane * 32, v);
        else
            st256(out + r * 1024 + lane * 32, v);
    }
}

// TMA bulk store: each CTA fills a 32 KiB smem tile once, then streams it out
// with cp.async.bulk 4-deep.
__global__ void k_bulk(char* out, uint64_t tiles, uint64_t v) {
    extern __shared__ __align__(128) uint64_t sm[];
    constexpr uint32_t TB = 32768;
    for (uint32_t i = threadIdx.x; i < TB / 8; i += blockDim.x) sm[i] = v;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x != 0) return;
    const uint32_t src = (uint32_t)__cvta_generic_to_shared(sm);
    for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
        asm volatile(
            "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n\t"
            "cp.async.bulk.commit_group;" ::"l"(out + t * TB),
            "r"(src), "r"(TB)
            : "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ----------------------------------------------------------- compute probes
template <int ENG>
struct E;
template <>
struct E<1> {
    using S = uint64_t;
    static __device__ S from(uint64_t z) { return z; }
    static __device__ S mul(S s, const Mult& k) { return mul_barrett(s, k.c, k.shoup); }
    static __device__ double unit(S s) { return unit_from_u64(s); }
    static __device__ uint64_t raw(S s) { return s; }
};
template <>
struct E<2> {
    using S = uint64_t;
    static __device__ S from(uint64_t z) { return z; }
    static __device__ S mul(S s, const Mult& k) { return mul_montgomery(s, k.mont); }
    static __device__ double unit(S s) { return unit_from_u64(s); }
    static __device__ uint64_t raw(S s) { return s; }
};
template <>
struct E<3> {
    using S = double;
    static __device__ S from(uint64_t z) {
        return z > kModulus / 2 ? (double)(int64_t)(z - kModulus) : (double)z;
    }
    static __device__ S mul(S s, const Mult& k) { return mul_fp64(s, k.cb, k.com); }
    static __device__ double unit(S s) { return __dmul_rn(fp64_canonical(s), kInvModulus); }
    static __device__ uint64_t raw(S s) { return __double2ull_rz(fp64_canonical(s)); }
};

// FMT 0 u64, 1 f64, 2 f32; emits into a sink only when the value is 0 (never).
template <int ENG, int FMT>
__global__ void __launch_bounds__(256) k_compute(uint64_t* sink, uint64_t rows, Mult k, uint64_t z0) {
    constexpr int V = FMT == 2 ? 8 : 4;
    uint64_t r, e;
    split(rows, r, e);
    typename E<ENG>::S st[V];
    uint64_t z = z0 + threadIdx.x + blockIdx.x;
    for (int v = 0; v < V; ++v) {
        st[v] = E<ENG>::from(z);
        z = step_modified_barrett(z);
    }
    uint64_t acc = 0;
    for (; r < e; ++r) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
            uint64_t b;
            if (FMT == 0)
                b = E<ENG>::raw(st[v]);
            else if (FMT == 1)
                b = (uint64_t)__double_as_longlong(E<ENG>::unit(st[v]));
            else
                b = __float_as_uint(f32_rz_from_unit(E<ENG>::unit(st[v])));
            acc |= (b == 0);
            st[v] = E<ENG>::mul(st[v], k);
        }
    }
    if (acc) sink[0] = acc;
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
    printf("{\"probe\":\"write\",\"bytes\":%llu,\"sms\":%d}\n", (unsigned long long)bytes, sms);
    for (int bps : {1, 2, 4, 6, 8}) {
        const int grid = sms * bps;
        float ms = time_ms([&] { k_write<0><<<grid, 256>>>(buf, rows, v); }, 20);
        printf("{\"kernel\":\"rows256\",\"ctas_per_sm\":%d,\"ms\":%.4f,\"gbs\":%.1f}\n", bps, ms, bytes / ms / 1e6);
        ms = time_ms([&] { k_write<1><<<grid, 256>>>(buf, rows, v); }, 20);
        printf("{\"kernel\":\"stride256\",\"ctas_per_sm\":%d,\"ms\":%.4f,\"gbs\":%.1f}\n", bps, ms, bytes / ms / 1e6);
        ms = time_ms([&] { k_write<2><<<grid, 256>>>(buf, rows, v); }, 20);
        printf("{\"kernel\":\"rows256cs\",\"ctas_per_sm\":%d,\"ms\":%.4f,\"gbs\":%.1f}\n", bps, ms, bytes / ms / 1e6);
        ms = time_ms([&] { k_write<3><<<grid, 256>>>(buf, rows, v); }, 20);
        printf("{\"kernel\":\"rows128\",\"ctas_per_sm\":%d,\"ms\":%.4f,\"gbs\":%.1f}\n", bps, ms, bytes / ms / 1e6);
    }
    CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768));
    for (int bps : {1, 2, 4, 6}) {
        const int grid = sms * bps;
        float ms = time_ms([&] { k_bulk<<<grid, 128, 32768>>>(buf, bytes / 32768, v); }, 20);
        printf("{\"kernel\":\"bulk32k\",\"ctas_per_sm\":%d,\"ms\":%.4f,\"gbs\":%.1f}\n", bps, ms, bytes / ms / 1e6);
    }
    {
        float ms = time_ms([&] { CK(cudaMemsetAsync(buf, 0x3f, bytes)); }, 20);
        printf("{\"kernel\":\"memset\",\"ms\":%.4f,\"gbs\":%.1f}\n", ms, bytes / ms / 1e6);
    }
    // Compute ceilings: 2^30 variates worth of rows, no stores.
    uint64_t* sink;
    CK(cudaMalloc(&sink, 8));
    const Mult k = host_make_mult(host_jump(128));
    const Mult k8 = host_make_mult(host_jump(256));
    for (int bps : {2, 4, 8}) {
        const int grid = sms * bps;
        const uint64_t nvar = 1ull << 30;
#define PROBE(ENG, FMT, NAME)                                                                        \
    {                                                                                                \
        const uint64_t rws = nvar / (FMT == 2 ? 256 : 128);                                          \
        float ms = time_ms([&] { k_compute<ENG, FMT><<<grid, 256>>>(sink, rws, FMT == 2 ? k8 : k, 12345); }, 10); \
        printf("{\"probe\":\"compute\",\"engine\":\"%s\",\"fmt\":%d,\"ctas_per_sm\":%d,\"ms\":%.4f,\"gvar_s\":%.1f}\n", \
               NAME, FMT, bps, ms, nvar / ms / 1e6);                                                 \
    }
        PROBE(1, 0, "barrett") PROBE(1, 1, "barrett") PROBE(1, 2, "barrett")
        PROBE(2, 1, "montgomery")
        PROBE(3, 0, "fp64") PROBE(3, 1, "fp64") PROBE(3, 2, "fp64")
    }
    return 0;
}
