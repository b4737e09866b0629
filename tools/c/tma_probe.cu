// TMA 2D load probe (exploration): encodes a u32 [256 x 256] map and loads one
// 32 x 32 box into shared memory, variants by argv[1]:
//   0: SWIZZLE_NONE, __grid_constant__ map   1: SWIZZLE_128B, __grid_constant__ map
//   2: SWIZZLE_128B, map in global memory    3: as 1 with the smem dst 1024-aligned by __align__
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

using Enc = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                         const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                         CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ void body(uint64_t desc, uint32_t* out, int x0) {
    __shared__ __align__(1024) uint32_t tile[32 * 32];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(4096));
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(su(tile)), "l"(desc), "r"(x0), "r"(64), "r"(su(&bar)) : "memory");
    }
    asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(su(&bar)));
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = tile[i];
}
__global__ void k_param(const __grid_constant__ CUtensorMap m, uint32_t* out, int x0) { body(reinterpret_cast<uint64_t>(&m), out, x0); }
__global__ void k_global(const CUtensorMap* m, uint32_t* out, int x0) { body(reinterpret_cast<uint64_t>(m), out, x0); }

int main(int argc, char** argv) {
    int v = argc > 1 ? atoi(argv[1]) : 0;
    int x0 = argc > 2 ? atoi(argv[2]) : 32;
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    printf("entry point %p q=%d\n", fn, (int)q);
    uint32_t* src; uint32_t* out;
    cudaMalloc(&src, 256 * 256 * 4); cudaMalloc(&out, 4096);
    uint32_t* h = (uint32_t*)malloc(256 * 256 * 4);
    for (int i = 0; i < 65536; ++i) h[i] = i;
    cudaMemcpy(src, h, 256 * 256 * 4, cudaMemcpyHostToDevice);
    CUtensorMap m;
    cuuint64_t dims[2] = {256, 256}, strides[1] = {1024};
    cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
    CUresult r = ((Enc)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           v == 0 ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    if (v == 2) {
        CUtensorMap* dm; cudaMalloc(&dm, sizeof(m)); cudaMemcpy(dm, &m, sizeof(m), cudaMemcpyHostToDevice);
        k_global<<<1, 128>>>(dm, out, x0);
    } else {
        k_param<<<1, 128>>>(m, out, x0);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("variant %d x0 %d: %s\n", v, x0, cudaGetErrorString(e));
    uint32_t o[1024];
    cudaMemcpy(o, out, 4096, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int r2 = 0; r2 < 32; ++r2) for (int c = 0; c < 32; ++c) {
        int chunk = c / 4, pos = v == 0 ? r2 * 32 + c : r2 * 32 + ((chunk ^ (r2 & 7)) * 4) + c % 4;
        if (o[pos] != (uint32_t)((64 + r2) * 256 + x0 + c)) ++bad;
    }
    printf("variant %d: %d mismatches\n", v, bad);
    return 0;
}
