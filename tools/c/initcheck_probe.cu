// Does compute-sanitizer initcheck see 256-bit stores (st.global.v4.b64,
// SASS STG.E.256)? Buffer A is written with 256-bit stores, buffer B with
// 64-bit stores; both are then copied to the host.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__global__ void k256(uint64_t* p, int n4) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n4)
        asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p + 4 * t), "l"(1ull * t), "l"(2ull),
                     "l"(3ull), "l"(4ull)
                     : "memory");
}

__global__ void k64(uint64_t* p, int n) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) p[t] = t;
}

int main() {
    const int n = 1 << 16;
    uint64_t *a, *b;
    cudaMalloc(&a, n * 8);
    cudaMalloc(&b, n * 8);
    k256<<<n / 4 / 256, 256>>>(a, n / 4);
    k64<<<n / 256, 256>>>(b, n);
    static uint64_t h[1 << 16];
    cudaMemcpy(h, b, n * 8, cudaMemcpyDeviceToHost);
    std::printf("64-bit buffer copied\n");
    cudaMemcpy(h, a, n * 8, cudaMemcpyDeviceToHost);
    std::printf("256-bit buffer copied (h[4] = %llu)\n", (unsigned long long)h[4]);
    return 0;
}
