// Does compute-sanitizer synccheck accept a named barrier reached from two
// different code locations (pacer warp vs worker warps)? Variant 0: separate
// bar.sync instructions per role (k_fill_paced today); variant 1: one common
// bar.sync at the end of each round.
#include <cuda_runtime.h>
#include <cstdio>

__global__ void k_split(int rounds, int* out) {
    const int warp = threadIdx.x >> 5;
    if (warp == 8) {
        for (int k = 0; k < rounds; ++k) {
            __syncwarp();
            asm volatile("bar.sync 1, 288;" ::: "memory");
        }
        return;
    }
    int acc = 0;
    for (int k = 0; k < rounds; ++k) {
        acc += k * threadIdx.x;
        asm volatile("bar.sync 1, 288;" ::: "memory");
        out[blockIdx.x * 256 + threadIdx.x] = acc;
    }
}

__global__ void k_common(int rounds, int* out) {
    const int warp = threadIdx.x >> 5;
    int acc = 0;
    for (int k = 0; k < rounds; ++k) {
        if (warp != 8) acc += k * threadIdx.x;
        __syncwarp();
        asm volatile("bar.sync 1, 288;" ::: "memory");
        if (warp != 8) out[blockIdx.x * 256 + threadIdx.x] = acc;
    }
}

int main(int argc, char** argv) {
    int* out;
    cudaMalloc(&out, 64 * 256 * sizeof(int));
    const int v = argc > 1 ? argv[1][0] - '0' : 0;
    if (v == 0) k_split<<<64, 288>>>(5, out);
    else k_common<<<64, 288>>>(5, out);
    cudaError_t e = cudaDeviceSynchronize();
    std::printf("variant %d: %s\n", v, cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 1;
}
