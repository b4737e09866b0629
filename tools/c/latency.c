/* Per-call cost of bcn_fill for small fills (exploration tool): host enqueue
 * time per call and end-to-end time per call (enqueue + device) for a stream
 * of back-to-back async calls, plus the same for synchronous calls.
 *
 *   make -C tools/c latency && tools/c/latency
 */
#include <cuda_runtime.h>
#include <stdio.h>
#include <time.h>

#include "bcnrand_b200.h"

static double now_us(void) {
    struct timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return t.tv_sec * 1e6 + t.tv_nsec * 1e-3;
}

int main(void) {
    void* d = NULL;
    const uint64_t cap = 1ull << 27;
    if (cudaMalloc(&d, cap * 8) != cudaSuccess) return 1;
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    const uint64_t a0 = 5559060566555523ull + 100;
    const uint64_t sizes[] = {1000, 10000, 100000, 1000000, 10000000, 100000000};
    for (unsigned k = 0; k < sizeof(sizes) / sizeof(sizes[0]); ++k) {
        const uint64_t n = sizes[k];
        const int calls = n >= 10000000 ? 50 : 1000;
        for (int i = 0; i < 10; ++i)
            bcn_fill(d, cap, n, BCN_FORMAT_F64, 1, BCN_LAYOUT_CONTIGUOUS, a0, BCN_METHOD_BARRETT_MODIFIED,
                     (uint64_t)i * n, BCN_ENGINE_AUTO, 0, s);
        cudaStreamSynchronize(s);
        double t0 = now_us();
        for (int i = 0; i < calls; ++i)
            if (bcn_fill(d, cap, n, BCN_FORMAT_F64, 1, BCN_LAYOUT_CONTIGUOUS, a0, BCN_METHOD_BARRETT_MODIFIED,
                         (uint64_t)i * n, BCN_ENGINE_AUTO, 0, s)) {
                printf("error: %s\n", bcn_last_error());
                return 1;
            }
        double t1 = now_us();
        cudaStreamSynchronize(s);
        double t2 = now_us();
        for (int i = 0; i < calls / 10; ++i)
            bcn_fill(d, cap, n, BCN_FORMAT_F64, 1, BCN_LAYOUT_CONTIGUOUS, a0, BCN_METHOD_BARRETT_MODIFIED,
                     (uint64_t)i * n, BCN_ENGINE_AUTO, 0, NULL);
        double t3 = now_us();
        printf("{\"n\": %llu, \"enqueue_us\": %.2f, \"async_us_per_call\": %.2f, \"sync_us_per_call\": %.2f, "
               "\"async_gvariates_s\": %.2f}\n",
               (unsigned long long)n, (t1 - t0) / calls, (t2 - t0) / calls, (t3 - t2) / (calls / 10),
               n * calls / (t2 - t0) * 1e-3);
        fflush(stdout);
    }
    return 0;
}
