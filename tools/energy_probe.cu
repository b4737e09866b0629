// energy_probe.cu — sustained throughput and board power of single
// instruction classes (exploration tool): DFMA, DMUL+FRND (cvt.rni.f64),
// IMAD (32-bit), IMAD.WIDE (u64 mul.lo), LOP3/IADD (ALU), FFMA. Each kernel
// runs ~2 s of back-to-back launches; power is sampled with NVML by the host.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o energy_probe tools/energy_probe.cu -lnvidia-ml
#include <cuda_runtime.h>
#include <nvml.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <thread>
#include <vector>

constexpr int kIters = 4096;
constexpr int kChains = 8;

template <int KIND>
__global__ void __launch_bounds__(256) k_ops(unsigned long long* sink, double seed) {
    double d[kChains];
    uint64_t u[kChains];
    float f[kChains];
    for (int c = 0; c < kChains; ++c) {
        d[c] = seed + threadIdx.x + c;
        u[c] = static_cast<uint64_t>(seed) * 2654435761u + threadIdx.x * 97 + c;
        f[c] = static_cast<float>(seed) + c;
    }
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            if (KIND == 0) d[c] = __fma_rn(d[c], 0.999999999, 1e-9);                       // DFMA
            if (KIND == 1) d[c] = __dmul_rn(rint(d[c] * 1.0000001), 0.9999999);             // DMUL+FRND+DMUL
            if (KIND == 2) u[c] = static_cast<uint32_t>(u[c]) * 2654435761u + 12345u;       // IMAD 32
            if (KIND == 3) u[c] = u[c] * 0x9E3779B97F4A7C15ull + 1;                         // u64 mul.lo
            if (KIND == 4) u[c] = (u[c] ^ (u[c] >> 7)) + 0x3C6EF372u;                        // ALU
            if (KIND == 5) f[c] = __fmaf_rn(f[c], 0.9999999f, 1e-7f);                        // FFMA
        }
    }
    unsigned long long acc = 0;
    for (int c = 0; c < kChains; ++c)
        acc += static_cast<unsigned long long>(d[c]) + u[c] + static_cast<unsigned long long>(f[c]);
    if (acc == 42) sink[0] = acc;
}

int main() {
    nvmlInit();
    nvmlDevice_t h;
    nvmlDeviceGetHandleByIndex(0, &h);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * 8;
    const char* names[6] = {"dfma", "dmul_frnd_dmul", "imad32", "mul_lo_u64", "alu_xor_shift_add", "ffma"};
    // SASS instructions per chain step (approx, see cuobjdump): 1, 3, 1, 3, 3, 1
    for (int kind = 0; kind < 6; ++kind) {
        auto launch = [&] {
            switch (kind) {
                case 0: k_ops<0><<<grid, 256>>>(sink, 1.5); break;
                case 1: k_ops<1><<<grid, 256>>>(sink, 1.5); break;
                case 2: k_ops<2><<<grid, 256>>>(sink, 1.5); break;
                case 3: k_ops<3><<<grid, 256>>>(sink, 1.5); break;
                case 4: k_ops<4><<<grid, 256>>>(sink, 1.5); break;
                default: k_ops<5><<<grid, 256>>>(sink, 1.5); break;
            }
        };
        launch();
        cudaDeviceSynchronize();
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        std::vector<unsigned> pw, clk;
        const auto t_end = std::chrono::steady_clock::now() + std::chrono::milliseconds(2500);
        int launches = 0;
        float ms_total = 0;
        while (std::chrono::steady_clock::now() < t_end) {
            cudaEventRecord(a);
            for (int r = 0; r < 10; ++r) launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (std::chrono::steady_clock::now() > t_end - std::chrono::milliseconds(1200)) {
                ms_total += ms;
                launches += 10;
                unsigned p, c;
                nvmlDeviceGetPowerUsage(h, &p);
                nvmlDeviceGetClockInfo(h, NVML_CLOCK_SM, &c);
                pw.push_back(p);
                clk.push_back(c);
            }
        }
        double pmean = 0, cmean = 0;
        for (size_t i = 0; i < pw.size(); ++i) {
            pmean += pw[i];
            cmean += clk[i];
        }
        pmean /= pw.size() * 1000.0;
        cmean /= clk.size();
        const double steps = static_cast<double>(grid) * 256 * kIters * kChains * launches;
        const double rate = steps / (ms_total * 1e-3);
        printf("{\"kind\":\"%s\",\"chain_steps_per_s\":%.4g,\"power_w\":%.1f,\"sm_mhz\":%.0f,\"nJ_per_1e3_steps\":%.4f}\n",
               names[kind], rate, pmean, cmean, pmean / rate * 1e12);
        fflush(stdout);
        std::this_thread::sleep_for(std::chrono::milliseconds(1500));
    }
    // idle power reference
    std::this_thread::sleep_for(std::chrono::milliseconds(1000));
    unsigned p;
    nvmlDeviceGetPowerUsage(h, &p);
    printf("{\"kind\":\"idle\",\"power_w\":%.1f}\n", p / 1000.0);
    return 0;
}
