// bcnrand_device.cuh — header-only device API of the alpha_{2,3} generator
// for generate-and-consume inside user kernels ("the generated random numbers
// need not be stored in memory").
//
//   #include "bcnrand_device.cuh"
//   __global__ void k(...) {
//       bcn::dev::Stream s = bcn::dev::state_at(seed_index, k0 + tid * 4096);  // skip-ahead
//       for (int i = 0; i < 4096; ++i) use(s.next_unit());   // == par::fill element k0+tid*4096+i
//   }
//
// Semantics match the reference exactly: Stream{z} holds the state of
// gen::GeneratorState (generator.hpp:24-29); next() is gen::next with the
// modified Barrett step (modred.hpp:149-159, the paper's Fig. 3); next_unit()
// is to_unit_interval(next()) (generator.hpp:74-78); state_at(a, k) equals
// gen::state_at (generator.cpp:42-49), computed from the closed form
// z_k = m - 2^((a - 3^33 - 1 + 53 k) mod P) mod m with a square-and-multiply
// over exact products reduced by a 128-bit Barrett step (no tables, no host
// set-up, no 128-bit division). Seeds out of range are the caller's
// responsibility (validate on the host with bcn_seed_from_index).
//
// The header also compiles as plain C++ (host only), which is how the CPU
// test suite checks its arithmetic (tests/cpp/test_device_api_host.cpp).
#pragma once

#include <cstdint>

#if !defined(__CUDACC__)
#ifndef __host__
#define __host__
#endif
#ifndef __device__
#define __device__
#endif
#ifndef __forceinline__
#define __forceinline__ inline
#endif
#endif

namespace bcn {
namespace dev {

constexpr uint64_t kModulus = 5559060566555523ull;  // 3^33
constexpr uint64_t kPeriod = 3706040377703682ull;   // 2 * 3^32
constexpr uint64_t kMu = 0x33D9481681D79Dull;       // floor(2^106 / m)
constexpr uint64_t kMinSeedIndex = kModulus + 100;
constexpr uint64_t kMaxSeedIndex = 1ull << 53;

__host__ __device__ __forceinline__ uint64_t umulhi(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
    return __umul64hi(a, b);
#else
    return static_cast<uint64_t>((static_cast<unsigned __int128>(a) * b) >> 64);
#endif
}

// a b mod m for a, b < m by a Barrett step on the 105-bit product x = a b:
// q = floor(floor(x / 2^51) mu / 2^55) with mu = floor(2^106 / m). Writing
// x = x1 2^51 + x0 and mu = 2^106/m - d (0 <= d < 1),
//     x/m - x1 mu / 2^55 = x0/m + x1 d / 2^55 < 2^51/m + 2^53.6/2^55 < 0.8,
// so q is floor(x/m) or one less, r = x - q m lies in [0, 2m) (exact mod
// 2^64) and one conditional subtract finishes. ~20 integer instructions
// instead of a software 128-bit division.
__host__ __device__ __forceinline__ uint64_t mulmod(uint64_t a, uint64_t b) {
    const uint64_t lo = a * b, hi = umulhi(a, b);
    const uint64_t x1 = (hi << 13) | (lo >> 51);  // floor(x / 2^51) < 2^54
    const uint64_t q = (umulhi(x1, kMu) << 9) | ((x1 * kMu) >> 55);
    const uint64_t r = lo - q * kModulus;
    return r >= kModulus ? r - kModulus : r;
}

// 2^e mod m by square-and-multiply (generator.cpp:17-30 restated).
__host__ __device__ inline uint64_t pow2(uint64_t e) {
    e %= kPeriod;
    uint64_t r = 1, b = 2;
    while (e) {
        if (e & 1) r = mulmod(r, b);
        b = mulmod(b, b);
        e >>= 1;
    }
    return r;
}

// The paper's modified Barrett step z -> 2^53 z mod m, valid on [1, m).
__host__ __device__ __forceinline__ uint64_t step(uint64_t z) {
    const uint64_t hi = umulhi(z, kMu);
    const uint64_t lo = z * kMu;
    const uint64_t q3 = (hi << 11) | (lo >> 53);
    const uint64_t r = 0x20000000000000ull - ((q3 * kModulus) & 0x1FFFFFFFFFFFFFull);
    return r >= kModulus ? r - kModulus : r;
}

struct Stream {
    uint64_t z;  // current iterate (gen::GeneratorState::z)

    // gen::next: advance one step, return the new residue.
    __host__ __device__ __forceinline__ uint64_t next() { return z = step(z); }
    // to_unit_interval(next()): one RN multiply of the exact double.
    __host__ __device__ __forceinline__ double next_unit() {
        return static_cast<double>(next()) * (1.0 / 5559060566555523.0);
    }
    // Skip `k` further steps in O(log k).
    __host__ __device__ inline void skip(uint64_t k) {
        z = mulmod(z, pow2(static_cast<uint64_t>(
                          static_cast<unsigned __int128>(k % kPeriod) * 53u % kPeriod)));
    }
};

// gen::seed_from_index(a) (a in [kMinSeedIndex, kMaxSeedIndex]).
__host__ __device__ inline Stream seed_from_index(uint64_t a) {
    return Stream{kModulus - pow2(a - kModulus - 1)};
}

// gen::state_at(a, k): the state after k steps from seed_from_index(a).
__host__ __device__ inline Stream state_at(uint64_t a, uint64_t k) {
    const uint64_t e = ((a - kModulus - 1) % kPeriod +
                        static_cast<uint64_t>(static_cast<unsigned __int128>(k % kPeriod) * 53u % kPeriod)) %
                       kPeriod;
    return Stream{kModulus - pow2(e)};
}

}  // namespace dev
}  // namespace bcn
