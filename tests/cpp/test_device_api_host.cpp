// Host-side checks of include/bcnrand_device.cuh compiled as plain C++ (no
// GPU): the Barrett mulmod against exact 128-bit arithmetic on edge and random
// operands, the step against the paper's recurrence, and state_at / skip
// against sequential stepping and the reference goldens
// (test_generator.cpp:13-17). Prints "[device-api-host] ok" on success.
#include <cstdint>
#include <cstdio>
#include <random>

#include "bcnrand_device.cuh"

namespace {
int failures = 0;
void check(bool ok, const char* what, uint64_t a = 0, uint64_t b = 0) {
    if (!ok && failures++ < 10) std::printf("FAILED: %s (%llu, %llu)\n", what, (unsigned long long)a, (unsigned long long)b);
}
uint64_t ref_mulmod(uint64_t a, uint64_t b) {
    return static_cast<uint64_t>(static_cast<unsigned __int128>(a) * b % bcn::dev::kModulus);
}
}  // namespace

int main() {
    using namespace bcn::dev;
    const uint64_t m = kModulus;
    const uint64_t edges[] = {0, 1, 2, 3, m / 2, m / 2 + 1, m - 3, m - 2, m - 1, 1ull << 52, (1ull << 52) - 1,
                              m / 3, 2 * (m / 3), 3706040377703682ull, 4258649398211344ull};
    for (uint64_t a : edges)
        for (uint64_t b : edges)
            if (a < m && b < m) check(mulmod(a, b) == ref_mulmod(a, b), "mulmod edge", a, b);
    std::mt19937_64 rng(0x12061187);
    for (int i = 0; i < 20000000; ++i) {
        const uint64_t a = rng() % m, b = rng() % m;
        check(mulmod(a, b) == ref_mulmod(a, b), "mulmod random", a, b);
    }
    // products near multiples of m: a = k, b = m - small
    for (uint64_t k = 1; k < 200000; ++k) {
        const uint64_t b = m - 1 - (k % 7);
        check(mulmod(k, b) == ref_mulmod(k, b), "mulmod near-multiple", k, b);
    }
    // step == 2^53 z mod m
    for (int i = 0; i < 2000000; ++i) {
        const uint64_t z = 1 + rng() % (m - 1);
        check(step(z) == ref_mulmod(z, (1ull << 53) % m), "step", z);
    }
    // goldens (test_generator.cpp:13-17) and skip-ahead
    const uint64_t a0 = kMinSeedIndex;
    check(seed_from_index(a0).z == 4258649398211344ull, "z0(a0)");
    check(state_at(a0, 1).z == 2138759898642167ull, "z1");
    check(state_at(a0, 1000).z == 5492007519572011ull, "z1000");
    check(seed_from_index(kMaxSeedIndex).z == 1895384862748766ull, "z0(2^53)");
    Stream s = seed_from_index(a0);
    for (int i = 0; i < 1000; ++i) s.next();
    check(s.z == 5492007519572011ull, "1000 steps");
    for (int i = 0; i < 2000; ++i) {
        const uint64_t a = a0 + rng() % ((1ull << 53) - a0 + 1);
        const uint64_t k = rng();
        Stream t = state_at(a, k);
        Stream u = state_at(a, k - 17);
        u.skip(17);
        check(t.z == u.z, "skip composes", a, k);
        Stream v = state_at(a, k);
        for (int j = 0; j < 5; ++j) v.next();
        check(v.z == state_at(a, k + 5).z, "state_at vs next", a, k);
    }
    check(state_at(a0, kPeriod).z == seed_from_index(a0).z, "period");
    if (failures) {
        std::printf("[device-api-host] %d failures\n", failures);
        return 1;
    }
    std::printf("[device-api-host] ok\n");
    return 0;
}
