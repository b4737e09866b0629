#pragma once

// B200 drop-in for the reference header of the same name
// (/root/reference/proj/include/bcnrand/oracle.hpp, src/oracle.cpp:16-52):
// the reference's ground-truth mathematics, independent of the generator —
// the truncated fractional expansion of alpha_{2,3} = sum_k 1/(3^k 2^(3^k))
// and brute-force multiplicative orders modulo small powers of three. Host
// only and header-only; nothing on the fill path calls it (it exists so code
// and tests written against the reference's API, e.g. its
// tests/test_oracle.cpp, keep working). Not to be confused with this repo's
// own CPU checker under oracle/.

#include <cstdint>
#include <stdexcept>

namespace bcn::oracle {

// oracle.hpp: numerator / 3^denominator_power.
struct AlphaFraction {
    std::uint64_t numerator = 0;
    int denominator_power = 0;
};

// 3^j for j in [0, 33]; otherwise std::invalid_argument.
inline std::uint64_t pow3(int j) {
    if (j < 0 || j > 33) throw std::invalid_argument("pow3: exponent outside [0, 33]");
    std::uint64_t p = 1;
    for (int i = 0; i < j; ++i) p *= 3;
    return p;
}

namespace detail {
inline std::uint64_t mulmod(std::uint64_t a, std::uint64_t b, std::uint64_t m) {
    return static_cast<std::uint64_t>(static_cast<unsigned __int128>(a) * b % m);
}
inline std::uint64_t pow2_mod(std::uint64_t e, std::uint64_t m) {
    std::uint64_t r = 1 % m, b = 2 % m;
    for (; e; e >>= 1, b = mulmod(b, b, m))
        if (e & 1) r = mulmod(r, b, m);
    return r;
}
}  // namespace detail

// Fractional part of 2^n * alpha truncated to `terms` series terms, as a
// numerator over 3^terms: sum_{k=1..terms} (2^(n - 3^k) mod 3^k) 3^(terms-k)
// mod 3^terms. Requires 1 <= terms <= 33 and n > 3^terms (every retained
// exponent positive); otherwise std::invalid_argument.
inline AlphaFraction alpha_fraction(std::uint64_t n, int terms) {
    if (terms < 1 || terms > 33) throw std::invalid_argument("alpha_fraction: terms outside [1, 33]");
    const std::uint64_t top = pow3(terms);
    if (n <= top) throw std::invalid_argument("alpha_fraction: n must exceed 3^terms");
    std::uint64_t acc = 0;
    for (int k = 1; k <= terms; ++k) {
        const std::uint64_t mk = pow3(k);
        const std::uint64_t digit = detail::pow2_mod(n - mk, mk);  // 2^(n-3^k) mod 3^k
        acc = (acc + detail::mulmod(digit, pow3(terms - k), top)) % top;
    }
    return AlphaFraction{acc, terms};
}

// Least t > 0 with (2^base_exponent)^t == 1 (mod 3^modulus_power), by direct
// iteration; modulus_power in [2, 13], otherwise std::invalid_argument.
inline std::uint64_t multiplicative_order(unsigned base_exponent, int modulus_power) {
    if (modulus_power < 2 || modulus_power > 13)
        throw std::invalid_argument("multiplicative_order: modulus power outside [2, 13]");
    const std::uint64_t m = pow3(modulus_power);
    const std::uint64_t g = detail::pow2_mod(base_exponent, m);
    std::uint64_t x = g, t = 1;
    while (x != 1) {
        x = detail::mulmod(x, g, m);
        ++t;
    }
    return t;
}

}  // namespace bcn::oracle
