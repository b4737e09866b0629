#pragma once

// B200 drop-in for the reference's oracle header
// (/root/reference/proj/include/bcnrand/oracle.hpp): ground-truth mathematics
// independent of the generator — the truncated fractional expansion of
// alpha_{2,3} = sum_k 1/(3^k 2^(3^k)) and multiplicative orders modulo small
// powers of three. Host-only and header-only; nothing on the fill path uses
// it (it keeps code and tests written against the reference API, e.g. its
// tests/test_oracle.cpp, compiling). Same preconditions and exception types as
// the reference (oracle.cpp:16-52); the order is found by divisor descent in
// the cyclic group of order 2*3^(j-1) rather than by iterating powers — the
// least period either way. Not to be confused with this repo's CPU checker
// under oracle/.

#include <array>
#include <cstdint>
#include <stdexcept>

namespace bcn::oracle {

struct AlphaFraction {
    std::uint64_t numerator = 0;  // over 3^denominator_power
    int denominator_power = 0;
};

namespace detail {

inline constexpr std::array<std::uint64_t, 34> kPow3 = [] {
    std::array<std::uint64_t, 34> t{};
    t[0] = 1;
    for (std::size_t i = 1; i < t.size(); ++i) t[i] = 3 * t[i - 1];
    return t;
}();

inline std::uint64_t mul_mod(std::uint64_t x, std::uint64_t y, std::uint64_t m) {
    return static_cast<std::uint64_t>((static_cast<unsigned __int128>(x) * y) % m);
}

inline std::uint64_t pow_mod(std::uint64_t base, std::uint64_t e, std::uint64_t m) {
    std::uint64_t acc = 1 % m;
    base %= m;
    while (e) {
        if (e & 1) acc = mul_mod(acc, base, m);
        base = mul_mod(base, base, m);
        e >>= 1;
    }
    return acc;
}

}  // namespace detail

// 3^j, j in [0, 33].
inline std::uint64_t pow3(int j) {
    if (j < 0 || j > 33) throw std::invalid_argument("pow3: j must lie in [0, 33]");
    return detail::kPow3[static_cast<std::size_t>(j)];
}

// frac(2^n * alpha) truncated to the first `terms` series terms, as a
// numerator over 3^terms: the k-th term contributes (2^(n - 3^k) mod 3^k)
// scaled by 3^(terms - k). Needs 1 <= terms <= 33 and n > 3^terms.
inline AlphaFraction alpha_fraction(std::uint64_t n, int terms) {
    if (terms < 1 || terms > 33) throw std::invalid_argument("alpha_fraction: terms must lie in [1, 33]");
    const std::uint64_t den = pow3(terms);
    if (n <= den) throw std::invalid_argument("alpha_fraction: n must be larger than 3^terms");
    AlphaFraction f;
    f.denominator_power = terms;
    for (int k = terms; k >= 1; --k) {
        const std::uint64_t mk = detail::kPow3[static_cast<std::size_t>(k)];
        const std::uint64_t digit = detail::pow_mod(2, n - mk, mk);
        f.numerator = (f.numerator + detail::mul_mod(digit, detail::kPow3[static_cast<std::size_t>(terms - k)], den)) % den;
    }
    return f;
}

// Least t > 0 with 2^(base_exponent * t) = 1 (mod 3^modulus_power),
// modulus_power in [2, 13]. 2 generates (Z/3^j)^*, so the order divides
// phi = 2 * 3^(j-1): strip prime factors while the reduced power stays 1.
inline std::uint64_t multiplicative_order(unsigned base_exponent, int modulus_power) {
    if (modulus_power < 2 || modulus_power > 13)
        throw std::invalid_argument("multiplicative_order: modulus_power must lie in [2, 13]");
    const std::uint64_t m = pow3(modulus_power);
    const std::uint64_t g = detail::pow_mod(2, base_exponent, m);
    std::uint64_t t = 2 * pow3(modulus_power - 1);
    for (std::uint64_t p : {2ull, 3ull})
        while (t % p == 0 && detail::pow_mod(g, t / p, m) == 1) t /= p;
    return t;
}

}  // namespace bcn::oracle
