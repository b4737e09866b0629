#pragma once

// B200 drop-in for the reference header of the same name
// (/root/reference/proj/include/bcnrand/modred.hpp): the residue type, the
// constant table and its self-check, and the four host step functions of the
// reduction layer (modred.hpp:16-159). On the GPU the step is done by the
// engines behind include/bcnrand_b200.h; these host versions exist so code
// (and tests) written against the reference's modred API keep working. They
// are exact restatements of the reference's arithmetic contracts — every
// function returns (2^53 z) mod m for z in its domain, with the reference's
// preconditions — written independently (128-bit products instead of the
// reference's 32-bit-halves arithmetic).

#include <cstdint>
#include <stdexcept>
#include <string>

namespace bcn {

// modred.hpp:16-18
struct Residue {
    std::uint64_t value = 0;
};

namespace modred {

inline constexpr std::uint64_t kModulus = 5559060566555523ull;  // 3^33
inline constexpr std::uint64_t kTwo53 = std::uint64_t{1} << 53;

// modred.hpp:28-48: the constants every reduction uses.
struct ReductionConstants {
    std::uint64_t m;      // modulus 3^33
    std::uint64_t a_red;  // Schrage multiplier 2^25 (two stages make 2^53 with the 4 and 2 factors)
    std::uint64_t q;      // floor(m / a_red)
    std::uint64_t r;      // m mod a_red
    double qinv;          // 1 / q, for the floating-point quotient of the fast Schrage stage
    std::uint64_t mu;     // floor(2^106 / m), Barrett constant
    int k_bits;           // 53: 2^(k-1) <= m < 2^k
};

constexpr ReductionConstants constants() {
    return ReductionConstants{kModulus,
                              std::uint64_t{1} << 25,
                              kModulus >> 25,
                              kModulus & ((std::uint64_t{1} << 25) - 1),
                              1.0 / static_cast<double>(kModulus >> 25),
                              static_cast<std::uint64_t>((static_cast<unsigned __int128>(1) << 106) / kModulus),
                              53};
}

// High 64 bits of a * b (modred.hpp:57-67).
constexpr std::uint64_t wide_mul_hi(std::uint64_t a, std::uint64_t b) {
    return static_cast<std::uint64_t>((static_cast<unsigned __int128>(a) * b) >> 64);
}

// modred.cpp:27-41: true iff every entry is the value derived from 3^33.
inline bool verify_constants(const ReductionConstants& c) {
    std::uint64_t m = 1;
    for (int i = 0; i < 33; ++i) m *= 3;
    if (c.m != m || c.a_red != (std::uint64_t{1} << 25) || c.k_bits != 53) return false;
    if (c.q != m / c.a_red || c.r != m % c.a_red) return false;
    if (c.qinv != 1.0 / static_cast<double>(c.q)) return false;
    if (c.mu != static_cast<std::uint64_t>((static_cast<unsigned __int128>(1) << 106) / m)) return false;
    const std::uint64_t two_k = std::uint64_t{1} << c.k_bits;
    return m < two_k && two_k < 2 * m && 4 * c.a_red * c.a_red < m;
}

namespace detail {

inline void check_residue(std::uint64_t z, std::uint64_t m, const char* fn) {
    if (z >= m) throw std::domain_error(std::string(fn) + ": residue out of range");
}

// x * a_red mod m for 0 <= x < 4m by Schrage's decomposition m = a q + r
// (r < q): a (x mod q) - r floor(x / q) lies in (-m, a q), folded into [0, m).
// `fast` takes the quotient from the double reciprocal and repairs it.
inline std::uint64_t schrage_times_a(std::uint64_t x, const ReductionConstants& c, bool fast) {
    std::uint64_t t = fast ? static_cast<std::uint64_t>(static_cast<double>(x) * c.qinv) : x / c.q;
    if (fast) {  // repair the floating-point quotient to floor(x / q)
        while (t * c.q > x) --t;
        while ((t + 1) * c.q <= x) ++t;
    }
    const std::int64_t hi = static_cast<std::int64_t>((x - t * c.q) * c.a_red);
    const std::int64_t lo = static_cast<std::int64_t>(t * c.r);
    const auto m = static_cast<std::int64_t>(c.m);
    const std::int64_t v = (hi - lo) % m;
    return static_cast<std::uint64_t>(v < 0 ? v + m : v);
}

}  // namespace detail

// The exact oracle (modred.hpp:103-107): 128-bit product and remainder.
inline Residue reduce_ref(Residue z) {
    detail::check_residue(z.value, kModulus, "reduce_ref");
    return Residue{static_cast<std::uint64_t>((static_cast<unsigned __int128>(z.value) << 53) % kModulus)};
}

// L'Ecuyer / Schrage (modred.hpp:112-124): 2^53 z = 2^25 (2 * 2^25 (4 z)).
inline Residue lecuyer_step(Residue z, const ReductionConstants& c = constants()) {
    detail::check_residue(z.value, c.m, "lecuyer_step");
    const std::uint64_t a = detail::schrage_times_a(4 * z.value, c, false);
    return Residue{detail::schrage_times_a(2 * a, c, false)};
}

inline Residue lecuyer_step_fast(Residue z, const ReductionConstants& c = constants()) {
    detail::check_residue(z.value, c.m, "lecuyer_step_fast");
    const std::uint64_t a = detail::schrage_times_a(4 * z.value, c, true);
    return Residue{detail::schrage_times_a(2 * a, c, true)};
}

// Classic Barrett (modred.hpp:129-143): x = 2^53 z, q = floor(floor(x / 2^(k-1)) mu / 2^(k+1)),
// r = x - q m mod 2^(k+1), at most two corrections.
inline Residue barrett_step(Residue z, const ReductionConstants& c = constants()) {
    detail::check_residue(z.value, c.m, "barrett_step");
    const unsigned __int128 x = static_cast<unsigned __int128>(z.value) << 53;
    const auto x_top = static_cast<std::uint64_t>(x >> (c.k_bits - 1));
    const auto quot = static_cast<std::uint64_t>((static_cast<unsigned __int128>(x_top) * c.mu) >> (c.k_bits + 1));
    const std::uint64_t low_bits = (std::uint64_t{2} << c.k_bits) - 1;
    const std::uint64_t rem = (static_cast<std::uint64_t>(x) - quot * c.m) & low_bits;
    return Residue{rem % c.m};  // the reference's (at most two) corrections
}

// The paper's modified Barrett step (modred.hpp:149-159, Fig. 3):
// q = floor(z mu / 2^53) is floor(2^53 z / m) or one less, and the remainder
// needs only the low 53 bits: r = 2^53 - (q m mod 2^53), one correction.
// z = 0 is outside its domain (modred.hpp:150).
inline Residue barrett_modified_step(Residue z, const ReductionConstants& c = constants()) {
    if (z.value == 0) throw std::domain_error("barrett_modified_step: z = 0 not in domain");
    detail::check_residue(z.value, c.m, "barrett_modified_step");
    const auto quot = static_cast<std::uint64_t>((static_cast<unsigned __int128>(z.value) * c.mu) >> 53);
    const std::uint64_t rem = kTwo53 - ((quot * c.m) & (kTwo53 - 1));
    return Residue{rem >= c.m ? rem - c.m : rem};
}

}  // namespace modred
}  // namespace bcn
