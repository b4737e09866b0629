#pragma once

// B200 drop-in for /root/reference/proj/include/bcnrand/generator.hpp: the
// same names, signatures, argument meaning and exceptions, implemented over
// the C ABI of libbcnrand_b200.so (include/bcnrand_b200.h). Build user code
// with -I<repo>/include and link -lbcnrand_b200 instead of bcnrand_core.

#include <algorithm>
#include <cctype>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "bcnrand/modred.hpp"
#include "bcnrand_b200.h"

namespace bcn {
namespace b200 {

// Re-raises a C-ABI status as the reference's exception type.
inline void check(bcn_status st) {
    switch (st) {
        case BCN_OK: return;
        case BCN_ERR_INVALID_ARGUMENT: throw std::invalid_argument(bcn_last_error());
        case BCN_ERR_OUT_OF_RANGE: throw std::out_of_range(bcn_last_error());
        case BCN_ERR_DOMAIN: throw std::domain_error(bcn_last_error());
        default: throw std::runtime_error(bcn_last_error());
    }
}

}  // namespace b200

namespace gen {

// generator.hpp:17
enum class Method { Ref128, LEcuyer, Barrett, BarrettModified };

// generator.hpp:19-22
inline constexpr std::uint64_t kMinSeedIndex = modred::kModulus + 100;
inline constexpr std::uint64_t kMaxSeedIndex = std::uint64_t{1} << 53;
inline constexpr std::uint64_t kPeriod = 3706040377703682ull;  // 2 * 3^32
inline constexpr double kInvModulus = 1.0 / 5559060566555523.0;

// generator.hpp:24-29
struct GeneratorState {
    std::uint64_t seed_index = 0;
    Residue z;
    std::uint64_t k = 0;
    Method method = Method::BarrettModified;
};

// generator.hpp:33 — 2^e mod `modulus` (odd, below 2^63).
inline std::uint64_t modpow2(std::uint64_t exponent, std::uint64_t modulus) {
    std::uint64_t out = 0;
    b200::check(bcn_modpow2(exponent, modulus, &out));
    return out;
}

// generator.hpp:37 — rejects a outside [kMinSeedIndex, kMaxSeedIndex].
inline GeneratorState seed_from_index(std::uint64_t a, Method method = Method::BarrettModified) {
    std::uint64_t z0 = 0;
    b200::check(bcn_seed_from_index(a, &z0));
    return GeneratorState{a, Residue{z0}, 0, method};
}

// generator.hpp:42-43 — z_k = 2^(53 (k mod P)) z_0 mod m.
inline GeneratorState state_at(std::uint64_t a, std::uint64_t k,
                               Method method = Method::BarrettModified) {
    std::uint64_t z = 0;
    b200::check(bcn_state_at(a, k, &z));
    return GeneratorState{a, Residue{z}, k, method};
}

inline const char* method_name(Method m) {
    switch (m) {
        case Method::Ref128: return "Ref128";
        case Method::LEcuyer: return "LEcuyer";
        case Method::Barrett: return "Barrett";
        case Method::BarrettModified: return "BarrettModified";
    }
    return "?";
}

// Case-insensitive; unknown names are std::invalid_argument.
inline Method parse_method(const std::string& name) {
    std::string s(name);
    std::transform(s.begin(), s.end(), s.begin(),
                   [](unsigned char c) { return static_cast<char>(std::tolower(c)); });
    if (s == "ref128") return Method::Ref128;
    if (s == "lecuyer") return Method::LEcuyer;
    if (s == "barrett") return Method::Barrett;
    if (s == "barrettmodified") return Method::BarrettModified;
    throw std::invalid_argument("unknown method: " + name);
}

// generator.hpp:52-70. Every method computes the same residue; the modified
// Barrett method alone rejects z = 0 (modred.hpp:150), all reject z >= m.
inline Residue next(GeneratorState& state) {
    if (state.z.value == 0 && state.method != Method::BarrettModified) {
        ++state.k;
        return state.z;  // 2^53 * 0 mod m
    }
    std::uint64_t z = state.z.value;
    b200::check(bcn_next(&z));
    state.z.value = z;
    ++state.k;
    return state.z;
}

// generator.hpp:74-78 — double(z) * kInvModulus, z = 0 and z >= m rejected.
inline double to_unit_interval(Residue z) {
    double u = 0.0;
    b200::check(bcn_to_unit_interval(z.value, &u));
    return u;
}

}  // namespace gen
}  // namespace bcn
