#pragma once

// B200 drop-in for the reference header of the same name
// (/root/reference/proj/include/bcnrand/modred.hpp). Only the part of the
// reduction layer the generator fill path exposes is provided: the residue
// type, the modulus constants and the exact step oracle reduce_ref
// (modred.hpp:16-23, :103-107). The per-step CPU reduction kernels
// (L'Ecuyer, Barrett, modified Barrett) are replaced on the device by the
// engines behind include/bcnrand_b200.h and are not re-exported.

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

// (2^53 z) mod m through an exact 128-bit product; z >= m is a domain error
// (modred.hpp:103-107).
inline Residue reduce_ref(Residue z) {
    if (z.value >= kModulus) throw std::domain_error("reduce_ref: residue out of range");
    const auto wide = static_cast<unsigned __int128>(z.value) << 53;
    return Residue{static_cast<std::uint64_t>(wide % kModulus)};
}

}  // namespace modred
}  // namespace bcn
