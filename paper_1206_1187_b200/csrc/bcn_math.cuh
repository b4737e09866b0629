// bcn_math.cuh — modular arithmetic for the alpha_{2,3} generator, host and device.
//
// The generator (reference include/bcnrand/generator.hpp:3-9) is the LCG
//     z_{k+1} = 2^53 z_k mod m,   m = 3^33,
// seeded by z_0(a) = 2^(a-3^33) floor(m/2) mod m (generator.cpp:32-40).
// Because floor(m/2) = -2^-1 (mod m) and 2 is a primitive root mod 3^33
// (order P = 2*3^32), every state has the closed form
//     z_k(a) = m - (2^E mod m),   E = (a - 3^33 - 1 + 53 k) mod P.
// The fill path only ever needs (i) 2^E mod m for a seed (a windowed power,
// once per stream) and (ii) multiplication by a FIXED jump multiplier
// c_T = 2^(53 T) mod m (once per emitted variate). For (ii) three exact
// reductions are provided ("engines", chosen by measurement):
//
//   Barrett  (Shoup form)  q = hi64(z * floor(c 2^64 / m)); r = z c - q m; r -= m if r >= m
//   Montgomery (REDC)      r = (z c~ + (z c~ m' mod 2^64) m) / 2^64 with c~ = c 2^64 mod m
//   FP64     (exact)       balanced residues held in doubles; quotient by one DFMA
//                          against a magic constant, remainder by error-free products.
//
// All three are bit-exact on their whole domain (proofs in DESIGN.md §3); the
// paper's modified Barrett step (reference modred.hpp:149-159) is also kept
// for the T = 1 staged kernel.
#pragma once

#include <cstdint>

namespace bcn_b200 {

constexpr uint64_t kModulus = 5559060566555523ull;   // 3^33, modred.hpp:22
constexpr uint64_t kPeriod = 3706040377703682ull;    // 2*3^32, generator.hpp:21
constexpr uint64_t kMinSeed = kModulus + 100ull;      // generator.hpp:19
constexpr uint64_t kMaxSeed = 1ull << 53;             // generator.hpp:20
constexpr uint64_t kMu = 0x33D9481681D79Dull;         // floor(2^106/m), modred.hpp:44
constexpr uint64_t kHalfM = 2779530283277761ull;      // floor(m/2), generator.cpp:36
constexpr uint64_t kMontMPrime = 0x1BA97738C32954D5ull;  // -m^-1 mod 2^64
constexpr double kInvModulus = 1.0 / 5559060566555523.0;  // generator.hpp:22
constexpr double kModulusD = 5559060566555523.0;      // exact: m < 2^53
constexpr double kMagic = 6755399441055744.0;         // 1.5 * 2^52

constexpr int kPowWindows = 13;  // 13 x 4-bit windows cover E < P < 2^52

// ---------------------------------------------------------------- host exact
// a b mod m for a, b < m: a 128-bit Barrett step instead of a 128-bit
// division (q = floor(floor(ab / 2^51) mu / 2^55) is floor(ab/m) or one less;
// proof and CPU test with include/bcnrand_device.cuh's identical mulmod).
inline uint64_t host_mulmod(uint64_t a, uint64_t b) {
    const unsigned __int128 x = static_cast<unsigned __int128>(a) * b;
    const uint64_t x1 = static_cast<uint64_t>(x >> 51);
    const uint64_t q = static_cast<uint64_t>((static_cast<unsigned __int128>(x1) * kMu) >> 55);
    const uint64_t r = static_cast<uint64_t>(x) - q * kModulus;
    return r >= kModulus ? r - kModulus : r;
}
inline uint64_t host_pow2(uint64_t e) {  // 2^e mod m, e reduced mod P first
    e %= kPeriod;
    uint64_t r = 1, b = 2;
    while (e) {
        if (e & 1) r = host_mulmod(r, b);
        b = host_mulmod(b, b);
        e >>= 1;
    }
    return r;
}
// Shoup constant floor(c 2^64 / m) for a multiplier c < m.
inline uint64_t host_shoup(uint64_t c) {
    return static_cast<uint64_t>((static_cast<unsigned __int128>(c) << 64) / kModulus);
}
// Montgomery image c 2^64 mod m.
inline uint64_t host_mont(uint64_t c) {
    return static_cast<uint64_t>((static_cast<unsigned __int128>(c) << 64) % kModulus);
}
// (53 * x) mod P for any 64-bit x.
inline uint64_t host_mul53_mod_p(uint64_t x) {
    return static_cast<uint64_t>((static_cast<unsigned __int128>(x % kPeriod) * 53u) % kPeriod);
}
// Exponent of 2 for logical element 0 of a fill whose first state is
// next(state_at(a, k)): E0 = (a - 3^33 - 1 + 53 ((k mod P) + 1)) mod P.
inline uint64_t host_fill_e0(uint64_t a, uint64_t k) {
    const uint64_t base = (a - kModulus - 1) % kPeriod;
    const uint64_t kk = (k % kPeriod + 1) % kPeriod;
    return (base + host_mul53_mod_p(kk)) % kPeriod;
}
// Jump multiplier for T logical steps (T may be "negative" mod P).
inline uint64_t host_jump(uint64_t steps_mod_p) { return host_pow2(host_mul53_mod_p(steps_mod_p)); }

// ------------------------------------------------------------ multipliers
// Every engine consumes the same packed multiplier so kernels can be engine
// generic: c (canonical), its Shoup constant, its Montgomery image, and the
// FP64 pair (balanced value, RN(balanced/m)).
struct alignas(16) Mult {
    double cb;    // balanced multiplier (FP64 engine); cb, com first: one 16-byte load
    double com;   // RN(cb / m)
    uint64_t c;
    uint64_t shoup;
    uint64_t mont;
    int64_t cbi;  // balanced multiplier as an integer (mixed engine)
};

inline Mult host_make_mult(uint64_t c) {
    Mult k;
    k.c = c;
    k.shoup = host_shoup(c);
    k.mont = host_mont(c);
    const int64_t bal = c > kModulus / 2 ? static_cast<int64_t>(c) - static_cast<int64_t>(kModulus)
                                         : static_cast<int64_t>(c);
    k.cb = static_cast<double>(bal);  // exact: |bal| <= m/2 < 2^52
    k.com = k.cb / kModulusD;         // RN(c_bal / m)
    k.cbi = bal;
    return k;
}

// -------------------------------------------------------------- device math
#if defined(__CUDACC__)

// Barrett with a precomputed quotient constant (Shoup). For z < 2^64 and
// c < m: q in {floor(zc/m) - 1, floor(zc/m)}, so r = zc - qm in [0, 2m) and
// one conditional subtract lands in [0, m). Everything is mod 2^64 because
// r < 2m < 2^54.
__device__ __forceinline__ uint64_t mul_barrett(uint64_t z, uint64_t c, uint64_t cs) {
    const uint64_t q = __umul64hi(z, cs);
    const uint64_t r = z * c - q * kModulus;
    return r >= kModulus ? r - kModulus : r;
}

// Montgomery REDC by the constant's Montgomery image ct = c 2^64 mod m:
// REDC(z ct) = z c mod m. T = z ct < m^2, so (T + u m)/2^64 < 2m.
__device__ __forceinline__ uint64_t mul_montgomery(uint64_t z, uint64_t ct) {
    const uint64_t lo = z * ct;
    const uint64_t hi = __umul64hi(z, ct);
    const uint64_t u = lo * kMontMPrime;
    const uint64_t r = hi + __umul64hi(u, kModulus) + (lo != 0 ? 1ull : 0ull);
    return r >= kModulus ? r - kModulus : r;
}

// The paper's modified Barrett step z -> 2^53 z mod m (reference
// modred.hpp:149-159, Fig. 3). Valid for z in [1, m).
__device__ __forceinline__ uint64_t step_modified_barrett(uint64_t z) {
    const uint64_t hi = __umul64hi(z, kMu);
    const uint64_t lo = z * kMu;
    const uint64_t q3 = (hi << 11) | (lo >> 53);
    const uint64_t r2 = (q3 * kModulus) & 0x1FFFFFFFFFFFFFull;
    const uint64_t r = 0x20000000000000ull - r2;
    return r >= kModulus ? r - kModulus : r;
}

// Exact modular multiply on the FP64 pipe. State s is an integer-valued
// double with |s| <= 0.75 m; cb is the balanced multiplier (|cb| <= m/2) and
// com = RN(cb/m). Invariant and exactness proof: DESIGN.md §3.3.
__device__ __forceinline__ double mul_fp64(double s, double cb, double com) {
    const double p = __dmul_rn(s, cb);           // RN(s cb)
    const double e = __fma_rn(s, cb, -p);        // s cb - p, exact
    const double qm = __fma_rn(s, com, kMagic);  // MAGIC + rint(s cb / m + eta)
    const double q = __dsub_rn(qm, kMagic);      // exact integer quotient estimate
    const double t = __fma_rn(-q, kModulusD, p); // p - q m, exact (|.| < 2^53)
    return __dadd_rn(t, e);                      // s cb - q m, exact, |.| <= 0.7315 m
}

// Mixed-pipe exact modular multiply: the quotient comes from ONE DFMA (the
// same rint(s c_b / m + eta) as mul_fp64, read straight out of the magic
// constant's significand), the remainder from exact 64-bit integer products:
//     r = s c_b - q m  (mod 2^64),   q = bits(qm) - bits(MAGIC),
// with |r| <= 0.7315 m < 2^63, so the two's-complement value IS r (proof as
// for mul_fp64). The state keeps the integer and its exact
// double image (one I2F per step). Cost: 1 DFMA + ~7 IMAD/IADD + 1 I2F.
constexpr uint64_t kMagicBits = 0x4338000000000000ull;  // bits of 1.5 * 2^52
struct MixedState {
    int64_t s;
    double d;
};

__device__ __forceinline__ MixedState mul_mixed(MixedState x, double com, int64_t cbi) {
    const double qm = __fma_rn(x.d, com, kMagic);
    const uint64_t qb = static_cast<uint64_t>(__double_as_longlong(qm));
    const uint64_t r = static_cast<uint64_t>(x.s) * static_cast<uint64_t>(cbi) -
                       (qb - kMagicBits) * kModulus;
    const int64_t rs = static_cast<int64_t>(r);
    return MixedState{rs, __ll2double_rn(rs)};
}

// Canonical residue (as an exact double) of a balanced FP64 state: add m when
// the sign bit is set. The addend is built with integer ops on the high word
// (SHF + 2 LOP3) instead of a DSETP + 2 FSEL, keeping the FP64 pipe for the
// arithmetic (s is never -0: it is a nonzero unit).
__device__ __forceinline__ double fp64_canonical(double s) {
    const int hi = __double2hiint(s);
    const int mask = hi >> 31;  // all ones iff s < 0
    const double add = __hiloint2double(mask & __double2hiint(kModulusD), mask & __double2loint(kModulusD));
    return __dadd_rn(s, add);
}

// reference generator.hpp:74-78: double(z) * kInvModulus with one RN multiply.
__device__ __forceinline__ double unit_from_u64(uint64_t z) {
    return __dmul_rn(__ull2double_rn(z), kInvModulus);
}

// f32 format: RZ of the f64 variate, i.e. the top 24
// significand bits. For u in [2^-53, 1) the low 32 bits of (bits >> 29) hold
// ((e & 0x1FF) << 23) | mant23, and subtracting 896 << 23 mod 2^32 rebases the
// exponent (e - 1408 == e - 896 - 512, and 512 << 23 == 2^32).
__device__ __forceinline__ float f32_rz_from_unit(double u) {
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(u));
    const uint32_t lo = static_cast<uint32_t>(b), hi = static_cast<uint32_t>(b >> 32);
    const uint32_t f = __funnelshift_r(lo, hi, 29) - (896u << 23);
    return __uint_as_float(f);
}

#endif  // __CUDACC__

}  // namespace bcn_b200
