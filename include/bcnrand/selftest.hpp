#pragma once

// B200 drop-in for the reference header of the same name
// (/root/reference/proj/include/bcnrand/selftest.hpp, src/selftest.cpp:25-156):
// the eight built-in correctness checks behind `bcnrand selftest`, with the
// reference's check names and `fast` / constant-table parameters. The checks
// run on this library — the host reduction layer, the scalar generator API
// through the C ABI, GPU fills for the worker-invariance sweep and the GPU
// quality suite — so a passing run certifies the B200 build. Only the two
// modred.* checks use the caller's constant table, so a corrupted table is
// reported as a modred failure (tests/test_selftest.cpp).

#include <cstdint>
#include <cstdio>
#include <random>
#include <span>
#include <string>
#include <vector>

#include "bcnrand/generator.hpp"
#include "bcnrand/modred.hpp"
#include "bcnrand/oracle.hpp"
#include "bcnrand/parallel.hpp"
#include "bcnrand/quality.hpp"

namespace bcn::selftest {

// selftest.hpp
struct CheckResult {
    std::string name;
    bool pass = false;
    std::string detail;
};

namespace detail {

inline std::string counted(const char* what, std::uint64_t n) {
    char buf[96];
    std::snprintf(buf, sizeof(buf), "%llu %s", static_cast<unsigned long long>(n), what);
    return buf;
}

// The constant table against 3^33.
inline CheckResult constants_check(const modred::ReductionConstants& c) {
    return {"modred.constants", modred::verify_constants(c), "table derived from 3^33"};
}

// Every step kernel equals the 128-bit oracle on [1, E) and on R random residues.
inline CheckResult equivalence_check(bool fast, const modred::ReductionConstants& c) {
    const std::uint64_t exhaustive = fast ? 10000 : 100000, randoms = fast ? 100000 : 1000000;
    bool ok = true;
    auto agree = [&](std::uint64_t z) {
        const std::uint64_t want = modred::reduce_ref(Residue{z}).value;
        ok = ok && modred::lecuyer_step(Residue{z}, c).value == want &&
             modred::lecuyer_step_fast(Residue{z}, c).value == want &&
             modred::barrett_step(Residue{z}, c).value == want &&
             modred::barrett_modified_step(Residue{z}, c).value == want;
    };
    try {
        for (std::uint64_t z = 1; z < exhaustive && ok; ++z) agree(z);
        std::mt19937_64 rng(0x5E1F7E57ull);
        std::uniform_int_distribution<std::uint64_t> dist(1, modred::kModulus - 1);
        for (std::uint64_t i = 0; i < randoms && ok; ++i) agree(dist(rng));
    } catch (const std::exception&) {
        ok = false;  // a corrupted table can push a kernel out of its domain
    }
    return {"modred.equivalence", ok, counted("exhaustive + random residues", exhaustive + randoms)};
}

// state_at(a, k) equals k sequential next() calls from seed_from_index(a).
inline CheckResult skip_ahead_check(bool fast) {
    const int trials = fast ? 5 : 25;
    const std::uint64_t max_k = fast ? 20000 : 200000;
    std::mt19937_64 rng(0x5C1BA4EAull);
    bool ok = true;
    for (int t = 0; t < trials && ok; ++t) {
        const std::uint64_t a = gen::kMinSeedIndex + rng() % (gen::kMaxSeedIndex - gen::kMinSeedIndex + 1);
        const std::uint64_t k = rng() % max_k;
        gen::GeneratorState s = gen::seed_from_index(a);
        for (std::uint64_t i = 0; i < k; ++i) gen::next(s);
        ok = s.z.value == gen::state_at(a, k).z.value;
    }
    return {"generator.skip_ahead", ok, counted("random (a, k) trials", static_cast<std::uint64_t>(trials))};
}

// The four methods produce one stream (and it matches the default-table
// modified-Barrett kernel step by step).
inline CheckResult method_streams_check(bool fast) {
    const std::uint64_t n = fast ? 10000 : 100000;
    const gen::Method methods[] = {gen::Method::Ref128, gen::Method::LEcuyer, gen::Method::Barrett,
                                   gen::Method::BarrettModified};
    std::vector<gen::GeneratorState> s;
    for (gen::Method m : methods) s.push_back(gen::seed_from_index(gen::kMinSeedIndex, m));
    Residue z = s[0].z;
    bool ok = true;
    for (std::uint64_t i = 0; i < n && ok; ++i) {
        z = modred::barrett_modified_step(z);
        for (auto& st : s) ok = ok && gen::next(st).value == z.value;
    }
    return {"generator.method_streams", ok, counted("steps under all four methods", n)};
}

// The alpha-series expansion reproduces seed_from_index (Eq. 1-2).
inline CheckResult alpha_fraction_check() {
    bool ok = true;
    for (std::uint64_t a : {gen::kMinSeedIndex, modred::kModulus + std::uint64_t{987654321}, gen::kMaxSeedIndex})
        ok = ok && oracle::alpha_fraction(a, 33).numerator == gen::seed_from_index(a).z.value;
    return {"oracle.alpha_fraction", ok, "series expansion matches seed formula"};
}

// ord(2^53 mod 3^j) = 2 * 3^(j-1): the period law behind P = 2 * 3^32.
inline CheckResult period_law_check(bool fast) {
    const int max_j = fast ? 8 : 13;
    bool ok = true;
    for (int j = 2; j <= max_j && ok; ++j) ok = oracle::multiplicative_order(53, j) == 2 * oracle::pow3(j - 1);
    return {"oracle.period_law", ok, counted("moduli 3^2 .. 3^max checked", static_cast<std::uint64_t>(max_j - 1))};
}

// The logical fill (GPU) is identical for every worker count and layout.
inline CheckResult worker_invariance_check(bool fast) {
    const std::uint64_t n = fast ? 10000 : 100000;
    std::vector<double> ref(n), out(n);
    par::fill(ref, par::make_plan(n, 1, par::Layout::Contiguous), gen::kMinSeedIndex, gen::Method::BarrettModified);
    bool ok = true;
    for (unsigned w : {2u, 3u, 7u, 16u, 1000u}) {
        for (par::Layout layout : {par::Layout::Contiguous, par::Layout::Interleaved}) {
            const auto plan = par::make_plan(n, w, layout);
            par::fill(out, plan, gen::kMinSeedIndex, gen::Method::BarrettModified);
            const std::vector<double> logical =
                layout == par::Layout::Interleaved ? par::deinterleave(out, plan) : out;
            ok = ok && logical == ref;
        }
    }
    return {"parallel.worker_invariance", ok, counted("elements x 5 worker counts x 2 layouts", n)};
}

// The statistical smoke suite (GPU) on fresh output.
inline CheckResult quality_check(bool fast) {
    const std::uint64_t n = fast ? 200000 : 2000000;
    std::vector<double> u(n);
    std::vector<std::uint64_t> z(n);
    const auto plan = par::make_plan(n, 1, par::Layout::Contiguous);
    par::fill(u, plan, gen::kMinSeedIndex, gen::Method::BarrettModified);
    par::fill_residues(z, plan, gen::kMinSeedIndex, gen::Method::BarrettModified);
    std::vector<Residue> r(n);
    for (std::uint64_t i = 0; i < n; ++i) r[i].value = z[i];
    const auto chi = quality::chi_square_uniformity(u, 1000);
    const auto mono = quality::monobit_mantissa(r);
    const auto corr = quality::serial_correlation(u, 1);
    return {"quality.suite", chi.pass && mono.pass && corr.pass,
            counted("samples: chi-square, mantissa monobit, lag-1 correlation", n)};
}

}  // namespace detail

// selftest.hpp: every check, in the reference's order.
inline std::vector<CheckResult> run_all(bool fast = false,
                                        const modred::ReductionConstants& c = modred::constants()) {
    return {detail::constants_check(c),        detail::equivalence_check(fast, c),
            detail::skip_ahead_check(fast),    detail::method_streams_check(fast),
            detail::alpha_fraction_check(),    detail::period_law_check(fast),
            detail::worker_invariance_check(fast), detail::quality_check(fast)};
}

inline bool all_passed(std::span<const CheckResult> results) {
    for (const auto& r : results)
        if (!r.pass) return false;
    return true;
}

}  // namespace bcn::selftest
