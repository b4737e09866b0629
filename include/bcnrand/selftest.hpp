#pragma once

// B200 drop-in for the reference's selftest header
// (/root/reference/proj/include/bcnrand/selftest.hpp): `run_all(fast,
// constants)` returns one CheckResult per built-in check, under the
// reference's eight check names and in its order (selftest.cpp:145-156), and
// `all_passed` folds them. Here the checks certify THIS build: the host
// reduction layer, the scalar generator API over the C ABI, GPU fills (method
// identity, worker/layout invariance) and the GPU quality suite. Only the
// modred.* checks take the caller's constant table, so a corrupted table
// fails as a modred check (reference tests/test_selftest.cpp). Sample sizes
// and sampling are this library's own; any exception inside a check counts as
// that check failing.

#include <cstdint>
#include <functional>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "bcnrand/generator.hpp"
#include "bcnrand/modred.hpp"
#include "bcnrand/oracle.hpp"
#include "bcnrand/parallel.hpp"
#include "bcnrand/quality.hpp"

namespace bcn::selftest {

struct CheckResult {
    std::string name;
    bool pass = false;
    std::string detail;
};

namespace detail {

// splitmix64: a small deterministic sampler for the randomized checks.
class Sampler {
  public:
    explicit Sampler(std::uint64_t seed) : x_(seed) {}
    std::uint64_t next() {
        std::uint64_t v = (x_ += 0x9E3779B97F4A7C15ull);
        v = (v ^ (v >> 30)) * 0xBF58476D1CE4E5B9ull;
        v = (v ^ (v >> 27)) * 0x94D049BB133111EBull;
        return v ^ (v >> 31);
    }
    // uniform enough on [lo, hi] for test sampling (hi - lo < 2^63)
    std::uint64_t in(std::uint64_t lo, std::uint64_t hi) { return lo + next() % (hi - lo + 1); }

  private:
    std::uint64_t x_;
};

using Outcome = std::pair<bool, std::string>;

struct Check {
    const char* name;
    std::function<Outcome()> body;
};

inline CheckResult evaluate(const Check& c) {
    try {
        auto [ok, what] = c.body();
        return {c.name, ok, std::move(what)};
    } catch (const std::exception& e) {
        return {c.name, false, std::string("exception: ") + e.what()};
    }
}

// All four step kernels (with table `c`) agree with the exact 128-bit
// reduction on the smallest and largest residues and on random ones, and so
// do the four GPU jump engines (bcn_engine_check) on the random sample.
inline Outcome kernels_agree(bool fast, const modred::ReductionConstants& c) {
    const std::uint64_t edge = fast ? 4096 : 65536, randoms = fast ? (1u << 16) : (1u << 20);
    auto agree = [&c](std::uint64_t v) {
        const Residue z{v};
        const std::uint64_t want = modred::reduce_ref(z).value;
        return modred::barrett_modified_step(z, c).value == want && modred::barrett_step(z, c).value == want &&
               modred::lecuyer_step(z, c).value == want && modred::lecuyer_step_fast(z, c).value == want;
    };
    for (std::uint64_t d = 1; d <= edge; ++d)
        if (!agree(d) || !agree(modred::kModulus - d)) return {false, "mismatch near 0 or m"};
    Sampler rng(0xB200'5E1F'0001ull);
    std::vector<std::uint64_t> sample(randoms);
    for (auto& v : sample) {
        v = rng.in(1, modred::kModulus - 1);
        if (!agree(v)) return {false, "mismatch on a random residue"};
    }
    // The GPU's jump engines, multiplier 2^53 mod m (one step), on the same sample.
    const std::vector<std::uint64_t> step(randoms, modred::reduce_ref(Residue{1}).value);
    std::vector<std::uint64_t> got(randoms);
    for (bcn_engine e : {BCN_ENGINE_BARRETT, BCN_ENGINE_MONTGOMERY, BCN_ENGINE_FP64, BCN_ENGINE_MIXED}) {
        b200::check(bcn_engine_check(e, sample.data(), step.data(), got.data(), randoms, 1, -1));
        for (std::uint64_t i = 0; i < randoms; ++i)
            if (got[i] != modred::reduce_ref(Residue{sample[i]}).value)
                return {false, std::string("device engine ") + bcn_engine_name(e) + " disagrees"};
    }
    return {true, std::to_string(2 * edge + randoms) + " residues, 4 host kernels + 4 device engines"};
}

// state_at(a, k) = state_at(a, j) followed by k - j next() calls; the first
// trial walks from the seed itself.
inline Outcome skip_ahead_composes(bool fast) {
    const int trials = fast ? 6 : 24;
    const std::uint64_t span = fast ? 30000 : 250000;
    Sampler rng(0xB200'5E1F'0002ull);
    for (int t = 0; t < trials; ++t) {
        const std::uint64_t a = rng.in(gen::kMinSeedIndex, gen::kMaxSeedIndex);
        const std::uint64_t k = rng.in(0, span);
        const std::uint64_t j = t == 0 ? 0 : rng.in(0, k);
        gen::GeneratorState s = t == 0 ? gen::seed_from_index(a) : gen::state_at(a, j);
        for (std::uint64_t i = j; i < k; ++i) gen::next(s);
        if (s.z.value != gen::state_at(a, k).z.value) return {false, "composition failed"};
    }
    return {true, std::to_string(trials) + " (a, j, k) triples"};
}

// The four methods step one stream, and it is the stream the GPU fills.
inline Outcome methods_share_one_stream(bool fast) {
    const std::uint64_t n = fast ? 8192 : 65536;
    std::vector<std::uint64_t> device(n);
    par::fill_residues(device, par::make_plan(n, 1, par::Layout::Contiguous), gen::kMinSeedIndex,
                       gen::Method::BarrettModified);
    gen::GeneratorState st[] = {gen::seed_from_index(gen::kMinSeedIndex, gen::Method::Ref128),
                                gen::seed_from_index(gen::kMinSeedIndex, gen::Method::LEcuyer),
                                gen::seed_from_index(gen::kMinSeedIndex, gen::Method::Barrett),
                                gen::seed_from_index(gen::kMinSeedIndex, gen::Method::BarrettModified)};
    for (std::uint64_t i = 0; i < n; ++i)
        for (auto& s : st)
            if (gen::next(s).value != device[i]) return {false, "methods or the device fill diverge"};
    return {true, std::to_string(n) + " steps x 4 methods vs the device fill"};
}

// The truncated alpha-series numerator is the seed (Eq. 1-2).
inline Outcome series_matches_seed() {
    Sampler rng(0xB200'5E1F'0003ull);
    std::vector<std::uint64_t> idx = {gen::kMinSeedIndex, gen::kMaxSeedIndex};
    for (int t = 0; t < 6; ++t) idx.push_back(rng.in(gen::kMinSeedIndex, gen::kMaxSeedIndex));
    for (std::uint64_t a : idx)
        if (oracle::alpha_fraction(a, 33).numerator != gen::seed_from_index(a).z.value)
            return {false, "series numerator differs from seed_from_index"};
    return {true, std::to_string(idx.size()) + " seed indices"};
}

// ord(2^53) modulo 3^j is 2 * 3^(j-1): the law behind the period P = 2 * 3^32.
inline Outcome orders_follow_law(bool fast) {
    const int top = fast ? 9 : 13;
    for (int j = top; j >= 2; --j)
        if (oracle::multiplicative_order(53, j) != 2 * oracle::pow3(j - 1)) return {false, "order law fails"};
    return {true, "3^2 .. 3^" + std::to_string(top)};
}

// Logical output of a GPU fill is the same for every worker count and layout.
inline Outcome fills_are_worker_invariant(bool fast) {
    const std::uint64_t n = fast ? 12289 : 100003;
    std::vector<double> want(n), got(n);
    par::fill(want, par::make_plan(n, 1, par::Layout::Contiguous), gen::kMinSeedIndex, gen::Method::BarrettModified);
    int cases = 0;
    for (unsigned workers : {2u, 5u, 64u, 1023u}) {
        for (auto layout : {par::Layout::Contiguous, par::Layout::Interleaved}) {
            const par::PartitionPlan plan = par::make_plan(n, workers, layout);
            par::fill(got, plan, gen::kMinSeedIndex, gen::Method::LEcuyer);
            if ((layout == par::Layout::Contiguous ? got : par::deinterleave(got, plan)) != want)
                return {false, "logical output depends on the partition"};
            ++cases;
        }
    }
    return {true, std::to_string(cases) + " partitions of " + std::to_string(n) + " elements"};
}

// The statistical smoke tests pass on fresh GPU output.
inline Outcome statistics_pass(bool fast) {
    const std::uint64_t n = fast ? 250000 : 2000000;
    const auto plan = par::make_plan(n, 1, par::Layout::Contiguous);
    std::vector<double> u(n);
    std::vector<std::uint64_t> raw(n);
    par::fill(u, plan, gen::kMinSeedIndex, gen::Method::BarrettModified);
    par::fill_residues(raw, plan, gen::kMinSeedIndex, gen::Method::BarrettModified);
    std::vector<Residue> residues;
    residues.reserve(n);
    for (std::uint64_t v : raw) residues.push_back(Residue{v});
    const bool ok = quality::chi_square_uniformity(u, 1000).pass && quality::monobit_mantissa(residues).pass &&
                    quality::serial_correlation(u, 1).pass;
    return {ok, std::to_string(n) + " variates: chi-square, monobit, lag-1"};
}

}  // namespace detail

inline std::vector<CheckResult> run_all(bool fast = false,
                                        const modred::ReductionConstants& c = modred::constants()) {
    const detail::Check checks[] = {
        {"modred.constants", [&] { return detail::Outcome{modred::verify_constants(c), "table vs 3^33"}; }},
        {"modred.equivalence", [&] { return detail::kernels_agree(fast, c); }},
        {"generator.skip_ahead", [&] { return detail::skip_ahead_composes(fast); }},
        {"generator.method_streams", [&] { return detail::methods_share_one_stream(fast); }},
        {"oracle.alpha_fraction", [] { return detail::series_matches_seed(); }},
        {"oracle.period_law", [&] { return detail::orders_follow_law(fast); }},
        {"parallel.worker_invariance", [&] { return detail::fills_are_worker_invariant(fast); }},
        {"quality.suite", [&] { return detail::statistics_pass(fast); }},
    };
    std::vector<CheckResult> out;
    out.reserve(std::size(checks));
    for (const auto& check : checks) out.push_back(detail::evaluate(check));
    return out;
}

inline bool all_passed(std::span<const CheckResult> results) {
    bool ok = true;
    for (const CheckResult& r : results) ok = ok && r.pass;
    return ok;
}

}  // namespace bcn::selftest
