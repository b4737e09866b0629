// Tests of the C++ drop-in headers (include/bcnrand/*.hpp) on the GPU path:
// user code written against the reference API, compiled against this repo's
// headers and linked with libbcnrand_b200.so. Run by tests/test_dropin.py.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <cuda_runtime.h>

#include <cstring>
#include <vector>

#include "bcnrand/parallel.hpp"
#include "doctest.h"

using namespace bcn;

namespace {

std::vector<std::uint64_t> serial(std::uint64_t n, std::uint64_t a, std::uint64_t k0 = 0) {
    std::vector<std::uint64_t> out(n);
    auto s = gen::state_at(a, k0);
    for (auto& v : out) v = gen::next(s).value;
    return out;
}

}  // namespace

TEST_CASE("goldens through the drop-in generator API") {
    CHECK(gen::seed_from_index(gen::kMinSeedIndex).z.value == 4258649398211344ull);
    auto s = gen::seed_from_index(gen::kMinSeedIndex);
    CHECK(gen::next(s).value == 2138759898642167ull);
    CHECK(gen::state_at(gen::kMinSeedIndex, 1000).z.value == 5492007519572011ull);
    CHECK(gen::modpow2(106, modred::kModulus) == 5239873117944745ull);
    CHECK_THROWS_AS(gen::seed_from_index(gen::kMinSeedIndex - 1), std::out_of_range);
    CHECK_THROWS_AS(gen::to_unit_interval(Residue{0}), std::domain_error);
}

TEST_CASE("host span fill equals the serial stream for every layout and W") {
    const std::uint64_t n = 100003;
    const auto ref = serial(n, gen::kMinSeedIndex, 77);
    for (unsigned w : {1u, 3u, 8u, 1000u}) {
        for (auto layout : {par::Layout::Contiguous, par::Layout::Interleaved}) {
            const auto plan = par::make_plan(n, w, layout);
            std::vector<std::uint64_t> buf(n);
            par::fill_residues(buf, plan, gen::kMinSeedIndex, gen::Method::Barrett, 77);
            if (layout == par::Layout::Interleaved) buf = par::deinterleave(std::span<const std::uint64_t>(buf), plan);
            REQUIRE(buf == ref);
        }
    }
}

TEST_CASE("double fill bits equal to_unit_interval of the residues") {
    const std::uint64_t n = 4099;
    const auto ref = serial(n, gen::kMaxSeedIndex);
    std::vector<double> u(n);
    par::fill(u, par::make_plan(n, 5, par::Layout::Contiguous), gen::kMaxSeedIndex,
              gen::Method::BarrettModified);
    for (std::uint64_t i = 0; i < n; ++i) REQUIRE(u[i] == gen::to_unit_interval(Residue{ref[i]}));
}

TEST_CASE("device span fill (pointer from cudaMalloc) equals the host fill") {
    const std::uint64_t n = (1u << 22) + 17;
    double* d = nullptr;
    REQUIRE(cudaMalloc(&d, n * sizeof(double)) == cudaSuccess);
    const auto plan = par::make_plan(n, 1, par::Layout::Contiguous);
    par::fill(std::span<double>(d, n), plan, gen::kMinSeedIndex, gen::Method::BarrettModified, 5);
    std::vector<double> got(n), want(n);
    REQUIRE(cudaMemcpy(got.data(), d, n * sizeof(double), cudaMemcpyDeviceToHost) == cudaSuccess);
    par::fill(want, plan, gen::kMinSeedIndex, gen::Method::BarrettModified, 5);
    CHECK(std::memcmp(got.data(), want.data(), n * sizeof(double)) == 0);
    cudaFree(d);
}

TEST_CASE("errors surface as the reference's exception types") {
    std::vector<double> small(9);
    CHECK_THROWS_AS(par::fill(small, par::make_plan(10, 2, par::Layout::Contiguous), gen::kMinSeedIndex,
                              gen::Method::BarrettModified),
                    std::invalid_argument);
    std::vector<double> buf(10);
    CHECK_THROWS_AS(par::fill(buf, par::make_plan(10, 4, par::Layout::Interleaved), 12345,
                              gen::Method::BarrettModified),
                    std::out_of_range);
    CHECK_THROWS_AS(par::make_plan(0, 2, par::Layout::Contiguous), std::invalid_argument);
    CHECK_THROWS_AS(par::deinterleave(std::span<const double>(buf), par::make_plan(10, 2, par::Layout::Contiguous)),
                    std::invalid_argument);
    CHECK_THROWS_AS(gen::parse_method("mt19937"), std::invalid_argument);
}

TEST_CASE("float extension is RZ of the double") {
    const std::uint64_t n = 1000;
    std::vector<double> u(n);
    std::vector<float> f(n);
    const auto plan = par::make_plan(n, 1, par::Layout::Contiguous);
    par::fill(u, plan, gen::kMinSeedIndex, gen::Method::BarrettModified);
    par::fill_float(f, plan, gen::kMinSeedIndex, gen::Method::BarrettModified);
    for (std::uint64_t i = 0; i < n; ++i) {
        REQUIRE(static_cast<double>(f[i]) <= u[i]);
        REQUIRE(u[i] - static_cast<double>(f[i]) < u[i] * 1.2e-7);
        REQUIRE(f[i] < 1.0f);
    }
}
