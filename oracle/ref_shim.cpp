// ref_shim.cpp — extern "C" access to the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY. oracle/Makefile compiles the reference sources in
// place (/root/reference/proj/src/{modred,generator,parallel}.cpp) together
// with this file into oracle/_ref/libbcnref.so. Nothing from the reference is
// copied into this repo; this file only translates the reference's C++ API
// (include/bcnrand/generator.hpp, parallel.hpp) and its exceptions into plain
// C calls and status codes so tests/ and bench.py can drive it via ctypes:
//   0 ok, 1 std::invalid_argument, 2 std::out_of_range, 3 std::domain_error.
#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>

#include "bcnrand/generator.hpp"
#include "bcnrand/parallel.hpp"
#include "bcnrand/quality.hpp"

namespace {

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::out_of_range&) {  // derives from logic_error: test first
        return 2;
    } catch (const std::domain_error&) {
        return 3;
    } catch (const std::invalid_argument&) {
        return 1;
    }
}

bcn::gen::Method method_of(int m) { return static_cast<bcn::gen::Method>(m); }
bcn::par::Layout layout_of(int l) {
    return l == 0 ? bcn::par::Layout::Contiguous : bcn::par::Layout::Interleaved;
}

}  // namespace

extern "C" {

int bref_modpow2(uint64_t e, uint64_t modulus, uint64_t* out) {
    return guarded([&] { *out = bcn::gen::modpow2(e, modulus); });
}

int bref_seed_from_index(uint64_t a, int method, uint64_t* z0) {
    return guarded([&] { *z0 = bcn::gen::seed_from_index(a, method_of(method)).z.value; });
}

int bref_state_at(uint64_t a, uint64_t k, int method, uint64_t* z) {
    return guarded([&] { *z = bcn::gen::state_at(a, k, method_of(method)).z.value; });
}

// Walks `count` next() calls from state_at(a, k) and stores every residue.
int bref_walk(uint64_t a, uint64_t k, int method, uint64_t count, uint64_t* out) {
    return guarded([&] {
        auto s = bcn::gen::state_at(a, k, method_of(method));
        for (uint64_t i = 0; i < count; ++i) out[i] = bcn::gen::next(s).value;
    });
}

int bref_step(uint64_t z, int method, uint64_t* out) {
    return guarded([&] {
        bcn::gen::GeneratorState s{bcn::gen::kMinSeedIndex, bcn::Residue{z}, 0, method_of(method)};
        *out = bcn::gen::next(s).value;
    });
}

int bref_to_unit_interval(uint64_t z, double* u) {
    return guarded([&] { *u = bcn::gen::to_unit_interval(bcn::Residue{z}); });
}

int bref_make_plan(uint64_t n, unsigned workers, unsigned* eff, uint64_t* wpw) {
    return guarded([&] {
        const auto p = bcn::par::make_plan(n, workers, bcn::par::Layout::Contiguous);
        *eff = p.workers;
        *wpw = p.work_per_worker;
    });
}

int bref_physical_index(uint64_t n, unsigned workers, int layout, unsigned w, uint64_t i,
                        uint64_t* out) {
    return guarded([&] {
        const auto p = bcn::par::make_plan(n, workers, layout_of(layout));
        *out = p.physical_index(w, i);
    });
}

// par::fill (fmt 1) / par::fill_residues (fmt 0) into a caller buffer of
// `cap` items — parallel.cpp:101-111, one std::thread per plan worker.
int bref_fill(void* out, uint64_t cap, int fmt, uint64_t n, unsigned workers, int layout,
              uint64_t seed_index, int method, uint64_t base_offset) {
    return guarded([&] {
        const auto plan = bcn::par::make_plan(n, workers, layout_of(layout));
        if (fmt == 0) {
            bcn::par::fill_residues(std::span<std::uint64_t>(static_cast<std::uint64_t*>(out), cap),
                                    plan, seed_index, method_of(method), base_offset);
        } else {
            bcn::par::fill(std::span<double>(static_cast<double*>(out), cap), plan, seed_index,
                           method_of(method), base_offset);
        }
    });
}

int bref_deinterleave(const void* in, uint64_t cap, void* out, int fmt, uint64_t n,
                      unsigned workers, int layout) {
    return guarded([&] {
        const auto plan = bcn::par::make_plan(n, workers, layout_of(layout));
        if (fmt == 0) {
            auto v = bcn::par::deinterleave(
                std::span<const std::uint64_t>(static_cast<const std::uint64_t*>(in), cap), plan);
            std::memcpy(out, v.data(), v.size() * 8);
        } else {
            auto v = bcn::par::deinterleave(
                std::span<const double>(static_cast<const double*>(in), cap), plan);
            std::memcpy(out, v.data(), v.size() * 8);
        }
    });
}

// quality.hpp:27-37 — the reference smoke statistics (for the GPU suite's parity).
int bref_chi_square(const double* x, uint64_t n, int bins, double* stat, int* pass) {
    return guarded([&] {
        const auto r = bcn::quality::chi_square_uniformity(std::span<const double>(x, n), bins);
        *stat = r.statistic;
        *pass = r.pass;
    });
}

int bref_monobit(const uint64_t* z, uint64_t n, double* stat, int* pass) {
    return guarded([&] {
        const auto r = bcn::quality::monobit_mantissa(
            std::span<const bcn::Residue>(reinterpret_cast<const bcn::Residue*>(z), n));
        *stat = r.statistic;
        *pass = r.pass;
    });
}

int bref_serial_correlation(const double* x, uint64_t n, int lag, double* rho, int* pass) {
    return guarded([&] {
        const auto r = bcn::quality::serial_correlation(std::span<const double>(x, n), lag);
        *rho = r.statistic;
        *pass = r.pass;
    });
}

}  // extern "C"
