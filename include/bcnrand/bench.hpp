#pragma once

// B200 drop-in for the reference header of the same name
// (/root/reference/proj/include/bcnrand/bench.hpp, src/bench.cpp:102-289): the
// throughput harness API — BenchConfig / BenchReport / GuardError, run(),
// table and CSV writers — measured on the GPU through bcn_bench_fill.
//
// On the GPU the reference's step methods are the library's engines (methods
// never change the bits, bench.cpp:241-248): Ref128 -> the FP64 engine (the
// default exact engine), Barrett -> Barrett (Shoup), BarrettModified -> the
// paper's T=1 modified-Barrett design (staged engine), LEcuyer / LEcuyerFast
// -> Montgomery; Constant -> the Constant writer. exec_seconds is the median
// kernel time, total_seconds the median wall time of the synchronous call
// (launch + seeding + generation). Variant::Unrolled is accepted for API
// compatibility; the GPU kernels are unrolled either way.

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <ostream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "bcnrand/parallel.hpp"

namespace bcn::bench {

// bench.hpp
enum class Variant { Rolled, Unrolled };

inline Variant parse_variant(const std::string& name) {
    if (name == "rolled" || name == "Rolled") return Variant::Rolled;
    if (name == "unrolled" || name == "Unrolled") return Variant::Unrolled;
    throw std::invalid_argument("unknown variant: " + name);
}

struct BenchConfig {
    std::uint64_t n = 20'000'000;
    std::vector<std::string> methods;  // empty: the four kernels + Constant
    unsigned workers = 0;              // 0: default_workers()
    par::Layout layout = par::Layout::Contiguous;
    int repeats = 5;
    Variant variant = Variant::Rolled;
    std::uint64_t seed_index = gen::kMinSeedIndex;
    double min_run_seconds = 0.050;  // > 0: guard against runs too small to time (see run())
    bool check_output = true;        // timed output must equal an untimed fill
};

struct BenchReport {
    std::string method;
    std::uint64_t elements = 0;
    double exec_seconds = 0.0;
    double total_seconds = 0.0;
    double exec_rate_gnum = 0.0;
    double total_rate_gnum = 0.0;
    unsigned workers = 0;
    par::Layout layout = par::Layout::Contiguous;
};

struct GuardError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// BCN_THREADS if set and positive, else hardware concurrency (at least 1).
inline unsigned default_workers() {
    if (const char* v = std::getenv("BCN_THREADS")) {
        const long n = std::strtol(v, nullptr, 10);
        if (n > 0) return static_cast<unsigned>(n);
    }
    const unsigned hw = std::thread::hardware_concurrency();
    return hw ? hw : 1;
}

namespace detail {

// Library engine for a reference method name, -1 for Constant.
inline int engine_for(const std::string& method) {
    if (method == "Ref128") return BCN_ENGINE_FP64;
    if (method == "Barrett") return BCN_ENGINE_BARRETT;
    if (method == "BarrettModified") return BCN_ENGINE_STAGED;
    if (method == "LEcuyer" || method == "LEcuyerFast") return BCN_ENGINE_MONTGOMERY;
    if (method == "Constant") return -1;
    throw std::invalid_argument("unknown bench method: " + method);
}

inline BenchReport measure(const BenchConfig& cfg, const std::string& method, unsigned workers) {
    double exec = 0.0, total = 0.0;
    b200::check(bcn_bench_fill(cfg.n, workers, par::detail::layout_of(cfg.layout), cfg.seed_index,
                               engine_for(method), cfg.repeats, cfg.check_output ? 1 : 0, -1, &exec, &total));
    BenchReport r;
    r.method = method;
    r.elements = cfg.n;
    r.exec_seconds = exec;
    r.total_seconds = total;
    r.exec_rate_gnum = static_cast<double>(cfg.n) / exec / 1e9;
    r.total_rate_gnum = static_cast<double>(cfg.n) / total / 1e9;
    r.workers = workers;
    r.layout = cfg.layout;
    return r;
}

}  // namespace detail

// bench.cpp:201-261: validate, calibrate with the Constant writer, then one
// row per method. The guard (GuardError) keeps the reference's purpose — no
// rows from a run too small to time the memory system — in GPU terms: the
// reference demands >= min_run_seconds of one CPU Constant run, which no
// HBM-sized GPU run reaches (2^30 doubles take ~1.4 ms); here the calibration
// run must write more bytes than the device's L2 holds (otherwise it times
// the cache). min_run_seconds = 0 disables the guard as in the reference.
inline std::vector<BenchReport> run(const BenchConfig& config) {
    std::vector<std::string> methods = config.methods;
    if (methods.empty()) methods = {"Ref128", "LEcuyer", "Barrett", "BarrettModified", "Constant"};
    for (const auto& m : methods) detail::engine_for(m);  // reject unknown names before any work
    if (config.n == 0 || config.repeats < 1) throw std::invalid_argument("bench: n and repeats must be >= 1");
    const unsigned workers = config.workers ? config.workers : default_workers();
    const BenchReport calibration = detail::measure(config, "Constant", workers);
    if (config.min_run_seconds > 0.0 && config.n * sizeof(double) <= bcn_l2_bytes(-1))
        throw GuardError("bench: calibration run fits in the GPU's L2 cache; increase n");
    std::vector<BenchReport> reports;
    for (const auto& m : methods)
        reports.push_back(m == "Constant" ? calibration : detail::measure(config, m, workers));
    return reports;
}

inline void write_table(std::ostream& os, const std::vector<BenchReport>& reports) {
    char line[200];
    std::snprintf(line, sizeof(line), "%-16s %14s %12s %12s %12s %12s %8s %12s\n", "method", "elements",
                  "exec_s", "total_s", "exec_GNum/s", "total_GNum/s", "workers", "layout");
    os << line;
    for (const auto& r : reports) {
        std::snprintf(line, sizeof(line), "%-16s %14llu %12.6f %12.6f %12.4f %12.4f %8u %12s\n",
                      r.method.c_str(), static_cast<unsigned long long>(r.elements), r.exec_seconds,
                      r.total_seconds, r.exec_rate_gnum, r.total_rate_gnum, r.workers,
                      par::layout_name(r.layout));
        os << line;
    }
}

inline void write_csv(std::ostream& os, const std::vector<BenchReport>& reports) {
    os << "method,elements,exec_seconds,total_seconds,exec_rate_gnum,total_rate_gnum,workers,layout\n";
    for (const auto& r : reports) {
        char line[200];
        std::snprintf(line, sizeof(line), "%s,%llu,%.9g,%.9g,%.9g,%.9g,%u,%s\n", r.method.c_str(),
                      static_cast<unsigned long long>(r.elements), r.exec_seconds, r.total_seconds,
                      r.exec_rate_gnum, r.total_rate_gnum, r.workers, par::layout_name(r.layout));
        os << line;
    }
}

}  // namespace bcn::bench
