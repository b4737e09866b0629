#pragma once

// B200 drop-in for the reference's command-line surface
// (/root/reference/proj/include/bcnrand/cli.hpp, src/cli.cpp): `bcn::cli::run`
// with the subcommands gen, bench, selftest and seed-info, the same options,
// byte formats and exit codes (0 ok, 1 selftest failure, 2 usage, 3 I/O).
// The reference parses with the vendored CLI11 (absent from the reference
// tree); this header carries its own small parser. `gen` streams the output
// in chunks of --chunk items: each chunk is one GPU fill at base_offset =
// items done (make_plan(chunk, workers, layout)), restored to logical order
// unless --keep-physical, and written as little-endian raw-u64 / raw-f64 or
// "%.17g" text lines (formatted in parallel by bcn_format_text). A failed
// command leaves no partial output file. tools/bcnrand_main.cpp wraps it as
// the `bcnrand` executable.

#include <algorithm>
#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <map>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "bcnrand/bench.hpp"
#include "bcnrand/generator.hpp"
#include "bcnrand/parallel.hpp"
#include "bcnrand/selftest.hpp"

namespace bcn::cli {

namespace detail {

enum Exit : int { kOk = 0, kSelftestFailed = 1, kUsage = 2, kIo = 3 };

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// `--name value` options, `--flag` switches and positionals after the
// subcommand; anything not declared is a usage error.
class Args {
  public:
    Args(const std::vector<std::string>& tokens, const std::set<std::string>& valued,
         const std::set<std::string>& flags) {
        for (std::size_t i = 0; i < tokens.size(); ++i) {
            const std::string& t = tokens[i];
            if (t.rfind("--", 0) != 0) {
                positional_.push_back(t);
            } else if (flags.count(t)) {
                flags_.insert(t);
            } else if (valued.count(t)) {
                if (i + 1 >= tokens.size()) throw UsageError(t + " needs a value");
                values_[t] = tokens[++i];
            } else {
                throw UsageError("unknown option " + t);
            }
        }
    }
    bool has(const std::string& k) const { return values_.count(k) != 0; }
    bool flag(const std::string& k) const { return flags_.count(k) != 0; }
    std::string text(const std::string& k, const std::string& dflt) const {
        auto it = values_.find(k);
        return it == values_.end() ? dflt : it->second;
    }
    std::uint64_t number(const std::string& k, std::uint64_t dflt) const {
        auto it = values_.find(k);
        return it == values_.end() ? dflt : parse_u64(it->second, k);
    }
    const std::vector<std::string>& positional() const { return positional_; }

    static std::uint64_t parse_u64(const std::string& s, const std::string& what) {
        if (s.empty() || s.find_first_not_of("0123456789") != std::string::npos)
            throw UsageError(what + ": expected a non-negative integer, got '" + s + "'");
        errno = 0;
        char* end = nullptr;
        const unsigned long long v = std::strtoull(s.c_str(), &end, 10);
        if (errno == ERANGE) throw UsageError(what + ": value out of range");
        return static_cast<std::uint64_t>(v);
    }

  private:
    std::map<std::string, std::string> values_;
    std::set<std::string> flags_;
    std::vector<std::string> positional_;
};

// Output file removed again unless commit() is reached; empty path = stdout.
class Sink {
  public:
    explicit Sink(const std::string& path) : path_(path) {
        if (!path_.empty()) {
            f_ = std::fopen(path_.c_str(), "wb");
            if (!f_) throw IoError("cannot open output file: " + path_);
        }
    }
    Sink(const Sink&) = delete;
    Sink& operator=(const Sink&) = delete;
    void write(const void* data, std::size_t bytes) {
        if (path_.empty()) {
            std::cout.write(static_cast<const char*>(data), static_cast<std::streamsize>(bytes));
            if (!std::cout) throw IoError("write failed: <stdout>");
        } else if (bytes && std::fwrite(data, 1, bytes, f_) != bytes) {
            throw IoError("write failed: " + path_);
        }
    }
    void commit() {
        if (path_.empty()) {
            std::cout.flush();
            if (!std::cout) throw IoError("write failed: <stdout>");
        } else {
            const bool ok = std::fclose(f_) == 0;
            f_ = nullptr;
            if (!ok) throw IoError("write failed: " + path_);
        }
        committed_ = true;
    }
    ~Sink() {
        if (f_) std::fclose(f_);
        if (!committed_ && !path_.empty()) std::remove(path_.c_str());
    }

  private:
    std::string path_;
    std::FILE* f_ = nullptr;
    bool committed_ = false;
};

template <typename T>
void write_le(Sink& sink, const std::vector<T>& v) {
    static_assert(sizeof(T) == 8);
    std::vector<unsigned char> bytes(v.size() * 8);
    for (std::size_t i = 0; i < v.size(); ++i) {
        std::uint64_t x;
        std::memcpy(&x, &v[i], 8);
        for (int b = 0; b < 8; ++b) bytes[i * 8 + b] = static_cast<unsigned char>(x >> (8 * b));
    }
    sink.write(bytes.data(), bytes.size());
}

inline void write_text(Sink& sink, const std::vector<double>& v) {
    std::vector<char> text(v.size() * 25 + 1);
    std::uint64_t written = 0;
    b200::check(bcn_format_text(v.data(), v.size(), text.data(), text.size(), &written));
    sink.write(text.data(), written);
}

inline int gen_command(const Args& a) {
    if (!a.has("--n")) throw UsageError("gen: --n is required");
    const gen::Method method = gen::parse_method(a.text("--method", "BarrettModified"));
    const par::Layout layout = par::parse_layout(a.text("--layout", "contiguous"));
    const std::uint64_t requested = a.number("--workers", 0);
    const unsigned workers = requested ? static_cast<unsigned>(requested) : bench::default_workers();
    const std::uint64_t seed = a.number("--seed", gen::kMinSeedIndex);
    const std::uint64_t n = a.number("--n", 0), chunk = a.number("--chunk", std::uint64_t{1} << 22);
    const std::string format = a.text("--format", "text");
    if (seed < gen::kMinSeedIndex || seed > gen::kMaxSeedIndex)
        throw UsageError("gen: seed outside [" + std::to_string(gen::kMinSeedIndex) + ", " +
                         std::to_string(gen::kMaxSeedIndex) + "]");
    if (n == 0 || chunk == 0) throw UsageError("gen: --n and --chunk must be at least 1");
    if (format != "text" && format != "raw-f64" && format != "raw-u64")
        throw UsageError("gen: unknown format " + format);
    const bool logical = layout == par::Layout::Contiguous || !a.flag("--keep-physical");

    Sink sink(a.text("--out", ""));
    std::vector<double> u;
    std::vector<std::uint64_t> z;
    for (std::uint64_t done = 0; done < n;) {
        const std::uint64_t m = std::min(chunk, n - done);
        const par::PartitionPlan plan = par::make_plan(m, workers, layout);
        if (format == "raw-u64") {
            z.resize(m);
            par::fill_residues(z, plan, seed, method, done);
            write_le(sink, logical && layout == par::Layout::Interleaved ? par::deinterleave(z, plan) : z);
        } else {
            u.resize(m);
            par::fill(u, plan, seed, method, done);
            const std::vector<double>& ordered =
                logical && layout == par::Layout::Interleaved ? par::deinterleave(u, plan) : u;
            if (format == "raw-f64")
                write_le(sink, ordered);
            else
                write_text(sink, ordered);
        }
        done += m;
    }
    sink.commit();
    return kOk;
}

inline std::vector<std::string> split_list(const std::string& s) {
    std::vector<std::string> out;
    std::stringstream in(s);
    for (std::string item; std::getline(in, item, ',');)
        if (!item.empty()) out.push_back(item);
    return out;
}

inline int bench_command(const Args& a) {
    bench::BenchConfig cfg;
    cfg.n = a.number("--n", cfg.n);
    cfg.methods = split_list(a.text("--methods", ""));
    cfg.workers = static_cast<unsigned>(a.number("--workers", 0));
    cfg.layout = par::parse_layout(a.text("--layout", "contiguous"));
    cfg.repeats = static_cast<int>(a.number("--repeats", static_cast<std::uint64_t>(cfg.repeats)));
    cfg.variant = bench::parse_variant(a.text("--variant", "rolled"));
    cfg.seed_index = a.number("--seed", cfg.seed_index);
    const auto reports = bench::run(cfg);
    if (a.flag("--csv"))
        bench::write_csv(std::cout, reports);
    else
        bench::write_table(std::cout, reports);
    return kOk;
}

inline int selftest_command(const Args& a) {
    const auto results = selftest::run_all(a.flag("--fast"));
    std::size_t w = 0;
    for (const auto& r : results) w = std::max(w, r.name.size());
    for (const auto& r : results)
        std::cout << (r.pass ? "ok    " : "FAIL  ") << r.name << std::string(w + 2 - r.name.size(), ' ')
                  << r.detail << '\n';
    const bool ok = selftest::all_passed(results);
    std::cout << (ok ? "selftest: all checks passed" : "selftest: FAILED") << std::endl;
    return ok ? kOk : kSelftestFailed;
}

inline int seed_info_command(const Args& a) {
    if (a.positional().size() != 1) throw UsageError("seed-info: expected one index");
    const std::uint64_t idx = Args::parse_u64(a.positional()[0], "seed-info");
    if (idx < gen::kMinSeedIndex || idx > gen::kMaxSeedIndex)
        throw UsageError("seed-info: index outside [" + std::to_string(gen::kMinSeedIndex) + ", " +
                         std::to_string(gen::kMaxSeedIndex) + "]");
    const gen::GeneratorState st = gen::seed_from_index(idx);
    char u[40];
    std::snprintf(u, sizeof(u), "%.17g", gen::to_unit_interval(st.z));
    std::cout << "index a        = " << idx << '\n'
              << "a - 3^33       = " << idx - modred::kModulus << '\n'
              << "2^53 - a       = " << gen::kMaxSeedIndex - idx << '\n'
              << "z0             = " << st.z.value << '\n'
              << "z0 * 3^-33     = " << u << std::endl;
    return kOk;
}

inline void usage(std::ostream& os) {
    os << "usage: bcnrand <gen|bench|selftest|seed-info> [options]\n"
          "  gen --n N [--seed A] [--method Ref128|LEcuyer|Barrett|BarrettModified] [--workers W]\n"
          "      [--layout contiguous|interleaved] [--format text|raw-f64|raw-u64] [--out PATH]\n"
          "      [--keep-physical] [--chunk C]\n"
          "  bench [--n N] [--methods a,b,...] [--workers W] [--layout L] [--repeats R]\n"
          "      [--variant rolled|unrolled] [--seed A] [--csv]\n"
          "  selftest [--fast]\n"
          "  seed-info A\n";
}

}  // namespace detail

inline int run(int argc, const char* const* argv) {
    using namespace detail;
    std::vector<std::string> tokens(argv + (argc > 0 ? 1 : 0), argv + (argc > 0 ? argc : 0));
    if (tokens.empty() || tokens[0] == "--help" || tokens[0] == "-h") {
        usage(tokens.empty() ? std::cerr : std::cout);
        return tokens.empty() ? kUsage : kOk;
    }
    const std::string cmd = tokens[0];
    tokens.erase(tokens.begin());
    try {
        if (cmd == "gen")
            return gen_command(Args(tokens,
                                    {"--n", "--seed", "--method", "--workers", "--layout", "--format", "--out",
                                     "--chunk"},
                                    {"--keep-physical"}));
        if (cmd == "bench")
            return bench_command(Args(
                tokens, {"--n", "--methods", "--workers", "--layout", "--repeats", "--variant", "--seed"}, {"--csv"}));
        if (cmd == "selftest") return selftest_command(Args(tokens, {}, {"--fast"}));
        if (cmd == "seed-info") return seed_info_command(Args(tokens, {}, {}));
        throw UsageError("unknown subcommand '" + cmd + "'");
    } catch (const IoError& e) {
        std::cerr << "i/o error: " << e.what() << '\n';
        return kIo;
    } catch (const bench::GuardError& e) {
        std::cerr << e.what() << '\n';
        return kUsage;
    } catch (const UsageError& e) {
        std::cerr << "error: " << e.what() << '\n';
        usage(std::cerr);
        return kUsage;
    } catch (const std::exception& e) {  // invalid_argument, out_of_range, domain_error, ...
        std::cerr << "error: " << e.what() << '\n';
        return kUsage;
    }
}

}  // namespace bcn::cli
