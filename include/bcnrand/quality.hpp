#pragma once

// B200 drop-in for /root/reference/proj/include/bcnrand/quality.hpp: the
// statistical smoke suite computed on the GPU (bcn_chi_square_uniformity,
// bcn_monobit_mantissa, bcn_serial_correlation in include/bcnrand_b200.h).
// Same reports, preconditions and pass bands (quality.cpp:21-140).

#include <cmath>
#include <cstdint>
#include <iomanip>
#include <ostream>
#include <sstream>
#include <span>
#include <string>

#include "bcnrand/generator.hpp"

namespace bcn::quality {

// quality.hpp:16-22
struct QualityReport {
    std::string name;
    double statistic = 0.0;
    int dof = 0;
    bool pass = false;
    std::string threshold;
};

namespace detail {
inline std::string band(const char* lhs, double bound) {
    std::ostringstream o;
    o << lhs << " <= " << std::setprecision(4) << bound;
    return o.str();
}
}  // namespace detail

// quality.hpp:27 — two-sided chi-square over `bins` equal-width bins of (0,1).
inline QualityReport chi_square_uniformity(std::span<const double> samples, int bins) {
    double stat = 0.0;
    int dof = 0, pass = 0;
    b200::check(bcn_chi_square_uniformity(samples.data(), samples.size(), bins, &stat, &dof, &pass, -1,
                                          nullptr));
    QualityReport r;
    r.name = "chi_square_uniformity";
    r.statistic = stat;
    r.dof = dof;
    r.pass = pass != 0;
    r.threshold = detail::band(("|stat - " + std::to_string(dof) + "|").c_str(), 4.5 * std::sqrt(2.0 * dof));
    return r;
}

// quality.hpp:33 — one-frequencies of the top 48 mantissa bits.
inline QualityReport monobit_mantissa(std::span<const Residue> residues) {
    static_assert(sizeof(Residue) == sizeof(std::uint64_t));
    double stat = 0.0;
    int worst = 5, pass = 0;
    b200::check(bcn_monobit_mantissa(reinterpret_cast<const std::uint64_t*>(residues.data()), residues.size(),
                                     &stat, &worst, &pass, -1, nullptr));
    QualityReport r;
    r.name = "monobit_mantissa";
    r.statistic = stat;
    r.dof = 48;
    r.pass = pass != 0;
    r.threshold = detail::band("max |ones/n - 1/2|", 4.5 / (2.0 * std::sqrt(static_cast<double>(residues.size())))) +
                  ", worst bit " + std::to_string(worst);
    return r;
}

// quality.hpp:37 — Pearson correlation between samples `lag` apart.
inline QualityReport serial_correlation(std::span<const double> samples, int lag = 1) {
    double rho = 0.0;
    int pass = 0;
    b200::check(bcn_serial_correlation(samples.data(), samples.size(), lag, &rho, &pass, -1, nullptr));
    const std::uint64_t pairs = samples.size() - static_cast<std::uint64_t>(lag);
    QualityReport r;
    r.name = lag == 1 ? "lag1_correlation" : "lag" + std::to_string(lag) + "_correlation";
    r.statistic = rho;
    r.dof = static_cast<int>(pairs > (std::uint64_t{1} << 30) ? (1 << 30) : pairs);
    r.pass = pass != 0;
    r.threshold = detail::band("|rho|", 4.5 / std::sqrt(static_cast<double>(samples.size())));
    return r;
}

// quality.hpp:40-45: an aligned human-readable table, and one
// `name=… statistic=… dof=… pass=…` line per report for scripts.
inline void write_table(std::ostream& os, std::span<const QualityReport> reports) {
    const auto row = [&os](const std::string& a, const std::string& b, const std::string& c,
                           const std::string& d, const std::string& e) {
        os << std::left << std::setw(26) << a << std::right << std::setw(16) << b << std::setw(10) << c
           << std::setw(7) << d << "   " << e << '\n';
    };
    row("test", "statistic", "dof", "pass", "threshold");
    for (const QualityReport& r : reports) {
        std::ostringstream stat;
        stat << std::setprecision(7) << r.statistic;
        row(r.name, stat.str(), std::to_string(r.dof), r.pass ? "yes" : "no", r.threshold);
    }
}

inline void write_kv(std::ostream& os, std::span<const QualityReport> reports) {
    for (const QualityReport& r : reports) {
        std::ostringstream line;
        line << "name=" << r.name << " statistic=" << std::setprecision(17) << r.statistic << " dof=" << r.dof
             << " pass=" << std::boolalpha << r.pass << '\n';
        os << line.str();
    }
}

}  // namespace bcn::quality
