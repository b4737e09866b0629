#pragma once

// B200 drop-in for /root/reference/proj/include/bcnrand/parallel.hpp. The
// plan types and signatures are the reference's; fill / fill_residues run the
// sm_100a kernels through bcn_fill (include/bcnrand_b200.h) — the caller's
// span may be host memory (generated on the GPU, copied back in chunks) or a
// device pointer wrapped in a span. The logical result is bit-identical to the
// reference for every plan, layout and base_offset (tests/test_gpu_fill.py and
// the reference's own tests built against these headers, tests/test_dropin.py).

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "bcnrand/generator.hpp"

namespace bcn::par {

// parallel.hpp:15
enum class Layout { Contiguous, Interleaved };

namespace detail {
struct LayoutName {
    Layout layout;
    const char* text;
};
inline constexpr LayoutName kLayoutNames[] = {{Layout::Contiguous, "contiguous"},
                                              {Layout::Interleaved, "interleaved"}};
}  // namespace detail

inline const char* layout_name(Layout layout) {
    for (const auto& e : detail::kLayoutNames)
        if (e.layout == layout) return e.text;
    return "?";
}

// The lower-case names above; anything else is std::invalid_argument.
inline Layout parse_layout(const std::string& text) {
    for (const auto& e : detail::kLayoutNames)
        if (text == e.text) return e.layout;
    throw std::invalid_argument("parse_layout: no layout named '" + text + "'");
}

// parallel.hpp:17-38
struct PartitionPlan {
    std::uint64_t n = 0;
    unsigned workers = 1;
    std::uint64_t work_per_worker = 0;
    std::vector<std::uint64_t> start_offsets;
    Layout layout = Layout::Contiguous;
    std::uint64_t step = 1;

    std::uint64_t elements_for(unsigned w) const {
        const std::uint64_t start = start_offsets[w];
        return work_per_worker < n - start ? work_per_worker : n - start;
    }

    std::uint64_t physical_index(unsigned w, std::uint64_t i) const {
        std::uint64_t slot = 0;
        b200::check(bcn_physical_index(n, workers,
                                       layout == Layout::Contiguous ? BCN_LAYOUT_CONTIGUOUS
                                                                    : BCN_LAYOUT_INTERLEAVED,
                                       w, i, &slot));
        return slot;
    }
};

// parallel.hpp:42 — n = 0 or workers = 0 is std::invalid_argument.
inline PartitionPlan make_plan(std::uint64_t n, unsigned workers, Layout layout) {
    std::uint32_t effective = 0;
    std::uint64_t per_worker = 0;
    b200::check(bcn_make_plan(n, workers, &effective, &per_worker));
    PartitionPlan plan;
    plan.n = n;
    plan.workers = effective;
    plan.work_per_worker = per_worker;
    plan.layout = layout;
    plan.step = effective;
    plan.start_offsets.resize(effective);
    std::uint64_t start = 0;
    for (auto& s : plan.start_offsets) {
        s = start;
        start += per_worker;
    }
    return plan;
}

namespace detail {
inline bcn_layout layout_of(Layout l) {
    return l == Layout::Contiguous ? BCN_LAYOUT_CONTIGUOUS : BCN_LAYOUT_INTERLEAVED;
}
inline bcn_method method_of(gen::Method m) { return static_cast<bcn_method>(static_cast<int>(m)); }
}  // namespace detail

// parallel.hpp:48-49 — plan.n unit-interval variates; a buffer smaller than
// plan.n is std::invalid_argument before any work.
inline void fill(std::span<double> out, const PartitionPlan& plan, std::uint64_t seed_index,
                 gen::Method method, std::uint64_t base_offset = 0) {
    b200::check(bcn_fill(out.data(), out.size(), plan.n, BCN_FORMAT_F64, plan.workers,
                         detail::layout_of(plan.layout), seed_index, detail::method_of(method),
                         base_offset, BCN_ENGINE_AUTO, -1, nullptr));
}

// parallel.hpp:52-54 — the raw residues z_k.
inline void fill_residues(std::span<std::uint64_t> out, const PartitionPlan& plan,
                          std::uint64_t seed_index, gen::Method method,
                          std::uint64_t base_offset = 0) {
    b200::check(bcn_fill(out.data(), out.size(), plan.n, BCN_FORMAT_U64, plan.workers,
                         detail::layout_of(plan.layout), seed_index, detail::method_of(method),
                         base_offset, BCN_ENGINE_AUTO, -1, nullptr));
}

// Extension (no reference counterpart): float32 variates, RZ of the double.
inline void fill_float(std::span<float> out, const PartitionPlan& plan, std::uint64_t seed_index,
                       gen::Method method, std::uint64_t base_offset = 0) {
    b200::check(bcn_fill(out.data(), out.size(), plan.n, BCN_FORMAT_F32, plan.workers,
                         detail::layout_of(plan.layout), seed_index, detail::method_of(method),
                         base_offset, BCN_ENGINE_AUTO, -1, nullptr));
}

namespace detail {
// One device transpose (bcn_deinterleave); host spans are staged through the GPU.
template <typename Item>
std::vector<Item> to_logical_order(std::span<const Item> physical, const PartitionPlan& plan) {
    if (plan.layout == Layout::Contiguous)
        throw std::invalid_argument("deinterleave: plan layout is not Interleaved");
    if (physical.size() < plan.n) throw std::invalid_argument("deinterleave: buffer smaller than plan.n");
    std::vector<Item> logical(plan.n);
    b200::check(bcn_deinterleave(physical.data(), logical.data(), plan.n, plan.workers,
                                 static_cast<std::uint32_t>(sizeof(Item)), -1, nullptr));
    return logical;
}
}  // namespace detail

// parallel.hpp:58-60
inline std::vector<double> deinterleave(std::span<const double> buffer, const PartitionPlan& plan) {
    return detail::to_logical_order(buffer, plan);
}
inline std::vector<std::uint64_t> deinterleave(std::span<const std::uint64_t> buffer, const PartitionPlan& plan) {
    return detail::to_logical_order(buffer, plan);
}

}  // namespace bcn::par
