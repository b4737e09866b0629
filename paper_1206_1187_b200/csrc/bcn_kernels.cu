// bcn_kernels.cu — sm_100a kernels for the alpha_{2,3} generator fill path.
//
// Kernel inventory:
//   k_fill_paced<FMT, ENG, MODE>  the default 8-byte fill: grid-strided 1 KiB rows,
//                                 8 worker warps + 1 pacer warp per CTA metering the
//                                 stores to a target HBM write rate; MODE selects the
//                                 contiguous layout, the reference Layout::Interleaved,
//                                 or the Constant / noise writer.
//   k_fill_contig<FMT, ENG>       unpaced logical-order fill (f32, integer engines),
//                                 lane-interleaved jump streams, 256-bit stores,
//                                 persistent grid. Both contiguous kernels write the
//                                 partial first / last rows themselves (EdgeRow).
//   k_fill_interleaved<FMT, ENG>  unpaced Layout::Interleaved (per-stream row-crossing
//                                 multiplier).
//   k_fill_bulk<FMT, ENG>         FP64 jump streams staged in smem, TMA bulk stores.
//   k_fill_staged<FMT>            the paper's T=1 modified-Barrett step per thread,
//                                 tile staged in smem, TMA bulk store per tile.
//   k_fill_slots<FMT>             exact per-slot reference semantics (interleaved
//                                 heads/tails, u64-wrap corner cases); one seed per slot.
//   k_seed                        batched state_at / next walks (skip-ahead stress).
//   k_digest                      order-sensitive checksums for verification.
//   k_engine_check<ENG>           z * c^r mod m through one jump engine on arbitrary
//                                 operands (bcn_engine_check, engine self-check).
//   k_constant                    the unpaced Constant writer: identical access
//                                 pattern, fixed value (the paper's memory ceiling).
//   k_transpose, k_transpose_narrow
//                                 device deinterleave (Interleaved -> logical),
//                                 pipelined shared-memory tiles.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <algorithm>
#include <atomic>
#include <mutex>
#include <type_traits>

#include "bcn_kernels.cuh"

namespace bcn_b200 {

// --------------------------------------------------------------- seed tables
// g_pow[i][d] = {2^(d 16^i) mod m, Shoup(...)} for 13 4-bit windows.
__device__ uint64_t g_pow[kPowWindows][16][2];

// 2^E mod m for E < P: 13 table multiplies (12 Barrett/Shoup products).
__device__ __forceinline__ uint64_t dev_pow2(uint64_t e) {
    uint64_t acc = __ldg(&g_pow[0][e & 15][0]);
    e >>= 4;
#pragma unroll
    for (int i = 1; i < kPowWindows; ++i) {
        const unsigned d = static_cast<unsigned>(e & 15);
        e >>= 4;
        acc = mul_barrett(acc, __ldg(&g_pow[i][d][0]), __ldg(&g_pow[i][d][1]));
    }
    return acc;
}

// Canonical state with 2-exponent E: z = m - (2^E mod m), never 0.
__device__ __forceinline__ uint64_t dev_state_from_exp(uint64_t e) {
    return kModulus - dev_pow2(e);
}

// (e0 + 53 j) mod P for e0 < P and j < 2^40 (53 j < 2^46 < P).
__device__ __forceinline__ uint64_t dev_exp_at(uint64_t e0, uint64_t j) {
    uint64_t e = e0 + 53ull * j;
    return e >= kPeriod ? e - kPeriod : e;
}

// ------------------------------------------------------------------ engines
template <int ENG>
struct Eng;

template <>
struct Eng<kEngBarrett> {
    using State = uint64_t;
    static __device__ __forceinline__ State from_canonical(uint64_t z) { return z; }
    static __device__ __forceinline__ State mul(State s, const Mult& k) {
        return mul_barrett(s, k.c, k.shoup);
    }
    static __device__ __forceinline__ uint64_t raw(State s) { return s; }
    static __device__ __forceinline__ double unit(State s) { return unit_from_u64(s); }
};

template <>
struct Eng<kEngMontgomery> {
    using State = uint64_t;
    static __device__ __forceinline__ State from_canonical(uint64_t z) { return z; }
    static __device__ __forceinline__ State mul(State s, const Mult& k) {
        return mul_montgomery(s, k.mont);
    }
    static __device__ __forceinline__ uint64_t raw(State s) { return s; }
    static __device__ __forceinline__ double unit(State s) { return unit_from_u64(s); }
};

template <>
struct Eng<kEngFP64> {
    using State = double;  // balanced residue, |s| <= 0.75 m, integer valued
    static __device__ __forceinline__ State from_canonical(uint64_t z) {
        return z > kModulus / 2 ? static_cast<double>(static_cast<int64_t>(z - kModulus))
                                : static_cast<double>(z);
    }
    static __device__ __forceinline__ State mul(State s, const Mult& k) {
        return mul_fp64(s, k.cb, k.com);
    }
    static __device__ __forceinline__ uint64_t raw(State s) {
        return __double2ull_rz(fp64_canonical(s));
    }
    static __device__ __forceinline__ double unit(State s) {
        return __dmul_rn(fp64_canonical(s), kInvModulus);
    }
};

template <>
struct Eng<kEngMixed> {
    using State = MixedState;  // balanced integer + its exact double image
    static __device__ __forceinline__ State from_canonical(uint64_t z) {
        const int64_t b = z > kModulus / 2 ? static_cast<int64_t>(z - kModulus) : static_cast<int64_t>(z);
        return State{b, static_cast<double>(b)};
    }
    static __device__ __forceinline__ State mul(State s, const Mult& k) {
        return mul_mixed(s, k.com, k.cbi);
    }
    // Sign mask from the integer's high word: z = s + (s < 0 ? m : 0).
    static __device__ __forceinline__ uint64_t raw(State s) {
        const uint64_t mask = static_cast<uint64_t>(s.s >> 63);
        return static_cast<uint64_t>(s.s) + (mask & kModulus);
    }
    static __device__ __forceinline__ double unit(State s) {
        const uint64_t mask = static_cast<uint64_t>(s.s >> 63);
        const double add = __longlong_as_double(static_cast<long long>(
            mask & static_cast<uint64_t>(__double_as_longlong(kModulusD))));
        return __dmul_rn(__dadd_rn(s.d, add), kInvModulus);
    }
};

// Index-aware view of an engine: a lane's V streams may run on different
// engines (Hybrid below), so every operation takes the stream's index v
// inside the lane's vector. The loops over v are fully unrolled, so v is a
// constant and the per-stream choice folds away at compile time.
template <class E>
struct EI {
    using State = typename E::State;
    static __device__ __forceinline__ State from(uint64_t z, int) { return E::from_canonical(z); }
    static __device__ __forceinline__ State mul(State s, const Mult& k, int) { return E::mul(s, k); }
    static __device__ __forceinline__ uint64_t raw(State s, int) { return E::raw(s); }
    static __device__ __forceinline__ double unit(State s, int) { return E::unit(s); }
};

// Hybrid engine: streams v < KF of each lane on the FP64 engine (FP64 pipe),
// the rest on the Shoup-Barrett engine (IMAD + ALU pipes), so both pipes share
// the jump multiplies of one row. The state register
// holds the FP64 state's bits or the canonical residue.
template <int KF>
struct Hyb {};
template <int KF>
struct EI<Hyb<KF>> {
    using State = uint64_t;
    using F = Eng<kEngFP64>;
    using B = Eng<kEngBarrett>;
    static __device__ __forceinline__ double d(State s) { return __longlong_as_double(static_cast<long long>(s)); }
    static __device__ __forceinline__ State u(double x) { return static_cast<State>(__double_as_longlong(x)); }
    static __device__ __forceinline__ State from(uint64_t z, int v) {
        return v < KF ? u(F::from_canonical(z)) : B::from_canonical(z);
    }
    static __device__ __forceinline__ State mul(State s, const Mult& k, int v) {
        return v < KF ? u(F::mul(d(s), k)) : B::mul(s, k);
    }
    static __device__ __forceinline__ uint64_t raw(State s, int v) { return v < KF ? F::raw(d(s)) : B::raw(s); }
    static __device__ __forceinline__ double unit(State s, int v) { return v < KF ? F::unit(d(s)) : B::unit(s); }
};

// Engine id -> index-aware engine. Hybrid ids are kEngHybridBase + KF.
template <int ENG, bool HYB = (ENG >= kEngHybridBase)>
struct EngSel {
    using type = EI<Eng<ENG>>;
};
template <int ENG>
struct EngSel<ENG, true> {
    using type = EI<Hyb<ENG - kEngHybridBase>>;
};
template <int ENG>
using EngOf = typename EngSel<ENG>::type;

// --------------------------------------------------------------- formats
template <int FMT>
struct Fmt;
template <>
struct Fmt<kFmtU64> {
    static constexpr int kVec = 4;  // 4 x 8 B = one 256-bit store per lane
    using Item = uint64_t;
};
template <>
struct Fmt<kFmtF64> {
    static constexpr int kVec = 4;
    using Item = double;
};
template <>
struct Fmt<kFmtF32> {
    static constexpr int kVec = 8;  // 8 x 4 B
    using Item = float;
};

template <int FMT, class E>
__device__ __forceinline__ uint64_t emit_bits(typename E::State s, int v) {
    if constexpr (FMT == kFmtU64) {
        return E::raw(s, v);
    } else if constexpr (FMT == kFmtF64) {
        return static_cast<uint64_t>(__double_as_longlong(E::unit(s, v)));
    } else {
        return static_cast<uint64_t>(__float_as_uint(f32_rz_from_unit(E::unit(s, v))));
    }
}

// The emitted bits of N streams. (An f32 conversion with one FP64 op instead
// of two — the canonical add folded into the scaling FMA, y = RN(s kInv +
// [s < 0]), exact except within 4 ulps of a 24-bit boundary, with a rare exact
// fallback — saved a DP op per variate but added ~3 integer ops and a branch:
// 5.09 vs 5.65 TB/s median, 5.78 vs 6.35 best, profiles/r02/ab_f32_conversion.jsonl.)
template <int FMT, class E, int N>
__device__ __forceinline__ void emit_vec(const typename E::State (&st)[N], uint64_t (&bits)[N]) {
#pragma unroll
    for (int v = 0; v < N; ++v) bits[v] = emit_bits<FMT, E>(st[v], v);
}

// 32-byte store: st.global.v4.b64 / v8.b32 -> SASS STG.E.256 on sm_100a.
__device__ __forceinline__ void st256(void* p, const uint64_t (&v)[4]) {
    asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(v[0]), "l"(v[1]),
                 "l"(v[2]), "l"(v[3])
                 : "memory");
}

template <int FMT>
__device__ __forceinline__ void pack_store(void* p, const uint64_t (&bits)[Fmt<FMT>::kVec]) {
    uint64_t w[4];
    if constexpr (Fmt<FMT>::kVec == 4) {
#pragma unroll
        for (int i = 0; i < 4; ++i) w[i] = bits[i];
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) w[i] = bits[2 * i] | (bits[2 * i + 1] << 32);
    }
    st256(p, w);
}

// One partial row (EdgeRow), written by a whole warp: each lane seeds its V
// elements (one windowed power + T=1 steps), converts them with the canonical
// path (bit-identical to every engine) and stores the in-range ones.
template <int FMT>
__device__ __forceinline__ void fill_edge_row(const EdgeRow& er, unsigned lane) {
    constexpr int V = Fmt<FMT>::kVec;
    using Item = typename Fmt<FMT>::Item;
    const uint32_t t0 = lane * V;
    uint64_t z = dev_state_from_exp(dev_exp_at(er.e0, t0));
    uint64_t bits[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
        if constexpr (FMT == kFmtU64)
            bits[v] = z;
        else if constexpr (FMT == kFmtF64)
            bits[v] = static_cast<uint64_t>(__double_as_longlong(unit_from_u64(z)));
        else
            bits[v] = __float_as_uint(f32_rz_from_unit(unit_from_u64(z)));
        if (v + 1 < V) z = step_modified_barrett(z);
    }
    char* p = static_cast<char*>(er.base) + t0 * sizeof(Item);
    if (t0 >= er.lo && t0 + V <= er.hi) {
        pack_store<FMT>(p, bits);
    } else {
#pragma unroll
        for (int v = 0; v < V; ++v)
            if (t0 + v >= er.lo && t0 + v < er.hi) {
                if constexpr (sizeof(Item) == 8)
                    reinterpret_cast<uint64_t*>(p)[v] = bits[v];
                else
                    reinterpret_cast<uint32_t*>(p)[v] = static_cast<uint32_t>(bits[v]);
            }
    }
}

// Warps 0 and 1 of CTA 0 write the head / tail edge rows, if any.
template <int FMT>
__device__ __forceinline__ void fill_edges(const EdgeRow (&edge)[2]) {
    const unsigned warp = threadIdx.x >> 5;
    if (blockIdx.x == 0 && warp < 2 && edge[warp].base) fill_edge_row<FMT>(edge[warp], threadIdx.x & 31);
}

// Splits `rows` over `nw` warps: warp w gets [begin, end).
__device__ __forceinline__ void warp_rows(uint64_t rows, uint64_t nw, uint64_t w, uint64_t& begin,
                                          uint64_t& end) {
    const uint64_t q = rows / nw, r = rows % nw;
    begin = w * q + (w < r ? w : r);
    end = begin + q + (w < r ? 1 : 0);
}

// ---------------------------------------------------------- contiguous fill
// A "row" is 32 lanes x kVec consecutive elements (1 KiB). Lane l holds kVec
// independent streams at elements row*ROW + l*kVec + v; every row each stream
// is multiplied by 2^(53 ROW) mod m. Consecutive lanes store consecutive
// 32-byte sectors, so every warp store is one fully coalesced 1 KiB write.
template <int FMT, int ENG>
__global__ void __launch_bounds__(kContigThreads) k_fill_contig(const ContigArgs a) {
    using E = EngOf<ENG>;
    constexpr int V = Fmt<FMT>::kVec;
    constexpr uint64_t ROW = 32ull * V;
    const unsigned lane = threadIdx.x & 31;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
    const uint64_t w = static_cast<uint64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    // Row order: contiguous per-warp ranges, or grid-strided (warp w writes rows
    // w, w+nw, ...; all warps sweep the buffer together, which keeps the DRAM
    // write stream local). jump_row advances a stream by `step` rows.
    uint64_t r, r_end, step;
    if (a.stride_order) {
        r = w;
        r_end = a.rows;
        step = nw;
    } else {
        warp_rows(a.rows, nw, w, r, r_end);
        step = 1;
    }
    fill_edges<FMT>(a.edge);
    if (r >= r_end) return;

    // Seed: one windowed power per lane, then T=1 steps for the lane's vector.
    typename E::State st[V];
    {
        uint64_t z = dev_state_from_exp(dev_exp_at(a.e0, r * ROW + lane * V));
#pragma unroll
        for (int v = 0; v < V; ++v) {
            st[v] = E::from(z, v);
            if (v + 1 < V) z = step_modified_barrett(z);
        }
    }
    const Mult k = a.jump_row;
    char* p = static_cast<char*>(a.out) + (r * ROW + lane * V) * sizeof(typename Fmt<FMT>::Item);
    constexpr uint64_t kRowBytes = ROW * sizeof(typename Fmt<FMT>::Item);
    const uint64_t pstep = step * kRowBytes;
#pragma unroll 2
    for (; r < r_end; r += step) {
        uint64_t bits[V];
        emit_vec<FMT, E>(st, bits);
        pack_store<FMT>(p, bits);
#pragma unroll
        for (int v = 0; v < V; ++v) st[v] = E::mul(st[v], k, v);
        p += pstep;
    }
}

// ------------------------------------------------------- paced contiguous fill
// HBM write efficiency on B200 collapses when SM stores oversubscribe the
// memory system (measured: ~6.3-6.4 TB/s back-to-back vs ~7.3-7.5 TB/s when
// the offered load is held just under capacity; profiles/r01/write_probe*.jsonl).
// This variant meters its own stores in real time: each CTA has 8 worker warps
// and one pacer warp. Workers generate their next 1 KiB row while the pacer
// waits on %globaltimer; every `gap` ns the pacer releases named barrier 1 and
// each worker stores the row it has ready. Rows are grid-strided (worker w of
// nwk writes rows w, w+nwk, ...), so the whole grid sweeps the buffer as one
// ordered stream at the target rate. With CONST the worker stores a fixed
// pattern (the paced Constant writer).
__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Shared-memory mbarriers of the pacer handshake (PTX mbarrier.*, sm_90+).
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
                 "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
                 : "memory");
}
// Blocks until the phase with parity `parity` has completed (try_wait sleeps
// in hardware between probes).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "BCN_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra BCN_WAIT;\n}" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
        "r"(parity)
        : "memory");
}

template <int FMT, int ENG, int MODE>
__global__ void __launch_bounds__(kPacedThreads) k_fill_paced(const PacedArgs a) {
    using E = EngOf<ENG>;
    constexpr bool CONST = MODE == kPacedConstant;
    constexpr bool INTER = MODE == kPacedInterleaved;  // per-stream row-crossing multiplier
    constexpr bool INTER_SEED = INTER || MODE == kPacedInterleavedFixed;
    constexpr int V = Fmt<FMT>::kVec;
    constexpr int H = paced_rows_per_round(FMT, CONST);  // rows per worker per round
    constexpr uint64_t ROW = 32ull * V;
    constexpr int kWorkers = kPacedThreads / 32 - 1;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t nwk = static_cast<uint64_t>(gridDim.x) * kWorkers;
    const uint64_t first = static_cast<uint64_t>(blockIdx.x) * kWorkers;
    // Worker w writes 1 KiB rows (ROW slots) at slots w*ROW + (H*k + h)*D,
    // h < H, for D = nwk*ROW (grid-strided rows; a round covers H*nwk rows) or
    // the interleaved super-row length a.row_stride (a multiple of the width
    // and of the 32-byte chunk; workers whose row would start past it idle).
    const uint64_t D = a.row_stride ? a.row_stride : nwk * ROW;
    const uint64_t N = a.rows * ROW;  // slots
    const uint64_t first_slot = first * ROW;
    const uint32_t rounds = first_slot < N && first_slot < D
                                ? static_cast<uint32_t>(((N - first_slot + D - 1) / D + H - 1) / H)
                                : 0;
    if constexpr (!CONST && !INTER_SEED) fill_edges<FMT>(a.edge);
    if (rounds == 0) return;  // uniform across the CTA
    // Interleaved: the two jump multipliers in shared memory, so a stream picks
    // its multiplier with one indexed (broadcast) load instead of selects.
    __shared__ Mult jumps[2];
    if constexpr (INTER) {
        if (threadIdx.x == 0) {
            jumps[0] = a.jump;
            jumps[1] = a.jump_wrap;
        }
    }
    // Pacer handshake on two shared-memory mbarriers. `release` completes one
    // phase per round when the pacer (one thread) arrives at the round's
    // scheduled time; `consumed` completes when all 8 worker warps have passed
    // that round's release, and the pacer waits for it before releasing the
    // next round, so no worker is ever more than one phase behind (the parity
    // waits stay unambiguous). Workers compute their next rows while the pacer
    // waits and store as soon as the release and their data are ready. (A
    // "ready" handshake — release only once every worker has computed the
    // round, r01's bar.sync semantics — serialises compute, two mbarrier
    // wake-ups and the stores: 4.8 TB/s whatever the target; metering in SM
    // cycles instead of %globaltimer ns did not raise the power-capped rate:
    // profiles/r02/pace_modes.jsonl.) Every thread reaches the one
    // __syncthreads() below (which also publishes `jumps`) from the same
    // instruction: synccheck-clean (profiles/r02/sanitizers.txt), unlike r01's
    // split aligned bar.sync.
    __shared__ uint64_t bar_release, bar_consumed;
    if (threadIdx.x == 0) {
        mbar_init(&bar_release, 1);
        mbar_init(&bar_consumed, kWorkers);
    }
    __syncthreads();
    if (warp == kWorkers) {
        // Pacer: release round k no earlier than t0 + k * gap (staggering the
        // CTAs' schedules or releasing each worker separately measured no
        // better, profiles/r01/timeline_stagger.jsonl).
        if (lane != 0) return;
        const uint64_t t0 = global_ns();
        for (uint32_t k = 0; k < rounds; ++k) {
            if (k > 0) mbar_wait(&bar_consumed, (k - 1) & 1);
            if (a.gap_q8) {
                const uint64_t target = t0 + ((static_cast<uint64_t>(k) * a.gap_q8) >> 8);
                uint64_t now = global_ns();
                while (now < target) {
                    const uint64_t d = target - now;
                    __nanosleep(d > 2048 ? 1024u : static_cast<unsigned>(d >> 1));
                    now = global_ns();
                }
            }
            mbar_arrive(&bar_release);
        }
        return;
    }
    const uint64_t w = first + warp;
    // Rows this lane's chunk takes part in (its chunk is whole or absent in
    // every row: D and N are multiples of the 32-byte chunk).
    const uint64_t w_slot = w * ROW + lane * V;
    const uint32_t count = w_slot < D && w_slot < N ? static_cast<uint32_t>((N - w_slot + D - 1) / D) : 0;
    typename E::State st[H][V];
    // interleaved: worker index of each stream's slot (< width < 2^32). A
    // stream stays in the same physical row iff col < same_below; col then
    // advances by adv_b, otherwise by adv_b - width (mod 2^32).
    uint32_t col[INTER ? H : 1][INTER ? V : 1];
    const uint32_t same_below = static_cast<uint32_t>(a.width - a.adv_b);
    const uint32_t adv_same = static_cast<uint32_t>(a.adv_b);
    const uint32_t adv_wrap = static_cast<uint32_t>(a.adv_b - a.width);
    // Constant writer pattern: a.e0 everywhere, or (a.q0 != 0, exploration)
    // fixed per-thread random words, to separate data-toggling power from
    // generator power.
    uint64_t pat[CONST ? H : 1][CONST ? V : 1];
    if constexpr (CONST) {
#pragma unroll
        for (int h = 0; h < H; ++h)
#pragma unroll
            for (int v = 0; v < V; ++v) {
                uint64_t x = a.q0 + 0x9e3779b97f4a7c15ull *
                                        ((static_cast<uint64_t>(blockIdx.x) * kPacedThreads + threadIdx.x) * (H * V) + h * V + v + 1);
                x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
                x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
                pat[h][v] = a.q0 ? (x ^ (x >> 31)) : a.e0;
            }
    }
    if (!CONST) {
#pragma unroll
        for (int h = 0; h < H; ++h) {
            if constexpr (INTER_SEED) {
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const uint64_t q = a.q0 + w_slot + h * D + v;
                    const uint64_t c = q % a.width;
                    if constexpr (INTER) col[h][v] = static_cast<uint32_t>(c);
                    const uint64_t j = c * a.wpw + a.i_base + q / a.width;
                    st[h][v] = E::from(dev_state_from_exp(dev_exp_at(a.e0, j)), v);
                }
            } else {
                uint64_t z = dev_state_from_exp(dev_exp_at(a.e0, w_slot + h * D));
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    st[h][v] = E::from(z, v);
                    if (v + 1 < V) z = step_modified_barrett(z);
                }
            }
        }
    }
    char* p = static_cast<char*>(a.out) + w_slot * sizeof(typename Fmt<FMT>::Item);
    const uint64_t hstep = D * sizeof(typename Fmt<FMT>::Item);
    const Mult k = a.jump;
    uint32_t r = 0;  // this worker's rows done
    for (uint32_t rd = 0; rd < rounds; ++rd, r += H) {
        uint64_t bits[H][V];
#pragma unroll
        for (int h = 0; h < H; ++h) {
            if constexpr (CONST) {
#pragma unroll
                for (int v = 0; v < V; ++v) bits[h][v] = pat[h][v];
            } else {
                emit_vec<FMT, E>(st[h], bits[h]);
            }
        }
        // Interleaved: this round's multiplier of every stream, loaded before
        // the pacer barrier so the shared-memory latency overlaps the wait.
        Mult sel[INTER ? H : 1][INTER ? V : 1];
        if constexpr (INTER) {
#pragma unroll
            for (int h = 0; h < H; ++h)
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const bool same = col[h][v] < same_below;
                    sel[h][v] = jumps[same ? 0 : 1];
                    col[h][v] += same ? adv_same : adv_wrap;
                }
        }
        mbar_wait(&bar_release, rd & 1);
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_consumed);
        if (r + H <= count) {
#pragma unroll
            for (int h = 0; h < H; ++h) pack_store<FMT>(p + h * hstep, bits[h]);
        } else {
#pragma unroll
            for (int h = 0; h < H; ++h)
                if (r + h < count) pack_store<FMT>(p + h * hstep, bits[h]);
        }
        if constexpr (INTER) {
#pragma unroll
            for (int h = 0; h < H; ++h)
#pragma unroll
                for (int v = 0; v < V; ++v) st[h][v] = E::mul(st[h][v], sel[h][v], v);
        } else if constexpr (!CONST) {
#pragma unroll
            for (int h = 0; h < H; ++h)
#pragma unroll
                for (int v = 0; v < V; ++v) st[h][v] = E::mul(st[h][v], k, v);
        }
        p += H * hstep;
    }
}

// -------------------------------------------------------- interleaved fill
template <int FMT, int ENG>
__global__ void __launch_bounds__(kContigThreads) k_fill_interleaved(const InterleavedArgs a) {
    using E = EngOf<ENG>;
    constexpr int V = Fmt<FMT>::kVec;
    constexpr uint64_t ROW = 32ull * V;
    const unsigned lane = threadIdx.x & 31;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
    const uint64_t w = static_cast<uint64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    uint64_t r, r_end;
    warp_rows(a.rows, nw, w, r, r_end);
    if (r >= r_end) return;

    typename E::State st[V];
    uint32_t col[V];  // worker index of each stream's current slot (see k_fill_paced)
    const uint32_t same_below = static_cast<uint32_t>(a.width - a.adv_b);
    const uint32_t adv_same = static_cast<uint32_t>(a.adv_b);
    const uint32_t adv_wrap = static_cast<uint32_t>(a.adv_b - a.width);
#pragma unroll
    for (int v = 0; v < V; ++v) {
        const uint64_t q = a.q0 + r * ROW + lane * V + v;
        col[v] = static_cast<uint32_t>(q % a.width);
        const uint64_t j = col[v] * a.wpw + a.i_base + q / a.width;
        st[v] = E::from(dev_state_from_exp(dev_exp_at(a.e0, j)), v);
    }
    char* p = static_cast<char*>(a.out) + (r * ROW + lane * V) * sizeof(typename Fmt<FMT>::Item);
    constexpr uint64_t kRowBytes = ROW * sizeof(typename Fmt<FMT>::Item);
    for (; r < r_end; ++r) {
        uint64_t bits[V];
        emit_vec<FMT, E>(st, bits);
        pack_store<FMT>(p, bits);
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const bool same = col[v] < same_below;
            st[v] = E::mul(st[v], same ? a.jump_same : a.jump_wrap, v);
            col[v] += same ? adv_same : adv_wrap;
        }
        p += kRowBytes;
    }
}

// ------------------------------------------------------------- slot fill
// Exact reference semantics for arbitrary slots: physical slot p -> (w, i)
// (parallel.cpp:24-33) -> state after i+1 steps from state_at(a, B + start_w)
// with B + start_w wrapping mod 2^64 exactly as the reference's u64 does.
__device__ __forceinline__ void slot_to_worker(const SlotArgs& a, uint64_t p, uint64_t& w,
                                               uint64_t& i) {
    if (a.layout == 0) {
        w = p / a.wpw;
        i = p % a.wpw;
        return;
    }
    const uint64_t last_start = static_cast<uint64_t>(a.workers - 1) * a.wpw;
    const uint64_t short_count = a.n - last_start < a.wpw ? a.n - last_start : a.wpw;
    const uint64_t main = short_count * a.workers;
    if (p < main) {
        w = p % a.workers;
        i = p / a.workers;
    } else {
        const uint64_t q = p - main, width = a.workers - 1;
        w = q % width;
        i = short_count + q / width;
    }
}

template <int FMT>
__global__ void __launch_bounds__(128) k_fill_slots(const SlotArgs a) {
    const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= a.count) return;
    uint64_t w, i;
    slot_to_worker(a, a.slot0 + t, w, i);
    const uint64_t kw = a.base_offset + w * a.wpw;  // wraps mod 2^64 like the reference
    const uint64_t steps = (kw % kPeriod + (i % kPeriod) + 1) % kPeriod;
    const uint64_t e = (a.a_exp + (53ull * steps) % kPeriod) % kPeriod;
    const uint64_t z = dev_state_from_exp(e);
    using Item = typename Fmt<FMT>::Item;
    Item* out = static_cast<Item*>(a.out) + t;
    if constexpr (FMT == kFmtU64) {
        *out = z;
    } else if constexpr (FMT == kFmtF64) {
        *out = unit_from_u64(z);
    } else {
        *out = f32_rz_from_unit(unit_from_u64(z));
    }
}

// ----------------------------------------------------------- staged (TMA)
// The paper's design (Fig. 3/4): each thread advances its own
// logically contiguous run with the T=1 modified Barrett step. Runs are
// written to shared memory at their logical positions (stride L words, L odd
// => conflict-free) and the whole tile leaves with ONE cp.async.bulk
// (TMA bulk store, SASS UBLKCP) issued by one thread; two tiles in flight.
template <int FMT>
__global__ void __launch_bounds__(kStagedThreads) k_fill_staged(const StagedArgs a) {
    using Item = typename Fmt<FMT>::Item;
    constexpr int L = kStagedL;
    constexpr uint32_t TILE = kStagedThreads * L;
    constexpr uint32_t TILE_BYTES = TILE * sizeof(Item);
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const unsigned tid = threadIdx.x;
    uint64_t tile = blockIdx.x;
    if (tile >= a.tiles) return;
    uint64_t z = dev_state_from_exp(dev_exp_at(a.e0, tile * TILE + tid * L));
    int b = 0;
    for (; tile < a.tiles; tile += gridDim.x, b ^= 1) {
        if (tid == 0) {
            // The bulk store issued two tiles ago read from this buffer.
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        }
        __syncthreads();
        Item* const tile_buf = reinterpret_cast<Item*>(smem_raw + b * TILE_BYTES);
        Item* t = tile_buf + tid * L;
#pragma unroll
        for (int i = 0; i < L; ++i) {
            if constexpr (FMT == kFmtU64) {
                t[i] = z;
            } else if constexpr (FMT == kFmtF64) {
                t[i] = unit_from_u64(z);
            } else {
                t[i] = f32_rz_from_unit(unit_from_u64(z));
            }
            z = step_modified_barrett(z);
        }
        // Make generic-proxy smem writes visible to the async (TMA) proxy.
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            const uint32_t src = static_cast<uint32_t>(__cvta_generic_to_shared(tile_buf));
            char* dst = static_cast<char*>(a.out) + tile * TILE_BYTES;
            asm volatile(
                "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n\t"
                "cp.async.bulk.commit_group;" ::"l"(dst),
                "r"(src), "r"(TILE_BYTES)
                : "memory");
        }
        z = mul_barrett(z, a.jump_next.c, a.jump_next.shoup);
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ------------------------------------------------- bulk (TMA) jump fill
// Jump-stream generation staged through shared memory and written with one
// TMA bulk store (cp.async.bulk, SASS UBLKCP) per 16 KiB tile. Each CTA owns
// a contiguous row range; warp w produces rows w and w+8 of every 16-row
// tile, so each of its streams advances by 16 rows per tile (one multiplier).
// Within a row a lane owns two 16-byte chunks (c*512 + lane*16 bytes), which
// makes both smem stores of the warp conflict-free.
template <int FMT, int ENG>
__global__ void __launch_bounds__(kContigThreads) k_fill_bulk(const ContigArgs a) {
    using E = EngOf<ENG>;
    using Item = typename Fmt<FMT>::Item;
    constexpr int EPC = 16 / sizeof(Item);           // elements per 16-byte chunk
    constexpr uint64_t ROW = 1024 / sizeof(Item);    // elements per 1 KiB row
    constexpr uint32_t TILE_ROWS = kBulkTileRows;    // 16
    constexpr uint32_t TILE_BYTES = TILE_ROWS * 1024;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    uint64_t r0, r1;  // this CTA's rows
    {
        const uint64_t q = a.rows / gridDim.x, rem = a.rows % gridDim.x;
        r0 = blockIdx.x * q + (blockIdx.x < rem ? blockIdx.x : rem);
        r1 = r0 + q + (blockIdx.x < rem ? 1 : 0);
    }
    if (r0 >= r1) return;
    // States: [h][c][j] for rows r0 + warp + 8h, chunk c, element j.
    typename E::State st[2][2][EPC];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const uint64_t j0 = (r0 + warp + 8 * h) * ROW + c * (32 * EPC) + lane * EPC;
            uint64_t z = dev_state_from_exp(dev_exp_at(a.e0, j0));
#pragma unroll
            for (int j = 0; j < EPC; ++j) {
                st[h][c][j] = E::from(z, j);
                if (j + 1 < EPC) z = step_modified_barrett(z);
            }
        }
    const Mult k = a.jump_row;  // 2^(53 * 16 rows) mod m for this kernel
    char* gout = static_cast<char*>(a.out);
    uint32_t it = 0;
    for (uint64_t t0 = r0; t0 < r1; t0 += TILE_ROWS, ++it) {
        const uint32_t b = it % kBulkStages;
        unsigned char* tile = smem_raw + b * TILE_BYTES;
        if (it >= kBulkStages && threadIdx.x == 0)
            asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kBulkStages - 1) : "memory");
        __syncthreads();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t row = warp + 8 * h;
            if (t0 + row < r1) {
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    uint64_t bits[EPC];
#pragma unroll
                    for (int j = 0; j < EPC; ++j) bits[j] = emit_bits<FMT, E>(st[h][c][j], j);
                    uint64_t w0, w1;
                    if constexpr (EPC == 2) {
                        w0 = bits[0];
                        w1 = bits[1];
                    } else {
                        w0 = bits[0] | (bits[1] << 32);
                        w1 = bits[2] | (bits[3] << 32);
                    }
                    const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(
                        tile + row * 1024 + c * 512 + lane * 16));
                    asm volatile("st.shared.v2.b64 [%0], {%1, %2};" ::"r"(sa), "l"(w0), "l"(w1)
                                 : "memory");
                }
            }
#pragma unroll
            for (int c = 0; c < 2; ++c)
#pragma unroll
                for (int j = 0; j < EPC; ++j) st[h][c][j] = E::mul(st[h][c][j], k, j);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint64_t nrows = r1 - t0 < TILE_ROWS ? r1 - t0 : TILE_ROWS;
            const uint32_t src = static_cast<uint32_t>(__cvta_generic_to_shared(tile));
            asm volatile(
                "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n\t"
                "cp.async.bulk.commit_group;" ::"l"(gout + t0 * 1024),
                "r"(src), "r"(static_cast<uint32_t>(nrows * 1024))
                : "memory");
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// -------------------------------------------------------- seed / walks
// SeedArgs.steps == 0: out[t] = state_at(a[t], k[t]) (generator.cpp:42-49).
// steps > 0: out[t*steps + s] = the (s+1)-th next() from that state.
__global__ void __launch_bounds__(256) k_seed(const SeedArgs a) {
    // Walk outputs: 32-byte vector stores per thread when steps % 4 == 0 and
    // the output is 32-byte aligned; otherwise staged 8 steps at a time in
    // shared memory ([thread][8], padded) so the block writes each thread's
    // 64-byte pieces with 8 lanes per piece.
    constexpr int kChunk = 8;
    __shared__ uint64_t stage[256][kChunk + 1];
    const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x;
    const uint64_t t = t0 + threadIdx.x;
    bool live = t < a.count;
    uint64_t z = 0;
    if (live) {
        const uint64_t idx = a.a[t];
        if (idx < kMinSeed || idx > kMaxSeed) {
            *a.error = 1;
            live = false;
        } else {
            const uint64_t ae = (idx - kModulus - 1) % kPeriod;
            const uint64_t e = (ae + (53ull * (a.k[t] % kPeriod)) % kPeriod) % kPeriod;
            z = dev_state_from_exp(e);
        }
    }
    if (a.steps == 0) {
        if (live) a.out[t] = z;
        return;
    }
    if (a.steps % 4 == 0 && reinterpret_cast<uintptr_t>(a.out) % 32 == 0) {
        // Each thread's walk is one contiguous run of steps * 8 bytes: write it
        // with 32-byte vector stores (every store fills whole sectors; L2
        // assembles the lines), no staging or cross-thread validity lookups.
        if (!live) return;
        uint64_t* dst = a.out + t * a.steps;
        for (uint32_t s = 0; s < a.steps; s += 4) {
            uint64_t v[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) v[i] = z = step_modified_barrett(z);
            st256(dst + s, v);
        }
        return;
    }
    const uint64_t nthreads = a.count - t0 < blockDim.x ? a.count - t0 : blockDim.x;
    for (uint32_t s0 = 0; s0 < a.steps; s0 += kChunk) {
        const uint32_t len = a.steps - s0 < kChunk ? a.steps - s0 : kChunk;
        for (uint32_t s = 0; s < len; ++s) {
            if (live) z = step_modified_barrett(z);
            stage[threadIdx.x][s] = z;
        }
        __syncthreads();
        for (uint32_t e = threadIdx.x; e < nthreads * len; e += blockDim.x) {
            const uint32_t th = e / len, s = e - th * len;
            const uint64_t src = a.a[t0 + th];
            if (src >= kMinSeed && src <= kMaxSeed)
                a.out[(t0 + th) * a.steps + s0 + s] = stage[th][s];
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------- digest
// 8 loads in flight per thread per pass (unguarded when the pass is whole);
// the sums are order-independent mod 2^64, so the result does not depend on
// the grid.
template <typename T>
__device__ __forceinline__ void digest_t(const DigestArgs& a, unsigned long long& s, unsigned long long& ws,
                                         unsigned long long& x) {
    constexpr int U = 8;
    const T* buf = static_cast<const T*>(a.buf);
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i0 < a.n; i0 += U * stride) {
        uint64_t v[U];
        if (i0 + (U - 1) * stride < a.n) {
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = buf[i0 + u * stride];
        } else {
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = i0 + u * stride < a.n ? buf[i0 + u * stride] : 0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t g = i0 + u * stride + a.index_base;
            s += v[u];
            ws += (g + 1) * v[u];
            x ^= v[u] * (2 * g + 1);
        }
    }
}

// Engine self-check: out[i] = z[i] * c[i]^chain mod m through one jump
// engine, intermediate states kept in the engine's own (possibly balanced,
// non-canonical) representation — exactness over the engine's whole reachable
// domain, independent of the multipliers a fill happens to use.
template <int ENG>
__global__ void __launch_bounds__(256) k_engine_check(const uint64_t* z, const Mult* mult, uint64_t* out,
                                                      uint64_t n, uint32_t chain) {
    using E = EngOf<ENG>;
    for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < n; i += gridDim.x * 256ull) {
        const Mult k = mult[i];
        typename E::State st = E::from(z[i], 0);
        for (uint32_t r = 0; r < chain; ++r) st = E::mul(st, k, 0);
        out[i] = E::raw(st, 0);
    }
}

__global__ void __launch_bounds__(256) k_digest(const DigestArgs a) {
    unsigned long long s = 0, ws = 0, x = 0;
    if (a.itemsize == 8)
        digest_t<uint64_t>(a, s, ws, x);
    else
        digest_t<uint32_t>(a, s, ws, x);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        ws += __shfl_xor_sync(0xffffffffu, ws, o);
        x ^= __shfl_xor_sync(0xffffffffu, x, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&a.out[0], s);
        atomicAdd(&a.out[1], ws);
        atomicXor(&a.out[2], x);
    }
}

// ------------------------------------------------------------- constant
// The reference's Constant baseline (bench.cpp:60-63): the same
// rows-per-warp split and 256-bit lane stores as k_fill_contig, fixed value.
__global__ void __launch_bounds__(kContigThreads) k_constant(const ConstArgs a) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
    const uint64_t w = static_cast<uint64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    uint64_t r, r_end, step;
    if (a.stride_order) {
        r = w;
        r_end = a.rows;
        step = nw;
    } else {
        warp_rows(a.rows, nw, w, r, r_end);
        step = 1;
    }
    const uint64_t v[4] = {a.value, a.value, a.value, a.value};
    char* p = static_cast<char*>(a.out) + r * 1024 + lane * 32;
#pragma unroll 4
    for (; r < r_end; r += step, p += step * 1024) st256(p, v);
}

// ------------------------------------------------------------ transpose
// Device deinterleave of one Interleaved region: the region is a row-major
// [rows x width] matrix M[i][w] at physical slot p0; logical position of
// M[i][w] is w*wpw + i_base + i. 32x32 smem tiles keep both sides coalesced.
// Both kernels are persistent and software-pipelined: the next tile's loads
// are issued into registers before the current tile is written out of shared
// memory, so every SM keeps reads and writes in flight at once.
//
// Wide regions (width > kNarrowMaxWidth workers): 64-row x 512-byte tiles of
// the [rows x width] region (64 workers of u64, 128 of u32). Loads run along
// tile rows (512-byte runs of the input, 16 or 32 per thread), the tile sits in
// shared memory with an odd pitch (conflict-free column reads for 4- and
// 8-byte items), and stores run along tile columns: each worker's 64
// consecutive logical items leave as one run.
constexpr unsigned kNarrowMaxWidth = 128;

template <typename T, int ROWS = 64, int BYTES = 512, int HALO = 0, int NT = 256, int PADJ = 0>
struct WideTile {
    static constexpr int kThreads = NT;
    static constexpr int kRows = ROWS;
    static constexpr int kHalo = HALO;                                  // rows loaded above the tile
    static constexpr int kTileRows = ROWS + HALO;
    static constexpr int kCols = BYTES / static_cast<int>(sizeof(T));  // workers
    // Odd pitch: conflict-free column reads of single items. Halo tiles of
    // 4-byte items whose run length is 1 mod 4 add PADJ = 2 (see the quad
    // gathers in transpose_wide_body).
    static constexpr int kPitch = kCols + 1 + PADJ;
    static constexpr int kLoads = kTileRows * kCols / NT;             // per thread
    static_assert(kCols <= NT && NT % kCols == 0 && kTileRows % (NT / kCols) == 0, "tile shape");
};

// Tile t -> (first worker, first row).
template <class G>
__device__ __forceinline__ void wide_origin(const TransposeArgs& a, uint64_t t, uint64_t ntw, uint64_t nrb,
                                            uint64_t& w0, uint64_t& i0) {
    if (a.order) {
        w0 = (t / nrb) * G::kCols;
        i0 = (t % nrb) * G::kRows;
    } else {
        w0 = (t % ntw) * G::kCols;
        i0 = (t / ntw) * G::kRows;
    }
}

// Rows [i0 - kHalo, i0 + kRows) x workers [w0, w0 + kCols) into registers
// (zeros outside the region).
template <typename T, class G>
__device__ __forceinline__ void wide_load(const TransposeArgs& a, uint64_t t, uint64_t ntw, uint64_t nrb,
                                          T (&v)[G::kLoads]) {
    const T* in = static_cast<const T*>(a.in);
    uint64_t w0, i0;
    wide_origin<G>(a, t, ntw, nrb, w0, i0);
    const int64_t top = static_cast<int64_t>(i0) - G::kHalo;
    const T* src = in + static_cast<int64_t>(a.p0) + top * static_cast<int64_t>(a.width) + static_cast<int64_t>(w0);
    constexpr int kRowStep = G::kThreads / G::kCols;  // rows a thread advances per load
    const int r = threadIdx.x / G::kCols, c = threadIdx.x % G::kCols;
    if (w0 + G::kCols <= a.width && top >= 0 && i0 + G::kRows <= a.rows) {
        const T* p = src + static_cast<uint64_t>(r) * a.width + c;
        const uint64_t step = kRowStep * a.width;
#pragma unroll
        for (int j = 0; j < G::kLoads; ++j) v[j] = p[j * step];
    } else {
#pragma unroll
        for (int j = 0; j < G::kLoads; ++j) {
            const int64_t rr = r + kRowStep * j;
            v[j] = (top + rr >= 0 && top + rr < static_cast<int64_t>(a.rows) && w0 + c < a.width)
                       ? src[rr * static_cast<int64_t>(a.width) + c]
                       : T(0);
        }
    }
}

// HALO = 0: every worker's run leaves in tile-row blocks [i0, i0 + kRows).
// HALO = L = 32 / itemsize (sector-aligned stores): worker w's block is shifted
// down by delta_w = (its output offset at i0) mod L items, so each block starts
// on a 32-byte sector of the output and every sector is written whole by ONE
// tile. Unaligned runs otherwise split sectors between two tiles written at
// different times, and HBM turns each partial sector into a read-modify-write:
// runs misaligned to 32-byte sectors cost 23% (u64) / 35% (u32) of the rate
// (profiles/r02/deinterleave_alignment.jsonl). The tile loads HALO extra rows
// above i0 for the shifted blocks; the first block starts at row 0 and the last
// one runs to the region end.
template <typename T, int ROWS, int BYTES, int HALO, int NT, int PADJ>
__device__ __forceinline__ void transpose_wide_body(const TransposeArgs& a) {
    using G = WideTile<T, ROWS, BYTES, HALO, NT, PADJ>;
    extern __shared__ __align__(16) unsigned char wide_smem[];
    T* tile = reinterpret_cast<T*>(wide_smem);
    T* out = static_cast<T*>(a.out);
    const uint64_t ntw = (a.width + G::kCols - 1) / G::kCols;
    const uint64_t nrb = (a.rows + G::kRows - 1) / G::kRows;
    const uint64_t ntiles = ntw * nrb;
    constexpr int kRowStep = NT / G::kCols;
    const int r = threadIdx.x / G::kCols, c = threadIdx.x % G::kCols;
    constexpr int P = G::kPitch;
    T v[G::kLoads];
    uint64_t t = blockIdx.x;
    if (t < ntiles) wide_load<T, G>(a, t, ntw, nrb, v);
    for (; t < ntiles; t += gridDim.x) {
#pragma unroll
        for (int j = 0; j < G::kLoads; ++j) tile[(r + kRowStep * j) * P + c] = v[j];
        __syncthreads();
        if (t + gridDim.x < ntiles) wide_load<T, G>(a, t + gridDim.x, ntw, nrb, v);  // prefetch
        uint64_t w0, i0;
        wide_origin<G>(a, t, ntw, nrb, w0, i0);
        const int i = threadIdx.x % G::kRows;  // item within the worker's run
        const int wq = threadIdx.x / G::kRows;  // first worker of this thread
        if constexpr (HALO == 0) {
            T* dst = out + w0 * a.wpw + a.i_base + i0;
            if (w0 + G::kCols <= a.width && i0 + G::kRows <= a.rows) {
#pragma unroll 8
                for (int wl = wq; wl < G::kCols; wl += NT / G::kRows)
                    dst[wl * a.wpw + i] = tile[i * G::kPitch + wl];
            } else {
                for (int wl = wq; wl < G::kCols; wl += NT / G::kRows)
                    if (w0 + wl < a.width && i0 + i < a.rows) dst[wl * a.wpw + i] = tile[i * G::kPitch + wl];
            }
        } else {
            // Worker w0 + wl: block [j0, j1) of its run, j0 = i0 - delta on a
            // sector (0 for the first block), j1 = the next block's j0 (the
            // region end for the last block, which may hold up to kRows + L - 1
            // items). In tile rows (row 0 = item i0 - kHalo) the block is
            // [s0, e); the per-quad arithmetic is 32-bit.
            const bool last = i0 + G::kRows >= a.rows;
            const uint32_t nw = static_cast<uint32_t>(a.width - w0 < static_cast<uint64_t>(G::kCols) ? a.width - w0 : G::kCols);
            const uint64_t base0 = w0 * a.wpw + a.i_base;  // item 0 of worker w0
            const uint32_t phase0 = static_cast<uint32_t>((a.out_mod + base0 + i0) & (HALO - 1));
            const uint32_t wpw_mod = static_cast<uint32_t>(a.wpw & (HALO - 1));
            const uint32_t e_last = static_cast<uint32_t>(a.rows - i0) + HALO;  // used when `last`
            const uint64_t q0 = base0 + i0 - HALO;  // item of tile row 0 (mod 2^64; only rows >= s0 are touched)
            {
                // 16-byte stores of E = 16 / itemsize items. Quads of E rows
                // start where the output address is 16-byte aligned (tile row
                // a0 = HALO - delta mod E, which differs between workers); a
                // warp takes 4 workers x 8 consecutive quads, so each store
                // instruction writes four whole 128-byte lines. The gathers
                // are conflict-free for even wpw and 2-way for odd wpw with
                // the pitch the launcher picks (PADJ; exhaustive check over
                // run phases; 8 workers x 4 quads is conflict-free at pitch 130
                // but its 64-byte store segments measured 13-18% slower).
                // Quads cut by the block ends fall back to single items.
                constexpr int E = 16 / static_cast<int>(sizeof(T));
                constexpr int kQ = G::kTileRows / E;  // quads per worker
                static_assert(kQ % 8 == 0 && G::kCols % 4 == 0, "warp = 4 workers x 8 quads");
                constexpr int kWarpSteps = G::kCols * kQ / 32;
                const unsigned lane = threadIdx.x & 31;
#pragma unroll 2
                for (int ws = threadIdx.x >> 5; ws < kWarpSteps; ws += NT / 32) {
                    const uint32_t wl = 4 * (ws % (G::kCols / 4)) + (lane >> 3);
                    const uint32_t kq = 8 * (ws / (G::kCols / 4)) + (lane & 7);
                    if (wl >= nw) continue;
                    const uint32_t delta = (phase0 + wl * wpw_mod) & (HALO - 1);
                    const uint32_t s0 = i0 != 0 ? HALO - delta : HALO;
                    const uint32_t e = last ? e_last : G::kRows + HALO - delta;
                    const uint32_t r0 = ((HALO - delta) & (E - 1)) + E * kq;
                    if (r0 >= e || r0 + E <= s0) continue;
                    T* p = out + (q0 + static_cast<uint64_t>(wl) * a.wpw + r0);
                    const T* t0 = tile + r0 * P + wl;
                    if (r0 >= s0 && r0 + E <= e) {
                        if constexpr (E == 4) {
                            const uint32_t x0 = t0[0], x1 = t0[P], x2 = t0[2 * P], x3 = t0[3 * P];
                            asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(x0), "r"(x1), "r"(x2),
                                         "r"(x3)
                                         : "memory");
                        } else {
                            const uint64_t x0 = t0[0], x1 = t0[P];
                            asm volatile("st.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(x0), "l"(x1) : "memory");
                        }
                    } else {
                        for (uint32_t c = 0; c < static_cast<uint32_t>(E); ++c)
                            if (r0 + c >= s0 && r0 + c < e) p[c] = t0[c * P];
                    }
                }
            }
        }
        __syncthreads();
    }
}

// The wide kernel. __launch_bounds__ without a minimum-blocks argument: with
// one, ptxas spends more registers (the 4-byte narrow tile went from 124 to 168,
// one CTA per SM instead of two, -10%).
template <typename T, int ROWS, int BYTES, int HALO, int NT = 256, int PADJ = 0>
__global__ void __launch_bounds__(NT) k_transpose(const TransposeArgs a) {
    transpose_wide_body<T, ROWS, BYTES, HALO, NT, PADJ>(a);
}

// Narrow regions (width <= kNarrowMaxWidth workers for 4-byte items, <= 85
// for 8-byte items; transpose_t): tiles of R whole rows
// (R*width <= kNarrowItems slots, R a multiple of 64, or of 16 when W > 64) are one contiguous span
// of the input, read fully coalesced (kNarrowItems/256 loads per thread),
// scattered into shared memory as [width][R] with an odd pitch (row = slot /
// width by a multiply-high), and each worker's R consecutive logical items
// leave as one run (all warps on one worker for width < 8, one worker per
// warp otherwise).
template <typename T, unsigned KITEMS = 8192>
struct NarrowTile {
    static constexpr unsigned kItems = KITEMS;  // slots per tile (default 64 / 32 KiB)
    static constexpr unsigned kLoads = kItems / 256;
    // Rows per tile: as many whole rows as fit, a multiple of 64 (512-byte
    // output runs for u64) — except for W in (64, 128], where that leaves 64
    // rows and 50-99% of the tile (W = 100: 6400 of 8192 slots); there a
    // multiple of 16 (W = 100: 80 rows) is 2-10% faster for u64 and 5-16% for
    // u32 (one exception: u64 W = 65, 11% slower). A multiple of 16 for every
    // W measured 1-5% slower at W = 7 and 33 (profiles/r01/deinterleave_rows16*.jsonl).
    static __host__ __device__ constexpr unsigned rows(unsigned width) {
        return width > 64 ? kItems / width / 16 * 16 : kItems / width / 64 * 64;
    }
    // Rows per tile with `halo` extra rows above it (k_transpose_narrow_h).
    static __host__ __device__ constexpr unsigned rows_halo(unsigned width, unsigned halo) {
        return (kItems / width - halo) / 16 * 16;
    }
};

template <typename T, unsigned NT = 256, unsigned KITEMS = 8192>
__device__ __forceinline__ void narrow_load(const TransposeArgs& a, uint64_t r0, unsigned items,
                                            T (&v)[KITEMS / NT]) {
    using G = NarrowTile<T, KITEMS>;
    constexpr unsigned kLoads = G::kItems / NT;
    const T* src = static_cast<const T*>(a.in) + a.p0 + r0 * a.width;
    if (items == G::kItems) {
#pragma unroll
        for (unsigned j = 0; j < kLoads; ++j) v[j] = src[threadIdx.x + NT * j];
    } else {
#pragma unroll
        for (unsigned j = 0; j < kLoads; ++j) {
            const unsigned q = threadIdx.x + NT * j;
            v[j] = q < items ? src[q] : T(0);
        }
    }
}

// Narrow tiles with sector-aligned worker blocks (the narrow counterpart of
// k_transpose<..., HALO>): tile t holds rows [t*R - H, t*R + R) (H = one
// 32-byte sector of items, loaded as one contiguous span with the R rows), and
// worker w's block [t*R - delta_w, t*R + R - delta_w) starts on a sector of
// its output run, so no sector is split between two tiles (split sectors
// become HBM read-modify-writes: u64 W = 65 / 85 at 2^30 items lose 26 / 17%).
// R + H whole rows fit the kItems-slot span; R is a multiple of 16. W >= 8.
template <typename T, unsigned NT = 256>
__global__ void __launch_bounds__(NT) k_transpose_narrow_h(const TransposeArgs a) {
    using G = NarrowTile<T>;
    constexpr unsigned H = 32 / sizeof(T);
    extern __shared__ __align__(16) unsigned char narrow_smem[];
    T* tile = reinterpret_cast<T*>(narrow_smem);
    T* out = static_cast<T*>(a.out);
    const unsigned W = static_cast<unsigned>(a.width);
    const unsigned R = G::rows_halo(W, H);
    const unsigned P = a.pitch ? a.pitch : ((R + H) | 1);
    const uint64_t M = ((1ull << 32) + W - 1) / W;
    const uint64_t ntiles = (a.rows + R - 1) / R;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // Loaded span of tile t: rows [start, end), smem row = row - (t*R - H).
    auto span = [&](uint64_t t, uint64_t& start, unsigned& items, unsigned& off) {
        const uint64_t top = t * R;  // + H
        start = top >= H ? top - H : 0;
        const uint64_t end = top + R < a.rows ? top + R : a.rows;
        items = static_cast<unsigned>((end - start) * W);
        off = static_cast<unsigned>(start + H - top);
    };
    constexpr unsigned kLoads = G::kItems / NT;
    T v[kLoads];
    uint64_t t = blockIdx.x;
    uint64_t start;
    unsigned items, off;
    if (t < ntiles) {
        span(t, start, items, off);
        narrow_load<T, NT>(a, start, items, v);
    }
    for (; t < ntiles; t += gridDim.x) {
        span(t, start, items, off);
#pragma unroll
        for (unsigned j = 0; j < kLoads; ++j) {
            const unsigned q = threadIdx.x + NT * j;
            if (q < items) {
                const unsigned row = static_cast<unsigned>((q * M) >> 32);
                tile[(q - row * W) * P + row + off] = v[j];
            }
        }
        __syncthreads();
        const uint64_t tn = t + gridDim.x;
        if (tn < ntiles) {
            uint64_t s2;
            unsigned i2, o2;
            span(tn, s2, i2, o2);
            narrow_load<T, NT>(a, s2, i2, v);  // prefetch
        }
        const uint64_t i0 = t * R;
        const bool last = i0 + R >= a.rows;
        const uint32_t e_last = static_cast<uint32_t>(a.rows - i0) + H;
        const uint64_t base_t = a.i_base + i0;
        const uint32_t wpw_mod = static_cast<uint32_t>(a.wpw & (H - 1));
        const uint32_t phase_t = static_cast<uint32_t>((a.out_mod + base_t) & (H - 1));
        for (unsigned col = warp; col < W; col += NT / 32) {
            const uint32_t delta = (phase_t + col * wpw_mod) & (H - 1);
            const uint32_t s0 = i0 != 0 ? H - delta : H;
            const uint32_t e = last ? e_last : R + H - delta;
            // rows [s0, e) of the column; a plain loop (an unrolled one with
            // per-column trip counts cost ~50 instructions of remainder logic
            // per column: 2.2x the plain kernel's instruction count)
            T* d = out + (col * a.wpw + base_t - H + s0);
            const T* sm = tile + col * P + s0;
            const uint32_t len = e - s0;
#pragma unroll 1
            for (uint32_t i = lane; i < len; i += 32) d[i] = sm[i];
        }
        __syncthreads();
    }
}

template <typename T, unsigned NT, unsigned KITEMS>
__device__ __forceinline__ void transpose_narrow_body(const TransposeArgs& a) {
    using G = NarrowTile<T, KITEMS>;
    extern __shared__ __align__(16) unsigned char narrow_smem[];
    T* tile = reinterpret_cast<T*>(narrow_smem);
    T* out = static_cast<T*>(a.out);
    const unsigned W = static_cast<unsigned>(a.width);
    const unsigned R = G::rows(W);  // rows per tile
    const unsigned P = a.pitch ? a.pitch : (R | 1);  // smem pitch (narrow_pitch)
    // slot / W == (slot * M) >> 32 exactly for slot < 2^32 / W, M = ceil(2^32 / W)
    const uint64_t M = ((1ull << 32) + W - 1) / W;
    const uint64_t ntiles = (a.rows + R - 1) / R;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    auto rows_of = [&](uint64_t t) {
        return static_cast<unsigned>(a.rows - t * R < R ? a.rows - t * R : R);
    };
    constexpr unsigned kLoads = G::kItems / NT;
    T v[kLoads];
    uint64_t t = blockIdx.x;
    if (t < ntiles) narrow_load<T, NT, KITEMS>(a, t * R, rows_of(t) * W, v);
    for (; t < ntiles; t += gridDim.x) {
        const unsigned nr = rows_of(t), items = nr * W;
#pragma unroll
        for (unsigned j = 0; j < kLoads; ++j) {
            const unsigned q = threadIdx.x + NT * j;
            if (q < items) {
                const unsigned row = static_cast<unsigned>((q * M) >> 32);
                tile[(q - row * W) * P + row] = v[j];
            }
        }
        __syncthreads();
        const uint64_t tn = t + gridDim.x;
        if (tn < ntiles) narrow_load<T, NT, KITEMS>(a, tn * R, rows_of(tn) * W, v);  // prefetch
        T* dst = out + a.i_base + t * R;
        if (W < 8) {
            for (unsigned col = 0; col < W; ++col)
                for (unsigned i = threadIdx.x; i < nr; i += NT) dst[col * a.wpw + i] = tile[col * P + i];
        } else {
            for (unsigned col = warp; col < W; col += NT / 32) {
                T* d = dst + col * a.wpw;
                const T* s = tile + col * P;
#pragma unroll 4
                for (unsigned i = lane; i < nr; i += 32) d[i] = s[i];
            }
        }
        __syncthreads();
    }
}

template <typename T, unsigned NT = 256, unsigned KITEMS = 8192>
__global__ void __launch_bounds__(NT) k_transpose_narrow(const TransposeArgs a) {
    transpose_narrow_body<T, NT, KITEMS>(a);
}

// ============================================================ launchers
std::atomic<uint64_t> g_launches{0};

uint64_t launch_count() { return g_launches.load(); }

namespace {

cudaError_t counted(cudaError_t e) {
    if (e == cudaSuccess) g_launches.fetch_add(1);
    return e;
}

// Hybrid engine ids kEngHybridBase + KF: KF FP64 streams per lane vector, the
// rest Barrett (instantiated for 1 <= KF < V).
template <int FMT, class F>
bool hybrid_dispatch(int engine, F&& f) {
    constexpr int V = Fmt<FMT>::kVec;
    switch (engine - kEngHybridBase) {
        case 1: f(std::integral_constant<int, 1>{}); return true;
        case 2: f(std::integral_constant<int, 2>{}); return true;
        case 3: f(std::integral_constant<int, 3>{}); return true;
        default: break;
    }
    if constexpr (V == 8) {
        switch (engine - kEngHybridBase) {
            case 4: f(std::integral_constant<int, 4>{}); return true;
            case 5: f(std::integral_constant<int, 5>{}); return true;
            case 6: f(std::integral_constant<int, 6>{}); return true;
            case 7: f(std::integral_constant<int, 7>{}); return true;
            default: break;
        }
    }
    return false;
}

template <int FMT>
cudaError_t contig_fmt(int engine, const ContigArgs& a, int grid, int block, cudaStream_t s) {
    switch (engine) {
        case kEngBarrett:
            k_fill_contig<FMT, kEngBarrett><<<grid, block, 0, s>>>(a);
            break;
        case kEngMontgomery:
            k_fill_contig<FMT, kEngMontgomery><<<grid, block, 0, s>>>(a);
            break;
        case kEngFP64:
            k_fill_contig<FMT, kEngFP64><<<grid, block, 0, s>>>(a);
            break;
        case kEngMixed:
            k_fill_contig<FMT, kEngMixed><<<grid, block, 0, s>>>(a);
            break;
        default:
            if (!hybrid_dispatch<FMT>(engine, [&](auto kf) {
                    k_fill_contig<FMT, kEngHybridBase + decltype(kf)::value><<<grid, block, 0, s>>>(a);
                }))
                return cudaErrorInvalidValue;
    }
    return counted(cudaGetLastError());
}

template <int FMT>
cudaError_t inter_fmt(int engine, const InterleavedArgs& a, int grid, int block, cudaStream_t s) {
    switch (engine) {
        case kEngBarrett:
            k_fill_interleaved<FMT, kEngBarrett><<<grid, block, 0, s>>>(a);
            break;
        case kEngMontgomery:
            k_fill_interleaved<FMT, kEngMontgomery><<<grid, block, 0, s>>>(a);
            break;
        case kEngFP64:
            k_fill_interleaved<FMT, kEngFP64><<<grid, block, 0, s>>>(a);
            break;
        case kEngMixed:
            k_fill_interleaved<FMT, kEngMixed><<<grid, block, 0, s>>>(a);
            break;
        default:
            return cudaErrorInvalidValue;
    }
    return counted(cudaGetLastError());
}

template <class K>
int occupancy(K kernel, int block, size_t smem = 0) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, block, smem) != cudaSuccess) n = 1;
    return n > 0 ? n : 1;
}

}  // namespace

cudaError_t launch_contig(int fmt, int engine, const ContigArgs& a, int grid, int block,
                          cudaStream_t s) {
    switch (fmt) {
        case kFmtU64: return contig_fmt<kFmtU64>(engine, a, grid, block, s);
        case kFmtF64: return contig_fmt<kFmtF64>(engine, a, grid, block, s);
        case kFmtF32: return contig_fmt<kFmtF32>(engine, a, grid, block, s);
    }
    return cudaErrorInvalidValue;
}

namespace {
template <int FMT, int MODE>
cudaError_t paced_mode(int engine, const PacedArgs& a, int grid, cudaStream_t s) {
    // Only the FP64-pipe engines are paced (bcn_capi.cu: paced()); the integer
    // engines are compute-bound below the write path and run unpaced.
    switch (engine) {
        case kEngFP64: k_fill_paced<FMT, kEngFP64, MODE><<<grid, kPacedThreads, 0, s>>>(a); break;
        case kEngMixed: k_fill_paced<FMT, kEngMixed, MODE><<<grid, kPacedThreads, 0, s>>>(a); break;
        default:
            if (MODE != kPacedContiguous ||
                !hybrid_dispatch<FMT>(engine, [&](auto kf) {
                    k_fill_paced<FMT, kEngHybridBase + decltype(kf)::value, kPacedContiguous>
                        <<<grid, kPacedThreads, 0, s>>>(a);
                }))
                return cudaErrorInvalidValue;
    }
    return counted(cudaGetLastError());
}

template <int FMT>
cudaError_t paced_fmt(int engine, const PacedArgs& a, int grid, cudaStream_t s) {
    if (engine == -1) {
        k_fill_paced<FMT, kEngBarrett, kPacedConstant><<<grid, kPacedThreads, 0, s>>>(a);
        return counted(cudaGetLastError());
    }
    switch (a.mode) {
        case kPacedInterleaved: return paced_mode<FMT, kPacedInterleaved>(engine, a, grid, s);
        case kPacedInterleavedFixed: return paced_mode<FMT, kPacedInterleavedFixed>(engine, a, grid, s);
        default: return paced_mode<FMT, kPacedContiguous>(engine, a, grid, s);
    }
}
}  // namespace

cudaError_t launch_paced(int fmt, int engine, const PacedArgs& a, int grid, cudaStream_t s) {
    switch (fmt) {
        case kFmtU64: return paced_fmt<kFmtU64>(engine, a, grid, s);
        case kFmtF64: return paced_fmt<kFmtF64>(engine, a, grid, s);
        case kFmtF32: return paced_fmt<kFmtF32>(engine, a, grid, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_interleaved(int fmt, int engine, const InterleavedArgs& a, int grid, int block,
                               cudaStream_t s) {
    switch (fmt) {
        case kFmtU64: return inter_fmt<kFmtU64>(engine, a, grid, block, s);
        case kFmtF64: return inter_fmt<kFmtF64>(engine, a, grid, block, s);
        case kFmtF32: return inter_fmt<kFmtF32>(engine, a, grid, block, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_slots(int fmt, const SlotArgs& a, cudaStream_t s) {
    if (a.count == 0) return cudaSuccess;
    const unsigned grid = static_cast<unsigned>((a.count + 127) / 128);
    switch (fmt) {
        case kFmtU64: k_fill_slots<kFmtU64><<<grid, 128, 0, s>>>(a); break;
        case kFmtF64: k_fill_slots<kFmtF64><<<grid, 128, 0, s>>>(a); break;
        case kFmtF32: k_fill_slots<kFmtF32><<<grid, 128, 0, s>>>(a); break;
        default: return cudaErrorInvalidValue;
    }
    return counted(cudaGetLastError());
}

cudaError_t launch_staged(int fmt, const StagedArgs& a, int grid, cudaStream_t s) {
    const size_t smem = 2ull * kStagedThreads * kStagedL * format_itemsize(fmt);
    switch (fmt) {
        case kFmtU64:
            cudaFuncSetAttribute(k_fill_staged<kFmtU64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem));
            k_fill_staged<kFmtU64><<<grid, kStagedThreads, smem, s>>>(a);
            break;
        case kFmtF64:
            cudaFuncSetAttribute(k_fill_staged<kFmtF64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem));
            k_fill_staged<kFmtF64><<<grid, kStagedThreads, smem, s>>>(a);
            break;
        case kFmtF32:
            cudaFuncSetAttribute(k_fill_staged<kFmtF32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem));
            k_fill_staged<kFmtF32><<<grid, kStagedThreads, smem, s>>>(a);
            break;
        default:
            return cudaErrorInvalidValue;
    }
    return counted(cudaGetLastError());
}

cudaError_t launch_bulk(int fmt, const ContigArgs& a, int grid, cudaStream_t s) {
    const int smem = kBulkStages * kBulkTileRows * 1024;
    switch (fmt) {
        case kFmtU64:
            cudaFuncSetAttribute(k_fill_bulk<kFmtU64, kEngFP64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            k_fill_bulk<kFmtU64, kEngFP64><<<grid, kContigThreads, smem, s>>>(a);
            break;
        case kFmtF64:
            cudaFuncSetAttribute(k_fill_bulk<kFmtF64, kEngFP64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            k_fill_bulk<kFmtF64, kEngFP64><<<grid, kContigThreads, smem, s>>>(a);
            break;
        case kFmtF32:
            cudaFuncSetAttribute(k_fill_bulk<kFmtF32, kEngFP64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            k_fill_bulk<kFmtF32, kEngFP64><<<grid, kContigThreads, smem, s>>>(a);
            break;
        default:
            return cudaErrorInvalidValue;
    }
    return counted(cudaGetLastError());
}

int bulk_blocks_per_sm(int fmt) {
    const size_t smem = static_cast<size_t>(kBulkStages) * kBulkTileRows * 1024;
    switch (fmt) {
        case kFmtU64: return occupancy(k_fill_bulk<kFmtU64, kEngFP64>, kContigThreads, smem);
        case kFmtF64: return occupancy(k_fill_bulk<kFmtF64, kEngFP64>, kContigThreads, smem);
        case kFmtF32: return occupancy(k_fill_bulk<kFmtF32, kEngFP64>, kContigThreads, smem);
    }
    return 1;
}

cudaError_t launch_seed(const SeedArgs& a, cudaStream_t s) {
    if (a.count == 0) return cudaSuccess;
    k_seed<<<static_cast<unsigned>((a.count + 255) / 256), 256, 0, s>>>(a);
    return counted(cudaGetLastError());
}

cudaError_t launch_engine_check(int engine, const uint64_t* z, const Mult* mult, uint64_t* out, uint64_t n,
                                uint32_t chain, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 148ull * 16));
    switch (engine) {
        case kEngBarrett: k_engine_check<kEngBarrett><<<grid, 256, 0, s>>>(z, mult, out, n, chain); break;
        case kEngMontgomery: k_engine_check<kEngMontgomery><<<grid, 256, 0, s>>>(z, mult, out, n, chain); break;
        case kEngFP64: k_engine_check<kEngFP64><<<grid, 256, 0, s>>>(z, mult, out, n, chain); break;
        case kEngMixed: k_engine_check<kEngMixed><<<grid, 256, 0, s>>>(z, mult, out, n, chain); break;
        default: return cudaErrorInvalidValue;
    }
    return counted(cudaGetLastError());
}

cudaError_t launch_digest(const DigestArgs& a, int grid, cudaStream_t s) {
    k_digest<<<grid, 256, 0, s>>>(a);
    return counted(cudaGetLastError());
}

cudaError_t launch_constant(const ConstArgs& a, int grid, int block, cudaStream_t s) {
    k_constant<<<grid, block, 0, s>>>(a);
    return counted(cudaGetLastError());
}

namespace {
template <typename T, int ROWS, int BYTES, int HALO, int NT = 256, int PADJ = 0>
cudaError_t transpose_wide_nt(const TransposeArgs& a, int sms, cudaStream_t s) {
    constexpr auto kernel = k_transpose<T, ROWS, BYTES, HALO, NT, PADJ>;
    using G = WideTile<T, ROWS, BYTES, HALO, NT, PADJ>;
    const size_t smem = static_cast<size_t>(G::kTileRows) * G::kPitch * sizeof(T);
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    const uint64_t nrb = (a.rows + G::kRows - 1) / G::kRows;
    const uint64_t tiles = ((a.width + G::kCols - 1) / G::kCols) * nrb;
    const uint64_t cap = static_cast<uint64_t>(sms) * occupancy(kernel, NT, smem);
    const uint64_t grid = std::min(tiles, cap);
    // Tile order: with few row blocks per worker (very wide regions: short
    // per-worker runs), walking row blocks fastest keeps every worker's whole
    // output run in flight at once: +8-33% at W >= 20000, +2-3% at W = 5000,
    // 4-30% slower when a worker has thousands of row blocks (W <= 1000 at
    // 2^28 items; profiles/r01/deinterleave_tile_order.jsonl).
    TransposeArgs b = a;
    b.order = nrb <= 4 * grid ? 1u : 0u;
    kernel<<<static_cast<unsigned>(grid), NT, smem, s>>>(b);
    return counted(cudaGetLastError());
}

// Threads per wide CTA: 512 for 8-byte regions of at most 104 workers (one
// mostly empty 128-worker column block; W = 86 / 100: +11 / +5%), 256
// otherwise (512 measured -6 to -9% at W = 120 / 127 and mixed for u32;
// profiles/r02/deinterleave_wide_threads.jsonl).
// BCN_DEINT_WIDE_THREADS = 256 | 512 forces one (A/B switch).
template <typename T>
int wide_threads(uint64_t width) {
    static const int env = [] {
        const char* v = std::getenv("BCN_DEINT_WIDE_THREADS");
        return v ? static_cast<int>(std::strtol(v, nullptr, 10)) : 0;
    }();
    if (env) return env;
    return sizeof(T) == 8 && width <= 104 ? 512 : 256;
}

template <typename T, int ROWS, int BYTES, int HALO>
cudaError_t transpose_wide_h(const TransposeArgs& a, int sms, cudaStream_t s) {
    if (wide_threads<T>(a.width) == 512) return transpose_wide_nt<T, ROWS, BYTES, HALO, 512>(a, sms, s);
    // 4-byte halo tiles with a run length of 1 mod 4: pitch + 2 halves the
    // quad-gather bank conflicts (4-way -> 2-way; 3 mod 4 is 2-way already).
    if constexpr (HALO != 0 && sizeof(T) == 4)
        if (a.wpw % 4 == 1) return transpose_wide_nt<T, ROWS, BYTES, HALO, 256, 2>(a, sms, s);
    return transpose_wide_nt<T, ROWS, BYTES, HALO, 256>(a, sms, s);
}

// Sector-aligned blocks suffice: runs aligned to 32-byte sectors but not to
// 128-byte lines lose only 5-15%, and line-aligned halo blocks (L = 128 B,
// 96 + 32 / 112 + 16 rows) measured 3-25% slower than sector-aligned ones
// (profiles/r02/deinterleave_u32_width_and_line_halo.jsonl). The halo tiles keep the register footprint of the
// plain ones for 4-byte items (120 + 8 rows: 2 CTAs per SM) and add 4 rows
// for 8-byte items (1 CTA per SM either way).
template <typename T, int ROWS, int BYTES>
cudaError_t transpose_wide(const TransposeArgs& a, int sms, cudaStream_t s) {
    constexpr int L = 32 / static_cast<int>(sizeof(T));
    constexpr int kRowsH = ROWS >= 128 ? ROWS - L : ROWS;
    // Runs that keep whole sectors at tile boundaries stay on the plain
    // kernel; so do 8-byte runs on a 16-byte (half-sector) boundary, which
    // measured faster plain (W = 200 / 10^6 at 2^30: 5.7 / 5.4 vs 4.6 / 4.7 TB/s)
    // while 8-byte-aligned runs gain 2-18% with the halo blocks
    // (profiles/r02/deinterleave_alignment.jsonl).
    // Short regions (a few blocks per run: < 256 rows for 4-byte, < 1024 for
    // 8-byte items) and 8-byte regions narrower than two worker blocks also
    // measured faster plain (-6 to -18% with halo blocks at W = 86 / 100 and
    // W = 10^6 with 268 rows).
    constexpr uint64_t kNeed = sizeof(T) == 8 ? 2 : L;
    const bool aligned_runs = (a.wpw % kNeed == 0) && ((a.out_mod + a.i_base) % kNeed == 0);
    const bool halo_pays = sizeof(T) == 4 ? a.rows >= 256 : (a.rows >= 1024 && a.width >= 256);
    // (the 4-byte quad mapping needs a multiple of 32 tile rows)
    constexpr bool kHaloShape = (kRowsH + L) % (8 * 16 / sizeof(T)) == 0;
    if constexpr (kHaloShape) {
        static const int mode = [] {  // BCN_DEINT_ALIGN: 0 never, 1 misaligned runs (default), 2 always
            const char* v = std::getenv("BCN_DEINT_ALIGN");
            return v ? static_cast<int>(std::strtol(v, nullptr, 10)) : 1;
        }();
        if (mode == 2 || (!aligned_runs && halo_pays && mode == 1))
            return transpose_wide_h<T, kRowsH, BYTES, L>(a, sms, s);
    }
    return transpose_wide_h<T, ROWS, BYTES, 0>(a, sms, s);
}

// Shared-memory pitch of a narrow 4-byte tile: the scatter writes slot q of
// the span to tile[(q % W) * P + q / W], so for W < 32 one warp touches
// several tile rows and the default odd pitch R | 1 (== 1 mod 32 for R a
// multiple of 64) puts (c, r) and (c + 1, r - 1) in one bank. Where that
// costs >= 5-way conflicts on average (W = 5, 6, 7) take the pad (W * pad
// within the kNarrowMaxWidth spare items) with the fewest conflicts over every
// warp alignment: +11 / +20 / +18% there. Re-pitching milder cases measured
// 1-6% slower (W = 3, 4, 8-16), so they keep R | 1
// (profiles/r01/deinterleave_pitch_u32_abba.jsonl, ABBA order, 4 reps).
unsigned narrow_conflicts_u32(unsigned W, unsigned P) {
    unsigned cost = 0;
    for (unsigned start = 0; start < W; ++start) {
        unsigned count[32] = {}, worst = 0;
        for (unsigned l = 0; l < 32; ++l) {
            const unsigned q = start + l;
            worst = std::max(worst, ++count[((q % W) * P + q / W) % 32]);
        }
        cost += worst;
    }
    return cost;  // summed over the W warp alignments
}

unsigned narrow_pitch_u32(unsigned W, unsigned R) {
    if (W >= 32 || narrow_conflicts_u32(W, R | 1) < 5 * W) return R | 1;
    unsigned best = R | 1, best_cost = ~0u;
    for (unsigned pad = 1; pad * W <= kNarrowMaxWidth; ++pad) {
        const unsigned cost = narrow_conflicts_u32(W, R + pad);
        if (cost < best_cost) {
            best_cost = cost;
            best = R + pad;
        }
    }
    return best;
}

// BCN_DEINT_TMA=1 routes aligned wide regions through the TMA tile mover
// (bcn_deint_tma.cu). Off by default: on the regions it can take (rows and runs
// whole 16-byte chunks) it measured 5.5-5.7 TB/s against 5.9-6.2 for the
// register pipeline (profiles/r02/deinterleave_tma_vs_registers.jsonl).
bool tma_deinterleave_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("BCN_DEINT_TMA");
        return v && v[0] == '1';
    }();
    return on;
}

// Narrow widths above this take 16384-slot tiles on 512 threads (twice the
// rows per tile, halving the sectors split between tiles): 4-byte items from
// W = 16, +2-26% (2^30 items: W = 63 / 85 / 100 / 116: +16 / +16 / +26 /
// +14%); W = 9 -2 to -5%; 8-byte items 0 to -6%, so they keep 8192 slots
// (profiles/r02/deinterleave_narrow_big_tiles.jsonl). Knobs
// BCN_DEINT_NARROW_BIG_MIN_U32 / _U64 override (A/B switch).
template <typename T>
unsigned narrow_big_min() {
    static const unsigned v = [] {
        const char* e = std::getenv(sizeof(T) == 4 ? "BCN_DEINT_NARROW_BIG_MIN_U32" : "BCN_DEINT_NARROW_BIG_MIN_U64");
        return e ? static_cast<unsigned>(std::strtoul(e, nullptr, 10)) : (sizeof(T) == 4 ? 15u : 0x7fffffffu);
    }();
    return v;
}

// BCN_DEINT_NARROW_HALO=0 disables the sector-aligned narrow tiles (A/B switch).
bool narrow_halo_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("BCN_DEINT_NARROW_HALO");
        return !(v && v[0] == '0');
    }();
    return on;
}

// Threads per narrow CTA: 512 for 8-byte items (twice the warps on the same
// 64 KiB tile: +7-10% at W = 2 / 16 / 31 / 33 / 64, equal elsewhere), 256 for
// 4-byte items (512 measured 0-6% slower; profiles/r02/deinterleave_narrow_threads.jsonl).
// BCN_DEINT_NARROW_THREADS=256|512 overrides (A/B switch).
template <typename T>
int narrow_threads() {
    static const int nt = [] {
        const char* v = std::getenv("BCN_DEINT_NARROW_THREADS");
        return v ? static_cast<int>(std::strtol(v, nullptr, 10)) : (sizeof(T) == 8 ? 512 : 256);
    }();
    return nt;
}

template <typename T>
cudaError_t transpose_t(const TransposeArgs& a, cudaStream_t s, bool allow_tma) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // Narrow row tiles up to W = 128 for 4-byte items; 8-byte items switch to
    // the wide 128-worker (1 KiB) tiles from W = 86: one partly filled column
    // block with 1 KiB output runs beats 80-112-row narrow tiles there
    // (W = 100: 5.4 vs 4.9 TB/s, W = 120: 5.8 vs 4.8, W = 128: 5.85 vs 5.5;
    // crossover at W ~ 86; profiles/r01/deinterleave_narrow_vs_wide.jsonl).
    // 4-byte items: narrow tiles up to W = 128 with the 16384-slot tiles
    // (with 8192-slot tiles the crossover was W = 116: W = 120 / 124 / 127
    // went wide, +16-26%; profiles/r02/deinterleave_u32_crossover.jsonl,
    // deinterleave_narrow_big_tiles.jsonl).
    // BCN_DEINT_U32_NARROW_MAX overrides the crossover (exploration).
    static const uint64_t narrow_max_u32 = [] {
        const char* v = std::getenv("BCN_DEINT_U32_NARROW_MAX");
        return v ? static_cast<uint64_t>(std::strtoul(v, nullptr, 10)) : uint64_t{128};
    }();
    const uint64_t narrow_max = sizeof(T) == 8 ? 85 : narrow_max_u32;
    // Sector-aligned narrow tiles for 8-byte items with W >= 40 whose worker
    // runs are not sector-aligned: +4 / +13 / +36 / +20% at W = 48 / 63 / 65 /
    // 85 (2^30 items), +-1% below W = 40. 4-byte items measured 7-38% slower
    // with them even with a lean store loop: the 8 halo rows and the
    // rounding of R to 16 cut the rows per 8192-slot tile (W = 116: 48 + 8
    // rows against 64), so they keep the plain tiles
    // (profiles/r02/deinterleave_narrow_halo_ab.jsonl, deinterleave_narrow_halo_u32_lean.jsonl).
    constexpr uint64_t kSector = 32 / sizeof(T);
    const bool narrow_halo = sizeof(T) == 8 && a.width >= 40 && a.width <= narrow_max && narrow_halo_enabled() &&
                             (a.wpw % kSector != 0 || (a.out_mod + a.i_base) % kSector != 0);
    if (narrow_halo) {
        using G = NarrowTile<T>;
        const size_t smemh = (G::kItems + kNarrowMaxWidth) * sizeof(T);
        const uint64_t rows_per_tile = G::rows_halo(static_cast<unsigned>(a.width), kSector);
        const uint64_t tiles = (a.rows + rows_per_tile - 1) / rows_per_tile;
        TransposeArgs b = a;
        b.pitch = 0;
        if (narrow_threads<T>() == 512) {
            cudaFuncSetAttribute(k_transpose_narrow_h<T, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smemh));
            const uint64_t cap = static_cast<uint64_t>(sms) * occupancy(k_transpose_narrow_h<T, 512>, 512, smemh);
            k_transpose_narrow_h<T, 512><<<static_cast<unsigned>(std::min(tiles, cap)), 512, smemh, s>>>(b);
        } else {
            cudaFuncSetAttribute(k_transpose_narrow_h<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smemh));
            const uint64_t cap = static_cast<uint64_t>(sms) * occupancy(k_transpose_narrow_h<T>, 256, smemh);
            k_transpose_narrow_h<T><<<static_cast<unsigned>(std::min(tiles, cap)), 256, smemh, s>>>(b);
        }
    } else if (a.width > narrow_big_min<T>() && a.width <= narrow_max) {
        // 16384-slot tiles on 512 threads (twice the rows per tile)
        using G = NarrowTile<T, 16384>;
        const size_t smem = (G::kItems + kNarrowMaxWidth) * sizeof(T);
        const uint64_t rows_per_tile = G::rows(static_cast<unsigned>(a.width));
        const uint64_t tiles = (a.rows + rows_per_tile - 1) / rows_per_tile;
        TransposeArgs b = a;
        b.pitch = sizeof(T) == 4 ? narrow_pitch_u32(static_cast<unsigned>(a.width), static_cast<unsigned>(rows_per_tile)) : 0;
        cudaFuncSetAttribute(k_transpose_narrow<T, 512, 16384>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        const uint64_t cap = static_cast<uint64_t>(sms) * occupancy(k_transpose_narrow<T, 512, 16384>, 512, smem);
        k_transpose_narrow<T, 512, 16384><<<static_cast<unsigned>(std::min(tiles, cap)), 512, smem, s>>>(b);
    } else if (a.width <= narrow_max) {
        using G = NarrowTile<T>;
        const size_t smem = (G::kItems + kNarrowMaxWidth) * sizeof(T);
        const uint64_t rows_per_tile = G::rows(static_cast<unsigned>(a.width));
        const uint64_t tiles = (a.rows + rows_per_tile - 1) / rows_per_tile;
        TransposeArgs b = a;
        b.pitch = sizeof(T) == 4 ? narrow_pitch_u32(static_cast<unsigned>(a.width), static_cast<unsigned>(rows_per_tile)) : 0;
        if (narrow_threads<T>() == 512) {
            cudaFuncSetAttribute(k_transpose_narrow<T, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem));
            const uint64_t cap = static_cast<uint64_t>(sms) * occupancy(k_transpose_narrow<T, 512>, 512, smem);
            k_transpose_narrow<T, 512><<<static_cast<unsigned>(std::min(tiles, cap)), 512, smem, s>>>(b);
        } else {
            cudaFuncSetAttribute(k_transpose_narrow<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem));
            const uint64_t cap = static_cast<uint64_t>(sms) * occupancy(k_transpose_narrow<T>, 256, smem);
            k_transpose_narrow<T><<<static_cast<unsigned>(std::min(tiles, cap)), 256, smem, s>>>(b);
        }
    } else {
        // Wide regions move through the TMA tile mover (bcn_deint_tma.cu) when
        // its tensor maps can describe them.
        if (allow_tma && tma_deinterleave_enabled()) {
            bool used = false;
            const cudaError_t e = launch_transpose_tma(a, sms, s, &used);
            if (e != cudaSuccess || used) return e;
        }
        // Tile shape sweep (profiles/r01/deinterleave_tiles.jsonl): 128-row
        // tiles win everywhere; 8-byte items prefer 1 KiB input runs unless
        // the last tile column would be mostly empty (e.g. W = 129).
        // 4-byte items likewise fall back from 512-byte (128-worker) to
        // 256-byte (64-worker) tiles when the last tile column would be mostly
        // empty (u32 W = 129: 0.54 ms with 128-worker tiles). 256-row u32
        // tiles (1 KiB output runs) measured no better
        // (profiles/r01/deinterleave_u32_256row_negative.jsonl).
        static const int shape = [] {  // exploration knob: force one wide tile shape
            const char* v = std::getenv("BCN_DEINT_WIDE");
            return v ? static_cast<int>(std::strtol(v, nullptr, 10)) : 0;
        }();
        switch (shape) {
            case 1: return transpose_wide<T, 128, 1024>(a, sms, s);
            case 2: return transpose_wide<T, 64, 1024>(a, sms, s);
            case 3: return transpose_wide<T, 32, 1024>(a, sms, s);
            case 4:
                if constexpr (sizeof(T) == 8) return transpose_wide<T, 64, 2048>(a, sms, s);
                break;
            case 5:
                if constexpr (sizeof(T) == 8) return transpose_wide<T, 32, 2048>(a, sms, s);
                break;
            case 6: return transpose_wide<T, 128, 512>(a, sms, s);
            default: break;
        }
        const uint64_t cover128 = (a.width + 127) / 128 * 128, cover64 = (a.width + 63) / 64 * 64;
        const bool wide_cols = cover128 * 10 <= cover64 * 11;
        if constexpr (sizeof(T) == 8) {
            if (wide_cols) return transpose_wide<T, 128, 1024>(a, sms, s);
            return transpose_wide<T, 128, 512>(a, sms, s);
        } else {
            if (wide_cols) return transpose_wide<T, 128, 512>(a, sms, s);
            return transpose_wide<T, 128, 256>(a, sms, s);
        }
    }
    return counted(cudaGetLastError());
}
}  // namespace

cudaError_t launch_transpose(const TransposeArgs& a, cudaStream_t s) {
    if (a.rows == 0 || a.width == 0) return cudaSuccess;
    return a.itemsize == 8 ? transpose_t<uint64_t>(a, s, true) : transpose_t<uint32_t>(a, s, true);
}

cudaError_t launch_transpose_registers(const TransposeArgs& a, cudaStream_t s) {
    if (a.rows == 0 || a.width == 0) return cudaSuccess;
    return a.itemsize == 8 ? transpose_t<uint64_t>(a, s, false) : transpose_t<uint32_t>(a, s, false);
}

int contig_blocks_per_sm(int fmt, int engine, int block) {
#define BCN_OCC(F)                                                                   \
    switch (engine) {                                                                \
        case kEngBarrett: return occupancy(k_fill_contig<F, kEngBarrett>, block);    \
        case kEngMontgomery: return occupancy(k_fill_contig<F, kEngMontgomery>, block); \
        case kEngFP64: return occupancy(k_fill_contig<F, kEngFP64>, block);          \
        case kEngMixed: return occupancy(k_fill_contig<F, kEngMixed>, block);        \
        default: {                                                                   \
            int n = 1;                                                               \
            hybrid_dispatch<F>(engine, [&](auto kf) {                                \
                n = occupancy(k_fill_contig<F, kEngHybridBase + decltype(kf)::value>, block); \
            });                                                                      \
            return n;                                                                \
        }                                                                            \
    }
    switch (fmt) {
        case kFmtU64: BCN_OCC(kFmtU64) break;
        case kFmtF64: BCN_OCC(kFmtF64) break;
        case kFmtF32: BCN_OCC(kFmtF32) break;
    }
#undef BCN_OCC
    return 1;
}

int interleaved_blocks_per_sm(int fmt, int engine, int block) {
#define BCN_OCC(F)                                                                        \
    switch (engine) {                                                                     \
        case kEngBarrett: return occupancy(k_fill_interleaved<F, kEngBarrett>, block);    \
        case kEngMontgomery: return occupancy(k_fill_interleaved<F, kEngMontgomery>, block); \
        case kEngFP64: return occupancy(k_fill_interleaved<F, kEngFP64>, block);          \
        case kEngMixed: return occupancy(k_fill_interleaved<F, kEngMixed>, block);        \
    }
    switch (fmt) {
        case kFmtU64: BCN_OCC(kFmtU64) break;
        case kFmtF64: BCN_OCC(kFmtF64) break;
        case kFmtF32: BCN_OCC(kFmtF32) break;
    }
#undef BCN_OCC
    return 1;
}

cudaError_t upload_tables() {
    static std::mutex mu;
    static bool done[64] = {};
    int dev = 0;
    cudaError_t err = cudaGetDevice(&dev);
    if (err != cudaSuccess) return err;
    std::lock_guard<std::mutex> lock(mu);
    if (dev >= 0 && dev < 64 && done[dev]) return cudaSuccess;
    static uint64_t host_tab[kPowWindows][16][2];
    static bool built = false;
    if (!built) {
        for (int i = 0; i < kPowWindows; ++i) {
            // 2^(16^i) mod m, then its powers d = 0..15.
            const uint64_t base = host_pow2(static_cast<uint64_t>(1) << (4 * i));
            uint64_t v = 1;
            for (int d = 0; d < 16; ++d) {
                host_tab[i][d][0] = v;
                host_tab[i][d][1] = host_shoup(v);
                v = host_mulmod(v, base);
            }
        }
        built = true;
    }
    err = cudaMemcpyToSymbol(g_pow, host_tab, sizeof(host_tab));
    if (err == cudaSuccess && dev >= 0 && dev < 64) done[dev] = true;
    return err;
}

}  // namespace bcn_b200
