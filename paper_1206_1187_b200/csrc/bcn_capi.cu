// bcn_capi.cu — the extern "C" boundary (include/bcnrand_b200.h).
//
// Host responsibilities: validate exactly like the reference (before any
// device work), translate the reference's plan semantics (make_plan,
// physical_index, base_offset wrap) into affine exponent segments and
// interleaved regions, and launch the sm_100a kernels of bcn_kernels.cu.
// Host output buffers are filled by generating chunks on the device and
// copying them back (two streams, generation overlapped with D2H).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#if defined(__x86_64__)
#include <emmintrin.h>
#endif

#include "bcnrand_b200.h"
#include "bcn_kernels.cuh"

using namespace bcn_b200;

namespace {

thread_local std::string g_last_error;

bcn_status fail(bcn_status st, const std::string& msg) {
    g_last_error = msg;
    return st;
}

bcn_status cuda_fail(cudaError_t e, const char* where) {
    return fail(BCN_ERR_CUDA, std::string(where) + ": " + cudaGetErrorName(e) + " (" +
                                  cudaGetErrorString(e) + ")");
}

#define BCN_CUDA(call)                                   \
    do {                                                 \
        cudaError_t e_ = (call);                         \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

// ----------------------------------------------------------- plan (host)
// reference parallel.cpp:35-52 / :19-33
struct Plan {
    uint64_t n = 0;
    uint64_t wpw = 0;
    uint32_t workers = 1;
    int layout = 0;
    uint64_t elements_for(uint32_t w) const {
        const uint64_t start = static_cast<uint64_t>(w) * wpw;
        return std::min(wpw, n - start);
    }
    uint64_t short_count() const { return elements_for(workers - 1); }
};

bcn_status make_plan(uint64_t n, uint32_t workers, int layout, Plan* p) {
    if (n == 0) return fail(BCN_ERR_INVALID_ARGUMENT, "make_plan: n must be at least 1");
    if (workers == 0) return fail(BCN_ERR_INVALID_ARGUMENT, "make_plan: workers must be at least 1");
    p->n = n;
    p->wpw = (n + workers - 1) / workers;
    p->workers = static_cast<uint32_t>((n + p->wpw - 1) / p->wpw);
    p->layout = layout;
    return BCN_OK;
}

bcn_status check_seed(uint64_t a) {
    if (a < kMinSeed || a > kMaxSeed)
        return fail(BCN_ERR_OUT_OF_RANGE, "seed_from_index: index outside [3^33+100, 2^53]");
    return BCN_OK;
}

// ------------------------------------------------------- device context
struct DevCtx {
    bool init = false;
    int sms = 148;
    cudaStream_t stream = nullptr;    // internal stream for stream == NULL calls
    cudaStream_t copy[2] = {nullptr, nullptr};
    void* scratch[2] = {nullptr, nullptr};  // device chunks for host outputs
    void* pinned[2] = {nullptr, nullptr};   // pinned staging for pageable outputs
    size_t chunk_bytes = 0;
    unsigned long long* digest = nullptr;
    int* flag = nullptr;
    void* qscratch = nullptr;         // quality-suite counts / partial sums (grows)
    size_t qscratch_bytes = 0;
    std::map<int, int> occ;           // (interleaved*1024 + fmt*64 + engine) -> blocks per SM
    std::mutex occ_mu;                // guards occ
    std::mutex mu;                    // serialises host-buffer fills on this device
    std::mutex small_mu;              // serialises users of digest / flag / qscratch
    // Automatic write pacing (calibrate_pace): this device's target and the
    // sweep it came from.
    std::once_flag pace_once;
    double pace_cal = kDefaultPaceGBs;
    int pace_src = BCN_PACE_DEFAULT;
    std::vector<std::pair<double, double>> pace_curve;  // (target, achieved) GB/s
};

std::mutex g_ctx_mu;
std::map<int, DevCtx*> g_ctx;

double pace_gbs(DevCtx* c);
std::atomic<double>& pace_setting();

bcn_status get_ctx_nocal(int device, DevCtx** out) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        return fail(BCN_ERR_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
    if (device < 0 || device >= count)
        return fail(BCN_ERR_INVALID_ARGUMENT, "device ordinal out of range");
    BCN_CUDA(cudaSetDevice(device));
    std::lock_guard<std::mutex> lock(g_ctx_mu);
    DevCtx*& c = g_ctx[device];
    if (!c) c = new DevCtx();
    if (!c->init) {
        BCN_CUDA(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device));
        BCN_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        BCN_CUDA(cudaStreamCreateWithFlags(&c->copy[0], cudaStreamNonBlocking));
        BCN_CUDA(cudaStreamCreateWithFlags(&c->copy[1], cudaStreamNonBlocking));
        BCN_CUDA(cudaMalloc(&c->digest, 3 * sizeof(unsigned long long)));
        BCN_CUDA(cudaMalloc(&c->flag, sizeof(int)));
        BCN_CUDA(upload_tables());
        c->init = true;
    }
    *out = c;
    return BCN_OK;
}

bcn_status get_ctx(int device, DevCtx** out) {
    bcn_status st = get_ctx_nocal(device, out);
    // Automatic pacing: measure this device's target once, at context
    // initialisation, so no fill (or timed region) pays for it later.
    if (!st && pace_setting().load() < 0.0) pace_gbs(*out);
    return st;
}

// Restores the calling thread's current device on scope exit: entry points
// switch to the buffer's device (get_ctx) but must not leave the caller's
// CUDA state (e.g. PyTorch's current device) changed.
class DeviceGuard {
  public:
    DeviceGuard() {
        if (cudaGetDevice(&prev_) != cudaSuccess) {
            cudaGetLastError();
            prev_ = -1;
        }
    }
    ~DeviceGuard() {
        int now = -1;
        if (prev_ >= 0 && cudaGetDevice(&now) == cudaSuccess && now != prev_) cudaSetDevice(prev_);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;

  private:
    int prev_ = -1;
};

// Device scratch of at least `bytes` for the quality suite (caller holds small_mu).
bcn_status quality_scratch(DevCtx* c, size_t bytes, void** out) {
    if (c->qscratch_bytes < bytes) {
        if (c->qscratch) BCN_CUDA(cudaFree(c->qscratch));
        c->qscratch = nullptr;
        c->qscratch_bytes = 0;
        BCN_CUDA(cudaMalloc(&c->qscratch, bytes));
        c->qscratch_bytes = bytes;
    }
    *out = c->qscratch;
    return BCN_OK;
}

// Stream of a call on device memory. stream != NULL: the caller's stream
// (ordering against the caller's other work is the caller's business).
// stream == NULL: the library's internal stream, after every earlier piece of
// work on the device has finished, so a synchronous call sees all prior
// writes to its buffers whatever stream made them, like the reference's
// synchronous functions.
bcn_status caller_stream(DevCtx* c, void* stream, cudaStream_t* s) {
    if (stream) {
        *s = static_cast<cudaStream_t>(stream);
        return BCN_OK;
    }
    BCN_CUDA(cudaDeviceSynchronize());
    *s = c->stream;
    return BCN_OK;
}

// Hybrid engine split: FP64 streams per lane vector (the rest run Barrett);
// BCN_HYBRID_KF overrides it for exploration (1 <= KF < streams per lane).
int hybrid_kf(int fmt) {
    static const long env = [] {
        const char* v = std::getenv("BCN_HYBRID_KF");
        return v ? std::strtol(v, nullptr, 10) : 0L;
    }();
    const int vec = fmt == kFmtF32 ? 8 : 4;
    if (env >= 1 && env < vec) return static_cast<int>(env);
    return vec - 1;
}

int resolve_engine(int engine, int fmt) {
    if (engine == kEngHybrid) return kEngHybridBase + hybrid_kf(fmt);
    if (engine != kEngAuto) return engine;
    return kEngFP64;  // measured best (profiles/)
}

bool is_hybrid(int engine) { return engine >= kEngHybridBase; }

int blocks_per_sm(DevCtx* c, int fmt, int engine, bool interleaved) {
    const int key = (interleaved ? 1024 : 0) + fmt * 64 + engine;
    std::lock_guard<std::mutex> lock(c->occ_mu);
    auto it = c->occ.find(key);
    if (it != c->occ.end()) return it->second;
    const int n = interleaved ? interleaved_blocks_per_sm(fmt, engine, kContigThreads)
                              : contig_blocks_per_sm(fmt, engine, kContigThreads);
    c->occ[key] = n;
    return n;
}

// Launch tuning (bcn_set_launch_config): CTAs per SM for the persistent
// fill grids (0 = as many as fit) and the row order of the contiguous kernels.
std::atomic<int> g_ctas_per_sm{0};
std::atomic<int> g_row_order{1};
// Write pacing (bcn_set_write_pacing): target HBM write rate of the paced
// contiguous kernels in GB/s — < 0: automatic (each device's calibrated
// target, calibrate_pace), 0: unpaced, else fixed — and their CTAs per SM.
constexpr double kMinPaceGBs = 100.0;  // lower fixed targets would stall a launch for seconds
std::atomic<double> g_pace_gbs{-1.0};
std::atomic<int> g_pace_cps{kDefaultPaceCps};
std::atomic<int> g_pace_formats{(1 << kFmtU64) | (1 << kFmtF64)};
std::atomic<double>& pace_setting() { return g_pace_gbs; }

// CTAs of the paced grid: ctas_per_sm x SMs, or BCN_PACE_GRID (an
// exploration override: total CTAs, e.g. to leave SMs idle under a power cap).
// The interleaved kernel does ~20 instructions per variate against ~15 for the
// contiguous one and needs more worker warps per SM to keep up with the pacer
// (profiles/r01/interleaved_cps.jsonl, TB/s with 1 / 2 / 3 CTAs per SM:
// W = 7: 5.0 / 5.6 / 6.3; W = 64...100003: 5.2-5.5 / 5.8-6.0 / 5.7-5.9).
// The Mixed engine (~1 DFMA + 8 integer ops per step) likewise needs 2 CTAs
// per SM (profiles/r01/tune_engines_cps.jsonl: 5.8 TB/s with 1, 7.05 with 2).
uint64_t paced_grid(const DevCtx* c, int engine, uint64_t interleaved_width = 0) {
    static const long env = [] {
        const char* v = std::getenv("BCN_PACE_GRID");
        return v ? std::strtol(v, nullptr, 10) : 0L;
    }();
    if (env > 0) return static_cast<uint64_t>(env);
    int cps = g_pace_cps.load();
    if (interleaved_width) cps = std::max(interleaved_width <= 32 ? 3 : 2, cps);
    if (engine == kEngMixed) cps = std::max(2, cps);
    return static_cast<uint64_t>(c->sms) * cps;
}

// Pacing only helps a kernel that can outrun the write path. The integer
// engines (Barrett ~26, Montgomery ~30 instructions per variate) are
// compute-bound below it and run faster unpaced at full occupancy (paced at
// 1..4 CTAs per SM: Barrett 3.9-5.6 TB/s, Montgomery 3.3-4.5,
// tune_engines_cps.jsonl; unpaced: 6.1 / 4.8, ab_f64.jsonl).
bool paced(DevCtx* c, int fmt, int engine) {
    return (g_pace_formats.load() >> fmt & 1) && (engine == kEngFP64 || engine == kEngMixed || is_hybrid(engine)) &&
           pace_gbs(c) > 0.0;
}

// Pacer period (ns x 256) for `bytes_per_round` at `gbs` (1 GB/s == 1 byte/ns;
// gbs >= kMinPaceGBs keeps this far below 2^64).
uint64_t pace_gap_q8_bytes(double bytes_per_round, double gbs) {
    return static_cast<uint64_t>(256.0 * bytes_per_round / std::max(gbs, kMinPaceGBs));
}

// One round of a grid-strided paced grid writes grid * 8 workers * H rows * 1 KiB.
uint64_t pace_gap_q8(int grid, double gbs, int fmt, bool constant = false) {
    return pace_gap_q8_bytes(1024.0 * grid * (kPacedThreads / 32 - 1) * paced_rows_per_round(fmt, constant), gbs);
}

int grid_for_rows(DevCtx* c, int fmt, int engine, bool interleaved, uint64_t rows) {
    int per_sm = blocks_per_sm(c, fmt, engine, interleaved);
    const int want = g_ctas_per_sm.load();
    if (want > 0 && want < per_sm) per_sm = want;
    const uint64_t persistent = static_cast<uint64_t>(c->sms) * per_sm;
    const uint64_t needed = (rows + (kContigThreads / 32) - 1) / (kContigThreads / 32);
    return static_cast<int>(std::max<uint64_t>(1, std::min(persistent, needed)));
}

uint64_t mod_p(unsigned __int128 x) { return static_cast<uint64_t>(x % kPeriod); }

// Exponent of 2 (mod P) for logical element j when every element from 0 is on
// one affine segment whose first state is next(state_at(a, k0)).
uint64_t exp_add(uint64_t e, uint64_t j) { return mod_p(static_cast<unsigned __int128>(e) + mod_p(static_cast<unsigned __int128>(j) * 53u)); }

// Jump multiplier for a signed number of logical steps.
Mult mult_for_steps(__int128 steps) {
    __int128 s = steps % static_cast<__int128>(kPeriod);
    if (s < 0) s += kPeriod;
    return host_make_mult(host_jump(static_cast<uint64_t>(s)));
}

// ------------------------------------------------------------- launching
struct FillJob {
    const Plan* plan;
    int fmt;
    int engine;
    uint64_t a;
    uint64_t base_offset;
    uint64_t a_exp;  // (a - 3^33 - 1) mod P
    DevCtx* ctx;
    cudaStream_t stream;
};

cudaError_t enqueue_slots(const FillJob& j, char* dptr, uint64_t slot0, uint64_t count) {
    if (count == 0) return cudaSuccess;
    SlotArgs s;
    s.out = dptr;
    s.slot0 = slot0;
    s.count = count;
    s.n = j.plan->n;
    s.wpw = j.plan->wpw;
    s.workers = j.plan->workers;
    s.layout = j.plan->layout;
    s.a_exp = j.a_exp;
    s.base_offset = j.base_offset;
    return launch_slots(j.fmt, s, j.stream);
}

// Physical slots [slot0, slot0+count) whose logical exponents are affine:
// slot slot0 + x has exponent (e_first + 53 x) mod P.
cudaError_t enqueue_affine(const FillJob& j, char* dptr, uint64_t slot0, uint64_t count,
                           uint64_t e_first) {
    const int isz = format_itemsize(j.fmt);
    if (count == 0) return cudaSuccess;
    const uint64_t addr = reinterpret_cast<uint64_t>(dptr);
    if (j.engine == kEngStaged) {
        const uint64_t tile = static_cast<uint64_t>(kStagedThreads) * kStagedL;
        const uint64_t head = std::min<uint64_t>(count, ((16 - addr % 16) % 16) / isz);
        const uint64_t tiles = (count - head) / tile;
        cudaError_t e = enqueue_slots(j, dptr, slot0, head);
        if (e != cudaSuccess) return e;
        if (tiles) {
            StagedArgs s;
            s.out = dptr + head * isz;
            s.tiles = tiles;
            s.e0 = exp_add(e_first, head);
            const int grid = static_cast<int>(std::min<uint64_t>(tiles, static_cast<uint64_t>(j.ctx->sms) * 3));
            s.jump_next = mult_for_steps(static_cast<__int128>(grid) * tile - kStagedL);
            e = launch_staged(j.fmt, s, grid, j.stream);
            if (e != cudaSuccess) return e;
        }
        const uint64_t done = head + tiles * tile;
        return enqueue_slots(j, dptr + done * isz, slot0 + done, count - done);
    }
    const uint64_t row = 32ull * (32 / isz);
    if (j.engine != kEngBulk) {
        // Whole rows from the 32-byte aligned address at or below dptr; the
        // partial first / last rows are written by the same kernel
        // (EdgeRow), so a range is exactly one launch.
        const uint64_t lo = (addr % 32) / isz;  // elements of the first row before dptr
        char* base = dptr - lo * isz;
        EdgeRow edge[2] = {};
        uint64_t consumed = 0;
        if (lo) {
            consumed = std::min<uint64_t>(count, row - lo);
            edge[0] = EdgeRow{base, exp_add(e_first, kPeriod - lo), static_cast<uint32_t>(lo),
                              static_cast<uint32_t>(lo + consumed)};
            base += row * isz;
        }
        const uint64_t rows = (count - consumed) / row;
        const uint64_t tail = (count - consumed) % row;
        if (tail)
            edge[1] = EdgeRow{base + rows * row * isz, exp_add(e_first, consumed + rows * row), 0,
                              static_cast<uint32_t>(tail)};
        ContigArgs c{};
        c.out = base;
        c.rows = rows;
        c.e0 = exp_add(e_first, consumed);
        c.edge[0] = edge[0];
        c.edge[1] = edge[1];
        if (paced(j.ctx, j.fmt, j.engine)) {
            // Paced path (by default for the 8-byte formats; f32 with the
            // FP64 engine is FP64-pipe bound below the write roof).
            constexpr uint64_t kWorkers = kPacedThreads / 32 - 1;
            const uint64_t want = paced_grid(j.ctx, j.engine);
            const int grid = static_cast<int>(std::max<uint64_t>(1, std::min(want, (rows + kWorkers - 1) / kWorkers)));
            PacedArgs pa{};
            pa.out = c.out;
            pa.rows = rows;
            pa.e0 = c.e0;
            pa.jump = mult_for_steps(static_cast<__int128>(row) * grid * kWorkers * paced_rows_per_round(j.fmt));
            pa.gap_q8 = pace_gap_q8(grid, pace_gbs(j.ctx), j.fmt);
            pa.mode = kPacedContiguous;
            pa.edge[0] = edge[0];
            pa.edge[1] = edge[1];
            return launch_paced(j.fmt, j.engine, pa, grid, j.stream);
        }
        const int grid = grid_for_rows(j.ctx, j.fmt, j.engine, false, std::max<uint64_t>(rows, 1));
        c.stride_order = static_cast<uint32_t>(g_row_order.load());
        const uint64_t step_rows = c.stride_order ? static_cast<uint64_t>(grid) * (kContigThreads / 32) : 1;
        c.jump_row = mult_for_steps(static_cast<__int128>(row) * step_rows);
        return launch_contig(j.fmt, j.engine, c, grid, kContigThreads, j.stream);
    }
    const uint64_t head = std::min<uint64_t>(count, ((32 - addr % 32) % 32) / isz);
    const uint64_t rows = (count - head) / row;
    cudaError_t e = enqueue_slots(j, dptr, slot0, head);
    if (e != cudaSuccess) return e;
    if (rows) {
        ContigArgs c{};
        c.out = dptr + head * isz;
        c.rows = rows;
        c.e0 = exp_add(e_first, head);
        {
            // Streams advance one 16-row tile per step (k_fill_bulk).
            c.jump_row = mult_for_steps(static_cast<__int128>(row) * kBulkTileRows);
            const uint64_t tiles = (rows + kBulkTileRows - 1) / kBulkTileRows;
            const uint64_t persistent = static_cast<uint64_t>(j.ctx->sms) * bulk_blocks_per_sm(j.fmt);
            const int grid = static_cast<int>(std::max<uint64_t>(1, std::min(persistent, tiles)));
            e = launch_bulk(j.fmt, c, grid, j.stream);
        }
        if (e != cudaSuccess) return e;
    }
    const uint64_t done = head + rows * row;
    return enqueue_slots(j, dptr + done * isz, slot0 + done, count - done);
}

// Interleaved region slots: region-relative slots [q_begin, q_begin+count)
// of a region of `width` workers starting at element i_base; dptr is slot
// q_begin; slot0 is its global physical slot (for the slot kernel).
cudaError_t enqueue_region(const FillJob& j, char* dptr, uint64_t slot0, uint64_t q_begin,
                           uint64_t count, uint64_t width, uint64_t i_base, uint64_t e_elem0) {
    const Plan& p = *j.plan;
    if (width == 1) {
        // Worker 0 only: logical j = i_base + q, affine.
        return enqueue_affine(j, dptr, slot0, count, exp_add(e_elem0, i_base + q_begin));
    }
    const int isz = format_itemsize(j.fmt);
    // The staged paths are contiguous-only; interleaved regions use the
    // matching direct-store engine.
    const int engine = j.engine == kEngStaged ? kEngBarrett
                       : (j.engine == kEngBulk || is_hybrid(j.engine)) ? kEngFP64
                                                                        : j.engine;
    const uint64_t addr = reinterpret_cast<uint64_t>(dptr);
    const uint64_t row = 32ull * (32 / isz);
    const uint64_t head = std::min<uint64_t>(count, ((32 - addr % 32) % 32) / isz);
    const uint64_t rows = (count - head) / row;
    cudaError_t e = enqueue_slots(j, dptr, slot0, head);
    if (e != cudaSuccess) return e;
    if (rows) {
        InterleavedArgs r;
        r.out = dptr + head * isz;
        r.rows = rows;
        r.q0 = q_begin + head;
        r.width = width;
        r.i_base = i_base;
        r.wpw = p.wpw;
        r.e0 = e_elem0;
        const uint64_t adv_a = row / width;
        r.adv_b = row % width;
        // Same physical row: w += b, i += a -> logical += b*wpw + a.
        r.jump_same = mult_for_steps(static_cast<__int128>(r.adv_b) * p.wpw + adv_a);
        // Crossing a physical row: w += b - width, i += a + 1.
        r.jump_wrap = mult_for_steps((static_cast<__int128>(r.adv_b) - static_cast<__int128>(width)) *
                                         static_cast<__int128>(p.wpw) +
                                     adv_a + 1);
        constexpr uint64_t kWorkers = kPacedThreads / 32 - 1;
        // Column-stable super-rows: the region is cut into super-rows of L
        // slots, L a multiple of both the width and the 32-byte chunk (lcm x
        // k0, the largest that fits the grid's workers); worker w writes the
        // 1 KiB block at w * row of every super-row (the last block of a
        // super-row is partial, whole chunks; workers past it idle). A slot
        // and the same slot one super-row later hold the same worker column,
        // L / width elements apart, so every stream steps by ONE multiplier —
        // the contiguous kernel's arithmetic with interleaved seeding — for
        // any width whose lcm fits: u64 up to ~37k workers with 1 CTA per SM,
        // ~113k with 3. Taken with the fewest CTAs per SM (1..3) at which
        // >= 95% of the workers have a block: W = 125 / 250 / 1001 at 1 CTA
        // per SM, +6 / +3 / +2% over r01's modes; W = 5003 with 92.5% at 1 CTA
        // per SM measured 3% slower than two multipliers, so it takes 2
        // (profiles/r02/interleaved_super.jsonl). Otherwise the two-multiplier
        // mode below.
        const uint64_t chunk = 32 / isz;
        const uint64_t lcm = width / std::gcd(width, chunk) * chunk;
        const int H = paced_rows_per_round(j.fmt);
        uint64_t sr_grid = 0, sr_len = 0;
        for (int cps = 1; cps <= 3 && !sr_grid; ++cps) {
            const uint64_t nwk = static_cast<uint64_t>(j.ctx->sms) * cps * kWorkers;
            const uint64_t k0 = row * nwk / lcm;
            const uint64_t L = k0 * lcm;
            if (k0 && (L + row - 1) / row * 100 >= nwk * 95) {
                sr_grid = static_cast<uint64_t>(j.ctx->sms) * cps;
                sr_len = L;
            }
        }
        if (paced(j.ctx, j.fmt, engine) && sr_grid) {
            const uint64_t n_slots = rows * row;
            const uint64_t busy = (std::min(sr_len, n_slots) + row - 1) / row;  // workers with a block
            const uint64_t grid = std::min(sr_grid, (busy + kWorkers - 1) / kWorkers);
            PacedArgs pa{};
            pa.out = r.out;
            pa.rows = rows;
            pa.e0 = r.e0;
            pa.gap_q8 = pace_gap_q8_bytes(static_cast<double>(H) * std::min(sr_len, n_slots) * isz, pace_gbs(j.ctx));
            pa.mode = kPacedInterleavedFixed;
            pa.q0 = r.q0;
            pa.width = width;
            pa.i_base = i_base;
            pa.wpw = p.wpw;
            pa.row_stride = sr_len;
            pa.jump = mult_for_steps(static_cast<__int128>(H) * (sr_len / width));
            e = launch_paced(j.fmt, engine, pa, static_cast<int>(grid), j.stream);
        } else if (paced(j.ctx, j.fmt, engine)) {
            // Paced, grid-strided: each stream advances nwk rows = S slots per round.
            const uint64_t want = paced_grid(j.ctx, engine, width);
            const int grid = static_cast<int>(std::max<uint64_t>(1, std::min(want, (rows + kWorkers - 1) / kWorkers)));
            const unsigned __int128 S =
                static_cast<unsigned __int128>(row) * grid * kWorkers * paced_rows_per_round(j.fmt);
            const uint64_t a_s = static_cast<uint64_t>(S / width), b_s = static_cast<uint64_t>(S % width);
            PacedArgs pa{};
            pa.out = r.out;
            pa.rows = rows;
            pa.e0 = r.e0;
            pa.gap_q8 = pace_gap_q8(grid, pace_gbs(j.ctx), j.fmt);
            pa.mode = kPacedInterleaved;
            pa.q0 = r.q0;
            pa.width = width;
            pa.i_base = i_base;
            pa.wpw = p.wpw;
            pa.adv_b = b_s;
            pa.jump = mult_for_steps(static_cast<__int128>(b_s) * p.wpw + a_s);
            pa.jump_wrap = mult_for_steps((static_cast<__int128>(b_s) - static_cast<__int128>(width)) *
                                              static_cast<__int128>(p.wpw) +
                                          a_s + 1);
            e = launch_paced(j.fmt, engine, pa, grid, j.stream);
        } else {
            const int grid = grid_for_rows(j.ctx, j.fmt, engine, true, rows);
            e = launch_interleaved(j.fmt, engine, r, grid, kContigThreads, j.stream);
        }
        if (e != cudaSuccess) return e;
    }
    const uint64_t done = head + rows * row;
    return enqueue_slots(j, dptr + done * isz, slot0 + done, count - done);
}

// Writes physical slots [p0, p1) of the plan into dptr (dptr == slot p0).
cudaError_t enqueue_range(const FillJob& j, char* dptr, uint64_t p0, uint64_t p1) {
    const Plan& p = *j.plan;
    const int isz = format_itemsize(j.fmt);
    const uint64_t last_start = static_cast<uint64_t>(p.workers - 1) * p.wpw;
    const bool wraps = j.base_offset > UINT64_MAX - last_start;
    if (p.layout == 0) {
        // Affine segments: workers whose k_w = B + start_w does not wrap, then
        // those that do (reference u64 arithmetic, parallel.cpp:63-64).
        uint64_t cut = p.n;  // first slot of the wrapped segment
        if (wraps) {
            const unsigned __int128 room = (static_cast<unsigned __int128>(1) << 64) - j.base_offset;
            const uint64_t wstar = static_cast<uint64_t>((room + p.wpw - 1) / p.wpw);
            cut = std::min<uint64_t>(p.n, wstar * p.wpw);
        }
        const uint64_t e_seg0 = host_fill_e0(j.a, j.base_offset);
        if (p0 < cut) {
            const uint64_t end = std::min(p1, cut);
            cudaError_t e = enqueue_affine(j, dptr, p0, end - p0, exp_add(e_seg0, p0));
            if (e != cudaSuccess) return e;
        }
        if (p1 > cut) {
            const uint64_t begin = std::max(p0, cut);
            const uint64_t e_seg1 = host_fill_e0(j.a, j.base_offset + cut);  // wrapped k
            return enqueue_affine(j, dptr + (begin - p0) * isz, begin, p1 - begin,
                                  exp_add(e_seg1, begin - cut));
        }
        return cudaSuccess;
    }
    if (wraps) return enqueue_slots(j, dptr, p0, p1 - p0);  // exact, slow, rare
    const uint64_t e0 = host_fill_e0(j.a, j.base_offset);
    const uint64_t sc = p.short_count();
    const uint64_t main = sc * p.workers;
    if (p0 < main) {
        const uint64_t end = std::min(p1, main);
        cudaError_t e = enqueue_region(j, dptr, p0, p0, end - p0, p.workers, 0, e0);
        if (e != cudaSuccess) return e;
    }
    if (p1 > main) {
        const uint64_t begin = std::max(p0, main);
        return enqueue_region(j, dptr + (begin - p0) * isz, begin, begin - main, p1 - begin,
                              p.workers - 1, sc, e0);
    }
    return cudaSuccess;
}

bcn_status validate_enums(int fmt, int layout, int method, int engine) {
    if (fmt < 0 || fmt > 2) return fail(BCN_ERR_INVALID_ARGUMENT, "fill: unknown format");
    if (layout < 0 || layout > 1) return fail(BCN_ERR_INVALID_ARGUMENT, "fill: unknown layout");
    if (method < 0 || method > 3) return fail(BCN_ERR_INVALID_ARGUMENT, "fill: unknown method");
    if (engine < 0 || engine > 7) return fail(BCN_ERR_INVALID_ARGUMENT, "fill: unknown engine");
    return BCN_OK;
}

bcn_status ensure_scratch(DevCtx* c, size_t bytes, bool pinned) {
    if (c->chunk_bytes < bytes) {
        for (int i = 0; i < 2; ++i) {
            if (c->scratch[i]) cudaFree(c->scratch[i]);
            if (c->pinned[i]) cudaFreeHost(c->pinned[i]);
            c->scratch[i] = c->pinned[i] = nullptr;
        }
        c->chunk_bytes = bytes;
    }
    for (int i = 0; i < 2; ++i) {
        if (!c->scratch[i]) BCN_CUDA(cudaMalloc(&c->scratch[i], c->chunk_bytes));
        if (pinned && !c->pinned[i]) BCN_CUDA(cudaMallocHost(&c->pinned[i], c->chunk_bytes));
    }
    return BCN_OK;
}

// Host copy pool: drains pinned staging buffers into pageable user memory
// with several threads (one thread reaches ~15 GB/s, well below the D2H rate;
// first-touch page faults of a fresh buffer are also spread across threads).
// Streaming (non-temporal) copy: the destination lines are written without
// being read first (no read-for-ownership), which cuts host DRAM traffic of a
// pinned -> pageable drain from ~4x to ~3x the payload. SSE2 is baseline x86-64.
void copy_stream(char* dst, const char* src, size_t bytes) {
#if defined(__x86_64__)
    size_t head = (16 - reinterpret_cast<uintptr_t>(dst) % 16) % 16;
    if (head > bytes) head = bytes;
    std::memcpy(dst, src, head);
    dst += head;
    src += head;
    bytes -= head;
    const size_t vec = bytes / 64 * 64;
    for (size_t i = 0; i < vec; i += 64) {
        const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
        const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 16));
        const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 32));
        const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 48));
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 16), b);
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 32), c);
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 48), d);
    }
    _mm_sfence();
    std::memcpy(dst + vec, src + vec, bytes - vec);
#else
    std::memcpy(dst, src, bytes);
#endif
}

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v ? static_cast<int>(std::strtol(v, nullptr, 10)) : dflt;
}

class CopyPool {
  public:
    CopyPool() {
        // One thread per core (up to 32) with streaming stores: 42 GB/s into a
        // pageable buffer on the 16-core B200 host against 29 GB/s for 8
        // threads of plain memcpy (profiles/r01/host_fill_copy.jsonl).
        // BCN_COPY_THREADS / BCN_COPY_NT=0 override (exploration knobs).
        unsigned hw = std::thread::hardware_concurrency();
        nthreads_ = hw == 0 ? 4 : std::min(32u, std::max(2u, hw));
        const int want = env_int("BCN_COPY_THREADS", 0);
        if (want > 0) nthreads_ = static_cast<unsigned>(std::min(64, want));
        streaming_ = env_int("BCN_COPY_NT", 1) != 0;
        for (unsigned t = 1; t < nthreads_; ++t) workers_.emplace_back([this, t] { loop(t); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> l(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& w : workers_) w.join();
    }
    // memcpy split into nthreads_ slices; returns when all slices are done.
    void copy(void* dst, const void* src, size_t bytes) {
        if (bytes < (4u << 20) || nthreads_ == 1) {
            std::memcpy(dst, src, bytes);
            return;
        }
        std::lock_guard<std::mutex> one_at_a_time(call_mu_);
        std::unique_lock<std::mutex> l(mu_);
        dst_ = static_cast<char*>(dst);
        src_ = static_cast<const char*>(src);
        bytes_ = bytes;
        pending_ = nthreads_ - 1;
        ++gen_;
        l.unlock();
        cv_.notify_all();
        slice(0);
        l.lock();
        done_cv_.wait(l, [this] { return pending_ == 0; });
    }

  private:
    void slice(unsigned t) {
        const size_t per = (bytes_ / nthreads_ + 63) & ~size_t{63};
        const size_t b = std::min(bytes_, per * t), e = std::min(bytes_, b + per);
        const size_t end = t + 1 == nthreads_ ? bytes_ : e;
        if (end > b) {
            if (streaming_)
                copy_stream(dst_ + b, src_ + b, end - b);
            else
                std::memcpy(dst_ + b, src_ + b, end - b);
        }
    }
    void loop(unsigned t) {
        uint64_t seen = 0;
        for (;;) {
            std::unique_lock<std::mutex> l(mu_);
            cv_.wait(l, [&] { return stop_ || gen_ != seen; });
            if (stop_) return;
            seen = gen_;
            l.unlock();
            slice(t);
            l.lock();
            if (--pending_ == 0) done_cv_.notify_one();
        }
    }
    unsigned nthreads_ = 1;
    bool streaming_ = false;
    std::vector<std::thread> workers_;
    std::mutex mu_, call_mu_;
    std::condition_variable cv_, done_cv_;
    bool stop_ = false;
    uint64_t gen_ = 0;
    unsigned pending_ = 0;
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    size_t bytes_ = 0;
};

CopyPool& copy_pool() {
    static CopyPool pool;
    return pool;
}

// Host output: generate chunks on the device, D2H on alternating streams.
bcn_status fill_host(FillJob& j, char* out, bool out_pinned) {
    DevCtx* c = j.ctx;
    std::lock_guard<std::mutex> lock(c->mu);
    // On an early (error) return no DMA into the caller's buffer or the
    // staging buffers may still be in flight: drain both copy streams.
    struct Drain {
        DevCtx* c;
        ~Drain() {
            cudaStreamSynchronize(c->copy[0]);
            cudaStreamSynchronize(c->copy[1]);
        }
    } drain{c};
    const int isz = format_itemsize(j.fmt);
    const uint64_t chunk_items = (64ull << 20) / isz;  // 64 MiB per chunk
    bcn_status st = ensure_scratch(c, chunk_items * isz, !out_pinned);
    if (st) return st;
    const uint64_t n = j.plan->n;
    const uint64_t nchunks = (n + chunk_items - 1) / chunk_items;
    for (uint64_t k = 0; k < nchunks; ++k) {
        const int b = static_cast<int>(k & 1);
        const uint64_t p0 = k * chunk_items, p1 = std::min(n, p0 + chunk_items);
        j.stream = c->copy[b];
        cudaError_t e = enqueue_range(j, static_cast<char*>(c->scratch[b]), p0, p1);
        if (e != cudaSuccess) return cuda_fail(e, "fill kernel launch");
        void* dst = out_pinned ? static_cast<void*>(out + p0 * isz) : c->pinned[b];
        BCN_CUDA(cudaMemcpyAsync(dst, c->scratch[b], (p1 - p0) * isz, cudaMemcpyDeviceToHost, c->copy[b]));
        if (!out_pinned) {
            // Drain the previous chunk from its staging buffer while this one copies.
            if (k >= 1) {
                const int pb = b ^ 1;
                const uint64_t q0 = (k - 1) * chunk_items, q1 = std::min(n, q0 + chunk_items);
                BCN_CUDA(cudaStreamSynchronize(c->copy[pb]));
                copy_pool().copy(out + q0 * isz, c->pinned[pb], (q1 - q0) * isz);
            }
        }
    }
    BCN_CUDA(cudaStreamSynchronize(c->copy[0]));
    BCN_CUDA(cudaStreamSynchronize(c->copy[1]));
    if (!out_pinned && nchunks >= 1) {
        const uint64_t k = nchunks - 1;
        const uint64_t q0 = k * chunk_items, q1 = n;
        copy_pool().copy(out + q0 * isz, c->pinned[k & 1], (q1 - q0) * isz);
    }
    return BCN_OK;
}

// Automatic pacing target of one device: the paced f64 fill (FP64 engine,
// the default 8-byte path) timed over a sweep of targets on a 2 GiB scratch
// buffer, 100 GB/s apart from just below its unpaced rate upwards. Below the
// write path's knee the kernel holds its target; above it the rate falls back
// towards the unpaced ~6.2 TB/s (profiles/r01/write_probe8.jsonl,
// r02/pace_modes.jsonl: 7.07 / 7.22 / 6.90 TB/s at 7200 / 7400 / 7600). The
// target is the sweep's best point; the sweep stops 3 points after the rate
// last rose. ~30 ms, once per device and process, at context initialisation.
// Stream-capture safe: the thread switches to relaxed capture mode and uses
// its own stream.
void calibrate_pace(DevCtx* c) {
    c->pace_cal = kDefaultPaceGBs;
    c->pace_src = BCN_PACE_DEFAULT;
    if (env_int("BCN_PACE_CALIBRATE", 1) == 0) return;
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    if (cudaThreadExchangeStreamCaptureMode(&mode) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    struct Scope {
        cudaStreamCaptureMode mode;
        void* buf = nullptr;
        cudaEvent_t ev[2] = {nullptr, nullptr};
        ~Scope() {
            if (buf) cudaFree(buf);
            for (cudaEvent_t e : ev)
                if (e) cudaEventDestroy(e);
            cudaThreadExchangeStreamCaptureMode(&mode);
            cudaGetLastError();
        }
    } sc{mode};
    constexpr uint64_t kItems = 1ull << 28;  // 2 GiB of doubles
    constexpr uint64_t kRow = 128;
    if (cudaMalloc(&sc.buf, kItems * 8) != cudaSuccess || cudaEventCreate(&sc.ev[0]) != cudaSuccess ||
        cudaEventCreate(&sc.ev[1]) != cudaSuccess)
        return;
    constexpr uint64_t kWorkers = kPacedThreads / 32 - 1;
    const int grid = c->sms * g_pace_cps.load();
    PacedArgs pa{};
    pa.out = sc.buf;
    pa.rows = kItems / kRow;
    pa.e0 = 0;
    pa.jump = mult_for_steps(static_cast<__int128>(kRow) * grid * kWorkers * paced_rows_per_round(kFmtF64));
    pa.mode = kPacedContiguous;
    bool ok = true;
    auto rate = [&](double gbs) -> double {  // GB/s over 3 launches after 1 warm-up
        pa.gap_q8 = gbs > 0.0 ? pace_gap_q8(grid, gbs, kFmtF64) : 0;
        ok = ok && launch_paced(kFmtF64, kEngFP64, pa, grid, c->stream) == cudaSuccess;
        ok = ok && cudaEventRecord(sc.ev[0], c->stream) == cudaSuccess;
        for (int i = 0; i < 3; ++i) ok = ok && launch_paced(kFmtF64, kEngFP64, pa, grid, c->stream) == cudaSuccess;
        ok = ok && cudaEventRecord(sc.ev[1], c->stream) == cudaSuccess;
        ok = ok && cudaEventSynchronize(sc.ev[1]) == cudaSuccess;
        float ms = 0.0f;
        ok = ok && cudaEventElapsedTime(&ms, sc.ev[0], sc.ev[1]) == cudaSuccess && ms > 0.0f;
        return ok ? 3.0 * kItems * 8 / ms / 1e6 : 0.0;
    };
    const double unpaced = rate(0.0);
    std::vector<std::pair<double, double>> curve;
    double best_t = 0.0, best_a = unpaced;
    int since_best = 0;
    for (double t = std::floor(unpaced / 100.0) * 100.0; ok && t <= 9000.0 && since_best < 3; t += 100.0) {
        const double a = rate(t);
        curve.emplace_back(t, a);
        if (a > best_a) {
            best_a = a;
            best_t = t;
            since_best = 0;
        } else {
            ++since_best;
        }
    }
    if (!ok || unpaced <= 0.0) return;
    c->pace_curve = curve;
    c->pace_cal = best_t;  // 0: pacing never beat the unpaced kernel
    c->pace_src = BCN_PACE_CALIBRATED;
}

double pace_gbs(DevCtx* c) {
    const double s = g_pace_gbs.load();
    if (s >= 0.0) return s;
    std::call_once(c->pace_once, [c] { calibrate_pace(c); });
    return c->pace_cal;
}

enum class PtrKind { Device, PinnedHost, PageableHost };

bcn_status classify(const void* p, int* device, PtrKind* kind) {
    cudaPointerAttributes attr;
    cudaError_t e = cudaPointerGetAttributes(&attr, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *kind = PtrKind::PageableHost;
        return BCN_OK;
    }
    switch (attr.type) {
        case cudaMemoryTypeDevice:
        case cudaMemoryTypeManaged:
            if (*device < 0) *device = attr.device;
            if (attr.device != *device)
                return fail(BCN_ERR_INVALID_ARGUMENT, "fill: device pointer belongs to another device");
            *kind = PtrKind::Device;
            return BCN_OK;
        case cudaMemoryTypeHost:
            *kind = PtrKind::PinnedHost;
            return BCN_OK;
        default:
            *kind = PtrKind::PageableHost;
            return BCN_OK;
    }
}

bcn_status do_fill(void* out, uint64_t capacity, uint64_t n, int fmt, uint32_t workers, int layout,
                   uint64_t seed_index, int method, uint64_t base_offset, int engine, int device,
                   void* stream) {
    DeviceGuard guard;
    Plan plan;
    bcn_status st = make_plan(n, workers, layout, &plan);
    if (st) return st;
    if ((st = validate_enums(fmt, layout, method, engine))) return st;
    if (capacity < plan.n) return fail(BCN_ERR_INVALID_ARGUMENT, "fill: buffer smaller than plan.n");
    if (!out) return fail(BCN_ERR_INVALID_ARGUMENT, "fill: null output buffer");
    if ((st = check_seed(seed_index))) return st;
    if (plan.n >= (1ull << 40)) return fail(BCN_ERR_INVALID_ARGUMENT, "fill: n must be below 2^40 per call");
    const int isz = format_itemsize(fmt);
    if (reinterpret_cast<uintptr_t>(out) % isz)
        return fail(BCN_ERR_INVALID_ARGUMENT, "fill: buffer not aligned to its item size");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        return fail(BCN_ERR_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
    }
    PtrKind kind;
    int dev = device;
    if ((st = classify(out, &dev, &kind))) return st;
    if (dev < 0) dev = 0;
    DevCtx* c = nullptr;
    if ((st = get_ctx(dev, &c))) return st;
    FillJob j;
    j.plan = &plan;
    j.fmt = fmt;
    j.engine = resolve_engine(engine, fmt);
    j.a = seed_index;
    j.base_offset = base_offset;
    j.a_exp = (seed_index - kModulus - 1) % kPeriod;
    j.ctx = c;
    if (kind != PtrKind::Device) return fill_host(j, static_cast<char*>(out), kind == PtrKind::PinnedHost);
    if ((st = caller_stream(c, stream, &j.stream))) return st;
    cudaError_t e = enqueue_range(j, static_cast<char*>(out), 0, plan.n);
    if (e != cudaSuccess) return cuda_fail(e, "fill kernel launch");
    if (!stream) BCN_CUDA(cudaStreamSynchronize(c->stream));
    return BCN_OK;
}

// Device view of a caller buffer for the read-only quality kernels: device
// pointers are used in place, host buffers are copied into a temporary.
struct DeviceInput {
    const void* ptr = nullptr;
    void* owned = nullptr;
    ~DeviceInput() {
        if (owned) cudaFree(owned);
    }
};

bcn_status stage_input(const void* buf, size_t bytes, int* device, DeviceInput* in, DevCtx** ctx,
                       cudaStream_t* s, void* stream) {
    PtrKind kind;
    bcn_status st = classify(buf, device, &kind);
    if (st) return st;
    if (*device < 0) *device = 0;
    if ((st = get_ctx(*device, ctx))) return st;
    if ((st = caller_stream(*ctx, stream, s))) return st;
    if (kind == PtrKind::Device) {
        in->ptr = buf;
        return BCN_OK;
    }
    BCN_CUDA(cudaMalloc(&in->owned, bytes));
    BCN_CUDA(cudaMemcpyAsync(in->owned, buf, bytes, cudaMemcpyHostToDevice, *s));
    in->ptr = in->owned;
    return BCN_OK;
}

}  // namespace

// ===================================================================== C ABI
extern "C" {

int bcn_abi_version(void) { return BCN_ABI_VERSION; }

const char* bcn_last_error(void) { return g_last_error.c_str(); }

const char* bcn_engine_name(int engine) {
    switch (engine) {
        case BCN_ENGINE_AUTO: return "auto";
        case BCN_ENGINE_BARRETT: return "barrett";
        case BCN_ENGINE_MONTGOMERY: return "montgomery";
        case BCN_ENGINE_FP64: return "fp64";
        case BCN_ENGINE_STAGED: return "staged";
        case BCN_ENGINE_BULK: return "bulk";
        case BCN_ENGINE_MIXED: return "mixed";
        case BCN_ENGINE_HYBRID: return "hybrid";
    }
    return "?";
}

uint64_t bcn_l2_bytes(int device) {
    int bytes = 0;
    if (cudaDeviceGetAttribute(&bytes, cudaDevAttrL2CacheSize, device < 0 ? 0 : device) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return static_cast<uint64_t>(bytes);
}

int bcn_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int bcn_auto_engine(bcn_format format) { return resolve_engine(kEngAuto, format); }

uint64_t bcn_launch_count(void) { return launch_count(); }

bcn_status bcn_set_write_pacing(double target_gbs, int ctas_per_sm, int format_mask) {
    if (std::isnan(target_gbs) || target_gbs > 1e5 || (target_gbs > 0.0 && target_gbs < kMinPaceGBs) ||
        ctas_per_sm < 1 || ctas_per_sm > 7 || format_mask < 0 || format_mask > 7)
        return fail(BCN_ERR_INVALID_ARGUMENT,
                    "set_write_pacing: target_gbs < 0 (automatic), 0 (unpaced) or in [100, 1e5]; "
                    "ctas_per_sm in [1,7], format_mask in [0,7]");
    g_pace_gbs.store(target_gbs < 0.0 ? -1.0 : target_gbs);
    g_pace_cps.store(ctas_per_sm);
    g_pace_formats.store(format_mask);
    return BCN_OK;
}

double bcn_write_pacing(void) { return g_pace_gbs.load(); }

void bcn_get_write_pacing(double* target_gbs, int* ctas_per_sm, int* format_mask) {
    if (target_gbs) *target_gbs = g_pace_gbs.load();
    if (ctas_per_sm) *ctas_per_sm = g_pace_cps.load();
    if (format_mask) *format_mask = g_pace_formats.load();
}

bcn_status bcn_device_write_pacing(int device, double* target_gbs, int* source) {
    if (!target_gbs || !source) return fail(BCN_ERR_INVALID_ARGUMENT, "device_write_pacing: null output");
    DeviceGuard guard;
    DevCtx* c = nullptr;
    bcn_status st = get_ctx(device < 0 ? 0 : device, &c);
    if (st) return st;
    const double setting = g_pace_gbs.load();
    *target_gbs = pace_gbs(c);
    *source = *target_gbs == 0.0 ? BCN_PACE_UNPACED : setting >= 0.0 ? BCN_PACE_USER : c->pace_src;
    return BCN_OK;
}

bcn_status bcn_pace_calibration(int device, double* targets, double* achieved, int capacity, int* count) {
    if (!count || capacity < 0 || (capacity > 0 && (!targets || !achieved)))
        return fail(BCN_ERR_INVALID_ARGUMENT, "pace_calibration: bad output arrays");
    DeviceGuard guard;
    DevCtx* c = nullptr;
    bcn_status st = get_ctx_nocal(device < 0 ? 0 : device, &c);
    if (st) return st;
    std::call_once(c->pace_once, [c] { calibrate_pace(c); });
    *count = static_cast<int>(c->pace_curve.size());
    for (int i = 0; i < capacity && i < *count; ++i) {
        targets[i] = c->pace_curve[static_cast<size_t>(i)].first;
        achieved[i] = c->pace_curve[static_cast<size_t>(i)].second;
    }
    return BCN_OK;
}

bcn_status bcn_set_launch_config(int ctas_per_sm, int row_order) {
    if (ctas_per_sm < 0 || ctas_per_sm > 32 || row_order < 0 || row_order > 1)
        return fail(BCN_ERR_INVALID_ARGUMENT, "set_launch_config: ctas_per_sm in [0,32], row_order 0|1");
    g_ctas_per_sm.store(ctas_per_sm);
    g_row_order.store(row_order);
    return BCN_OK;
}

bcn_status bcn_modpow2(uint64_t e, uint64_t modulus, uint64_t* out) {
    // generator.cpp:17-30
    if (!out) return fail(BCN_ERR_INVALID_ARGUMENT, "modpow2: null output");
    if (modulus % 2 == 0) return fail(BCN_ERR_INVALID_ARGUMENT, "modpow2: modulus must be odd");
    if (modulus >= (1ull << 63)) return fail(BCN_ERR_INVALID_ARGUMENT, "modpow2: modulus must be below 2^63");
    uint64_t r = 1 % modulus, b = 2 % modulus;
    while (e) {
        if (e & 1) r = static_cast<uint64_t>(static_cast<unsigned __int128>(r) * b % modulus);
        b = static_cast<uint64_t>(static_cast<unsigned __int128>(b) * b % modulus);
        e >>= 1;
    }
    *out = r;
    return BCN_OK;
}

bcn_status bcn_seed_from_index(uint64_t a, uint64_t* z0) {
    // generator.cpp:32-40
    if (!z0) return fail(BCN_ERR_INVALID_ARGUMENT, "seed_from_index: null output");
    bcn_status st = check_seed(a);
    if (st) return st;
    *z0 = host_mulmod(host_pow2(a - kModulus), kHalfM);
    return BCN_OK;
}

bcn_status bcn_state_at(uint64_t a, uint64_t k, uint64_t* z) {
    // generator.cpp:42-49
    if (!z) return fail(BCN_ERR_INVALID_ARGUMENT, "state_at: null output");
    bcn_status st = check_seed(a);
    if (st) return st;
    const uint64_t z0 = host_mulmod(host_pow2(a - kModulus), kHalfM);
    *z = host_mulmod(host_pow2(host_mul53_mod_p(k)), z0);
    return BCN_OK;
}

bcn_status bcn_next(uint64_t* z) {
    // generator.hpp:52-70 (all methods agree; modred.hpp:150 rejects z = 0)
    if (!z) return fail(BCN_ERR_INVALID_ARGUMENT, "next: null state");
    if (*z == 0) return fail(BCN_ERR_DOMAIN, "barrett_modified_step: z = 0 not in domain");
    if (*z >= kModulus) return fail(BCN_ERR_DOMAIN, "barrett_modified_step: residue out of range");
    *z = static_cast<uint64_t>((static_cast<unsigned __int128>(*z) << 53) % kModulus);
    return BCN_OK;
}

bcn_status bcn_to_unit_interval(uint64_t z, double* u) {
    // generator.hpp:74-78
    if (!u) return fail(BCN_ERR_INVALID_ARGUMENT, "to_unit_interval: null output");
    if (z == 0) return fail(BCN_ERR_DOMAIN, "to_unit_interval: z = 0 maps outside (0,1)");
    if (z >= kModulus) return fail(BCN_ERR_DOMAIN, "to_unit_interval: residue out of range");
    *u = static_cast<double>(z) * kInvModulus;
    return BCN_OK;
}

bcn_status bcn_make_plan(uint64_t n, uint32_t workers, uint32_t* eff_workers,
                         uint64_t* work_per_worker) {
    Plan p;
    bcn_status st = make_plan(n, workers, 0, &p);
    if (st) return st;
    if (eff_workers) *eff_workers = p.workers;
    if (work_per_worker) *work_per_worker = p.wpw;
    return BCN_OK;
}

bcn_status bcn_physical_index(uint64_t n, uint32_t workers, bcn_layout layout, uint32_t w,
                              uint64_t i, uint64_t* slot) {
    Plan p;
    bcn_status st = make_plan(n, workers, layout, &p);
    if (st) return st;
    if (!slot) return fail(BCN_ERR_INVALID_ARGUMENT, "physical_index: null output");
    if (w >= p.workers || i >= p.elements_for(w))
        return fail(BCN_ERR_INVALID_ARGUMENT, "physical_index: (w, i) outside the plan");
    if (layout == BCN_LAYOUT_CONTIGUOUS) {
        *slot = static_cast<uint64_t>(w) * p.wpw + i;
    } else {
        const uint64_t sc = p.short_count();
        *slot = i < sc ? i * p.workers + w : sc * p.workers + (i - sc) * (p.workers - 1) + w;
    }
    return BCN_OK;
}

bcn_status bcn_fill(void* out, uint64_t capacity, uint64_t n, bcn_format format, uint32_t workers,
                    bcn_layout layout, uint64_t seed_index, bcn_method method, uint64_t base_offset,
                    bcn_engine engine, int device, void* stream) {
    return do_fill(out, capacity, n, format, workers, layout, seed_index, method, base_offset,
                   engine, device, stream);
}

bcn_status bcn_bench_fill(uint64_t n, uint32_t workers, bcn_layout layout, uint64_t seed_index,
                          int engine, int repeats, int check_output, int device,
                          double* exec_seconds, double* total_seconds) {
    // bench.cpp:102-142 / :241-248, measured on the device.
    if (!exec_seconds || !total_seconds) return fail(BCN_ERR_INVALID_ARGUMENT, "bench_fill: null output");
    if (n == 0 || repeats < 1) return fail(BCN_ERR_INVALID_ARGUMENT, "bench_fill: n and repeats must be >= 1");
    if (engine < -1 || engine > 7) return fail(BCN_ERR_INVALID_ARGUMENT, "bench_fill: unknown engine");
    DeviceGuard guard;
    DevCtx* c = nullptr;
    bcn_status st = get_ctx(device < 0 ? 0 : device, &c);
    if (st) return st;
    struct Buffers {
        void* p[2] = {nullptr, nullptr};
        cudaEvent_t ev[2] = {nullptr, nullptr};
        ~Buffers() {
            for (void* q : p)
                if (q) cudaFree(q);
            for (cudaEvent_t e : ev)
                if (e) cudaEventDestroy(e);
        }
    } b;
    const size_t bytes = n * sizeof(double);
    BCN_CUDA(cudaMalloc(&b.p[0], bytes + 1024));
    BCN_CUDA(cudaEventCreate(&b.ev[0]));
    BCN_CUDA(cudaEventCreate(&b.ev[1]));
    const int dev = device < 0 ? 0 : device;
    cudaStream_t s = c->stream;
    std::vector<double> exec(static_cast<size_t>(repeats)), total(static_cast<size_t>(repeats));
    for (int r = 0; r < repeats; ++r) {
        BCN_CUDA(cudaStreamSynchronize(s));
        const auto t0 = std::chrono::steady_clock::now();
        BCN_CUDA(cudaEventRecord(b.ev[0], s));
        if (engine == -1) {
            const uint64_t rows_bytes = bytes / 1024 * 1024;
            if (rows_bytes) {
                st = bcn_fill_constant(b.p[0], rows_bytes, 0x3FE0000000000000ull, dev, s);
                if (st) return st;
            }
        } else {
            st = do_fill(b.p[0], n, n, BCN_FORMAT_F64, workers, layout, seed_index, BCN_METHOD_BARRETT_MODIFIED, 0,
                         engine, dev, s);
            if (st) return st;
        }
        BCN_CUDA(cudaEventRecord(b.ev[1], s));
        BCN_CUDA(cudaEventSynchronize(b.ev[1]));
        total[static_cast<size_t>(r)] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        float ms = 0.0f;
        BCN_CUDA(cudaEventElapsedTime(&ms, b.ev[0], b.ev[1]));
        exec[static_cast<size_t>(r)] = std::min(static_cast<double>(ms) * 1e-3, total[static_cast<size_t>(r)]);
    }
    auto median = [](std::vector<double>& v) {
        std::sort(v.begin(), v.end());
        return v.size() % 2 ? v[v.size() / 2] : 0.5 * (v[v.size() / 2 - 1] + v[v.size() / 2]);
    };
    *exec_seconds = median(exec);
    *total_seconds = median(total);
    if (check_output && engine != -1) {
        BCN_CUDA(cudaMalloc(&b.p[1], bytes));
        st = do_fill(b.p[1], n, n, BCN_FORMAT_F64, workers, layout, seed_index, BCN_METHOD_BARRETT_MODIFIED, 0,
                     BCN_ENGINE_AUTO, dev, s);
        if (st) return st;
        uint64_t d0[3], d1[3];
        if ((st = bcn_digest(b.p[0], n, 8, 0, d0, dev, s))) return st;
        if ((st = bcn_digest(b.p[1], n, 8, 0, d1, dev, s))) return st;
        if (d0[0] != d1[0] || d0[1] != d1[1] || d0[2] != d1[2])
            return fail(BCN_ERR_DOMAIN, "bench_fill: timed output differs from an untimed fill");
    }
    return BCN_OK;
}

bcn_status bcn_fill_multi(void* const* outs, const uint64_t* capacities, const int* devices, int ndev,
                          uint64_t n, bcn_format format, uint64_t seed_index, uint64_t base_offset,
                          bcn_engine engine, void* const* streams) {
    if (!outs || !capacities || !devices || ndev <= 0)
        return fail(BCN_ERR_INVALID_ARGUMENT, "fill_multi: no devices");
    Plan plan;
    bcn_status st = make_plan(n, static_cast<uint32_t>(ndev), 0, &plan);
    if (st) return st;
    if ((st = validate_enums(format, 0, 3, engine))) return st;
    if ((st = check_seed(seed_index))) return st;
    if (plan.wpw >= (1ull << 40))
        return fail(BCN_ERR_INVALID_ARGUMENT, "fill_multi: n must be below 2^40 per device");
    const int isz = format_itemsize(format);
    // Every shard is validated before any device work (like bcn_fill's
    // capacity check): a short or misplaced buffer is invalid_argument, never
    // an out-of-bounds write.
    for (uint32_t g = 0; g < plan.workers; ++g) {
        if (!outs[g]) return fail(BCN_ERR_INVALID_ARGUMENT, "fill_multi: null shard buffer");
        if (capacities[g] < plan.elements_for(g))
            return fail(BCN_ERR_INVALID_ARGUMENT, "fill_multi: shard " + std::to_string(g) +
                                                      " buffer smaller than its shard of make_plan(n, ndev)");
        if (reinterpret_cast<uintptr_t>(outs[g]) % isz)
            return fail(BCN_ERR_INVALID_ARGUMENT, "fill_multi: shard buffer not aligned to its item size");
    }
    for (uint32_t g = 0; g < plan.workers; ++g) {
        int dev = devices[g];
        PtrKind kind;
        if ((st = classify(outs[g], &dev, &kind))) return st;
        if (kind != PtrKind::Device)
            return fail(BCN_ERR_INVALID_ARGUMENT, "fill_multi: shard buffers must be device memory");
        for (uint32_t h = 0; h < g; ++h)
            if (devices[h] == devices[g] && streams && streams[h] != streams[g])
                return fail(BCN_ERR_INVALID_ARGUMENT, "fill_multi: shards on one device need one stream");
    }
    DeviceGuard guard;
    std::vector<bcn_status> res(plan.workers, BCN_OK);
    std::vector<std::string> msg(plan.workers);
    std::vector<std::thread> pool;
    for (uint32_t g = 0; g < plan.workers; ++g) {
        pool.emplace_back([&, g] {
            DevCtx* c = nullptr;
            bcn_status s = get_ctx(devices[g], &c);
            cudaStream_t cs = nullptr;
            // The caller's stream for this device, or (NULL) the internal
            // stream after the device drains, so the shard writes are ordered
            // after every earlier use of the buffer (bcn_fill's rule).
            if (!s) s = caller_stream(c, streams ? streams[g] : nullptr, &cs);
            if (!s) {
                FillJob j;
                j.plan = &plan;
                j.fmt = format;
                j.engine = resolve_engine(engine, format);
                j.a = seed_index;
                j.base_offset = base_offset;
                j.a_exp = (seed_index - kModulus - 1) % kPeriod;
                j.ctx = c;
                j.stream = cs;
                const uint64_t p0 = static_cast<uint64_t>(g) * plan.wpw;
                cudaError_t e = enqueue_range(j, static_cast<char*>(outs[g]), p0, p0 + plan.elements_for(g));
                if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
                if (e != cudaSuccess) s = cuda_fail(e, "fill_multi shard");
            }
            res[g] = s;
            msg[g] = g_last_error;
        });
    }
    for (auto& t : pool) t.join();
    for (uint32_t g = 0; g < plan.workers; ++g)
        if (res[g]) return fail(res[g], "device " + std::to_string(devices[g]) + ": " + msg[g]);
    return BCN_OK;
}

bcn_status bcn_deinterleave(const void* in, void* out, uint64_t n, uint32_t workers,
                            uint32_t itemsize, int device, void* stream) {
    DeviceGuard guard;
    Plan p;
    bcn_status st = make_plan(n, workers, 1, &p);
    if (st) return st;
    if (!in || !out) return fail(BCN_ERR_INVALID_ARGUMENT, "deinterleave: null buffer");
    if (itemsize != 4 && itemsize != 8) return fail(BCN_ERR_INVALID_ARGUMENT, "deinterleave: itemsize must be 4 or 8");
    PtrKind kin, kout;
    int dev = device;
    if ((st = classify(in, &dev, &kin))) return st;
    if ((st = classify(out, &dev, &kout))) return st;
    if ((kin == PtrKind::Device) != (kout == PtrKind::Device))
        return fail(BCN_ERR_INVALID_ARGUMENT, "deinterleave: mixed host/device buffers");
    if (dev < 0) dev = 0;
    DevCtx* c = nullptr;
    if ((st = get_ctx(dev, &c))) return st;
    cudaStream_t s;
    if ((st = caller_stream(c, stream, &s))) return st;
    const void* din = in;
    void* dout = out;
    const size_t bytes = n * itemsize;
    // Host buffers: staged through one device temporary, freed (after the
    // stream drains) on every exit path.
    struct Temp {
        void* p = nullptr;
        cudaStream_t s = nullptr;
        ~Temp() {
            if (p) {
                cudaStreamSynchronize(s);
                cudaFree(p);
            }
        }
    } tmp;
    tmp.s = s;
    if (kin != PtrKind::Device) {
        if (n >= (1ull << 40)) return fail(BCN_ERR_INVALID_ARGUMENT, "deinterleave: n must be below 2^40 per call");
        BCN_CUDA(cudaMalloc(&tmp.p, 2 * bytes));
        BCN_CUDA(cudaMemcpyAsync(tmp.p, in, bytes, cudaMemcpyHostToDevice, s));
        din = tmp.p;
        dout = static_cast<char*>(tmp.p) + bytes;
    }
    const uint64_t sc = p.short_count();
    TransposeArgs t;
    t.in = din;
    t.out = dout;
    t.wpw = p.wpw;
    t.itemsize = itemsize;
    t.order = 0;  // chosen per region by the launcher
    t.pitch = 0;
    t.in_items = n;
    t.out_mod = (reinterpret_cast<uintptr_t>(dout) / itemsize) % (128 / itemsize);
    // Region 1: rows [0, sc) of all workers; region 2: the remaining
    // wpw - sc elements of workers 0..W-2 (parallel.cpp:24-33). One
    // persistent-grid launch per region.
    for (int region = 0; region < 2; ++region) {
        const uint64_t rows = region == 0 ? sc : p.wpw - sc;
        const uint64_t width = region == 0 ? p.workers : p.workers - 1;
        if (rows == 0 || width == 0) continue;
        t.p0 = region == 0 ? 0 : sc * p.workers;
        t.rows = rows;
        t.width = width;
        t.i_base = region == 0 ? 0 : sc;
        cudaError_t e = launch_transpose(t, s);
        if (e != cudaSuccess) return cuda_fail(e, "deinterleave launch");
    }
    if (tmp.p) {
        BCN_CUDA(cudaMemcpyAsync(out, dout, bytes, cudaMemcpyDeviceToHost, s));
        BCN_CUDA(cudaStreamSynchronize(s));
    } else if (!stream) {
        BCN_CUDA(cudaStreamSynchronize(s));
    }
    return BCN_OK;
}

bcn_status bcn_seed_states(const uint64_t* a, const uint64_t* k, uint64_t* out, uint64_t count,
                           uint32_t steps, int device, void* stream) {
    DeviceGuard guard;
    if (!a || !k || !out) return fail(BCN_ERR_INVALID_ARGUMENT, "seed_states: null buffer");
    if (count == 0) return BCN_OK;
    int dev = device;
    PtrKind kind;
    bcn_status st = classify(out, &dev, &kind);
    if (st) return st;
    if (kind != PtrKind::Device) return fail(BCN_ERR_INVALID_ARGUMENT, "seed_states: buffers must be device memory");
    for (const void* in : {static_cast<const void*>(a), static_cast<const void*>(k)}) {
        if ((st = classify(in, &dev, &kind))) return st;
        if (kind != PtrKind::Device)
            return fail(BCN_ERR_INVALID_ARGUMENT, "seed_states: buffers must be device memory");
    }
    DevCtx* c = nullptr;
    if ((st = get_ctx(dev, &c))) return st;
    std::lock_guard<std::mutex> scratch_lock(c->small_mu);
    cudaStream_t s;
    if ((st = caller_stream(c, stream, &s))) return st;
    BCN_CUDA(cudaMemsetAsync(c->flag, 0, sizeof(int), s));
    SeedArgs sa{a, k, out, count, steps, c->flag};
    cudaError_t e = launch_seed(sa, s);
    if (e != cudaSuccess) return cuda_fail(e, "seed_states launch");
    int flag = 0;
    BCN_CUDA(cudaMemcpyAsync(&flag, c->flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    BCN_CUDA(cudaStreamSynchronize(s));
    if (flag) return fail(BCN_ERR_OUT_OF_RANGE, "seed_from_index: index outside [3^33+100, 2^53]");
    return BCN_OK;
}

bcn_status bcn_digest(const void* buf, uint64_t n, uint32_t itemsize, uint64_t index_base,
                      uint64_t d[3], int device, void* stream) {
    DeviceGuard guard;
    if (!buf || !d) return fail(BCN_ERR_INVALID_ARGUMENT, "digest: null buffer");
    if (itemsize != 4 && itemsize != 8) return fail(BCN_ERR_INVALID_ARGUMENT, "digest: itemsize must be 4 or 8");
    int dev = device;
    PtrKind kind;
    bcn_status st = classify(buf, &dev, &kind);
    if (st) return st;
    if (kind != PtrKind::Device) return fail(BCN_ERR_INVALID_ARGUMENT, "digest: buffer must be device memory");
    DevCtx* c = nullptr;
    if ((st = get_ctx(dev, &c))) return st;
    std::lock_guard<std::mutex> scratch_lock(c->small_mu);
    cudaStream_t s;
    if ((st = caller_stream(c, stream, &s))) return st;
    BCN_CUDA(cudaMemsetAsync(c->digest, 0, 3 * sizeof(unsigned long long), s));
    DigestArgs da{buf, n, itemsize, index_base, c->digest};
    if (n) {
        const int grid = static_cast<int>(std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(c->sms) * 8));
        cudaError_t e = launch_digest(da, grid, s);
        if (e != cudaSuccess) return cuda_fail(e, "digest launch");
    }
    unsigned long long h[3];
    BCN_CUDA(cudaMemcpyAsync(h, c->digest, sizeof(h), cudaMemcpyDeviceToHost, s));
    BCN_CUDA(cudaStreamSynchronize(s));
    for (int i = 0; i < 3; ++i) d[i] = h[i];
    return BCN_OK;
}

bcn_status bcn_engine_check(bcn_engine engine, const uint64_t* z, const uint64_t* c, uint64_t* out,
                            uint64_t count, uint32_t chain, int device) {
    DeviceGuard guard;
    if (engine != BCN_ENGINE_BARRETT && engine != BCN_ENGINE_MONTGOMERY && engine != BCN_ENGINE_FP64 &&
        engine != BCN_ENGINE_MIXED)
        return fail(BCN_ERR_INVALID_ARGUMENT, "engine_check: not a jump engine");
    if (!z || !c || !out) return fail(BCN_ERR_INVALID_ARGUMENT, "engine_check: null buffer");
    if (count > (1ull << 26)) return fail(BCN_ERR_INVALID_ARGUMENT, "engine_check: count above 2^26");
    std::vector<Mult> mults(count);
    for (uint64_t i = 0; i < count; ++i) {
        if (z[i] >= kModulus || c[i] >= kModulus)
            return fail(BCN_ERR_DOMAIN, "engine_check: residue or multiplier out of range");
        mults[i] = host_make_mult(c[i]);
    }
    if (count == 0) return BCN_OK;
    DevCtx* ctx = nullptr;
    bcn_status st = get_ctx(device < 0 ? 0 : device, &ctx);
    if (st) return st;
    struct Buffers {
        void* p = nullptr;
        ~Buffers() {
            if (p) cudaFree(p);
        }
    } b;
    const size_t zb = count * 8, mb = count * sizeof(Mult);
    BCN_CUDA(cudaMalloc(&b.p, 2 * zb + mb));
    auto* dz = static_cast<uint64_t*>(b.p);
    auto* dout = dz + count;
    auto* dm = reinterpret_cast<Mult*>(dout + count);  // 16-byte aligned: 2 * count * 8 bytes in
    const cudaStream_t s = ctx->stream;
    BCN_CUDA(cudaMemcpyAsync(dz, z, zb, cudaMemcpyHostToDevice, s));
    BCN_CUDA(cudaMemcpyAsync(dm, mults.data(), mb, cudaMemcpyHostToDevice, s));
    cudaError_t e = launch_engine_check(engine, dz, dm, dout, count, chain, s);
    if (e != cudaSuccess) return cuda_fail(e, "engine_check launch");
    BCN_CUDA(cudaMemcpyAsync(out, dout, zb, cudaMemcpyDeviceToHost, s));
    BCN_CUDA(cudaStreamSynchronize(s));
    return BCN_OK;
}

namespace {
// The Constant writer and its noise variant (bcn_fill_constant / bcn_fill_noise).
bcn_status constant_writer(const char* what, void* out, uint64_t nbytes, uint64_t pattern,
                           uint64_t noise_seed, int device, void* stream) {
    DeviceGuard guard;
    if (!out) return fail(BCN_ERR_INVALID_ARGUMENT, std::string(what) + ": null buffer");
    if (reinterpret_cast<uintptr_t>(out) % 32 || nbytes % 1024)
        return fail(BCN_ERR_INVALID_ARGUMENT, std::string(what) + ": needs 32-byte alignment and whole 1 KiB rows");
    int dev = device;
    PtrKind kind;
    bcn_status st = classify(out, &dev, &kind);
    if (st) return st;
    if (kind != PtrKind::Device) return fail(BCN_ERR_INVALID_ARGUMENT, std::string(what) + ": buffer must be device memory");
    DevCtx* c = nullptr;
    if ((st = get_ctx(dev, &c))) return st;
    cudaStream_t s;
    if ((st = caller_stream(c, stream, &s))) return st;
    cudaError_t e;
    const double pace = pace_gbs(c);
    if (pace > 0.0 || noise_seed) {
        // The Constant writer under the same metering as the paced fill.
        constexpr uint64_t kWorkers = kPacedThreads / 32 - 1;
        const uint64_t rows = nbytes / 1024;
        const uint64_t want = static_cast<uint64_t>(c->sms) * g_pace_cps.load();
        const int grid = static_cast<int>(std::max<uint64_t>(1, std::min(want, (rows + kWorkers - 1) / kWorkers)));
        PacedArgs pa{};
        pa.out = out;
        pa.rows = rows;
        pa.e0 = pattern;
        pa.gap_q8 = pace > 0.0 ? pace_gap_q8(grid, pace, kFmtU64, true) : 0;
        pa.mode = kPacedConstant;
        pa.q0 = noise_seed;  // != 0: per-thread pseudo-random words instead of `pattern`
        e = launch_paced(kFmtU64, -1, pa, grid, s);
    } else {
        ConstArgs ca{out, nbytes / 1024, pattern, static_cast<uint32_t>(g_row_order.load())};
        const int grid = grid_for_rows(c, kFmtF64, kEngBarrett, false, ca.rows);
        e = launch_constant(ca, grid, kContigThreads, s);
    }
    if (e != cudaSuccess) return cuda_fail(e, what);
    if (!stream) BCN_CUDA(cudaStreamSynchronize(s));
    return BCN_OK;
}
}  // namespace

bcn_status bcn_fill_constant(void* out, uint64_t nbytes, uint64_t pattern, int device, void* stream) {
    return constant_writer("fill_constant", out, nbytes, pattern, 0, device, stream);
}

bcn_status bcn_fill_noise(void* out, uint64_t nbytes, uint64_t seed, int device, void* stream) {
    if (seed == 0) return fail(BCN_ERR_INVALID_ARGUMENT, "fill_noise: seed must be non-zero");
    return constant_writer("fill_noise", out, nbytes, 0, seed, device, stream);
}

}  // extern "C"

// ------------------------------------------------------------ quality suite
namespace {
constexpr uint64_t kMaxQualityItems = 1ull << 40;  // keeps n * 8 far from overflow
}

extern "C" {

bcn_status bcn_chi_square_uniformity(const double* samples, uint64_t n, int bins, double* statistic,
                                     int* dof, int* pass, int device, void* stream) {
    DeviceGuard guard;
    // quality.cpp:21-54 (same preconditions, same formula on exact counts)
    if (!statistic || !dof || !pass) return fail(BCN_ERR_INVALID_ARGUMENT, "chi_square: null output");
    if (n == 0) return fail(BCN_ERR_INVALID_ARGUMENT, "chi_square: no samples");
    if (bins < 2) return fail(BCN_ERR_INVALID_ARGUMENT, "chi_square: need at least 2 bins");
    const double expected = static_cast<double>(n) / bins;
    if (expected < 20.0) return fail(BCN_ERR_INVALID_ARGUMENT, "chi_square: expected count per bin below 20");
    if (!samples) return fail(BCN_ERR_INVALID_ARGUMENT, "chi_square: null samples");
    if (n >= kMaxQualityItems) return fail(BCN_ERR_INVALID_ARGUMENT, "chi_square: n must be below 2^40");
    DeviceInput in;
    DevCtx* c = nullptr;
    cudaStream_t s;
    int dev = device;
    bcn_status st = stage_input(samples, n * sizeof(double), &dev, &in, &c, &s, stream);
    if (st) return st;
    std::lock_guard<std::mutex> scratch_lock(c->small_mu);
    void* scratch = nullptr;
    if ((st = quality_scratch(c, static_cast<size_t>(bins) * 8, &scratch))) return st;
    auto* counts = static_cast<unsigned long long*>(scratch);
    BCN_CUDA(cudaMemsetAsync(counts, 0, static_cast<size_t>(bins) * 8, s));
    BCN_CUDA(cudaMemsetAsync(c->flag, 0, sizeof(int), s));
    const int grid = static_cast<int>(std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(c->sms) * 4));
    cudaError_t e = launch_chi_hist(static_cast<const double*>(in.ptr), n, bins, counts, c->flag, grid, s);
    if (e != cudaSuccess) return cuda_fail(e, "chi_square launch");
    std::vector<unsigned long long> h(static_cast<size_t>(bins));
    int flag = 0;
    BCN_CUDA(cudaMemcpyAsync(h.data(), counts, h.size() * 8, cudaMemcpyDeviceToHost, s));
    BCN_CUDA(cudaMemcpyAsync(&flag, c->flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    BCN_CUDA(cudaStreamSynchronize(s));
    if (flag) return fail(BCN_ERR_INVALID_ARGUMENT, "chi_square: sample outside (0,1)");
    double stat = 0.0;
    for (unsigned long long cnt : h) {
        const double d = static_cast<double>(cnt) - expected;
        stat += d * d / expected;
    }
    *dof = bins - 1;
    *statistic = stat;
    *pass = std::fabs(stat - *dof) <= 4.5 * std::sqrt(2.0 * *dof) ? 1 : 0;
    return BCN_OK;
}

bcn_status bcn_monobit_mantissa(const uint64_t* residues, uint64_t n, double* statistic, int* worst_bit,
                                int* pass, int device, void* stream) {
    DeviceGuard guard;
    // quality.cpp:56-90
    if (!statistic || !worst_bit || !pass) return fail(BCN_ERR_INVALID_ARGUMENT, "monobit: null output");
    if (n < 100000) return fail(BCN_ERR_INVALID_ARGUMENT, "monobit: need at least 1e5 residues");
    if (!residues) return fail(BCN_ERR_INVALID_ARGUMENT, "monobit: null residues");
    if (n >= kMaxQualityItems) return fail(BCN_ERR_INVALID_ARGUMENT, "monobit: n must be below 2^40");
    DeviceInput in;
    DevCtx* c = nullptr;
    cudaStream_t s;
    int dev = device;
    bcn_status st = stage_input(residues, n * 8, &dev, &in, &c, &s, stream);
    if (st) return st;
    std::lock_guard<std::mutex> scratch_lock(c->small_mu);
    void* scratch = nullptr;
    if ((st = quality_scratch(c, 53 * 8, &scratch))) return st;
    auto* ones = static_cast<unsigned long long*>(scratch);
    BCN_CUDA(cudaMemsetAsync(ones, 0, 53 * 8, s));
    BCN_CUDA(cudaMemsetAsync(c->flag, 0, sizeof(int), s));
    const int grid = static_cast<int>(std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(c->sms) * 4));
    cudaError_t e = launch_monobit(static_cast<const uint64_t*>(in.ptr), n, ones, c->flag, grid, s);
    if (e != cudaSuccess) return cuda_fail(e, "monobit launch");
    unsigned long long h[53];
    int flag = 0;
    BCN_CUDA(cudaMemcpyAsync(h, ones, sizeof(h), cudaMemcpyDeviceToHost, s));
    BCN_CUDA(cudaMemcpyAsync(&flag, c->flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    BCN_CUDA(cudaStreamSynchronize(s));
    if (flag) return fail(BCN_ERR_INVALID_ARGUMENT, "monobit: residue out of range");
    const double nn = static_cast<double>(n);
    double worst = 0.0;
    int wb = 5;
    for (int bit = 5; bit < 53; ++bit) {
        const double dev_ = std::fabs(static_cast<double>(h[bit]) / nn - 0.5);
        if (dev_ > worst) {
            worst = dev_;
            wb = bit;
        }
    }
    *statistic = worst;
    *worst_bit = wb;
    *pass = worst <= 4.5 / (2.0 * std::sqrt(nn)) ? 1 : 0;
    return BCN_OK;
}

bcn_status bcn_serial_correlation(const double* samples, uint64_t n, int lag, double* rho, int* pass,
                                  int device, void* stream) {
    DeviceGuard guard;
    // quality.cpp:92-118; per-block partial sums, fixed-order host reduction.
    if (!rho || !pass) return fail(BCN_ERR_INVALID_ARGUMENT, "serial_correlation: null output");
    if (lag < 1) return fail(BCN_ERR_INVALID_ARGUMENT, "serial_correlation: lag must be positive");
    if (n < 100000) return fail(BCN_ERR_INVALID_ARGUMENT, "serial_correlation: need at least 1e5 samples");
    if (!samples) return fail(BCN_ERR_INVALID_ARGUMENT, "serial_correlation: null samples");
    if (n >= kMaxQualityItems) return fail(BCN_ERR_INVALID_ARGUMENT, "serial_correlation: n must be below 2^40");
    // The reference reads past the span when lag >= n (quality.cpp:94); rejected here.
    if (static_cast<uint64_t>(lag) >= n)
        return fail(BCN_ERR_INVALID_ARGUMENT, "serial_correlation: lag must be below the sample count");
    DeviceInput in;
    DevCtx* c = nullptr;
    cudaStream_t s;
    int dev = device;
    bcn_status st = stage_input(samples, n * sizeof(double), &dev, &in, &c, &s, stream);
    if (st) return st;
    const uint64_t pairs = n - static_cast<uint64_t>(lag);
    constexpr int kGrid = 592;  // fixed: the reduction order does not depend on the device
    std::lock_guard<std::mutex> scratch_lock(c->small_mu);
    void* scratch = nullptr;
    if ((st = quality_scratch(c, kGrid * 5 * sizeof(double), &scratch))) return st;
    auto* part = static_cast<double*>(scratch);
    cudaError_t e = launch_lag_sums(static_cast<const double*>(in.ptr), pairs, static_cast<uint64_t>(lag), part,
                                    kGrid, s);
    if (e != cudaSuccess) return cuda_fail(e, "serial_correlation launch");
    std::vector<double> h(kGrid * 5);
    BCN_CUDA(cudaMemcpyAsync(h.data(), part, h.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    BCN_CUDA(cudaStreamSynchronize(s));
    double sum[5] = {0, 0, 0, 0, 0};
    for (int b = 0; b < kGrid; ++b)
        for (int k = 0; k < 5; ++k) sum[k] += h[b * 5 + k];
    const double np = static_cast<double>(pairs);
    const double vx = sum[2] / np - (sum[0] / np) * (sum[0] / np);
    const double vy = sum[3] / np - (sum[1] / np) * (sum[1] / np);
    const double cov = sum[4] / np - (sum[0] / np) * (sum[1] / np);
    const double r = (vx > 0.0 && vy > 0.0) ? cov / std::sqrt(vx * vy) : std::nan("");
    *rho = r;
    *pass = std::isfinite(r) && std::fabs(r) <= 4.5 / std::sqrt(static_cast<double>(n)) ? 1 : 0;
    return BCN_OK;
}

}  // extern "C"

// ------------------------------------------------------------ text format
extern "C" bcn_status bcn_format_text(const double* values, uint64_t n, char* out, uint64_t capacity,
                                      uint64_t* written) {
    // cli.cpp:127-131: one "%.17g\n" line per value. Formatted in parallel
    // slices into per-slice buffers, then concatenated in order.
    if ((!values && n) || !written || (!out && capacity)) return fail(BCN_ERR_INVALID_ARGUMENT, "format_text: null buffer");
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const uint64_t slices = std::min<uint64_t>(std::max<uint64_t>(1, n / 65536), hw);
    std::vector<std::string> parts(slices);
    std::vector<std::thread> pool;
    auto body = [&](uint64_t k) {
        const uint64_t b = n * k / slices, e = n * (k + 1) / slices;
        std::string& o = parts[k];
        o.reserve((e - b) * 24);
        char line[64];
        for (uint64_t i = b; i < e; ++i) {
            const int len = std::snprintf(line, sizeof(line), "%.17g\n", values[i]);
            o.append(line, static_cast<size_t>(len));
        }
    };
    for (uint64_t k = 1; k < slices; ++k) pool.emplace_back(body, k);
    body(0);
    for (auto& t : pool) t.join();
    uint64_t total = 0;
    for (const auto& p : parts) total += p.size();
    *written = total;
    if (total > capacity) return fail(BCN_ERR_INVALID_ARGUMENT, "format_text: output buffer too small");
    for (const auto& p : parts) {
        std::memcpy(out, p.data(), p.size());
        out += p.size();
    }
    return BCN_OK;
}
