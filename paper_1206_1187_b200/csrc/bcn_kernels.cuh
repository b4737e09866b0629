// bcn_kernels.cuh — launch-argument structs and launchers shared by the
// kernels (bcn_kernels.cu) and the C-ABI host layer (bcn_capi.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "bcn_math.cuh"

namespace bcn_b200 {

enum Format : int { kFmtU64 = 0, kFmtF64 = 1, kFmtF32 = 2 };
enum Engine : int {
    kEngAuto = 0,
    kEngBarrett = 1,
    kEngMontgomery = 2,
    kEngFP64 = 3,
    kEngStaged = 4,  // paper T=1 modified-Barrett runs, smem transpose, TMA bulk store
    kEngBulk = 5,    // FP64 jump streams, smem-staged 16 KiB tiles, TMA bulk store
    kEngMixed = 6,   // DFMA quotient + integer remainder (fewest FP64 ops)
    kEngHybrid = 7   // FP64 and Barrett streams side by side in every lane
};
// Internal ids of the hybrid engine's instantiations: kEngHybridBase + number
// of FP64 streams per lane vector (bcn_capi.cu: resolve_engine).
constexpr int kEngHybridBase = 16;

inline int format_itemsize(int fmt) { return fmt == kFmtF32 ? 4 : 8; }

// A partial row at either end of a contiguous range, written inside the main
// kernel (by warps 0 / 1 of CTA 0) instead of by extra launches: the row
// starts at the 32-byte aligned `base`, its element t has 2-exponent
// (e0 + 53 t) mod P, and only elements t in [lo, hi) are stored.
struct EdgeRow {
    void* base;  // nullptr: no edge row
    uint64_t e0;
    uint32_t lo, hi;
};

// Contiguous fast path: `rows` full rows of 32 lanes x 32 bytes starting at the
// 32-byte aligned `out`; element j of `out` has 2-exponent (e0 + 53 j) mod P.
struct ContigArgs {
    void* out;
    uint64_t rows;
    uint64_t e0;
    Mult jump_row;          // 2^(53 * elements per stream step) mod m
    uint32_t stride_order;  // 0: per-warp row ranges; 1: grid-strided rows
    EdgeRow edge[2];        // partial head / tail rows (or none)
};

// Paced contiguous fill (k_fill_paced): grid-strided rows metered to a
// target HBM write rate by one pacer warp per CTA.
// kPacedInterleavedFixed: an interleaved region whose per-round slot advance
// is a multiple of the width, so every stream stays in its worker column and
// steps by ONE multiplier (the contiguous kernel's stepping, interleaved seeding).
enum PacedMode : int { kPacedContiguous = 0, kPacedConstant = 1, kPacedInterleaved = 2, kPacedInterleavedFixed = 3 };
struct PacedArgs {
    void* out;        // 32-byte aligned
    uint64_t rows;    // rows of 32 lanes x 32 bytes
    uint64_t e0;      // exponent of element 0 (or the 8-byte pattern, Constant)
    Mult jump;        // per round: contiguous 2^(53 * H * nwk * ROW); interleaved: same-row advance
    uint64_t gap_q8;  // ns between CTA rounds, x256 (0 = unpaced)
    int mode;         // PacedMode (interleaved uses the fields below, as InterleavedArgs)
    uint64_t q0, width, i_base, wpw, adv_b;
    Mult jump_wrap;
    uint64_t row_stride;  // slots between a worker's consecutive rows (0: grid * 8 rows)
    EdgeRow edge[2];  // contiguous mode: partial head / tail rows (or none)
};

// Interleaved region fast path (reference Layout::Interleaved,
// parallel.cpp:24-33): physical slots q in [0, rows*ROW) of a region whose
// slot q0 + q sits at worker w = (q0 + q) % width, element
// i = i_base + (q0 + q) / width; logical index j = w * wpw + i.
struct InterleavedArgs {
    void* out;       // 32-byte aligned, physical slot q0 of the region
    uint64_t rows;
    uint64_t q0;     // region-relative slot of out[0]
    uint64_t width;  // workers per physical row in this region (W or W-1)
    uint64_t i_base;
    uint64_t wpw;
    uint64_t e0;     // exponent of logical element 0
    uint64_t adv_b;  // ROW mod width
    Mult jump_same;  // advance when w + adv_b < width
    Mult jump_wrap;  // advance when the lane crosses a physical row
};

// Generic per-slot path with the reference's exact semantics, including the
// u64 wrap of base_offset + start_w (parallel.cpp:63-64). One seed per slot.
struct SlotArgs {
    void* out;          // physical slot `slot0`
    uint64_t slot0;
    uint64_t count;
    uint64_t n;         // plan.n
    uint64_t wpw;       // plan.work_per_worker
    uint32_t workers;   // plan.workers (effective)
    int layout;         // 0 contiguous, 1 interleaved
    uint64_t a_exp;     // (a - 3^33 - 1) mod P
    uint64_t base_offset;
};

// Paper-style staged path: each thread runs L consecutive T=1 steps
// (modified Barrett), the CTA tile is assembled in shared memory in logical
// order and written with one TMA bulk store per tile.
struct StagedArgs {
    void* out;       // 16-byte aligned
    uint64_t tiles;  // full tiles
    uint64_t e0;
    Mult jump_next;  // 2^(53 (gridDim.x * TILE - L)) mod m
};

struct SeedArgs {
    const uint64_t* a;  // seed indices
    const uint64_t* k;  // skip-ahead offsets
    uint64_t* out;      // count * (steps ? steps : 1)
    uint64_t count;
    uint32_t steps;     // 0: state_at only; >0: emit next() `steps` times
    int* error;         // set to 1 when any a is out of range
};

struct DigestArgs {
    const void* buf;
    uint64_t n;
    uint32_t itemsize;
    uint64_t index_base;
    unsigned long long* out;  // [3] device accumulators
};

struct ConstArgs {
    void* out;
    uint64_t rows;  // rows of 32 lanes x 32 bytes
    uint64_t value; // bit pattern replicated (8 bytes)
    uint32_t stride_order;
};

struct TransposeArgs {
    const void* in;   // physical buffer
    void* out;        // logical buffer
    uint64_t p0;      // first physical slot of the region
    uint64_t rows;    // region rows (elements per worker in the region)
    uint64_t width;   // workers per row in the region
    uint64_t wpw;
    uint64_t i_base;  // element offset of the region inside each worker
    uint32_t itemsize;
    uint32_t order;   // wide tiles: 0 = worker blocks vary fastest, 1 = row blocks
    uint32_t pitch;   // narrow tiles: smem row pitch in items (0 = rows | 1)
    uint64_t in_items;  // items of the input buffer from `in` (bulk-copy bounds)
    uint64_t out_mod;   // (address of `out` / itemsize) mod (128 / itemsize): line phase of the output
};

// Launchers (bcn_kernels.cu). Each returns the launch error, if any.
cudaError_t launch_contig(int fmt, int engine, const ContigArgs& a, int grid, int block,
                          cudaStream_t s);
cudaError_t launch_interleaved(int fmt, int engine, const InterleavedArgs& a, int grid, int block,
                               cudaStream_t s);
// engine -1 = paced Constant writer (pattern in a.e0)
cudaError_t launch_paced(int fmt, int engine, const PacedArgs& a, int grid, cudaStream_t s);
cudaError_t launch_slots(int fmt, const SlotArgs& a, cudaStream_t s);
cudaError_t launch_staged(int fmt, const StagedArgs& a, int grid, cudaStream_t s);
cudaError_t launch_bulk(int fmt, const ContigArgs& a, int grid, cudaStream_t s);
cudaError_t launch_seed(const SeedArgs& a, cudaStream_t s);
cudaError_t launch_digest(const DigestArgs& a, int grid, cudaStream_t s);
cudaError_t launch_engine_check(int engine, const uint64_t* z, const Mult* mult, uint64_t* out, uint64_t n,
                                uint32_t chain, cudaStream_t s);
cudaError_t launch_constant(const ConstArgs& a, int grid, int block, cudaStream_t s);
cudaError_t launch_transpose(const TransposeArgs& a, cudaStream_t s);
// Register-pipelined transposes only (no TMA tile mover).
cudaError_t launch_transpose_registers(const TransposeArgs& a, cudaStream_t s);
// TMA tile mover for a wide region (bcn_deint_tma.cu); *used = false when the
// region cannot be described by its tensor maps (nothing launched).
cudaError_t launch_transpose_tma(const TransposeArgs& a, int sms, cudaStream_t s, bool* used);

// Quality smoke suite (bcn_quality.cu).
constexpr int kChiSmemBins = 16384;
cudaError_t launch_chi_hist(const double* u, uint64_t n, int bins, unsigned long long* counts, int* error,
                            int grid, cudaStream_t s);
cudaError_t launch_monobit(const uint64_t* z, uint64_t n, unsigned long long* ones, int* error, int grid,
                           cudaStream_t s);
cudaError_t launch_lag_sums(const double* x, uint64_t pairs, uint64_t lag, double* out, int grid,
                            cudaStream_t s);

// Kernels launched through this library so far (process-wide).
uint64_t launch_count();

// Uploads the windowed power table to the current device (idempotent per device).
cudaError_t upload_tables();

// Resident CTAs per SM for the contiguous kernel of (fmt, engine) at `block`.
int contig_blocks_per_sm(int fmt, int engine, int block);
int interleaved_blocks_per_sm(int fmt, int engine, int block);
int bulk_blocks_per_sm(int fmt);

constexpr int kStagedL = 15;          // odd: conflict-free strided smem stores
constexpr int kStagedThreads = 256;
constexpr int kContigThreads = 256;
constexpr int kPacedThreads = 288;  // 8 worker warps + 1 pacer warp
// Rows each paced worker stores per pacer round: 2 for the generating kernels
// of the 8-byte formats (8 independent streams per lane), 1 for f32 (already 8
// streams per lane) and for the Constant writer (no compute spreads its
// stores, and a 2-row burst per round measurably lowers HBM efficiency).
__host__ __device__ constexpr int paced_rows_per_round(int fmt, bool constant = false) {
    return (constant || fmt == kFmtF32) ? 1 : 2;
}
// Measured default pacing target for the 8-byte formats (DESIGN.md §5,
// profiles/r01/tune_pace.jsonl): FP64 engine f64/u64 reach ~7.08 TB/s at
// 7200 vs ~6.25 unpaced; above ~7.3 the write path starts to oversubscribe.
constexpr double kDefaultPaceGBs = 7200.0;
// CTAs per SM of the paced grid: 1 and 2 reach the same single-launch rate;
// under the board power cap 1 is ~1.3% faster sustained (profiles/r01/
// timeline_cps_pace.jsonl).
constexpr int kDefaultPaceCps = 1;
constexpr int kBulkTileRows = 16;  // 16 KiB per TMA bulk store
constexpr int kBulkStages = 3;     // tiles in flight per CTA

}  // namespace bcn_b200
