/*
 * bcnrand_b200.h — C ABI of the B200-native alpha_{2,3} generator.
 *
 * The reference (/root/reference/proj) is a C++20 header API with no FFI
 * layer. Each entry point below is the C-ABI replacement of one
 * reference function; the C++ drop-in headers in include/bcnrand/ re-export
 * the reference signatures on top of it.
 *
 * Conventions
 *  - Plain pointers and sizes only; no C++ or torch types cross this boundary.
 *  - Every call returns a bcn_status. Status codes map 1:1 onto the reference
 *    exception types (std::invalid_argument / out_of_range / domain_error);
 *    bcn_last_error() returns the message of the calling thread's last error.
 *  - Validation (seed range, n, workers, buffer size, alignment) happens
 *    BEFORE any device work, so an invalid seed never reaches a kernel (the
 *    reference aborts with std::terminate for W > 1).
 *  - `out` may be a device pointer (written in place on `stream`, or on an
 *    internal stream followed by a synchronize when stream == NULL) or a host
 *    pointer (pinned or pageable; generated on `device` and copied back in
 *    chunks; always synchronous).
 *  - There is no CPU fallback: with no usable CUDA device every generating
 *    call fails with BCN_ERR_CUDA.
 */
#ifndef BCNRAND_B200_H
#define BCNRAND_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BCN_ABI_VERSION 2

typedef enum bcn_status {
    BCN_OK = 0,
    BCN_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    BCN_ERR_OUT_OF_RANGE = 2,     /* std::out_of_range     */
    BCN_ERR_DOMAIN = 3,           /* std::domain_error     */
    BCN_ERR_CUDA = 4              /* device / driver failure (no reference analogue) */
} bcn_status;

/* Output item formats. U64 = raw residues (par::fill_residues), F64 =
 * to_unit_interval doubles (par::fill). F32 is an extension: RZ of the f64. */
typedef enum bcn_format { BCN_FORMAT_U64 = 0, BCN_FORMAT_F64 = 1, BCN_FORMAT_F32 = 2 } bcn_format;

/* reference include/bcnrand/parallel.hpp:15 */
typedef enum bcn_layout { BCN_LAYOUT_CONTIGUOUS = 0, BCN_LAYOUT_INTERLEAVED = 1 } bcn_layout;

/* reference include/bcnrand/generator.hpp:17. Every method yields identical
 * bits (test_generator.cpp:70-83); on the GPU it is validated and recorded,
 * and the device reduction is chosen by bcn_engine instead. */
typedef enum bcn_method {
    BCN_METHOD_REF128 = 0,
    BCN_METHOD_LECUYER = 1,
    BCN_METHOD_BARRETT = 2,
    BCN_METHOD_BARRETT_MODIFIED = 3
} bcn_method;

/* Device reduction engine. AUTO = the measured best. */
typedef enum bcn_engine {
    BCN_ENGINE_AUTO = 0,
    BCN_ENGINE_BARRETT = 1,    /* Shoup-form Barrett jump multiply         */
    BCN_ENGINE_MONTGOMERY = 2, /* Montgomery REDC jump multiply            */
    BCN_ENGINE_FP64 = 3,       /* exact FP64-pipe jump multiply            */
    BCN_ENGINE_STAGED = 4,     /* paper T=1 modified Barrett + TMA bulk store */
    BCN_ENGINE_BULK = 5,       /* FP64 jump streams staged in smem + TMA bulk store */
    BCN_ENGINE_MIXED = 6,      /* DFMA quotient + exact integer remainder   */
    BCN_ENGINE_HYBRID = 7      /* FP64 and Barrett streams side by side (FP64 + IMAD pipes) */
} bcn_engine;

/* ---- library ---------------------------------------------------------- */
int bcn_abi_version(void);
/* Message for the calling thread's most recent non-OK status ("" if none). */
const char* bcn_last_error(void);
/* Name of an engine ("auto", "barrett", "montgomery", "fp64", "staged", "bulk", "mixed"). */
const char* bcn_engine_name(int engine);
/* Number of visible CUDA devices (0 when none; never an error). */
int bcn_device_count(void);

/* L2 cache size of `device` in bytes (0 when there is no such device). */
uint64_t bcn_l2_bytes(int device);

/* ---- generator.hpp ------------------------------------------------------ */
/* generator.hpp:33 / generator.cpp:17-30 — 2^e mod `modulus` (odd, < 2^63). */
bcn_status bcn_modpow2(uint64_t e, uint64_t modulus, uint64_t* out);
/* generator.hpp:37 / generator.cpp:32-40 — z0 for seed index a. */
bcn_status bcn_seed_from_index(uint64_t a, uint64_t* z0);
/* generator.hpp:42-43 / generator.cpp:42-49 — z_k = 2^(53 (k mod P)) z0. */
bcn_status bcn_state_at(uint64_t a, uint64_t k, uint64_t* z);
/* generator.hpp:52-70 — one step of z (z in [1, m)). */
bcn_status bcn_next(uint64_t* z);
/* generator.hpp:74-78 — double(z) / 3^33 with one RN multiply. */
bcn_status bcn_to_unit_interval(uint64_t z, double* u);

/* ---- parallel.hpp ------------------------------------------------------- */
/* parallel.hpp:42 / parallel.cpp:35-52 — effective workers and ceil(n/W). */
bcn_status bcn_make_plan(uint64_t n, uint32_t workers, uint32_t* eff_workers,
                         uint64_t* work_per_worker);
/* parallel.cpp:24-33 — physical slot of worker w's element i. */
bcn_status bcn_physical_index(uint64_t n, uint32_t workers, bcn_layout layout, uint32_t w,
                              uint64_t i, uint64_t* slot);

/* parallel.hpp:48-49 (F64) and :52-54 (U64), plus F32.
 * Writes plan.n = n items (from make_plan(n, workers, layout)) for seed index
 * `seed_index`, worker w seeded by state_at(a, base_offset + w*wpw) exactly as
 * parallel.cpp:56-79. `capacity` is the buffer size in items (the span size);
 * capacity < n is std::invalid_argument before any work. Device pointers must
 * be aligned to the item size. */
bcn_status bcn_fill(void* out, uint64_t capacity, uint64_t n, bcn_format format,
                    uint32_t workers, bcn_layout layout, uint64_t seed_index, bcn_method method,
                    uint64_t base_offset, bcn_engine engine, int device, void* stream);

/* Multi-GPU fill from one host process: the logical range [0, n) is split with
 * make_plan(n, ndev) (contiguous shards) and shard g is written to outs[g]
 * (device memory of devices[g], capacities[g] items, >= the shard size, else
 * std::invalid_argument before any device work) with base_offset + its start,
 * one host thread per device, no collective. streams: NULL (each device drains,
 * then the library's stream) or one stream per shard (the caller orders).
 * Synchronous. The concatenation of the shards is bit-identical to a
 * single-device fill. */
bcn_status bcn_fill_multi(void* const* outs, const uint64_t* capacities, const int* devices, int ndev,
                          uint64_t n, bcn_format format, uint64_t seed_index, uint64_t base_offset,
                          bcn_engine engine, void* const* streams);

/* parallel.hpp:58-60 — de-interleave an Interleaved buffer of plan.n items
 * (itemsize 4 or 8) into logical order. Both pointers on `device` (or both
 * host). */
bcn_status bcn_deinterleave(const void* in, void* out, uint64_t n, uint32_t workers,
                            uint32_t itemsize, int device, void* stream);

/* Skip-ahead stress / seed-states kernel. Device arrays:
 * a[count] seed indices, k[count] offsets. steps == 0: out[t] =
 * state_at(a[t], k[t]); steps > 0: out[t*steps + s] = (s+1)-th next() from
 * that state. Any out-of-range a -> BCN_ERR_OUT_OF_RANGE (checked on device,
 * reported after the launch completes). Synchronous. */
bcn_status bcn_seed_states(const uint64_t* a, const uint64_t* k, uint64_t* out, uint64_t count,
                           uint32_t steps, int device, void* stream);

/* Order-sensitive digest of n items (itemsize 4 or 8) at a device pointer:
 * d[0] = sum x_i, d[1] = sum (index_base+i+1) x_i, d[2] = xor x_i (2(index_base+i)+1),
 * all mod 2^64 (sums combine across shards; NCCL ncclSum on ncclUint64). */
bcn_status bcn_digest(const void* buf, uint64_t n, uint32_t itemsize, uint64_t index_base,
                      uint64_t d[3], int device, void* stream);

/* Engine self-check (the device counterpart of the reference's kernel
 * equivalence check, modred.hpp:103-159 / test_modred.cpp:73-96):
 * out[i] = z[i] * c[i]^chain mod 3^33 computed by one jump engine (BARRETT,
 * MONTGOMERY, FP64 or MIXED), the state kept in the engine's own
 * representation between the `chain` multiplications. z[i] and c[i] in
 * [0, 3^33); host arrays of `count` <= 2^26 items. Synchronous. */
bcn_status bcn_engine_check(bcn_engine engine, const uint64_t* z, const uint64_t* c, uint64_t* out,
                            uint64_t count, uint32_t chain, int device);

/* The Constant writer (reference bench.cpp:60-63): identical geometry and
 * 256-bit stores as the contiguous fill, writing one fixed 8-byte pattern.
 * Device pointer, 32-byte aligned, nbytes a multiple of 1024. Asynchronous on
 * `stream` (synchronous when stream == NULL). The roofline denominator. */
bcn_status bcn_fill_constant(void* out, uint64_t nbytes, uint64_t pattern, int device,
                             void* stream);

/* Write-ceiling probe: the Constant writer's geometry and write pacing, but
 * each thread writes fixed pseudo-random words derived from `seed` (non-zero)
 * — data that toggles the HBM interface like generator output, which costs
 * measurably more power than a constant pattern. Same pointer rules and
 * stream semantics as bcn_fill_constant. Not part of the reference API. */
bcn_status bcn_fill_noise(void* out, uint64_t nbytes, uint64_t seed, int device, void* stream);

/* One row of the reference's throughput harness (bench::run, bench.cpp:102-142)
 * on the GPU: `repeats` fills of n doubles (plan make_plan(n, workers, layout),
 * seed index `seed_index`) into a device buffer on `device` with `engine`
 * (or, for engine == -1, the Constant writer over the same bytes rounded down
 * to whole 1 KiB rows). exec_seconds = median kernel time (CUDA events),
 * total_seconds = median wall time of the synchronous call (launch, setup and
 * generation). With check_output, the last timed output must equal a fill
 * with the default engine (compared by digest), else BCN_ERR_DOMAIN. */
bcn_status bcn_bench_fill(uint64_t n, uint32_t workers, bcn_layout layout, uint64_t seed_index,
                          int engine, int repeats, int check_output, int device,
                          double* exec_seconds, double* total_seconds);

/* Engine AUTO resolves to this engine for (format); exposed for benches. */
int bcn_auto_engine(bcn_format format);

/* Number of kernels this library has launched in the process (benches count
 * their own launches inside a timed region with it). */
uint64_t bcn_launch_count(void);

/* Process-wide launch tuning of the contiguous fill and Constant kernels:
 * CTAs per SM of the persistent grid (0 = as many as fit) and row order
 * (0 = per-warp contiguous row ranges, 1 = grid-strided rows, the default).
 * Output bits never depend on it. */
bcn_status bcn_set_launch_config(int ctas_per_sm, int row_order);

/* Process-wide HBM write pacing of the contiguous fill and Constant kernels.
 * B200 write efficiency drops when SM stores oversubscribe HBM; the paced
 * kernels meter their stores to a target rate (GB/s, per device) with one pacer
 * thread per CTA reading %globaltimer. target_gbs < 0: automatic (default) —
 * each device uses the target its context measured at initialisation (a short
 * sweep of the paced fill, 100 GB/s apart: the target with the highest
 * measured rate; BCN_PACE_CALIBRATE=0 skips the sweep and uses 7200); 0: unpaced;
 * otherwise a fixed target >= 100. ctas_per_sm in [1,7] (default 1: 8 worker
 * warps per SM — measured ~1.3% faster sustained than 2); format_mask: bit f
 * enables pacing for bcn_format f (default U64|F64 = 3). Output bits never
 * depend on it. */
bcn_status bcn_set_write_pacing(double target_gbs, int ctas_per_sm, int format_mask);
/* The pacing setting in GB/s (< 0 = automatic, 0 = unpaced). */
double bcn_write_pacing(void);
/* Where a device's effective pacing target comes from. */
typedef enum bcn_pace_source {
    BCN_PACE_UNPACED = 0,
    BCN_PACE_USER = 1,        /* bcn_set_write_pacing with a fixed target   */
    BCN_PACE_CALIBRATED = 2,  /* measured by this process on this device    */
    BCN_PACE_DEFAULT = 3      /* calibration disabled or failed: 7200 GB/s  */
} bcn_pace_source;
/* Effective pacing target of `device` (0 = unpaced) and its source; runs the
 * device's calibration first if it has not run yet. */
bcn_status bcn_device_write_pacing(int device, double* target_gbs, int* source);
/* The (target, achieved) GB/s points of `device`'s calibration sweep; *count
 * = number of points (at most `capacity` are written). */
bcn_status bcn_pace_calibration(int device, double* targets, double* achieved, int capacity, int* count);
/* Current pacing configuration (any pointer may be NULL). */
void bcn_get_write_pacing(double* target_gbs, int* ctas_per_sm, int* format_mask);

/* ---- quality.hpp: statistical smoke suite on the GPU ---
 * Host or device input pointers. Preconditions and formulas follow
 * quality.cpp:21-118; chi-square and monobit statistics are computed from
 * exact device counts (bit-identical to the reference), the lag correlation
 * from per-block partial sums reduced in a fixed order (deterministic). */
/* quality.hpp:27 — chi-square over `bins` equal bins of (0,1). */
bcn_status bcn_chi_square_uniformity(const double* samples, uint64_t n, int bins, double* statistic,
                                     int* dof, int* pass, int device, void* stream);
/* quality.hpp:33 — worst one-frequency deviation over bits 5..52 of floor(z 2^53/m). */
bcn_status bcn_monobit_mantissa(const uint64_t* residues, uint64_t n, double* statistic, int* worst_bit,
                                int* pass, int device, void* stream);
/* quality.hpp:37 — Pearson correlation of samples `lag` apart. */
bcn_status bcn_serial_correlation(const double* samples, uint64_t n, int lag, double* rho, int* pass,
                                  int device, void* stream);

/* cli.cpp:127-131 — the `gen --format text` rendering: one "%.17g\n" line per
 * value (host, multi-threaded). *written = bytes needed; capacity too small is
 * BCN_ERR_INVALID_ARGUMENT (24 bytes per value always suffice). */
bcn_status bcn_format_text(const double* values, uint64_t n, char* out, uint64_t capacity,
                           uint64_t* written);

#ifdef __cplusplus
}
#endif
#endif /* BCNRAND_B200_H */
