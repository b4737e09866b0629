/*
 * bcn_oracle.h — CPU restatement of the reference alpha_{2,3} generator path.
 *
 * TEST INFRASTRUCTURE ONLY. This is the parity checker for the CUDA product
 * path: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it. The product library
 * (paper_1206_1187_b200/libbcnrand_b200.so) never links or calls it.
 *
 * Every function restates the reference algorithm and cites the reference
 * file:line it follows (paths relative to /root/reference/proj). Parity of this
 * restatement is pinned two ways (see tests/test_oracle.py):
 *   - against the reference's own golden vectors (tests/test_modred.cpp:13-16,
 *     tests/test_generator.cpp:13-17, tests/test_cli.cpp:85) and the SURVEY
 *     Appendix A digests, and
 *   - against the reference itself compiled here into oracle/_ref/ (see
 *     oracle/Makefile), through tests/golden/ fixtures made by
 *     tests/golden/make_golden.py.
 */
#ifndef BCN_ORACLE_H
#define BCN_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes mirror the reference exception types. */
enum {
    BCNO_OK = 0,
    BCNO_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    BCNO_OUT_OF_RANGE = 2,     /* std::out_of_range     */
    BCNO_DOMAIN_ERROR = 3      /* std::domain_error     */
};

/* include/bcnrand/modred.hpp:22-23, generator.hpp:19-22 */
#define BCNO_MODULUS 5559060566555523ull
#define BCNO_PERIOD 3706040377703682ull
#define BCNO_MIN_SEED (BCNO_MODULUS + 100ull)
#define BCNO_MAX_SEED (1ull << 53)
#define BCNO_MU 0x33D9481681D79Dull

/* modred.hpp:103-107 — (2^53 z) mod m through an exact 128-bit product. */
int bcno_reduce_ref(uint64_t z, uint64_t* out);
/* modred.hpp:149-159 — the paper's modified Barrett step (default Method). */
int bcno_barrett_modified_step(uint64_t z, uint64_t* out);
/* generator.cpp:17-30 — 2^e mod modulus by square-and-multiply. */
int bcno_modpow2(uint64_t e, uint64_t modulus, uint64_t* out);
/* generator.cpp:32-40 — z0 = 2^(a-3^33) * floor(m/2) mod m. */
int bcno_seed_from_index(uint64_t a, uint64_t* z0);
/* generator.cpp:42-49 — z_k = 2^(53 (k mod P)) z0 mod m. */
int bcno_state_at(uint64_t a, uint64_t k, uint64_t* z);
/* generator.hpp:74-78 — double(z) * (1.0/3^33), one RN multiply. */
int bcno_to_unit_interval(uint64_t z, double* u);
/* f32 format (not in the reference; defined by this repo):
 * RZ(to_unit_interval(z)), i.e. the double rounded toward zero. */
int bcno_to_unit_float(uint64_t z, float* u);

/* parallel.cpp:35-52 — make_plan: wpw = ceil(n/W), effective W. */
int bcno_make_plan(uint64_t n, uint32_t workers, uint32_t* eff_workers, uint64_t* wpw);
/* parallel.cpp:19-22 */
uint64_t bcno_elements_for(uint64_t n, uint64_t wpw, uint32_t w);
/* parallel.cpp:24-33; layout 0 = Contiguous, 1 = Interleaved */
uint64_t bcno_physical_index(uint64_t n, uint32_t workers, uint64_t wpw, int layout,
                             uint32_t w, uint64_t i);

/* parallel.cpp:56-111 — fill / fill_residues with the plan's worker split.
 * fmt: 0 = raw u64 residues, 1 = f64, 2 = f32. out has room for n items.
 * threads: host threads to use (>=1); the result does not depend on it. */
int bcno_fill(void* out, uint64_t n, int fmt, uint32_t workers, int layout,
              uint64_t seed_index, uint64_t base_offset, uint32_t threads);
/* parallel.cpp:81-97 — inverse of the Interleaved scatter, itemsize 4 or 8. */
int bcno_deinterleave(const void* in, void* out, uint64_t n, uint32_t workers,
                      uint32_t itemsize);

/* Order-sensitive digests of a buffer of 8-byte (or 4-byte) items:
 * d[0] = sum x_i mod 2^64, d[1] = sum (i+1+index_base) x_i mod 2^64,
 * d[2] = xor of x_i * (2(i+index_base)+1) mod 2^64. */
void bcno_digest(const void* buf, uint64_t n, uint32_t itemsize, uint64_t index_base,
                 uint64_t d[3]);

/* Step one state with the reference's next() semantics (generator.hpp:52-70). */
int bcno_next(uint64_t* z);

/* Batched state_at (steps == 0: out[t] = state_at(a[t], k[t])) or walks
 * (out[t*steps + s] = (s+1)-th next() from it) — the C4 skip-ahead checker. */
int bcno_seed_batch(const uint64_t* a, const uint64_t* k, uint64_t* out, uint64_t count,
                    uint32_t steps);

#ifdef __cplusplus
}
#endif
#endif
