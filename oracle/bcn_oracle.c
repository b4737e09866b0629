/*
 * bcn_oracle.c — CPU restatement of the reference alpha_{2,3} fill path.
 *
 * TEST INFRASTRUCTURE ONLY (see bcn_oracle.h): the checker for the CUDA path,
 * never the thing measured or shipped. Reference paths are relative to
 * /root/reference/proj.
 */
#include "bcn_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

static uint64_t mulmod(uint64_t a, uint64_t b, uint64_t m) {
    /* generator.cpp:11-13 */
    return (uint64_t)((u128)a * b % m);
}

int bcno_reduce_ref(uint64_t z, uint64_t* out) {
    /* modred.hpp:103-107: require z < m, then (z << 53) % m in 128 bits. */
    if (z >= BCNO_MODULUS) return BCNO_DOMAIN_ERROR;
    *out = (uint64_t)(((u128)z << 53) % BCNO_MODULUS);
    return BCNO_OK;
}

int bcno_barrett_modified_step(uint64_t z, uint64_t* out) {
    /* modred.hpp:149-159: q3 = floor(mu z / 2^53); r = 2^53 - (q3 m mod 2^53);
     * one conditional subtract. z = 0 is outside the domain (modred.hpp:150). */
    if (z == 0 || z >= BCNO_MODULUS) return BCNO_DOMAIN_ERROR;
    const u128 prod = (u128)z * BCNO_MU;
    const uint64_t q3 = (uint64_t)(prod >> 53);
    const uint64_t r2 = (q3 * BCNO_MODULUS) & ((1ull << 53) - 1);
    uint64_t r = (1ull << 53) - r2;
    if (r >= BCNO_MODULUS) r -= BCNO_MODULUS;
    *out = r;
    return BCNO_OK;
}

int bcno_next(uint64_t* z) {
    /* generator.hpp:52-70 with the default Method::BarrettModified. */
    return bcno_barrett_modified_step(*z, z);
}

int bcno_modpow2(uint64_t e, uint64_t modulus, uint64_t* out) {
    /* generator.cpp:17-30 */
    if (modulus % 2 == 0) return BCNO_INVALID_ARGUMENT;
    if (modulus >= (1ull << 63)) return BCNO_INVALID_ARGUMENT;
    uint64_t result = 1 % modulus;
    uint64_t base = 2 % modulus;
    while (e != 0) {
        if (e & 1) result = mulmod(result, base, modulus);
        base = mulmod(base, base, modulus);
        e >>= 1;
    }
    *out = result;
    return BCNO_OK;
}

int bcno_seed_from_index(uint64_t a, uint64_t* z0) {
    /* generator.cpp:32-40 */
    if (a < BCNO_MIN_SEED || a > BCNO_MAX_SEED) return BCNO_OUT_OF_RANGE;
    const uint64_t half_m = 2779530283277761ull; /* floor(3^33 / 2) */
    uint64_t p;
    bcno_modpow2(a - BCNO_MODULUS, BCNO_MODULUS, &p);
    *z0 = mulmod(p, half_m, BCNO_MODULUS);
    return BCNO_OK;
}

int bcno_state_at(uint64_t a, uint64_t k, uint64_t* z) {
    /* generator.cpp:42-49: 53 (k mod P) < 2^63 never overflows. */
    uint64_t z0;
    int st = bcno_seed_from_index(a, &z0);
    if (st) return st;
    uint64_t hop;
    bcno_modpow2(53 * (k % BCNO_PERIOD), BCNO_MODULUS, &hop);
    *z = mulmod(hop, z0, BCNO_MODULUS);
    return BCNO_OK;
}

int bcno_to_unit_interval(uint64_t z, double* u) {
    /* generator.hpp:74-78: z = 0 and z >= m are rejected; one RN multiply. */
    if (z == 0 || z >= BCNO_MODULUS) return BCNO_DOMAIN_ERROR;
    const double inv = 1.0 / 5559060566555523.0; /* generator.hpp:22 */
    *u = (double)z * inv;
    return BCNO_OK;
}

static float f64_to_f32_rz(double d) {
    /* Round toward zero for a positive normal double in (0,1): keep the top 24
     * significand bits. Values here are >= 1/m ~ 1.8e-16, far above FLT_MIN. */
    uint64_t bits;
    memcpy(&bits, &d, 8);
    const uint32_t exp = (uint32_t)(bits >> 52) & 0x7FF;
    const uint32_t fbits = ((exp - 1023 + 127) << 23) | (uint32_t)((bits >> 29) & 0x7FFFFF);
    float f;
    memcpy(&f, &fbits, 4);
    return f;
}

int bcno_to_unit_float(uint64_t z, float* u) {
    double d;
    int st = bcno_to_unit_interval(z, &d);
    if (st) return st;
    *u = f64_to_f32_rz(d);
    return BCNO_OK;
}

int bcno_make_plan(uint64_t n, uint32_t workers, uint32_t* eff_workers, uint64_t* wpw) {
    /* parallel.cpp:35-52 */
    if (n == 0 || workers == 0) return BCNO_INVALID_ARGUMENT;
    const uint64_t w = (n + workers - 1) / workers;
    *wpw = w;
    *eff_workers = (uint32_t)((n + w - 1) / w);
    return BCNO_OK;
}

uint64_t bcno_elements_for(uint64_t n, uint64_t wpw, uint32_t w) {
    /* parallel.cpp:19-22 */
    const uint64_t start = (uint64_t)w * wpw;
    return wpw < n - start ? wpw : n - start;
}

uint64_t bcno_physical_index(uint64_t n, uint32_t workers, uint64_t wpw, int layout,
                             uint32_t w, uint64_t i) {
    /* parallel.cpp:24-33; `workers` is the effective count (plan.step). */
    if (layout == 0) return (uint64_t)w * wpw + i;
    const uint64_t short_count = bcno_elements_for(n, wpw, workers - 1);
    if (i < short_count) return i * workers + w;
    return short_count * workers + (i - short_count) * (workers - 1) + w;
}

/* Splits worker w's elements into [i0, i1) pieces so a plan with few workers
 * still uses all host threads; each piece seeds itself by skip-ahead, exactly
 * like a worker does (the result is a pure function of the logical index). */
typedef struct {
    void* out;
    uint64_t n, wpw, base_offset, seed_index;
    uint32_t workers, w;
    int fmt, layout;
    uint64_t i0, i1;
} piece_job;

static void* fill_piece(void* arg) {
    const piece_job* j = (const piece_job*)arg;
    /* State after i0 steps of worker w == state_at(a, start_w + i0) (the
     * reference's skip-ahead composition, test_generator.cpp:103-114); the k
     * argument wraps mod 2^64 exactly as base_offset + start_w does. */
    uint64_t z;
    bcno_state_at(j->seed_index, j->base_offset + (uint64_t)j->w * j->wpw, &z);
    if (j->i0) {
        uint64_t hop;
        bcno_modpow2(53 * (j->i0 % BCNO_PERIOD), BCNO_MODULUS, &hop);
        z = mulmod(hop, z, BCNO_MODULUS);
    }
    for (uint64_t i = j->i0; i < j->i1; ++i) {
        bcno_barrett_modified_step(z, &z);
        const uint64_t p = bcno_physical_index(j->n, j->workers, j->wpw, j->layout, j->w, i);
        if (j->fmt == 0) {
            ((uint64_t*)j->out)[p] = z;
        } else if (j->fmt == 1) {
            bcno_to_unit_interval(z, &((double*)j->out)[p]);
        } else {
            bcno_to_unit_float(z, &((float*)j->out)[p]);
        }
    }
    return NULL;
}

int bcno_fill(void* out, uint64_t n, int fmt, uint32_t workers, int layout,
              uint64_t seed_index, uint64_t base_offset, uint32_t threads) {
    uint32_t eff;
    uint64_t wpw;
    int st = bcno_make_plan(n, workers, &eff, &wpw);
    if (st) return st;
    if (fmt < 0 || fmt > 2 || layout < 0 || layout > 1) return BCNO_INVALID_ARGUMENT;
    if (seed_index < BCNO_MIN_SEED || seed_index > BCNO_MAX_SEED) return BCNO_OUT_OF_RANGE;
    if (threads == 0) threads = 1;
    /* Pieces: every worker is cut into ceil(threads/eff) pieces. */
    uint64_t per_worker = (threads + eff - 1) / eff;
    if (per_worker == 0) per_worker = 1;
    const uint64_t npieces = (uint64_t)eff * per_worker;
    piece_job* jobs = (piece_job*)calloc(npieces, sizeof(piece_job));
    uint64_t nj = 0;
    for (uint32_t w = 0; w < eff; ++w) {
        const uint64_t cnt = bcno_elements_for(n, wpw, w);
        const uint64_t step = (cnt + per_worker - 1) / per_worker;
        for (uint64_t i0 = 0; i0 < cnt; i0 += step) {
            piece_job* j = &jobs[nj++];
            j->out = out; j->n = n; j->wpw = wpw; j->base_offset = base_offset;
            j->seed_index = seed_index; j->workers = eff; j->w = w; j->fmt = fmt;
            j->layout = layout; j->i0 = i0; j->i1 = i0 + step < cnt ? i0 + step : cnt;
        }
    }
    if (threads == 1 || nj == 1) {
        for (uint64_t k = 0; k < nj; ++k) fill_piece(&jobs[k]);
    } else {
        /* Run pieces on `threads` threads, round-robin. */
        pthread_t* tid = (pthread_t*)calloc(threads, sizeof(pthread_t));
        for (uint64_t base = 0; base < nj; base += threads) {
            uint32_t started = 0;
            for (uint32_t t = 0; t < threads && base + t < nj; ++t) {
                pthread_create(&tid[t], NULL, fill_piece, &jobs[base + t]);
                ++started;
            }
            for (uint32_t t = 0; t < started; ++t) pthread_join(tid[t], NULL);
        }
        free(tid);
    }
    free(jobs);
    return BCNO_OK;
}

int bcno_deinterleave(const void* in, void* out, uint64_t n, uint32_t workers,
                      uint32_t itemsize) {
    /* parallel.cpp:81-97 (layout checked by the caller: this is the
     * Interleaved inverse). */
    uint32_t eff;
    uint64_t wpw;
    int st = bcno_make_plan(n, workers, &eff, &wpw);
    if (st) return st;
    if (itemsize != 4 && itemsize != 8) return BCNO_INVALID_ARGUMENT;
    for (uint32_t w = 0; w < eff; ++w) {
        const uint64_t cnt = bcno_elements_for(n, wpw, w);
        for (uint64_t i = 0; i < cnt; ++i) {
            const uint64_t p = bcno_physical_index(n, eff, wpw, 1, w, i);
            const uint64_t l = (uint64_t)w * wpw + i;
            memcpy((char*)out + l * itemsize, (const char*)in + p * itemsize, itemsize);
        }
    }
    return BCNO_OK;
}

void bcno_digest(const void* buf, uint64_t n, uint32_t itemsize, uint64_t index_base,
                 uint64_t d[3]) {
    uint64_t s = 0, ws = 0, x = 0;
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t v;
        if (itemsize == 8) {
            memcpy(&v, (const char*)buf + i * 8, 8);
        } else {
            uint32_t v32;
            memcpy(&v32, (const char*)buf + i * 4, 4);
            v = v32;
        }
        const uint64_t g = i + index_base;
        s += v;
        ws += (g + 1) * v;
        x ^= v * (2 * g + 1);
    }
    d[0] = s;
    d[1] = ws;
    d[2] = x;
}

int bcno_seed_batch(const uint64_t* a, const uint64_t* k, uint64_t* out, uint64_t count,
                    uint32_t steps) {
    for (uint64_t t = 0; t < count; ++t) {
        uint64_t z;
        int st = bcno_state_at(a[t], k[t], &z);
        if (st) return st;
        if (steps == 0) {
            out[t] = z;
            continue;
        }
        for (uint32_t s = 0; s < steps; ++s) {
            bcno_barrett_modified_step(z, &z);
            out[t * steps + s] = z;
        }
    }
    return BCNO_OK;
}
