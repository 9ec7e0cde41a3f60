/*
 * chase_gen.h — seeded synthetic carbon-intensity traces (harness inputs).
 *
 * This module holds NONE of the planner's arithmetic: it only produces the
 * inputs that the oracle (oracle/) and the product (paper_2303_02508_b200/)
 * both consume.  It is integer-only and counter-based, so the host and the
 * device produce bit-identical traces (every rank generates its own shard).
 *
 * Shape of the workload (DESIGN.md §5 "input recipe"):
 *   value(t) = mean + amp*sin_q[(phase0+t+shift) mod T]          (diurnal)
 *            + season*year_q[(t / T) mod 365]                     (seasonal drift)
 *            + sigma*IrwinHall4(hash(seed, trace, t))             (noise)
 * in units of 1/64 g/kWh, clamped to [0, 262143] (i.e. < 4096 g/kWh) and
 * stored as fp32 (exact: value_q * 2^-6 has <= 18 significant bits).
 * "paper" mode fixes mean 550, amp 150, sigma 10 g/kWh (S:520 at hourly T),
 * whose max over a day lands near the paper's 750 g/kWh.
 */
#ifndef CHASE_GEN_H
#define CHASE_GEN_H

#include <stdint.h>

#if defined(__CUDACC__)
#define CHASEGEN_HD __host__ __device__ __forceinline__
#else
#define CHASEGEN_HD static inline
#endif

#define CHASEGEN_MODE_RANDOM 0
#define CHASEGEN_MODE_PAPER  1
#define CHASEGEN_QMAX 262143   /* 4096*64 - 1 */

CHASEGEN_HD uint64_t chasegen_mix(uint64_t z) {          /* splitmix64 finaliser */
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

CHASEGEN_HD uint64_t chasegen_hash(uint64_t seed, uint64_t trace, uint32_t stream, uint32_t step) {
    uint64_t h = chasegen_mix(seed ^ 0xD1B54A32D192ED03ull);
    h = chasegen_mix(h ^ trace);
    h = chasegen_mix(h ^ (((uint64_t)stream << 32) | (uint64_t)step));
    return h;
}

typedef struct {
    int64_t mean_q, amp_q, sigma_q, season_q;
    int32_t shift;
} chasegen_params_t;

CHASEGEN_HD chasegen_params_t chasegen_params(uint64_t seed, uint64_t trace, int32_t mode, int32_t T) {
    chasegen_params_t p;
    if (mode == CHASEGEN_MODE_PAPER) {
        p.mean_q = 550 * 64; p.amp_q = 150 * 64; p.sigma_q = 10 * 64; p.season_q = 0; p.shift = 0;
        return p;
    }
    const uint32_t FULL = 0xFFFFFFFFu;
    uint64_t u0 = chasegen_hash(seed, trace, 1, FULL) >> 32;
    uint64_t u1 = chasegen_hash(seed, trace, 2, FULL) >> 32;
    uint64_t u2 = chasegen_hash(seed, trace, 3, FULL) >> 32;
    uint64_t u3 = chasegen_hash(seed, trace, 4, FULL) >> 32;
    uint64_t u4 = chasegen_hash(seed, trace, 5, FULL) >> 32;
    p.mean_q   = 6400 + (int64_t)(u0 % 44801u);                       /* U[100, 800] g/kWh */
    p.amp_q    = (p.mean_q * (int64_t)(3277 + u1 % 19661u)) >> 16;    /* U[0.05, 0.35]*mean */
    p.sigma_q  = (p.mean_q * (int64_t)(655 + u2 % 1966u)) >> 16;      /* U[0.01, 0.04]*mean */
    p.season_q = (p.mean_q * (int64_t)(u3 % 9831u)) >> 16;            /* U[0, 0.15]*mean   */
    p.shift    = (int32_t)(u4 % (uint64_t)T);
    return p;
}

/* value of step t (0-based within the trace) in 1/64 g/kWh.
 * sin_q[T]: round(2^30 sin(2 pi phi / T)); year_q[365]: round(2^30 cos(2 pi d / 365)). */
CHASEGEN_HD int32_t chasegen_value_q(const chasegen_params_t* p, uint64_t seed, uint64_t trace,
                                     int64_t t, int32_t T, int32_t phase0,
                                     const int32_t* sin_q, const int32_t* year_q) {
    int32_t phi = (int32_t)(((int64_t)phase0 + t + p->shift) % T);
    int32_t day = (int32_t)((((int64_t)phase0 + t) / T) % 365);
    int64_t v = p->mean_q;
    v += (p->amp_q * (int64_t)sin_q[phi]) >> 30;
    v += (p->season_q * (int64_t)year_q[day]) >> 30;
    uint64_t h = chasegen_hash(seed, trace, 7, (uint32_t)t);
    int64_t s = (int64_t)(h & 0xFFFF) + (int64_t)((h >> 16) & 0xFFFF)
              + (int64_t)((h >> 32) & 0xFFFF) + (int64_t)((h >> 48) & 0xFFFF) - 131070;
    v += (p->sigma_q * s) / 37837;            /* Irwin-Hall(4): sd = 65536/sqrt(3) */
    if (v < 0) v = 0;
    if (v > CHASEGEN_QMAX) v = CHASEGEN_QMAX;
    return (int32_t)v;
}

/* per-trace profile shape id (C4: "three profile shapes chosen per trace") */
CHASEGEN_HD int32_t chasegen_profile_id(uint64_t seed, uint64_t trace, int32_t n_profiles) {
    return (int32_t)((chasegen_hash(seed, trace, 9, 0xFFFFFFFFu) >> 32) % (uint64_t)n_profiles);
}

#endif
