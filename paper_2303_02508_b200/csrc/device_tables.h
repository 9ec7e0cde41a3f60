// device_tables.h — layout of the per-call constant tables that the host
// builds (envelope.cpp) and the kernels stage into shared memory.
//
// Blob = TablesHeader | phase S[T], C[T] (f64) | ProfileTable[n_prof] |
//        PairTable[n_prof * n_eta]     (pair index = p * n_eta + e)
#pragma once
#include <stddef.h>
#include <stdint.h>
#include <vector_types.h>      // double2, uint2
#include <vector_functions.h>  // make_double2

namespace chase {

constexpr int kMaxK = 32;          // CHASE_MAX_LIMITS
constexpr int kNB = 776;           // buckets per pair table (12 octaves x 64 + 2, padded to 8)
constexpr int kNBUsed = 770;       // bucket 0 = below range, 1..768 = table, 769 = above
constexpr int kSH = 14;            // hi32(y) >> 14 = sign | 11-bit exponent | 6 mantissa bits
constexpr int kZeroLine = 32;      // ProfileTable.line[32] = (0, 0): marks a deferred canonical window

// Bucket entry (uint2), compared on h = hi32(y) as a signed int (monotone in
// y for y >= 0; negative y has h < 0):
//   x = T1                          (hi32 of the "below" threshold)
//   y = below | above << 8 | delta << 16,  T2 = T1 + delta
//   p1 = h < T1  (=> y < t_lo),  p2 = h > T2  (=> y > t_hi)
//   k = p1 ? below : (p2 ? above : kZeroLine)
// FAST: T1 = INT32_MAX.  All-slow: T1 = INT32_MIN, above = kZeroLine.
// kZeroLine -> the canonical K-way Eq. 6 (deferred).  See DESIGN.md §6.

struct alignas(16) TablesHeader {
    int32_t T, n_prof, n_eta, n_pairs;
    int32_t off_phase, off_prof, off_pair, total_bytes;
    double delta;
    double reserved[3];
};

struct alignas(16) ProfileTable {
    double2 line[kMaxK + 1];  // (s_k = Thr_k * Delta, P_k); line[kZeroLine] = (0, 0)
    double thr[kMaxK];     // Thr_k
    int32_t K, reserved;
    double pmax;           // resolved MaxPower
    double smax;           // max_k s_k (bounds the samples done after n windows)
    double reserved2;
    int32_t limit_w[kMaxK];  // the power limits themselves (timeline rows)
};

struct alignas(16) PairTable {
    double a[kMaxK];       // a_k = eta * P_k
    double kbase;          // (1 - eta) * Pmax; Kc = kbase * MaxCI
    int32_t base;          // idx = clamp((hi32(y) >> kSH) - base, 0, kNBUsed - 1)
    int32_t k0;            // 1: Kc == 0 (eta == 1) -> y = x; 0: y = x * (1/Kc)
    int32_t n_test;        // entries with a threshold test (diagnostic)
    int32_t n_intervals;   // fast intervals (diagnostic)
    double y_min;          // a lower bound on every positive finite interval endpoint (before the
                           // shrink), +inf if none: bounds the error a key computation may make
                           // (the headline's one-fma key)
    double reserved;
    uint2 ent[kNB];
};

// The leading fields of PairTable (everything but the bucket entries): the
// headline kernel keeps only these in shared memory next to its own expanded
// entries, and hands them to helpers that never touch `ent`.
struct PairHead {
    double a[kMaxK];
    double kbase;
    int32_t base, k0, n_test, n_intervals;
    double y_min, reserved;
};
static_assert(offsetof(PairTable, ent) == sizeof(PairHead), "PairHead mirrors PairTable's head");
static_assert(offsetof(PairTable, kbase) == offsetof(PairHead, kbase), "PairHead layout");
static_assert(offsetof(PairTable, k0) == offsetof(PairHead, k0), "PairHead layout");
static_assert(offsetof(PairTable, y_min) == offsetof(PairHead, y_min), "PairHead layout");

static_assert(sizeof(TablesHeader) % 16 == 0, "header alignment");
static_assert(sizeof(ProfileTable) % 16 == 0, "profile alignment");
static_assert(sizeof(PairTable) % 16 == 0, "pair alignment");

inline int tables_bytes(int T, int n_prof, int n_eta) {
    int phase = ((2 * T * 8) + 15) / 16 * 16;
    return (int)sizeof(TablesHeader) + phase + n_prof * (int)sizeof(ProfileTable) +
           n_prof * n_eta * (int)sizeof(PairTable);
}

}  // namespace chase
