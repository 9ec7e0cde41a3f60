// envelope.h — host construction of the exact fast path for Eq. 6.
//
// For a fixed (profile, eta), cost_k(x) = (a_k x + Kc)/Thr_k is affine in the
// forecast x, and Kc = (1-eta)*Pmax*MaxCI only scales it: with y = x/Kc,
// cost_k = Kc * (a_k y + 1)/Thr_k.  So the argmin over k is a function of y
// alone whose breakpoints depend only on (profile, eta).  The builder finds,
// in long double, the y-intervals on which ONE line beats every other line by
// a relative margin of at least 64u (u = 2^-53); there the canonical fp64
// rule (three roundings per cost, error <= 3u) provably returns that line.
// Outside them (bands of ~1e-14 relative around each breakpoint, identical
// or nearly coincident lines) the kernel evaluates the canonical K-way rule.
// The intervals are then bucketed by the high bits of y's fp64 encoding.
#pragma once
#include <vector>

#include "device_tables.h"

namespace chase {

struct FastInterval {
    double lo, hi;   // y in [lo, hi] (after conservative shrinking) -> line k
    int k;
};

// Fill `out` (a, kbase, base, k0, slots, ent) for one (profile, eta) pair.
// Returns the fast intervals for diagnostics/tests.
std::vector<FastInterval> build_pair_table(int K, const double* avg_power, const double* thr,
                                           double eta, double pmax, PairTable* out);

}  // namespace chase
