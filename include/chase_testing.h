/*
 * chase_testing.h — host-only test hooks of libchase.so (not part of the
 * planner ABI).  They run the host half of the Eq. 6 fast path (the envelope
 * bucket table of DESIGN.md §6) exactly as the kernels consume it, so the CPU
 * test suite can check it against the oracle without a GPU.
 */
#ifndef CHASE_TESTING_H
#define CHASE_TESTING_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* For one (profile, eta) and per-trace MaxCI / Pmax, decide the limit index
 * of each forecast x[i] with the table lookup of the kernels: out[i] = index,
 * or -1 when the kernel would take the canonical K-way path.  Returns the
 * number of fast intervals of the table, or -1 on invalid arguments. */
int32_t chase_testing_envelope(int32_t K, const double* avg_power, const double* thr, double eta,
                               double pmax, double max_ci, int64_t n, const double* x, int32_t* out);

#ifdef __cplusplus
}
#endif
#endif
