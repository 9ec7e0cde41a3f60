// kernels.h — launch interface between the C ABI (chase_api.cpp) and the
// sm_100a kernels (kernels.cu).  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "chase.h"
#include "device_tables.h"

namespace chase {

constexpr int kThreads = 256;              // sweep CTA size
constexpr int kChunk = 36;                 // windows per thread per tile (4 x odd -> conflict-free LDS.128)
constexpr int kTileW = kThreads * kChunk;  // 9216 windows per tile
constexpr int kRecDoubles = 8;             // fit record: c0, ws, wc, wl, max_ci, status, ridge, kind
constexpr int kMaxEta = CHASE_MAX_ETA;

enum SweepMode { MODE_FUSED = 0, MODE_PREDICT = 1, MODE_REPLAY = 2 };

struct SweepParams {
    const void* traces;
    int64_t ld, n_traces;
    int32_t N, L, T, phase0, W, n_tiles;
    double delta;
    const double* records;        // [n][8] (FUSED / PREDICT)
    const uint8_t* tables;        // blob in the workspace
    int32_t tables_bytes;
    int32_t n_eta, n_prof;
    int32_t stage_bytes;          // per pipeline stage (trace tile + 64 B record slot)
    const uint8_t* profile_id;    // may be null
    const double* job;            // may be null
    double max_ci_fixed;          // > 0: fixed MaxCI
    const uint8_t* choice_in;     // REPLAY
    uint8_t* choice;              // FUSED out (may be null)
    int64_t ld_c;
    double* forecast;             // may be null (PREDICT: required)
    int64_t ld_f;
    chase_totals_t* per_trace;    // may be null
    double* cta_sums;             // [grid][n_eta][8]
    uint8_t* status;              // [n]
    chase_diag_t* diag;
};

struct FitParams {
    const void* traces;
    int64_t ld, n_traces;
    int32_t L, T, phase0, is_f64;
    double ridge, tol;
    const double* phase_tab;      // S[T], C[T] in the workspace blob
    double* records;              // [n][8]
    double* models_out;           // optional user copy [n][8]
    double* max_ci_out;           // optional [n]
};

struct PlanParams {
    const double* forecast;
    int64_t n_traces, W, ld_f;
    const uint8_t* tables;
    int32_t tables_bytes, n_eta, n_prof;
    const uint8_t* profile_id;
    const double* max_ci;         // per trace (when max_ci_fixed <= 0)
    double max_ci_fixed;
    uint8_t* choice;
    int64_t ld_c;
    chase_diag_t* diag;
};

// Shared-memory bytes of one sweep CTA for these shapes.
size_t sweep_smem_bytes(int tables_bytes, int T, int elem_size, int mode);
int sweep_stage_bytes(int elem_size);

cudaError_t launch_upload(const void* host, size_t bytes, void* dst, cudaStream_t s);
cudaError_t launch_fit(const FitParams& p, cudaStream_t s);
// grid_out receives the number of CTAs used (rows of cta_sums).
cudaError_t launch_sweep(int mode, bool f64, bool aligned, const SweepParams& p, int max_grid,
                         int* grid_out, cudaStream_t s);
cudaError_t launch_plan(const PlanParams& p, cudaStream_t s);
cudaError_t launch_finalize(const double* cta_sums, int grid, int n_eta, chase_sum_t* sum,
                            const uint8_t* status, int64_t n_traces, uint8_t* choice, int64_t ld_c,
                            int64_t W, int n_eta_choice, double* forecast, int64_t ld_f,
                            chase_diag_t* diag, cudaStream_t s);
cudaError_t launch_diag_reset(chase_diag_t* diag, cudaStream_t s);
uint64_t kernel_launches();
cudaError_t launch_accumulate(double* acc, const double* add, int n, cudaStream_t s);

}  // namespace chase
