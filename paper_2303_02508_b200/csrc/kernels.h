// kernels.h — launch interface between the C ABI (chase_api.cpp) and the
// sm_100a kernels (kernels.cu).  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "chase.h"
#include "device_tables.h"

namespace chase {

constexpr int kThreads = 192;              // sweep CTA size (6 independent warps; 12 per SM at <= 168 registers)
constexpr int kWarpsPerCta = kThreads / 32;
constexpr int kChunk = 36;                 // windows per lane per chunk (4 x odd -> conflict-free LDS.128)
constexpr int kWarpW = 32 * kChunk;        // 1152 windows per warp chunk
constexpr int kRecDoubles = 16;            // workspace record per trace (see below)
constexpr int kModelDoubles = 8;           // d_models row of chase_fit_forecast
constexpr int kRawDoubles = 8;             // per (eta, trace) replay raw result
constexpr int kMaxEta = CHASE_MAX_ETA;
constexpr int kFinThreads = 256;           // finalize CTA size

// Workspace record of trace i (written by fit_kernel, read by sweep/finalize):
//  [0] c0 [1] w_sin [2] w_cos [3] w_lag [4] max_ci(history) [5] status
//  [6] ridge [7] kind [8] m_base (baseline completion count, 0: J <= 0)
//  [9] Cb (baseline sum of c over the windows before w*_b; sweep writes)
//  [10..15] eta-0 scalars for the headline sweep: Kc, 1/Kc, J, profile,
//           windows-to-completion lower bound, resolved MaxCI
// Raw per (eta, trace) (sweep writes, finalize reads):
//  [0] E [1] C [2] S [3] f [4] w* [5] P_k* [6] c[w*] [7] done
enum SweepMode { MODE_FUSED = 0, MODE_PREDICT = 1, MODE_REPLAY = 2 };

struct SweepParams {
    const void* traces;
    int64_t ld, n_traces;
    int32_t N, L, T, phase0, W, n_chunks;
    double delta;
    double* records;              // [n][16]
    double* raw;                  // [n_eta][n][8]
    const uint8_t* tables;        // blob in the workspace
    int32_t tables_bytes;
    int32_t n_eta, n_prof;
    int32_t stage_bytes;          // per pipeline stage (trace chunk + record slot)
    // host-precomputed chunk geometry (kept in the constant bank, not registers)
    int32_t a0, off0, W_last, phase_step, phase_start;
    uint32_t bytes_full, bytes_last;
    const uint8_t* profile_id;    // may be null
    const double* job;            // may be null
    double max_ci_fixed;          // > 0: fixed MaxCI
    const uint8_t* choice_in;     // REPLAY
    uint8_t* choice;              // FUSED out (may be null)
    int64_t ld_c;
    double* forecast;             // may be null (PREDICT: required)
    int64_t ld_f;
    uint8_t* status;              // [n]
    chase_diag_t* diag;
    int64_t* bad_list;            // [n]: traces with status 4..7 (slot = old n_bad)
    const double* fc_in;          // rolling refit: forecasts [n][ld_fin] (null: fit-once fold)
    int64_t ld_fin;
    int32_t kc_last;              // headline kernel: windows per lane in the last chunk (4 mod 8)
    int32_t smem_total;           // headline kernel: dynamic shared memory planned by the host
    int32_t period;               // > 1: one decision per period of this many windows (headline kernel)
    int32_t k0len;                // headline kernel, periods: doubles of the closed-form horizon table per warp (0: none)
    int32_t refit;                // roll_fused_kernel: the refit stride R >= 1
    double ridge, tol;            // roll_fused_kernel: the fit's ridge and singular tolerance (exact fallback)
};

struct FitParams {
    const void* traces;
    int64_t ld, n_traces;
    int32_t L, T, phase0, is_f64, W, n_prof;
    int32_t baseline_only;        // 1: only the baseline count m (chase_replay)
    double ridge, tol;
    const uint8_t* tables;        // blob (phase table, profiles)
    const uint8_t* profile_id;
    const double* job;
    double* records;              // [n][16]
    double* models_out;           // optional user copy [n][8]
    double* max_ci_out;           // optional [n]
    double* prec;                 // workspace slot for the job-start phase record (phase_stride(64) doubles)
    int32_t n_eta;                // > 0: also the single-eta sweep's per-trace scalars (record [10..15])
    int32_t reserved;
    double max_ci_fixed;          // > 0: fixed MaxCI
};

struct FinalizeParams {
    const void* traces;
    int64_t ld, n_traces;
    int32_t L, W, n_eta, n_prof, is_f64;
    double delta;
    const double* records;
    const double* raw;
    const uint8_t* tables;
    const uint8_t* profile_id;
    const double* job;
    uint8_t* status;              // in: sweep status; out: final (incl. exhausted)
    chase_totals_t* per_trace;    // may be null
    double* block_sums;           // [grid][n_eta][8]
    chase_diag_t* diag;
    chase_sum_t* sum_direct;      // one-block launch: the block writes the per-eta sums itself
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

size_t sweep_smem_bytes(int tables_bytes, int T, int elem_size, int mode);
int sweep_stage_bytes(int elem_size);
int64_t finalize_grid(int64_t n_traces);

cudaError_t launch_upload(const void* host, size_t bytes, void* dst, cudaStream_t s, chase_diag_t* reset = nullptr);
cudaError_t launch_fit(const FitParams& p, cudaStream_t s);
// the specialised headline kernel applies (fp32, aligned, one eta, no forecast in/out); it also
// runs decision periods in place (p.period > 1), every other period path is forecast-first
bool headline_eligible(int mode, bool f64, bool aligned, const SweepParams& p);
cudaError_t launch_sweep(int mode, bool f64, bool aligned, const SweepParams& p, cudaStream_t s);
cudaError_t launch_plan(const PlanParams& p, cudaStream_t s);
// rolling refit (refit_stride >= 1): per-phase tables, then one thread per (trace, origin)
int roll_phase_doubles(int T, int L);
// forecast-evaluation sweep: walk-forward MAPE of the fit-once model and of persistence
// fc_in != null: the predictions are read from fc_in [n][ld_fin] (the SVR forecaster's)
cudaError_t launch_mape(const void* traces, bool f64, int64_t ld, int64_t n_traces, int N, int L, int T, int phase0,
                        const double* phase, const double* records, const double* fc_in, int64_t ld_fin, double* out,
                        int32_t* status, cudaStream_t s);
// epsilon-SVR forecaster (f2): per-trace SMO fit (warp per trace) into models [n][kSvrModelDoubles],
// then the per-period forecasts into forecast [n][ld_f]; records[.][5] is the status
constexpr int kSvrModelDoubles = 268;
cudaError_t launch_svr(const void* traces, bool f64, int64_t ld, int64_t n_traces, int N, int L, int T, int phase0,
                       int P, double C, double eps, double gamma, double tol, int max_iter, const double* phase,
                       double* records, double* models, double* forecast, int64_t ld_f, cudaStream_t s);
// timeline / audit rows of a planned replay, one warp per selected trace
cudaError_t launch_timeline(const void* traces, bool f64, int64_t ld, int64_t n_traces, int N, int L, int P,
                            int n_prof, double delta, const uint8_t* choice, int64_t ld_c, const double* forecast,
                            int64_t ld_f, const uint8_t* tables, const uint8_t* profile_id, const double* job,
                            const int64_t* ids, int64_t m, double* rows, double* summary, cudaStream_t s);
// SPEC --count-profiling: the profiling run's {time, energy, carbon} per trace
cudaError_t launch_profiling(const void* traces, bool f64, int64_t ld, int64_t n, int L, double delta,
                             const uint8_t* tables, int n_prof, const uint8_t* profile_id, double* out, cudaStream_t s);
// per-limit Eq. 6 cost vectors behind each period's decision (audit)
cudaError_t launch_period_costs(const double* forecast, int64_t ld_f, int64_t n_traces, int W, int P, int ld_k,
                                int n_prof, const uint8_t* tables, const uint8_t* profile_id, const double* max_ci,
                                double max_ci_fixed, const int64_t* ids, int64_t m, double* costs, cudaStream_t s);
// decision periods (period_steps > 1): one thread per (trace, period) writes the period's decision forecast
cudaError_t launch_periods(const void* traces, bool f64, int64_t ld, int64_t n_traces, int N, int L, int T, int phase0,
                           int P, const double* phase, const double* records, double* forecast, int64_t ld_f,
                           cudaStream_t s);
// rolling refit fused into the sweep (k2_roll.cuh): fp32, aligned, one eta, no forecast output, L <= 64,
// T <= 2048; returns false (nothing launched) when the shape is not covered
bool roll_fused_eligible(const SweepParams& p);
bool sweep_in_place(bool f64, bool aligned, int L, int T, int n_prof, int n_eta, bool rolling, bool periods,
                    int tables_bytes);
cudaError_t launch_roll_fused(const SweepParams& p, cudaStream_t s);
cudaError_t launch_rolling(const void* traces, bool f64, int64_t ld, int64_t n_traces, int N, int L, int T, int phase0,
                           int R, double ridge, double tol, const double* phase, double* ptab, double* records,
                           double max_ci_fixed, double* forecast, int64_t ld_f, cudaStream_t s);
// per-trace totals + fixed-order per-GPU sums (+ invalid-trace fix-up)
cudaError_t launch_finalize(const FinalizeParams& p, const int64_t* bad_list, chase_sum_t* sum, uint8_t* choice,
                            int64_t ld_c, int n_eta_choice, double* forecast, int64_t ld_f, chase_diag_t* diag,
                            cudaStream_t s);
cudaError_t launch_fixup(const uint8_t* status, const int64_t* bad_list, int64_t n_traces, uint8_t* choice,
                         int64_t ld_c, int64_t W, int n_eta_choice, double* forecast, int64_t ld_f,
                         chase_diag_t* diag, cudaStream_t s);
cudaError_t launch_diag_reset(chase_diag_t* diag, cudaStream_t s);
// chase_sweep_host: fold a chunk's diagnostics into acc (c0 = its first trace; c0 == 0 resets
// acc first); c0 < 0 copies acc back into `chunk` (the workspace's diagnostics)
cudaError_t launch_diag_merge(chase_diag_t* acc, chase_diag_t* chunk, int64_t c0, cudaStream_t s);
cudaError_t launch_diag_merge_eta(chase_diag_t* acc, const uint8_t* ws, size_t slice, size_t diag_off,
                                  size_t status_off, int n_eta, int64_t n, cudaStream_t s);
cudaError_t launch_accumulate(double* acc, const double* add, int n, cudaStream_t s);
uint64_t kernel_launches();

}  // namespace chase
