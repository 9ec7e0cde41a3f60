/*
 * chase.h — C ABI of libchase.so, the B200-native batched trace-replay
 * planner for Chase (arXiv 2303.02508, "carbon-aware DNN training").
 *
 * For every carbon-intensity trace and every decision window the planner
 *   (1) fits the paper's one-lag forecaster on the history before job start
 *       and predicts the window's intensity      (§3.1, Eq. 1-2),
 *   (2) takes the argmin of the eta-weighted carbon/time cost over the
 *       profiled power-limit table                 (§3.2, Eq. 6),
 *   (3) replays the chosen limits against the true intensity, accumulating
 *       time, energy and carbon, plus a max-power baseline (P:93-96, P:126,
 *       P:185).
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n; Q-numbers are the
 * readings of DESIGN.md §3.
 *
 * Conventions (all entry points)
 *  - Device pointers ("d_" prefix) are caller-owned CUDA device memory;
 *    host pointers are read during the call only and never retained.
 *  - Every call is asynchronous on `stream` (a cudaStream_t passed as void*;
 *    NULL = legacy default stream).  CHASE_OK means "validated and enqueued".
 *  - Argument/config violations are detected on the host before anything is
 *    enqueued and return CHASE_ERR_INVALID; chase_last_error() explains.
 *  - Data-dependent problems (a negative or non-finite intensity, MaxCI <= 0,
 *    an unsolvable fit, trace exhaustion) are recorded per trace in
 *    chase_totals_t.status and in the workspace diagnostics; read them with
 *    chase_diag_read().  Choices of invalid traces are 0xFF, their forecasts
 *    NaN, their totals zero, and they are excluded from chase_sum_t.
 *  - The library allocates no device memory: scratch lives in the caller's
 *    workspace (chase_workspace_bytes), which must stay untouched until the
 *    enqueued work completes.  No global device state is kept.
 *  - Thread-safety: calls on different workspaces may run concurrently.
 */
#ifndef CHASE_H
#define CHASE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CHASE_MAX_LIMITS   32   /* rows of a power profile                    */
#define CHASE_MAX_ETA      16   /* eta values per call                        */
#define CHASE_MAX_PROFILES  8   /* distinct profiles (per-trace model shapes) */
#define CHASE_MAX_PAIRS    32   /* n_profiles * n_eta                          */

typedef enum {
    CHASE_OK = 0,
    CHASE_ERR_INVALID = 2,          /* S:494 input/validation error            */
    CHASE_ERR_TRACE_EXHAUSTED = 3,  /* S:399, S:436 (per-trace status only)    */
    CHASE_ERR_DATA = 4,             /* S:29 negative / non-finite intensity    */
    CHASE_ERR_MAXCI = 5,            /* S:292 MaxCarbonIntensity must be > 0    */
    CHASE_ERR_FIT = 6,              /* S:135 rank-deficient after ridge        */
    CHASE_ERR_CHOICE = 7,           /* chase_replay: choice index out of range */
    CHASE_ERR_ZERO_ACTUAL = 8,      /* chase_forecast_mape: a zero intensity */
    CHASE_ERR_CUDA = 10,
    CHASE_ERR_NCCL = 11,
    CHASE_ERR_WORKSPACE = 12        /* workspace NULL, misaligned or too small */
} chase_status_t;

typedef enum { CHASE_F32 = 0, CHASE_F64 = 1 } chase_dtype_t;

/* D1 CarbonTrace: row-major [n_traces][ld] DEVICE matrix of
 * intensities in g/kWh; trace i step t at data[i*ld + t].  Step t = 0 is the
 * first history point; the job starts at step s0 = history_len, so
 * the decision windows are w = s0 .. n_steps-1 and W = n_steps - s0.
 *   ld*sizeof(elem) % 16 == 0 and data 16-byte aligned (bulk-copy rows);
 *   interval_s = Delta > 0 with 86400 % Delta == 0;
 *   phase0 = (start_time mod 86400)/Delta, the UTC-midnight phase of step 0
 *   (Q3). */
typedef struct {
    const void* data;
    int32_t dtype;               /* chase_dtype_t */
    int32_t interval_s;
    int64_t n_traces, n_steps, ld;
    int32_t phase0;
    int32_t reserved;
} chase_traces_t;

/* §3.1 forecaster (Eq. 1-2): least squares on (sin_time, cos_time, CI(t-1)). */
typedef struct {
    int32_t steps_per_day;       /* T = 86400/interval_s (Eq. 2)                   */
    int32_t history_len;         /* L: points before job start, L-1 >= 4 rows */
    int32_t refit_stride;        /* 0 = fit once at job start.
                                    R >= 1 = rolling refit: window w uses the model
                                    fitted on the L points before its origin
                                    r = s0 + R*floor((w-s0)/R) (Q1);
                                    MaxCI stays the job-start value.  The
                                    workspace then also holds an f64 forecast
                                    scratch of round_up(W,2) per trace.         */
    int32_t period_steps;        /* <= 1: a decision every trace step.
                                    P > 1: one decision per period of P steps
                                    (P:78-79), on the mean of the
                                    recursive forecast over the period
                                    (S:158-166); d_forecast then holds
                                    each window's decision value.  Needs
                                    refit_stride == 0; uses the same forecast
                                    scratch as the rolling refit.               */
    double  ridge_lambda;        /* 1e-8                                   */
    double  singular_tol;        /* 1e-12: Cholesky pivot <= tol*(L-1) -> ridge (Q6) */
    int32_t forecaster;          /* CHASE_FC_LINEAR (0): Eq. 1 least squares (§3.1).
                                    CHASE_FC_SVR (1): the epsilon-SVR with an RBF
                                    kernel on the same three features, z-scored on
                                    the fit window (Table 1's best model, P:162,
                                    P:171; SPEC fit_svr S:140-148), solved by SMO
                                    with second-order working-set selection
                                    (DESIGN §6.8).  Needs refit_stride == 0,
                                    history_len <= 64 and steps_per_day <= 8192;
                                    combines with period_steps.                  */
    int32_t svr_max_iter;        /* SMO iteration cap (>= 0; 10000 in the binding) */
    double  svr_C;               /* box constraint C > 0 (1.0)                     */
    double  svr_eps;             /* epsilon-tube half width >= 0, in z-units (0.1) */
    double  svr_gamma;           /* RBF gamma >= 0; 0 = 1/(#non-constant features)  */
    double  svr_tol;             /* KKT stopping tolerance > 0 (1e-3)              */
} chase_forecast_cfg_t;

enum { CHASE_FC_LINEAR = 0, CHASE_FC_SVR = 1 };

/* D2 PowerProfile, HOST memory, copied during the call.
 * limit_w strictly increasing, n_limits in [2, 32], avg_power_w > 0 and
 * <= 1.05*limit_w, throughput_sps > 0. */
typedef struct {
    int32_t n_limits;
    int32_t reserved;
    const int32_t* limit_w;
    const double* avg_power_w;
    const double* throughput_sps;
} chase_profile_t;

/* Eq. 6 constants, HOST memory. */
typedef struct {
    const double* eta;           /* n_eta values in [0, 1]                         */
    int32_t n_eta;               /* 1 .. 16                                        */
    int32_t reserved;
    double max_power_w;          /* > 0: fixed, >= every profile's largest limit;
                                    <= 0: each profile's largest limit     */
    double max_ci;               /* > 0: fixed MaxCarbonIntensity; <= 0: per trace,
                                    the max of its L history points  */
} chase_cost_cfg_t;

/* D9 per (trace, eta) result, 64 bytes. */
typedef struct {
    double time_s, energy_j, carbon_g, samples;
    double base_time_s, base_energy_j, base_carbon_g;  /* max-limit baseline */
    int32_t completion_window;   /* absolute step w* where the job completed, or -1 */
    int32_t status;              /* chase_status_t: 0, 3, 4, 5, 6 or 7             */
} chase_totals_t;

/* Per-eta sum over the status-0 traces of one call (one GPU's shard). */
typedef struct {
    double time_s, energy_j, carbon_g, samples;
    double base_time_s, base_energy_j, base_carbon_g;
    double n_ok;
} chase_sum_t;

/* Workspace diagnostics (read with chase_diag_read). */
typedef struct {
    int64_t first_bad_trace;     /* lowest trace index with status 4..7, or -1 */
    int32_t first_bad_status;
    int32_t reserved;
    uint64_t n_bad;              /* traces with status 4..7                     */
    uint64_t n_exhausted;        /* traces with status 3                        */
    uint64_t n_slow_windows;     /* (window, eta) decisions that took the
                                    canonical K-way Eq. 6 path (§8(a) a5)      */
    uint64_t kernel_path;        /* which sweep kernels the call ran (bits):
                                    CHASE_PATH_*, for tests and the bench      */
    uint64_t n_seq_periods;      /* decision periods (headline kernel) whose
                                    horizon ran step by step because the
                                    closed form declined         */
    uint64_t reserved2;
} chase_diag_t;

#define CHASE_PATH_HEADLINE   1u   /* sweep_fast_kernel<0>: fp32, aligned, one eta, no forecast output */
#define CHASE_PATH_H_PERIODS  2u   /* sweep_fast_kernel<PM > 0>: decision periods in the headline kernel */
#define CHASE_PATH_GENERAL    4u   /* sweep_kernel: every other shape (f64, multi-eta, forecast output) */
#define CHASE_PATH_FC_IN      8u   /* sweep_kernel reading precomputed forecasts (SVR, periods, rolling) */
#define CHASE_PATH_ROLL_FUSED 16u  /* rolling refit fused into the sweep (sliding moments) */

/* Bytes of device workspace needed by any entry point for these shapes
 * (n_profiles, n_eta >= 1).  Returns 0 on invalid arguments. */
size_t chase_workspace_bytes(const chase_traces_t* traces, const chase_forecast_cfg_t* fcfg,
                             int32_t n_profiles, int32_t n_eta);

/* §3.1 forecaster: fit Eq. 1 on the L history points of every trace (fit once,
 * or rolling per refit_stride) and write the one-step forecast of every
 * window, using the last OBSERVED intensity as the lag:
 *   d_forecast [n_traces][ld_f] f64, window w at column w - s0 (ld_f >= W);
 *   d_max_ci   [n_traces] f64 or NULL: max of the L history points;
 *   d_models   [n_traces][8] f64 or NULL: job-start model
 *              {c0, w_sin, w_cos, w_lag, max_ci, status, ridge, kind}
 *              with forecast = max(0, ((c0 + w_sin*S) + w_cos*C) + w_lag*lag).
 *              Must be NULL with the SVR forecaster (its dual lives in the
 *              workspace). */
chase_status_t chase_fit_forecast(const chase_traces_t* traces, const chase_forecast_cfg_t* fcfg,
                                  double* d_forecast, int64_t ld_f, double* d_max_ci,
                                  double* d_models, void* d_ws, size_t ws_bytes, void* stream);

/* Eq. 6 argmin for given forecasts (e.g. chase_fit_forecast's,
 * or the true trace for the oracle-forecast mode of S:434):
 *   d_forecast  [n_traces][ld_f] f64 (>= 0, finite; else the choice is 0xFF);
 *   d_profile_id [n_traces] u8 or NULL (all profile 0);
 *   d_max_ci    [n_traces] f64, required when cost->max_ci <= 0;
 *   d_choice    [n_eta][n_traces][ld_c] u8 out, ld_c >= round_up(W, 16) and a
 *               multiple of 16; bytes [W, round_up(W,16)) of a row are scratch.
 * Choice = first k minimising ((eta*P_k)*chat + ((1-eta)*Pmax)*MaxCI)/Thr_k in
 * IEEE fp64 (lowest limit on ties).  Bit-exact with that rule. */
chase_status_t chase_plan_power_limits(const double* d_forecast, int64_t n_traces, int64_t W,
                                       int64_t ld_f, const chase_profile_t* profiles,
                                       int32_t n_profiles, const uint8_t* d_profile_id,
                                       const chase_cost_cfg_t* cost, const double* d_max_ci,
                                       uint8_t* d_choice, int64_t ld_c,
                                       void* d_ws, size_t ws_bytes, void* stream);

/* Fixed-work replay: per (trace, eta) run the job of
 * d_job_samples[i] samples (<= 0 or NULL: run to the trace end) at the chosen
 * limits, stepwise carbon, pro-rata last window; baseline =
 * the largest limit.
 *   d_per_trace [n_eta][n_traces] or NULL;  d_sum [n_eta] (required). */
chase_status_t chase_replay(const chase_traces_t* traces, int32_t history_len,
                            const uint8_t* d_choice, int64_t ld_c, int32_t n_eta,
                            const chase_profile_t* profiles, int32_t n_profiles,
                            const uint8_t* d_profile_id, const double* d_job_samples,
                            chase_totals_t* d_per_trace, chase_sum_t* d_sum,
                            void* d_ws, size_t ws_bytes, void* stream);

/* The fused planner: fit + predict + Eq. 6 argmin + replay for every trace,
 * window and eta in one pass over the traces (the headline path).  Outputs
 * as above; d_choice / d_forecast / d_per_trace may be NULL.  d_sum is this
 * GPU's per-eta sum; for a multi-GPU sweep the caller all-reduces it (NCCL,
 * e.g. torch.distributed.all_reduce) — nccl_comm must be NULL.
 * A multi-eta call over at most 2368 fp32 traces with no forecast output (and
 * neither rolling refit nor SVR) runs as n_eta concurrent one-eta sweeps on
 * streams forked from and joined back into `stream`, each in its own slice of
 * d_ws (chase_workspace_bytes sizes for it); results are the same. */
chase_status_t chase_sweep(const chase_traces_t* traces, const chase_forecast_cfg_t* fcfg,
                           const chase_profile_t* profiles, int32_t n_profiles,
                           const uint8_t* d_profile_id, const chase_cost_cfg_t* cost,
                           const double* d_job_samples,
                           uint8_t* d_choice, int64_t ld_c, double* d_forecast, int64_t ld_f,
                           chase_totals_t* d_per_trace, chase_sum_t* d_sum,
                           void* nccl_comm, void* d_ws, size_t ws_bytes, void* stream);

/* Forecast-evaluation sweep (the walk-forward Table 1 experiment, P:159-161;
 * SPEC evaluate_models S:175-184, mape S:167-174): the Eq. 1 model fitted once
 * on the L history points predicts every window w = L..n_steps-1 from the TRUE
 * previous intensity (the first seeded by the last history point), and the
 * MAPE of those predictions and of persistence (p(w) = c[w-1]) is written per
 * trace:
 *   d_mape   [n_traces][2] f64 out: {MAPE linear, MAPE persistence} in percent,
 *            NaN where undefined;
 *   d_status [n_traces] int32 out or NULL: 0, 4 (negative / non-finite value),
 *            6 (fit failed) or 8 (a zero intensity: MAPE undefined).
 * fcfg->forecaster selects the model (CHASE_FC_SVR: the first column is the
 * SVR's MAPE, Table 1's comparison).  Needs refit_stride == 0,
 * period_steps <= 1 and steps_per_day <= 2048.  Predictions are bit-identical to the oracle's; the MAPE
 * sums agree to <= 1e-9 relative. */
chase_status_t chase_forecast_mape(const chase_traces_t* traces, const chase_forecast_cfg_t* fcfg, double* d_mape,
                                   int32_t* d_status, void* d_ws, size_t ws_bytes, void* stream);

/* Timeline / audit rows of a planned replay (SPEC emit_timeline S:413-421;
 * Figure 1/2) for m selected traces: one row per decision period
 * (period_steps <= 1: per window) from the job start,
 *   {period_start (absolute step), forecast_ci, actual_mean_ci, chosen_limit_w,
 *    avg_power_w, samples_done, energy_j, carbon_g}
 * with the fixed-work replay split by period: full windows count in full, the
 * completion window pro rata (its samples are J - samples before, so a row set
 * sums to J), later windows contribute nothing.
 *   d_choice    [n_traces][ld_c] u8 of ONE eta (e.g. chase_sweep's first eta
 *               plane), or NULL for the max-limit baseline;
 *   d_forecast  [n_traces][ld_f] f64 decision forecasts or NULL (rows get NaN);
 *   d_trace_ids [m] int64 trace indices, or NULL for traces 0..m-1; a row
 *               whose id lies outside [0, n_traces) is written as NaN (rows
 *               and summary), nothing outside the inputs is read;
 *   d_rows      [m][ceil(W/P)][8] f64 out, 16-byte aligned (rows leave by TMA bulk stores);
 *   d_summary   [m][4] f64 out or NULL: Eq. 3 next to the stepwise
 *               integration over the job's run:
 *               {stepwise carbon g, TTA*AvgPower*AvgCI carbon g, AvgPower W,
 *                time-weighted AvgCI g/kWh} (oracle_job_summary, <= 1e-9).
 * Rows match oracle_timeline (bit-identical for the dyadic synthetic inputs). */
chase_status_t chase_timeline(const chase_traces_t* traces, int32_t history_len, int32_t period_steps,
                              const uint8_t* d_choice, int64_t ld_c, const double* d_forecast, int64_t ld_f,
                              const chase_profile_t* profiles, int32_t n_profiles, const uint8_t* d_profile_id,
                              const double* d_job_samples, const int64_t* d_trace_ids, int64_t m, double* d_rows,
                              double* d_summary, void* d_ws, size_t ws_bytes, void* stream);

/* SPEC --count-profiling (DESIGN Q33): the cost of profiling the
 * power-limit table before the job, one trace step per limit in increasing
 * order over steps history_len-K .. history_len-1, each at that limit's
 * average power:
 *   d_out [n_traces][3] f64 out: {time s, energy J, carbon g}, to add to a
 *         replay's totals (chase_sweep's per-trace totals exclude profiling).
 * history_len >= the largest n_limits.  Workspace: chase_workspace_bytes(
 * traces, NULL, n_profiles, 1).  Bit-identical to oracle_profiling_overhead. */
chase_status_t chase_profiling_overhead(const chase_traces_t* traces, int32_t history_len,
                                        const chase_profile_t* profiles, int32_t n_profiles,
                                        const uint8_t* d_profile_id, double* d_out, void* d_ws, size_t ws_bytes,
                                        void* stream);

/* Per-limit cost vectors behind the decisions (SPEC PeriodDecision S:296-297;
 * Eq. 6), an audit output for m selected traces: for period j
 * (windows s0 + jP .. , period_steps <= 1: per window) and limit k,
 *   cost_k = ((eta*P_k)*chat + ((1-eta)*Pmax)*MaxCI) / Thr_k
 * (the canonical rule's operations, without the 1/3.6e6 of Eq. 6, Q12) at the
 * period's decision value chat = d_forecast[i][jP] (as chase_fit_forecast /
 * chase_sweep write it), eta = cost->eta[0], Pmax and MaxCI as chase_sweep
 * (d_max_ci: chase_fit_forecast's, required when cost->max_ci <= 0).  The
 * chosen limit is the first minimum of its row.
 *   d_costs [m][ceil(W/P)][ld_k] f64 out, ld_k >= the largest n_limits; the
 *           entries k >= the trace's n_limits are NaN, as are all entries of a
 *           NaN decision value (an invalid trace) and of a trace id outside
 *           [0, n_traces) in d_trace_ids.
 * Workspace: chase_workspace_bytes(traces, NULL, n_profiles, 1). */
chase_status_t chase_period_costs(const double* d_forecast, int64_t n_traces, int64_t W, int64_t ld_f,
                                  int32_t period_steps, const chase_profile_t* profiles, int32_t n_profiles,
                                  const uint8_t* d_profile_id, const chase_cost_cfg_t* cost, const double* d_max_ci,
                                  const int64_t* d_trace_ids, int64_t m, double* d_costs, int32_t ld_k, void* d_ws,
                                  size_t ws_bytes, void* stream);

/* End-to-end variant with HOST inputs (the public call a user makes when the
 * traces live in host memory; bench.py's "e2e" figure): streams chunks of
 * `chunk_traces` traces through a double-buffered device staging area with
 * the host->device copies on a second stream overlapping the fused kernels
 * of the previous chunk, and returns the per-eta sums in HOST memory.
 *   h_traces->data, h_profile_id, h_job_samples: host memory (pin it, e.g.
 *   cudaHostAlloc / torch pin_memory, for copy/compute overlap);
 *   d_staging: chase_sweep_host_staging_bytes() bytes of device memory;
 *   d_ws: chase_workspace_bytes() for a descriptor with n_traces = chunk_traces.
 * Synchronous: returns after h_sum is written.  Afterwards chase_diag_read(d_ws)
 * reports the whole call: counts summed over the chunks, first_bad_trace as
 * an index into h_traces. */
size_t chase_sweep_host_staging_bytes(const chase_traces_t* h_traces, int64_t chunk_traces, int32_t n_eta);
chase_status_t chase_sweep_host(const chase_traces_t* h_traces, const chase_forecast_cfg_t* fcfg,
                                const chase_profile_t* profiles, int32_t n_profiles,
                                const uint8_t* h_profile_id, const chase_cost_cfg_t* cost,
                                const double* h_job_samples, int64_t chunk_traces, chase_sum_t* h_sum,
                                void* d_staging, size_t staging_bytes, void* d_ws, size_t ws_bytes,
                                void* stream);

/* Number of kernels this thread has launched through the library so far
 * (bench.py reports the count inside its timed region as gpu_launches). */
uint64_t chase_kernel_launches(void);

/* Optional timing hook: when both are non-NULL cudaEvent_t handles, the next
 * calls record `start` / `stop` on their stream immediately around the
 * dominant kernel (the fused sweep, the replay or the plan kernel; with
 * refit_stride >= 1, the rolling refit kernel), so the caller can time that
 * kernel alone with CUDA events.  Pass NULLs to clear.
 * Thread-local. */
void chase_set_kernel_events(void* start, void* stop);

/* Copy the workspace diagnostics of the last call to the host (synchronises
 * `stream`). */
chase_status_t chase_diag_read(const void* d_ws, chase_diag_t* out, void* stream);

/* Thread-local text for the last CHASE_ERR_* returned on this thread. */
const char* chase_last_error(void);

/* Library build string (arch, version). */
const char* chase_version(void);

#ifdef __cplusplus
}
#endif
#endif
