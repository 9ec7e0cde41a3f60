// rolling.cuh — rolling refit forecaster (DESIGN Q1), included
// by kernels.cu inside its anonymous namespace.
//
// refit_stride R >= 1: window w is predicted by the model fitted on the L
// points before its refit origin r = s0 + R*floor((w - s0)/R) (rows
// t = r-L+1 .. r-1; P:67's "one day prior" applied at every origin),
// with MaxCI frozen at job start.  One thread per (trace, origin): the fit is
// oracle_fit's exact operation sequence (sequential two-pass moments, z-scored
// Gram, Cholesky with ridge fallback, un-standardisation), so forecasts are
// bit-identical to the oracle and choices stay bit-exact.
//
// The phase columns (sin, cos) of an origin's rows depend only on the phase
// rho = (phase0 + r - L) mod T of its first history point, so their means,
// sigmas, z-scores and the phase-only Gram entries G00, G10, G11 are computed
// once per rho (rolling_phase_kernel) with the very same sequential
// operations and read back per origin; each accumulator is its own sequential
// sum over rows, so splitting them off changes no rounding.  Per origin this
// leaves 2(L-1) divides (lag and target z-scores) instead of 4(L-1).

// One phase_record (fit.cuh) per first-point phase rho.
__host__ __device__ inline int roll_phase_stride(int L) { return phase_stride(L); }

__global__ void rolling_phase_kernel(const double* __restrict__ S, const double* __restrict__ Cc, int T, int L,
                                     double* __restrict__ tab) {
    const int rho = blockIdx.x * blockDim.x + threadIdx.x;
    if (rho >= T) return;
    phase_record(S, Cc, T, L, rho, tab + (int64_t)rho * phase_stride(L));
}

struct RollParams {
    const void* traces;
    int64_t ld, n_traces;
    int32_t N, L, T, phase0, R, n_orig;   // n_orig = ceil(W / R)
    double ridge, tol;
    const double* phase;                  // S[T], C[T] (workspace tables blob)
    const double* ptab;                   // rolling_phase_kernel output [T][stride]
    double* records;                      // [n][16]: status written (6) when an origin's fit fails
    double max_ci_fixed;
    double* forecast;                     // [n][ld_f]
    int64_t ld_f;
};

// Fit of one origin (history h[0..L), first-point phase rho): model in
// (c0, w[3]); returns the status (0 or CHASE_ERR_FIT; bad values are left to
// the sweep's validation of the whole trace).
template <typename E>
__device__ int rolling_fit(const E* h, int L, int T, int rho, const RollParams& p, double& c0, double* w) {
    double rec[kRecDoubles];
    fit_phase<E>(h, L, T, rho, p.ptab + (int64_t)rho * phase_stride(L), p.phase, p.phase + T, p.ridge, p.tol, rec);
    c0 = rec[0];
    w[0] = rec[1];
    w[1] = rec[2];
    w[2] = rec[3];
    return (int)rec[5] == CHASE_ERR_FIT ? CHASE_ERR_FIT : 0;
}

template <typename E>
#ifndef CHASE_ROLL_MINB
#define CHASE_ROLL_MINB 8  // 8 CTAs of 128 per SM (<= 64 registers): occupancy hides the fit's latency chains
#endif
__global__ void __launch_bounds__(128, CHASE_ROLL_MINB) rolling_forecast_kernel(const __grid_constant__ RollParams p) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= p.n_traces * (int64_t)p.n_orig) return;
    const int64_t i = idx / p.n_orig;
    const int o = (int)(idx - i * p.n_orig);
    const int L = p.L, T = p.T, s0 = L;
    const int r = s0 + o * p.R;
    const E* row = reinterpret_cast<const E*>(p.traces) + i * p.ld;
    const int rho = (int)(((int64_t)p.phase0 + r - L) % T);
    double c0 = 0.0, w[3];
    const int st = rolling_fit<E>(row + (r - L), L, T, rho, p, c0, w);
    if (st != 0) {
        // P:184 / S:292 precedence (DESIGN Q25): MaxCI <= 0 (5) outranks a failed fit (6);
        // a bad value anywhere (4) is found by the sweep's validation
        double* rec = p.records + i * kRecDoubles;
        const double maxci = p.max_ci_fixed > 0.0 ? p.max_ci_fixed : rec[4];
        if (rec[5] == 0.0 && maxci > 0.0) rec[5] = (double)CHASE_ERR_FIT;
    }
    const int w_end = min(r + p.R, p.N);
    const double* S = p.phase;
    const double* C = p.phase + T;
    int ph = (int)(((int64_t)p.phase0 + r) % T);
    double* out = p.forecast + i * p.ld_f + (r - s0);
    for (int wv = r; wv < w_end; ++wv) {
        // Eq. 1 with the observed lag, oracle_predict's rounding order
        const double A = __dadd_rn(__dadd_rn(c0, __dmul_rn(w[0], S[ph])), __dmul_rn(w[1], C[ph]));
        const double pr = __dadd_rn(A, __dmul_rn(w[2], (double)row[wv - 1]));
        out[wv - r] = pr > 0.0 ? pr : 0.0;
        ph = ph + 1 == T ? 0 : ph + 1;
    }
}

// ------------------------------------------------------------------ decision periods
// period_steps P > 1 ("the period between forecasts and power
// limit adjustments"): at each period start b = s0 + jP the fit-once model
// forecasts recursively over n = min(P, N - b) steps from the last observed
// value (SPEC forecast_horizon: prediction k is the lag of prediction k+1,
// clamped at 0), and Eq. 6 decides on the mean of those n forecasts.
// One thread per (trace, period) writes that decision value to the period's n
// windows; the FIN sweep then takes the same decision for each of them.
// oracle_plan_trace's operation order throughout (bit-identical).
struct PeriodParams {
    const void* traces;
    int64_t ld, n_traces;
    int32_t N, L, T, phase0, P, n_per;   // n_per = ceil(W / P)
    const double* phase;                 // S[T], C[T]
    const double* records;               // fit-once models [n][16]
    double* forecast;                    // [n][ld_f]: the decision value of every window
    int64_t ld_f;
};

template <typename E>
__global__ void __launch_bounds__(128) period_forecast_kernel(const __grid_constant__ PeriodParams p) {
    // one warp per (trace, group of 32 periods): lane j forecasts period 32g + j, then the
    // warp writes the group's decision values with coalesced stores (one period at a time)
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int n_grp = (p.n_per + 31) >> 5;
    if (wid >= p.n_traces * (int64_t)n_grp) return;
    const int64_t i = wid / n_grp;
    const int g = (int)(wid - i * n_grp);
    const int s0 = p.L, T = p.T, W = p.N - p.L;
    const int j = 32 * g + lane;
    const E* row = reinterpret_cast<const E*>(p.traces) + i * p.ld;
    const double* rec = p.records + i * kRecDoubles;
    const double c0 = rec[0], ws = rec[1], wc = rec[2], wl = rec[3];
    const double* S = p.phase;
    const double* C = p.phase + T;
    double chat = 0.0;
    if (j < p.n_per) {
        const int b = s0 + j * p.P;
        const int n = min(p.P, p.N - b);
        int ph = (int)(((int64_t)p.phase0 + b) % T);
        double prev = (double)row[b - 1], sum = 0.0;
        for (int k = 0; k < n; ++k) {
            const double A = __dadd_rn(__dadd_rn(c0, __dmul_rn(ws, S[ph])), __dmul_rn(wc, C[ph]));
            const double pr = __dadd_rn(A, __dmul_rn(wl, prev));
            const double f = pr > 0.0 ? pr : 0.0;
            sum = __dadd_rn(sum, f);
            prev = f;
            ph = ph + 1 == T ? 0 : ph + 1;
        }
        chat = __ddiv_rn(sum, (double)n);
    }
    double* out = p.forecast + i * p.ld_f;
    const int jmax = min(32, p.n_per - 32 * g);
    for (int jj = 0; jj < jmax; ++jj) {
        const double v = __shfl_sync(kFull, chat, jj);
        const int b = (32 * g + jj) * p.P;
        const int n = min(p.P, W - b);
        for (int k = lane; k < n; k += 32) out[b + k] = v;
    }
}
