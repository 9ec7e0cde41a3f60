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

// Per-rho record: [mu0, mu1, sg0, sg1, G00, G10, G11, ok] then z0[1..n], z1[1..n].
__host__ __device__ inline int roll_phase_stride(int L) { return 8 + 2 * (L - 1); }

__global__ void rolling_phase_kernel(const double* __restrict__ S, const double* __restrict__ Cc, int T, int L,
                                     double* __restrict__ tab) {
    const int rho = blockIdx.x * blockDim.x + threadIdx.x;
    if (rho >= T) return;
    const int n = L - 1;
    const double dn = (double)n;
    double* out = tab + (int64_t)rho * roll_phase_stride(L);
    double s0 = 0.0, s1 = 0.0;
    int ph = (rho + 1) % T;
    for (int i = 1; i <= n; ++i) {
        s0 = __dadd_rn(s0, S[ph]);
        s1 = __dadd_rn(s1, Cc[ph]);
        ph = ph + 1 == T ? 0 : ph + 1;
    }
    const double mu0 = __ddiv_rn(s0, dn), mu1 = __ddiv_rn(s1, dn);
    double q0 = 0.0, q1 = 0.0;
    ph = (rho + 1) % T;
    for (int i = 1; i <= n; ++i) {
        const double d0 = __dsub_rn(S[ph], mu0), d1 = __dsub_rn(Cc[ph], mu1);
        q0 = __dadd_rn(q0, __dmul_rn(d0, d0));
        q1 = __dadd_rn(q1, __dmul_rn(d1, d1));
        ph = ph + 1 == T ? 0 : ph + 1;
    }
    const double sg0 = __dsqrt_rn(__ddiv_rn(q0, dn)), sg1 = __dsqrt_rn(__ddiv_rn(q1, dn));
    const bool ok = sg0 > 0.0 && sg1 > 0.0;
    double G00 = 0.0, G10 = 0.0, G11 = 0.0;
    double* z0 = out + 8;
    double* z1 = z0 + n;
    ph = (rho + 1) % T;
    for (int i = 1; i <= n; ++i) {
        const double a = ok ? __ddiv_rn(__dsub_rn(S[ph], mu0), sg0) : 0.0;
        const double b = ok ? __ddiv_rn(__dsub_rn(Cc[ph], mu1), sg1) : 0.0;
        z0[i - 1] = a;
        z1[i - 1] = b;
        G00 = __dadd_rn(G00, __dmul_rn(a, a));
        G10 = __dadd_rn(G10, __dmul_rn(b, a));
        G11 = __dadd_rn(G11, __dmul_rn(b, b));
        ph = ph + 1 == T ? 0 : ph + 1;
    }
    out[0] = mu0;
    out[1] = mu1;
    out[2] = sg0;
    out[3] = sg1;
    out[4] = G00;
    out[5] = G10;
    out[6] = G11;
    out[7] = ok ? 1.0 : 0.0;
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
// (c0, w[3]); returns the status (0 or CHASE_ERR_FIT).
template <typename E>
__device__ int rolling_fit(const E* h, int L, int T, int rho, const RollParams& p, double& c0, double* w) {
    const int n = L - 1;
    const double dn = (double)n;
    w[0] = w[1] = w[2] = 0.0;
    bool constant = true;
    for (int i = 2; i <= n; ++i)
        if ((double)h[i] != (double)h[1]) { constant = false; break; }
    if (constant) {  // F2: intercept-only model
        c0 = (double)h[1];
        return 0;
    }
    const double* pt = p.ptab + (int64_t)rho * roll_phase_stride(L);
    double sl = 0.0, sy = 0.0;
    for (int i = 1; i <= n; ++i) {
        sl = __dadd_rn(sl, (double)h[i - 1]);
        sy = __dadd_rn(sy, (double)h[i]);
    }
    const double mu2 = __ddiv_rn(sl, dn), mu3 = __ddiv_rn(sy, dn);
    double ql = 0.0, qy = 0.0;
    for (int i = 1; i <= n; ++i) {
        const double d2 = __dsub_rn((double)h[i - 1], mu2), d3 = __dsub_rn((double)h[i], mu3);
        ql = __dadd_rn(ql, __dmul_rn(d2, d2));
        qy = __dadd_rn(qy, __dmul_rn(d3, d3));
    }
    const double sg2 = __dsqrt_rn(__ddiv_rn(ql, dn)), sg3 = __dsqrt_rn(__ddiv_rn(qy, dn));
    if (!(sg3 > 0.0)) {  // numerically constant target
        c0 = mu3;
        return 0;
    }
    if (pt[7] != 0.0 && sg2 > 0.0) {
        const double mu[4] = {pt[0], pt[1], mu2, mu3};
        const double sg[4] = {pt[2], pt[3], sg2, sg3};
        const double* z0 = pt + 8;
        const double* z1 = z0 + n;
        double h0 = 0.0, h1 = 0.0, h2 = 0.0, G20 = 0.0, G21 = 0.0, G22 = 0.0;
        for (int i = 1; i <= n; ++i) {
            const double a = __ldg(z0 + i - 1), b = __ldg(z1 + i - 1);
            const double z2 = __ddiv_rn(__dsub_rn((double)h[i - 1], mu2), sg2);
            const double u = __ddiv_rn(__dsub_rn((double)h[i], mu3), sg3);
            h0 = __dadd_rn(h0, __dmul_rn(a, u));
            h1 = __dadd_rn(h1, __dmul_rn(b, u));
            G20 = __dadd_rn(G20, __dmul_rn(z2, a));
            G21 = __dadd_rn(G21, __dmul_rn(z2, b));
            G22 = __dadd_rn(G22, __dmul_rn(z2, z2));
            h2 = __dadd_rn(h2, __dmul_rn(z2, u));
        }
        int status = 0, ridge_fired = 0;
        chol3_solve(pt[4], pt[5], pt[6], G20, G21, G22, h0, h1, h2, p.ridge, p.tol, dn, mu, sg, c0, w, status,
                    ridge_fired);
        return status;
    }
    // a zero-variance column: the general path of fit_one (cold)
    double rec[kRecDoubles];
    fit_one<E>(h, L, T, rho, p.phase, p.phase + T, p.ridge, p.tol, rec);
    c0 = rec[0];
    w[0] = rec[1];
    w[1] = rec[2];
    w[2] = rec[3];
    return (int)rec[5] == CHASE_ERR_FIT ? CHASE_ERR_FIT : 0;
}

template <typename E>
__global__ void __launch_bounds__(128) rolling_forecast_kernel(const __grid_constant__ RollParams p) {
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
