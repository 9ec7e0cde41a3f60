// fit.cuh — §3.1 forecaster fit (K1), included by kernels.cu.

// ------------------------------------------------------------------ fit (K1)
// §3.1: the model is fitted once per trace on its L history points c[0..L)
// ("one day prior").  One lane per trace, the same
// sequential order and rounding as oracle_fit (bit-identical records).
// Normal equations, Cholesky (ridge fallback) and un-standardisation for the
// 3-column case, unrolled: identical arithmetic to the general path.
// Cholesky of the standardised 3x3 Gram (ridge fallback), the two
// triangular solves and the un-standardisation of oracle_fit (DESIGN Q24).
__device__ __forceinline__ void chol3_solve(double G00, double G10, double G11, double G20, double G21, double G22,
                                            double h0, double h1, double h2, double ridge, double tol_rel, double dn,
                                            const double* mu, const double* sg, double& c0, double* w, int& status,
                                            int& ridge_fired) {
    const double tol = __dmul_rn(tol_rel, dn);
    double L00 = 0, L10 = 0, L20 = 0, L11 = 0, L21 = 0, L22 = 0;
    bool ok = false;
    for (int attempt = 0; attempt < 2 && !ok; ++attempt) {
        if (attempt == 1) {
            G00 = __dadd_rn(G00, ridge);
            G11 = __dadd_rn(G11, ridge);
            G22 = __dadd_rn(G22, ridge);
            ridge_fired = 1;
        }
        double d = G00;
        if (!(d > tol)) continue;
        L00 = __dsqrt_rn(d);
        L10 = __ddiv_rn(G10, L00);
        L20 = __ddiv_rn(G20, L00);
        d = __dsub_rn(G11, __dmul_rn(L10, L10));
        if (!(d > tol)) continue;
        L11 = __dsqrt_rn(d);
        L21 = __ddiv_rn(__dsub_rn(G21, __dmul_rn(L20, L10)), L11);
        d = __dsub_rn(__dsub_rn(G22, __dmul_rn(L20, L20)), __dmul_rn(L21, L21));
        if (!(d > tol)) continue;
        L22 = __dsqrt_rn(d);
        ok = true;
    }
    if (!ok) {
        status = CHASE_ERR_FIT;
        return;
    }
    const double zt0 = __ddiv_rn(h0, L00);
    const double zt1 = __ddiv_rn(__dsub_rn(h1, __dmul_rn(L10, zt0)), L11);
    const double zt2 = __ddiv_rn(__dsub_rn(__dsub_rn(h2, __dmul_rn(L20, zt0)), __dmul_rn(L21, zt1)), L22);
    const double b2 = __ddiv_rn(zt2, L22);
    const double b1 = __ddiv_rn(__dsub_rn(zt1, __dmul_rn(L21, b2)), L11);
    const double b0 = __ddiv_rn(__dsub_rn(__dsub_rn(zt0, __dmul_rn(L10, b1)), __dmul_rn(L20, b2)), L00);
    w[0] = __ddiv_rn(__dmul_rn(sg[3], b0), sg[0]);
    w[1] = __ddiv_rn(__dmul_rn(sg[3], b1), sg[1]);
    w[2] = __ddiv_rn(__dmul_rn(sg[3], b2), sg[2]);
    c0 = __dsub_rn(__dsub_rn(__dsub_rn(mu[3], __dmul_rn(w[0], mu[0])), __dmul_rn(w[1], mu[1])), __dmul_rn(w[2], mu[2]));
}

// Correctly rounded a/b for a fixed divisor b: y = RN(1/b) once, then per
// quotient q0 = RN(a y), r = fma(-q0, b, a) (exact), q = RN(q0 + r y) --
// Markstein's final step, which returns RN(a/b) when y = RN(1/b) and q0 is
// within an ulp, absent over/underflow (tools/div_probe.cu: 1.6e10 operand
// pairs, random, all-ones mantissas and fit-shaped, no mismatch with
// __ddiv_rn).  Three fp64 operations instead of a full divide.  Used where
// the operands come from fp32 traces (centred values over a sigma: far from
// the exponent limits); b outside [2^-900, 2^900] takes the plain divide.
struct RnDiv {
    double b, y;
    bool fast;
    __device__ __forceinline__ explicit RnDiv(double bb) {
        b = bb;
        y = __drcp_rn(bb);
        const double ab = fabs(bb);
        fast = ab > 0x1p-900 && ab < 0x1p900;
    }
    __device__ __forceinline__ double operator()(double a) const {
        if (!fast) return __ddiv_rn(a, b);
        const double q0 = __dmul_rn(a, y);
        return __fma_rn(__fma_rn(-q0, b, a), y, q0);
    }
};

template <typename E>
__device__ __forceinline__ void fit_solve3(const E* h, int n, int T, int phi0, const double* S, const double* Cc,
                                           double ridge, double tol_rel, const double* mu, const double* sg, double dn,
                                           double& c0, double* w, int& status, int& ridge_fired) {
    double G00 = 0, G10 = 0, G11 = 0, G20 = 0, G21 = 0, G22 = 0, h0 = 0, h1 = 0, h2 = 0;
    int ph = (phi0 + 1) % T;
    for (int i = 1; i <= n; ++i) {
        const double z0 = __ddiv_rn(__dsub_rn(S[ph], mu[0]), sg[0]);
        const double z1 = __ddiv_rn(__dsub_rn(Cc[ph], mu[1]), sg[1]);
        const double z2 = __ddiv_rn(__dsub_rn((double)h[i - 1], mu[2]), sg[2]);
        const double u = __ddiv_rn(__dsub_rn((double)h[i], mu[3]), sg[3]);
        G00 = __dadd_rn(G00, __dmul_rn(z0, z0));
        h0 = __dadd_rn(h0, __dmul_rn(z0, u));
        G10 = __dadd_rn(G10, __dmul_rn(z1, z0));
        G11 = __dadd_rn(G11, __dmul_rn(z1, z1));
        h1 = __dadd_rn(h1, __dmul_rn(z1, u));
        G20 = __dadd_rn(G20, __dmul_rn(z2, z0));
        G21 = __dadd_rn(G21, __dmul_rn(z2, z1));
        G22 = __dadd_rn(G22, __dmul_rn(z2, z2));
        h2 = __dadd_rn(h2, __dmul_rn(z2, u));
        ph = ph + 1 == T ? 0 : ph + 1;
    }
    chol3_solve(G00, G10, G11, G20, G21, G22, h0, h1, h2, ridge, tol_rel, dn, mu, sg, c0, w, status, ridge_fired);
}

template <typename E>
__device__ void fit_one(const E* h, int L, int T, int phi0, const double* S, const double* Cc, double ridge,
                        double tol_rel, double* rec) {
    const int n = L - 1;
    const double dn = (double)n;
    double maxci = (double)h[0];
    int bad = 0;
    for (int t = 0; t < L; ++t) {
        E v = h[t];
        bad |= bad_value(v);
        if ((double)v > maxci) maxci = (double)v;
    }
    double c0 = 0, w[3] = {0, 0, 0};
    int status = bad ? CHASE_ERR_DATA : 0, ridge_fired = 0, kind = 0;
    bool constant = true;
    for (int i = 2; i <= n; ++i)
        if ((double)h[i] != (double)h[1]) { constant = false; break; }
    if (status == 0 && constant) {
        kind = 1;
        c0 = (double)h[1];
    } else if (status == 0) {
        double sum[4] = {0, 0, 0, 0};
        for (int i = 1; i <= n; ++i) {
            int ph = (phi0 + i) % T;
            sum[0] = __dadd_rn(sum[0], S[ph]);
            sum[1] = __dadd_rn(sum[1], Cc[ph]);
            sum[2] = __dadd_rn(sum[2], (double)h[i - 1]);
            sum[3] = __dadd_rn(sum[3], (double)h[i]);
        }
        double mu[4], ss[4] = {0, 0, 0, 0}, sg[4];
        for (int j = 0; j < 4; ++j) mu[j] = __ddiv_rn(sum[j], dn);
        for (int i = 1; i <= n; ++i) {
            int ph = (phi0 + i) % T;
            double d0 = __dsub_rn(S[ph], mu[0]);
            double d1 = __dsub_rn(Cc[ph], mu[1]);
            double d2 = __dsub_rn((double)h[i - 1], mu[2]);
            double d3 = __dsub_rn((double)h[i], mu[3]);
            ss[0] = __dadd_rn(ss[0], __dmul_rn(d0, d0));
            ss[1] = __dadd_rn(ss[1], __dmul_rn(d1, d1));
            ss[2] = __dadd_rn(ss[2], __dmul_rn(d2, d2));
            ss[3] = __dadd_rn(ss[3], __dmul_rn(d3, d3));
        }
        for (int j = 0; j < 4; ++j) sg[j] = __dsqrt_rn(__ddiv_rn(ss[j], dn));
        if (!(sg[3] > 0.0)) {
            kind = 1;
            c0 = mu[3];
        } else if (sg[0] > 0.0 && sg[1] > 0.0 && sg[2] > 0.0) {
            // all three columns kept (the common case): the same operation
            // sequence as the general path below, with register-resident 3x3 state
            fit_solve3(h, n, T, phi0, S, Cc, ridge, tol_rel, mu, sg, dn, c0, w, status, ridge_fired);
        } else {
            int cols[3], m = 0;
            for (int j = 0; j < 3; ++j)
                if (sg[j] > 0.0) cols[m++] = j;
            double G[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}}, hv[3] = {0, 0, 0};
            for (int i = 1; i <= n; ++i) {
                int ph = (phi0 + i) % T;
                double x[3] = {S[ph], Cc[ph], (double)h[i - 1]};
                double z[3];
                for (int a = 0; a < m; ++a) z[a] = __ddiv_rn(__dsub_rn(x[cols[a]], mu[cols[a]]), sg[cols[a]]);
                double u = __ddiv_rn(__dsub_rn((double)h[i], mu[3]), sg[3]);
                for (int a = 0; a < m; ++a) {
                    for (int b = 0; b <= a; ++b) G[a][b] = __dadd_rn(G[a][b], __dmul_rn(z[a], z[b]));
                    hv[a] = __dadd_rn(hv[a], __dmul_rn(z[a], u));
                }
            }
            for (int a = 0; a < m; ++a)
                for (int b = 0; b < a; ++b) G[b][a] = G[a][b];
            const double tol = __dmul_rn(tol_rel, dn);
            double Lc[3][3];
            bool ok = false;
            for (int attempt = 0; attempt < 2 && !ok; ++attempt) {
                if (attempt == 1) {
                    for (int a = 0; a < m; ++a) G[a][a] = __dadd_rn(G[a][a], ridge);
                    ridge_fired = 1;
                }
                for (int a = 0; a < 3; ++a)
                    for (int b = 0; b < 3; ++b) Lc[a][b] = 0.0;
                ok = true;
                for (int j = 0; j < m && ok; ++j) {
                    double d = G[j][j];
                    for (int k = 0; k < j; ++k) d = __dsub_rn(d, __dmul_rn(Lc[j][k], Lc[j][k]));
                    if (!(d > tol)) { ok = false; break; }
                    Lc[j][j] = __dsqrt_rn(d);
                    for (int i = j + 1; i < m; ++i) {
                        double v = G[i][j];
                        for (int k = 0; k < j; ++k) v = __dsub_rn(v, __dmul_rn(Lc[i][k], Lc[j][k]));
                        Lc[i][j] = __ddiv_rn(v, Lc[j][j]);
                    }
                }
                if (m == 0) ok = true;
            }
            if (!ok) {
                status = CHASE_ERR_FIT;
            } else {
                double zt[3] = {0, 0, 0}, beta[3] = {0, 0, 0};
                for (int a = 0; a < m; ++a) {
                    double v = hv[a];
                    for (int b = 0; b < a; ++b) v = __dsub_rn(v, __dmul_rn(Lc[a][b], zt[b]));
                    zt[a] = __ddiv_rn(v, Lc[a][a]);
                }
                for (int a = m - 1; a >= 0; --a) {
                    double v = zt[a];
                    for (int b = a + 1; b < m; ++b) v = __dsub_rn(v, __dmul_rn(Lc[b][a], beta[b]));
                    beta[a] = __ddiv_rn(v, Lc[a][a]);
                }
                for (int a = 0; a < m; ++a) w[cols[a]] = __ddiv_rn(__dmul_rn(sg[3], beta[a]), sg[cols[a]]);
                c0 = mu[3];
                for (int a = 0; a < m; ++a) c0 = __dsub_rn(c0, __dmul_rn(w[cols[a]], mu[cols[a]]));
            }
        }
    }
    rec[0] = c0;
    rec[1] = w[0];
    rec[2] = w[1];
    rec[3] = w[2];
    rec[4] = maxci;
    rec[5] = (double)status;
    rec[6] = (double)ridge_fired;
    rec[7] = (double)kind;
}

// Phase columns of a fit whose first history point has phase rho (rows
// i = 1..n, phase (rho + i) mod T): their means, population sigmas, z-scores
// and the phase-only Gram entries G00, G10, G11, each computed with
// oracle_fit's own sequential operations.  Every accumulator of the fit is a
// separate sequential sum over the rows, so taking these from a table changes
// no rounding.  Record layout (phase_stride(L) doubles):
//   [mu0, mu1, sg0, sg1, G00, G10, G11, ok] z0[1..n] z1[1..n]
__host__ __device__ inline int phase_stride(int L) { return 8 + 2 * (L - 1); }

__device__ void phase_record(const double* S, const double* Cc, int T, int L, int rho, double* out) {
    const int n = L - 1;
    const double dn = (double)n;
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

// fit_one with the phase columns from a phase_record `pt` (same results,
// bit for bit, with half the divides): rec[0..7] as fit_one.
template <typename E>
__device__ void fit_phase(const E* h, int L, int T, int rho, const double* pt, const double* S, const double* Cc,
                          double ridge, double tol_rel, double* rec) {
    const int n = L - 1;
    const double dn = (double)n;
    double maxci = (double)h[0];
    int bad = 0;
    for (int t = 0; t < L; ++t) {
        const E v = h[t];
        bad |= bad_value(v);
        if ((double)v > maxci) maxci = (double)v;
    }
    double c0 = 0.0, w[3] = {0.0, 0.0, 0.0};
    int status = bad ? CHASE_ERR_DATA : 0, ridge_fired = 0, kind = 0;
    bool constant = true;
    for (int i = 2; i <= n; ++i)
        if ((double)h[i] != (double)h[1]) { constant = false; break; }
    if (status == 0 && constant) {  // F2: intercept-only model
        kind = 1;
        c0 = (double)h[1];
    } else if (status == 0) {
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
            kind = 1;
            c0 = mu3;
        } else if (pt[7] != 0.0 && sg2 > 0.0) {
            const double mu[4] = {pt[0], pt[1], mu2, mu3};
            const double sg[4] = {pt[2], pt[3], sg2, sg3};
            const double* z0 = pt + 8;
            const double* z1 = z0 + n;
            double h0 = 0.0, h1 = 0.0, h2 = 0.0, G20 = 0.0, G21 = 0.0, G22 = 0.0;
            const RnDiv d2(sg2), d3(sg3);
            for (int i = 1; i <= n; ++i) {
                const double a = z0[i - 1], b = z1[i - 1];
                // fp32 traces: the Markstein quotients (= the divide, bit for bit); fp64: the divide
                const double z2 = sizeof(E) == 4 ? d2(__dsub_rn((double)h[i - 1], mu2))
                                                 : __ddiv_rn(__dsub_rn((double)h[i - 1], mu2), sg2);
                const double u = sizeof(E) == 4 ? d3(__dsub_rn((double)h[i], mu3))
                                                : __ddiv_rn(__dsub_rn((double)h[i], mu3), sg3);
                h0 = __dadd_rn(h0, __dmul_rn(a, u));
                h1 = __dadd_rn(h1, __dmul_rn(b, u));
                G20 = __dadd_rn(G20, __dmul_rn(z2, a));
                G21 = __dadd_rn(G21, __dmul_rn(z2, b));
                G22 = __dadd_rn(G22, __dmul_rn(z2, z2));
                h2 = __dadd_rn(h2, __dmul_rn(z2, u));
            }
            chol3_solve(pt[4], pt[5], pt[6], G20, G21, G22, h0, h1, h2, ridge, tol_rel, dn, mu, sg, c0, w, status,
                        ridge_fired);
        } else {  // a zero-variance column: the general path (cold)
            fit_one<E>(h, L, T, rho, S, Cc, ridge, tol_rel, rec);
            return;
        }
    }
    rec[0] = c0;
    rec[1] = w[0];
    rec[2] = w[1];
    rec[3] = w[2];
    rec[4] = maxci;
    rec[5] = (double)status;
    rec[6] = (double)ridge_fired;
    rec[7] = (double)kind;
}

// The phase record of the fit-once job start (one thread, once per call).
__global__ void fit_phase_kernel(const uint8_t* tables, int T, int L, int phase0, double* out) {
    const TablesHeader* H = reinterpret_cast<const TablesHeader*>(tables);
    const double* ph = reinterpret_cast<const double*>(tables + H->off_phase);
    phase_record(ph, ph + T, T, L, phase0 % T, out);
}

// Fit kernel: stage the CTA's 128 histories (L <= 64) into smem with coalesced
// loads (odd row stride), one lane per trace runs the canonical fit; also the
// max-power baseline's completion count m: the first m with
// m*s_b >= J, s_b = Thr_{K-1}*Delta (exact for the dyadic inputs; DESIGN R3).
template <typename E>
__global__ void __launch_bounds__(128) fit_kernel(const __grid_constant__ FitParams p) {
    extern __shared__ __align__(16) uint8_t fsm[];
    E* hs = reinterpret_cast<E*>(fsm);
    double* tab = reinterpret_cast<double*>(fsm + round16(128 * 65 * (int)sizeof(E)));
    double* prec = tab + 2 * p.T;  // the phase record of phase0 (staged path: L <= 64)
    const TablesHeader* H = reinterpret_cast<const TablesHeader*>(p.tables);
    const int L = p.L, T = p.T;
    const int64_t first = (int64_t)blockIdx.x * 128;
    const E* tr = reinterpret_cast<const E*>(p.traces);
    const bool staged = !p.baseline_only && L <= 64;
    if (!p.baseline_only) {
        const double* ph = reinterpret_cast<const double*>(p.tables + H->off_phase);
        for (int q = threadIdx.x; q < 2 * T; q += blockDim.x) tab[q] = ph[q];
    }
    if (staged) {
        const int stride = L | 1;
        for (int q = threadIdx.x; q < 128 * L; q += blockDim.x) {
            int r = q / L, t = q - r * L;
            int64_t i = first + r;
            if (i < p.n_traces) hs[r * stride + t] = tr[i * p.ld + t];
        }
    }
    __syncthreads();
    if (staged) {  // the job-start phase record (fit_phase_kernel, once per call; one CTA: here)
        if (gridDim.x == 1) {
            if (threadIdx.x == 0) phase_record(tab, tab + T, T, L, p.phase0 % T, prec);
        } else {
            for (int q = threadIdx.x; q < phase_stride(L); q += blockDim.x) prec[q] = p.prec[q];
        }
    }
    __syncthreads();
    const int64_t i = first + threadIdx.x;
    if (i >= p.n_traces) return;
    double rec[kRecDoubles];
#pragma unroll
    for (int q = 0; q < kRecDoubles; ++q) rec[q] = 0.0;
    if (!p.baseline_only) {
        const E* h = staged ? hs + threadIdx.x * (L | 1) : tr + i * p.ld;
        if (staged) fit_phase<E>(h, L, T, p.phase0 % T, prec, tab, tab + T, p.ridge, p.tol, rec);
        else fit_one<E>(h, L, T, p.phase0 % T, tab, tab + T, p.ridge, p.tol, rec);
    }
    const double J = p.job ? p.job[i] : 0.0;
    int prof = 0;
    if (p.n_prof > 0) {
        prof = p.profile_id ? (int)p.profile_id[i] : 0;
        if (prof >= p.n_prof) prof = 0;
    }
    if (p.n_eta > 0 && !p.baseline_only) {
        // per-trace scalars of the single-eta sweep, one thread per trace here instead of a warp there:
        // [10] Kc = ((1-eta)*Pmax)*MaxCI   [11] 1/Kc (0: canonical path)   [12] J   [13] profile
        // [14] J/(1.000001*max_k s_k) (a lower bound on the windows to completion)   [15] MaxCI
        const PairTable* pt = reinterpret_cast<const PairTable*>(p.tables + H->off_pair) + prof * p.n_eta;
        const ProfileTable* pf = blob_profiles(p.tables) + prof;
        const double maxci = p.max_ci_fixed > 0.0 ? p.max_ci_fixed : rec[4];
        const double Kc = __dmul_rn(pt->kbase, maxci);
        rec[10] = Kc;
        rec[11] = per_trace_invK(pt, Kc);
        rec[12] = J;
        rec[13] = (double)prof;
        rec[14] = J > 0.0 ? __ddiv_rn(J, __dmul_rn(pf->smax, 1.000001)) : 0.0;
        rec[15] = maxci;
    }
    if (J > 0.0 && p.n_prof > 0) {
        const ProfileTable* pf = blob_profiles(p.tables) + prof;
        const double sb = pf->line[pf->K - 1].x;
        const double qv = __ddiv_rn(J, sb);
        int64_t m = qv < 4.0e15 ? (int64_t)ceil(qv) : (int64_t)p.W + 2;
        if (m < 1) m = 1;
        while (m > 1 && __dmul_rn((double)(m - 1), sb) >= J) --m;
        while (m <= (int64_t)p.W && __dmul_rn((double)m, sb) < J) ++m;
        if (m > (int64_t)p.W) m = (int64_t)p.W + 1;
        rec[8] = (double)m;
    }
    double* out = p.records + i * kRecDoubles;
#pragma unroll
    for (int q = 0; q < kRecDoubles; ++q) out[q] = rec[q];
    if (p.models_out) {
#pragma unroll
        for (int q = 0; q < kModelDoubles; ++q) p.models_out[i * kModelDoubles + q] = rec[q];
    }
    if (p.max_ci_out) p.max_ci_out[i] = rec[4];
}

