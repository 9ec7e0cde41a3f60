// svr.cuh — the epsilon-SVR forecaster (Table 1's best model,
// P:162; SPEC fit_svr S:140-148), included by kernels.cu inside its
// anonymous namespace.
//
// One thread per trace fits the RBF epsilon-SVR on the L history points with
// the oracle's algorithm, operation for operation: z-scored features and
// target (fit-window statistics), the kernel matrix, SMO on the 2n dual
// variables with second-order working-set selection, the bias from the free
// variables.  exp() is svr_exp, the same Cody-Waite + degree-13 Horner
// polynomial as oracle_rbf_exp, so every value is bit-identical.  One thread
// per window then predicts f(x) = sum_t coef_t K(z_t, z(x)) - rho, in the
// oracle's summation order, and the sweep plans on those forecasts (FIN).
constexpr int kSvrMaxN = 63;

// Model record per trace (doubles): z[63][3] | coef[63] | mu[4] | sigma[4] | gamma, rho | n, kind, keep0..2
constexpr int kSvrZ = 0, kSvrCoef = 3 * kSvrMaxN, kSvrMu = kSvrCoef + kSvrMaxN, kSvrSigma = kSvrMu + 4;
constexpr int kSvrGamma = kSvrSigma + 4, kSvrRho = kSvrGamma + 1, kSvrN = kSvrRho + 1, kSvrKind = kSvrN + 1;
constexpr int kSvrKeep = kSvrKind + 1, kSvrIters = kSvrKeep + 3, kSvrDoubles = (kSvrIters + 1 + 1) & ~1;

__device__ __forceinline__ double svr_exp(double x) {
    if (!(x <= 0.0)) return CUDART_NAN;
    if (x < -745.0) return 0.0;
    const double k = floor(__dadd_rn(__dmul_rn(x, 1.4426950408889634), 0.5));
    const double r = __dsub_rn(__dsub_rn(x, __dmul_rn(k, 6.93147180369123816490e-01)),
                               __dmul_rn(k, 1.90821492927058770002e-10));
    double q = 0x1.6124613a86d09p-33;
    q = __dadd_rn(__dmul_rn(q, r), 0x1.1eed8eff8d898p-29);
    q = __dadd_rn(__dmul_rn(q, r), 0x1.ae64567f544e4p-26);
    q = __dadd_rn(__dmul_rn(q, r), 0x1.27e4fb7789f5cp-22);
    q = __dadd_rn(__dmul_rn(q, r), 0x1.71de3a556c734p-19);
    q = __dadd_rn(__dmul_rn(q, r), 0x1.a01a01a01a01ap-16);
    q = __dadd_rn(__dmul_rn(q, r), 0x1.a01a01a01a01ap-13);
    q = __dadd_rn(__dmul_rn(q, r), 0x1.6c16c16c16c17p-10);
    q = __dadd_rn(__dmul_rn(q, r), 0x1.1111111111111p-7);
    q = __dadd_rn(__dmul_rn(q, r), 0x1.5555555555555p-5);
    q = __dadd_rn(__dmul_rn(q, r), 0x1.5555555555555p-3);
    q = __dadd_rn(__dmul_rn(q, r), 0.5);
    q = __dadd_rn(__dmul_rn(q, r), 1.0);
    q = __dadd_rn(__dmul_rn(q, r), 1.0);
    return ldexp(q, (int)k);
}

__device__ __forceinline__ double svr_rbf(const double* a, const double* b, double gamma) {
    const double d0 = __dsub_rn(a[0], b[0]), d1 = __dsub_rn(a[1], b[1]), d2 = __dsub_rn(a[2], b[2]);
    const double d = __dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2));
    return svr_exp(-__dmul_rn(gamma, d));
}

struct SvrParams {
    const void* traces;
    int64_t ld, n_traces;
    int32_t N, L, T, phase0, max_iter;
    int32_t P, n_per;      // decision period (>= 1) and periods per trace
    double C, eps, gamma, tol;
    const double* phase;   // S[T], C[T]
    double* models;        // [n][kSvrDoubles]
    double* records;       // fit records [n][16]: [5] status (the SVR resets the linear fit's 6)
    double* forecast;      // [n][ld_f]
    int64_t ld_f;
};

// (value, index) arg-extremum across the warp with the oracle's tie rule: the
// sequential scans update on `>=` / `<=`, so among equal values the LAST index wins.
__device__ __forceinline__ void warp_argmax_last(double& v, int& i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, i, o);
        if (ov > v || (ov == v && oi > i)) { v = ov; i = oi; }
    }
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Shared memory per warp (doubles): K[n*n] | alpha[2n] | G[2n] | z[3n] | u[n]
__host__ __device__ inline int svr_smem_doubles(int L) {
    const int n = L - 1;
    return n * n + 4 * n + 3 * n + n;
}

constexpr int kSvrWarps = 4;

// One warp per trace.  Every value is computed with the oracle's operations in
// the oracle's order; what runs in parallel is only independent work (kernel
// entries, the elementwise gradient update) and the arg-extremum scans, whose
// results do not depend on the scan order under the last-index tie rule.
// Sequential sums (moments, the bias) run on lane 0.
template <typename E>
__global__ void __launch_bounds__(32 * kSvrWarps) svr_fit_kernel(const __grid_constant__ SvrParams p) {
    extern __shared__ __align__(16) double svs[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t i = (int64_t)blockIdx.x * kSvrWarps + wid;
    if (i >= p.n_traces) return;
    double* rec = p.records + i * kRecDoubles;
    if (rec[5] == (double)CHASE_ERR_DATA) return;  // the history check is the fit's (fit_kernel)
    const int L = p.L, T = p.T, n = L - 1, l = 2 * n;
    double* K = svs + (size_t)wid * svr_smem_doubles(L);
    double* al = K + n * n;
    double* G = al + l;
    double* z = G + l;
    double* u = z + 3 * n;
    const E* h = reinterpret_cast<const E*>(p.traces) + i * p.ld;
    double* M = p.models + i * kSvrDoubles;
    const double* S = p.phase;
    const double* Cc = p.phase + T;
    const int phi0 = p.phase0 % T;
    const double dn = (double)n;
    // moments (lane 0, sequential as the oracle), broadcast through registers
    double mu[4], sg[4];
    if (lane == 0) {
        double sum[4] = {0.0, 0.0, 0.0, 0.0};
        for (int r = 1; r <= n; ++r) {
            const int ph = (phi0 + r) % T;
            sum[0] = __dadd_rn(sum[0], S[ph]);
            sum[1] = __dadd_rn(sum[1], Cc[ph]);
            sum[2] = __dadd_rn(sum[2], (double)h[r - 1]);
            sum[3] = __dadd_rn(sum[3], (double)h[r]);
        }
        for (int j = 0; j < 4; ++j) mu[j] = __ddiv_rn(sum[j], dn);
        double ss[4] = {0.0, 0.0, 0.0, 0.0};
        for (int r = 1; r <= n; ++r) {
            const int ph = (phi0 + r) % T;
            const double xv[4] = {S[ph], Cc[ph], (double)h[r - 1], (double)h[r]};
            for (int j = 0; j < 4; ++j) {
                const double d = __dsub_rn(xv[j], mu[j]);
                ss[j] = __dadd_rn(ss[j], __dmul_rn(d, d));
            }
        }
        for (int j = 0; j < 4; ++j) sg[j] = __dsqrt_rn(__ddiv_rn(ss[j], dn));
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        mu[j] = __shfl_sync(0xffffffffu, mu[j], 0);
        sg[j] = __shfl_sync(0xffffffffu, sg[j], 0);
    }
    rec[5] = 0.0;  // the SVR fit cannot fail for 2 <= n <= 63 (the linear fit's status does not apply)
    if (lane == 0) {
        M[kSvrN] = dn;
        for (int j = 0; j < 4; ++j) {
            M[kSvrMu + j] = mu[j];
            M[kSvrSigma + j] = sg[j];
        }
    }
    if (!(sg[3] > 0.0)) {  // constant target: the constant
        if (lane == 0) M[kSvrKind] = 1.0;
        return;
    }
    bool keep[3];
    int kept = 0;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        keep[j] = sg[j] > 0.0;
        kept += keep[j];
    }
    const double gamma = p.gamma > 0.0 ? p.gamma : (kept > 0 ? __ddiv_rn(1.0, (double)kept) : 1.0);
    for (int r = lane; r < n; r += 32) {
        const int ph = (phi0 + r + 1) % T;
        const double xv[3] = {S[ph], Cc[ph], (double)h[r]};
#pragma unroll
        for (int j = 0; j < 3; ++j) z[3 * r + j] = keep[j] ? __ddiv_rn(__dsub_rn(xv[j], mu[j]), sg[j]) : 0.0;
        u[r] = __ddiv_rn(__dsub_rn((double)h[r + 1], mu[3]), sg[3]);
    }
    __syncwarp();
    for (int q = lane; q < n * n; q += 32) {
        const int a = q / n, b = q - a * n;
        K[q] = svr_rbf(z + 3 * a, z + 3 * b, gamma);
    }
    for (int t = lane; t < l; t += 32) {
        al[t] = 0.0;
        G[t] = t < n ? __dsub_rn(p.eps, u[t]) : __dadd_rn(p.eps, u[t - n]);
    }
    __syncwarp();
    const double C = p.C, TAU = 1e-12;
    int it = 0;
    for (;;) {
        // second-order working-set selection
        double Gmax = -CUDART_INF;
        int wi = -1;
        for (int t = lane; t < l; t += 32) {
            const double v = t < n ? (al[t] < C ? -G[t] : CUDART_NAN) : (al[t] > 0.0 ? G[t] : CUDART_NAN);
            if (v >= Gmax) { Gmax = v; wi = t; }  // NaN: not eligible
        }
        warp_argmax_last(Gmax, wi);
        double Gmax2 = -CUDART_INF, obj = CUDART_INF;
        int wj = -1;
        if (wi >= 0) {
            const double yi = wi < n ? 1.0 : -1.0;
            const int ri = wi < n ? wi : wi - n;
            const double Kii = K[ri * n + ri];
            for (int t = lane; t < l; t += 32) {
                const double yt = t < n ? 1.0 : -1.0;
                const int rt = t < n ? t : t - n;
                const double Qit = __dmul_rn(__dmul_rn(yi, yt), K[ri * n + rt]);
                const double Gt = G[t], at = al[t];
                if (t < n ? at > 0.0 : at < C) {
                    const double gv = t < n ? Gt : -Gt;
                    const double gd = t < n ? __dadd_rn(Gmax, Gt) : __dsub_rn(Gmax, Gt);
                    if (gv >= Gmax2) Gmax2 = gv;
                    if (gd > 0.0) {
                        const double kk = __dadd_rn(Kii, K[rt * n + rt]);
                        const double yq = __dmul_rn(__dmul_rn(2.0, yi), Qit);
                        const double qc = t < n ? __dsub_rn(kk, yq) : __dadd_rn(kk, yq);
                        const double od = -__ddiv_rn(__dmul_rn(gd, gd), qc > 0.0 ? qc : TAU);
                        if (od <= obj) { wj = t; obj = od; }
                    }
                }
            }
            Gmax2 = warp_max(Gmax2);
            double nobj = -obj;  // min with the last index == max of the negation with the last index
            warp_argmax_last(nobj, wj);
        }
        if (__dadd_rn(Gmax, Gmax2) < p.tol || wj < 0) break;
        if (it >= p.max_iter) break;
        ++it;
        // analytic pair update (every lane, identical values)
        const double yi = wi < n ? 1.0 : -1.0, yj = wj < n ? 1.0 : -1.0;
        const int ri = wi < n ? wi : wi - n, rj = wj < n ? wj : wj - n;
        const double Qij = __dmul_rn(__dmul_rn(yi, yj), K[ri * n + rj]);
        const double ai = al[wi], aj = al[wj];
        double nai = ai, naj = aj;
        if (yi != yj) {
            double qc = __dadd_rn(__dadd_rn(K[ri * n + ri], K[rj * n + rj]), __dmul_rn(2.0, Qij));
            if (qc <= 0.0) qc = TAU;
            const double delta = __ddiv_rn(__dsub_rn(-G[wi], G[wj]), qc);
            const double diff = __dsub_rn(ai, aj);
            nai = __dadd_rn(ai, delta);
            naj = __dadd_rn(aj, delta);
            if (diff > 0.0) { if (naj < 0.0) { naj = 0.0; nai = diff; } }
            else { if (nai < 0.0) { nai = 0.0; naj = -diff; } }
            if (diff > 0.0) { if (nai > C) { nai = C; naj = __dsub_rn(C, diff); } }
            else { if (naj > C) { naj = C; nai = __dadd_rn(C, diff); } }
        } else {
            double qc = __dsub_rn(__dadd_rn(K[ri * n + ri], K[rj * n + rj]), __dmul_rn(2.0, Qij));
            if (qc <= 0.0) qc = TAU;
            const double delta = __ddiv_rn(__dsub_rn(G[wi], G[wj]), qc);
            const double sm = __dadd_rn(ai, aj);
            nai = __dsub_rn(ai, delta);
            naj = __dadd_rn(aj, delta);
            if (sm > C) { if (nai > C) { nai = C; naj = __dsub_rn(sm, C); } }
            else { if (naj < 0.0) { naj = 0.0; nai = sm; } }
            if (sm > C) { if (naj > C) { naj = C; nai = __dsub_rn(sm, C); } }
            else { if (nai < 0.0) { nai = 0.0; naj = sm; } }
        }
        const double dai = __dsub_rn(nai, ai), daj = __dsub_rn(naj, aj);
        __syncwarp();
        if (lane == 0) {
            al[wi] = nai;
            al[wj] = naj;
        }
        for (int t = lane; t < l; t += 32) {
            const double yt = t < n ? 1.0 : -1.0;
            const int rt = t < n ? t : t - n;
            const double Qti = __dmul_rn(__dmul_rn(yt, yi), K[rt * n + ri]);
            const double Qtj = __dmul_rn(__dmul_rn(yt, yj), K[rt * n + rj]);
            G[t] = __dadd_rn(G[t], __dadd_rn(__dmul_rn(Qti, dai), __dmul_rn(Qtj, daj)));
        }
        __syncwarp();
    }
    if (lane == 0) {  // bias: mean y*G over the free variables (sequential), else the bounds' midpoint
        double ub = CUDART_INF, lb = -CUDART_INF, sfree = 0.0;
        int nfree = 0;
        for (int t = 0; t < l; ++t) {
            const double yt = t < n ? 1.0 : -1.0;
            const double yG = __dmul_rn(yt, G[t]);
            if (al[t] >= C) { if (yt < 0.0) ub = fmin(ub, yG); else lb = fmax(lb, yG); }
            else if (al[t] <= 0.0) { if (yt > 0.0) ub = fmin(ub, yG); else lb = fmax(lb, yG); }
            else { ++nfree; sfree = __dadd_rn(sfree, yG); }
        }
        M[kSvrRho] = nfree > 0 ? __ddiv_rn(sfree, (double)nfree) : __ddiv_rn(__dadd_rn(ub, lb), 2.0);
        M[kSvrGamma] = gamma;
        M[kSvrIters] = (double)it;
        M[kSvrKind] = 0.0;
        for (int j = 0; j < 3; ++j) M[kSvrKeep + j] = keep[j] ? 1.0 : 0.0;
    }
    for (int r = lane; r < n; r += 32) {
        for (int j = 0; j < 3; ++j) M[kSvrZ + 3 * r + j] = z[3 * r + j];
        M[kSvrCoef + r] = __dsub_rn(al[r], al[r + n]);
    }
}

// oracle_svr_predict for window w of trace i (thread per window).
__device__ __forceinline__ double svr_predict(const double* M, double s, double c, double lag) {
    if (M[kSvrKind] != 0.0) return M[kSvrMu + 3] > 0.0 ? M[kSvrMu + 3] : 0.0;
    const double xv[3] = {s, c, lag};
    double zq[3];
    for (int j = 0; j < 3; ++j)
        zq[j] = M[kSvrKeep + j] != 0.0 ? __ddiv_rn(__dsub_rn(xv[j], M[kSvrMu + j]), M[kSvrSigma + j]) : 0.0;
    const int n = (int)M[kSvrN];
    const double gamma = M[kSvrGamma];
    double f = 0.0;
    for (int t = 0; t < n; ++t) f = __dadd_rn(f, __dmul_rn(M[kSvrCoef + t], svr_rbf(M + kSvrZ + 3 * t, zq, gamma)));
    f = __dsub_rn(f, M[kSvrRho]);
    const double pr = __dadd_rn(M[kSvrMu + 3], __dmul_rn(M[kSvrSigma + 3], f));
    return pr > 0.0 ? pr : 0.0;
}

// One thread per (trace, decision period): the recursive horizon of
// oracle_plan_trace (prediction k is the lag of prediction k+1, from the last
// observed value), its mean written to every window of the period.  P = 1 is
// the one-step forecast with the observed lag.
template <typename E>
__global__ void __launch_bounds__(256) svr_forecast_kernel(const __grid_constant__ SvrParams p) {
    const int W = p.N - p.L, P = p.P;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= p.n_traces * (int64_t)p.n_per) return;
    const int64_t i = idx / p.n_per;
    const int b = (int)(idx - i * p.n_per) * P;
    if (p.records[i * kRecDoubles + 5] != 0.0) return;  // bad history: no model (the sweep reports it)
    const E* row = reinterpret_cast<const E*>(p.traces) + i * p.ld;
    const double* M = p.models + i * kSvrDoubles;
    const int n = W - b < P ? W - b : P;
    double prev = (double)row[p.L + b - 1], sum = 0.0;
    int ph = (int)(((int64_t)p.phase0 + p.L + b) % p.T);
    for (int k = 0; k < n; ++k) {
        const double f = svr_predict(M, p.phase[ph], p.phase[p.T + ph], prev);
        sum = __dadd_rn(sum, f);
        prev = f;
        ph = ph + 1 == p.T ? 0 : ph + 1;
    }
    const double chat = __ddiv_rn(sum, (double)n);
    double* out = p.forecast + i * p.ld_f + b;
    for (int k = 0; k < n; ++k) out[k] = chat;
}
