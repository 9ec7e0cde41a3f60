// svr.cuh — the epsilon-SVR forecaster (Table 1's best model,
// P:162; SPEC fit_svr S:140-148), included by kernels.cu inside its
// anonymous namespace.
//
// One warp per trace fits the RBF epsilon-SVR on the L history points with
// the oracle's algorithm (libsvm's, as scikit-learn runs it; DESIGN Q31):
// z-scored features and target (fit-window statistics), the training kernel
// matrix rounded to single precision (libsvm's Qfloat cache), SMO on the 2n
// dual variables with second-order working-set selection, the bias from the
// free variables.  exp() is svr_exp_neg, this library's own table exp
// (<= 2 ulp of libm's; the oracle uses libm's), so a training kernel entry
// equals the oracle's unless the two exps straddle a single-precision rounding
// boundary (~1e-8 of the entries).  One thread per window (or period) then
// predicts f(x) = sum_t coef_t K(z_t, z(x)) - rho in double precision (fma);
// the forecasts agree with the oracle's to ~1e-13, within the 1e-9 bar.
constexpr int kSvrMaxN = 63;

// Model record per trace (doubles): z[63][3] | coef[63] | mu[4] | sigma[4] | gamma, rho | n, kind, keep0..2
constexpr int kSvrZ = 0, kSvrCoef = 3 * kSvrMaxN, kSvrMu = kSvrCoef + kSvrMaxN, kSvrSigma = kSvrMu + 4;
constexpr int kSvrGamma = kSvrSigma + 4, kSvrRho = kSvrGamma + 1, kSvrN = kSvrRho + 1, kSvrKind = kSvrN + 1;
constexpr int kSvrKeep = kSvrKind + 1, kSvrIters = kSvrKeep + 3, kSvrDoubles = (kSvrIters + 1 + 1) & ~1;

// The table exp's scalar constants in the constant bank (the fma's take them
// as c[][] operands): 64/ln2, (ln2/64)_hi, (ln2/64)_lo, 1/5!, 1/4!, 1/3!,
// 1/2, 1, 1.
__constant__ double c_svr_exp[9] = {0x1.71547652b82fep+6, 0x1.62e42feep-7, 0x1.a39ef35793c76p-39,
                                    0x1.1111111111111p-7, 0x1.5555555555555p-5, 0x1.5555555555555p-3,
                                    0.5, 1.0, 1.0};
// 2^(j/64), the doubles nearest the exact values (this library's own table), in global
// memory: indexed by data (a constant-bank read would serialise the lanes);
// the forecast kernel stages them in shared memory.
__device__ const double g_svr_exp2[64] = {
    0x1.0000000000000p+0, 0x1.02c9a3e778061p+0, 0x1.059b0d3158574p+0, 0x1.0874518759bc8p+0,
    0x1.0b5586cf9890fp+0, 0x1.0e3ec32d3d1a2p+0, 0x1.11301d0125b51p+0, 0x1.1429aaea92de0p+0,
    0x1.172b83c7d517bp+0, 0x1.1a35beb6fcb75p+0, 0x1.1d4873168b9aap+0, 0x1.2063b88628cd6p+0,
    0x1.2387a6e756238p+0, 0x1.26b4565e27cddp+0, 0x1.29e9df51fdee1p+0, 0x1.2d285a6e4030bp+0,
    0x1.306fe0a31b715p+0, 0x1.33c08b26416ffp+0, 0x1.371a7373aa9cbp+0, 0x1.3a7db34e59ff7p+0,
    0x1.3dea64c123422p+0, 0x1.4160a21f72e2ap+0, 0x1.44e086061892dp+0, 0x1.486a2b5c13cd0p+0,
    0x1.4bfdad5362a27p+0, 0x1.4f9b2769d2ca7p+0, 0x1.5342b569d4f82p+0, 0x1.56f4736b527dap+0,
    0x1.5ab07dd485429p+0, 0x1.5e76f15ad2148p+0, 0x1.6247eb03a5585p+0, 0x1.6623882552225p+0,
    0x1.6a09e667f3bcdp+0, 0x1.6dfb23c651a2fp+0, 0x1.71f75e8ec5f74p+0, 0x1.75feb564267c9p+0,
    0x1.7a11473eb0187p+0, 0x1.7e2f336cf4e62p+0, 0x1.82589994cce13p+0, 0x1.868d99b4492edp+0,
    0x1.8ace5422aa0dbp+0, 0x1.8f1ae99157736p+0, 0x1.93737b0cdc5e5p+0, 0x1.97d829fde4e50p+0,
    0x1.9c49182a3f090p+0, 0x1.a0c667b5de565p+0, 0x1.a5503b23e255dp+0, 0x1.a9e6b5579fdbfp+0,
    0x1.ae89f995ad3adp+0, 0x1.b33a2b84f15fbp+0, 0x1.b7f76f2fb5e47p+0, 0x1.bcc1e904bc1d2p+0,
    0x1.c199bdd85529cp+0, 0x1.c67f12e57d14bp+0, 0x1.cb720dcef9069p+0, 0x1.d072d4a07897cp+0,
    0x1.d5818dcfba487p+0, 0x1.da9e603db3285p+0, 0x1.dfc97337b9b5fp+0, 0x1.e502ee78b3ff6p+0,
    0x1.ea4afa2a490dap+0, 0x1.efa1bee615a27p+0, 0x1.f50765b6e4540p+0, 0x1.fa7c1819e90d8p+0,
};

// q * 2^e (t in [0.99, 2)) rounded once (ldexp).  For
// e >= -1021 the product is normal and exact, so e is added to the exponent
// field (integer pipe); below that (rare) two multiplications, the first
// exact, the second rounding the exact value once.
__device__ __forceinline__ double svr_scale2k(double q, int ki) {
    if (ki >= -1021) return __hiloint2double(__double2hiint(q) + (ki << 20), __double2loint(q));
    return __dmul_rn(__dmul_rn(q, 0x1p-600), __hiloint2double((ki + 600 + 1023) << 20, 0));
}

// The uncommon keys of svr_exp_neg: y = -0 (x = +0), NaN or negative y
// (x > 0 or NaN: NaN), y > 745 (0), and y in (707, 745] (a result that may be
// subnormal: the general scaling).
__device__ __noinline__ double svr_exp_rare(unsigned long long v, double t, int k) {
    if (v == 0x8000000000000000ull) return svr_scale2k(t, k >> 6);
    if (!(v <= 0x7FF0000000000000ull)) return CUDART_NAN;
    if (v > 0x4087480000000000ull) return 0.0;
    return svr_scale2k(t, k >> 6);
}

// exp(-y): kd = 64 e + j the integer nearest 64 y/ln2, Cody-Waite reduction
// by ln2/64, the degree-5 Taylor polynomial of exp(r) (|r| <= ln2/128) in
// Horner form (fma), times 2^(j/64) from the table at `tab` (shared or global
// memory), scaled by 2^e; <= 2 ulp of libm (DESIGN Q31).  kd
// comes from the 1.5*2^52 shift, whose low word is kd (no F2I), and
// kd = 64 e + j splits with a mask and a shift.  The common keys, y in
// [+0, 707], are one unsigned compare of the bit pattern (integer pipe; the
// fp64 pipe is this kernel's bound) and need no further guard: x >= -707
// gives e >= -1021, a normal result, scaled by an exponent-field add.
// The six non-trivial constants of the exp held in registers for a kernel's
// lifetime (the moves through inline asm keep the compiler from re-reading
// them from the constant bank inside the term loop).
struct SvrExpK {
    double c[6];
    __device__ __forceinline__ SvrExpK() {
#pragma unroll
        for (int j = 0; j < 6; ++j) asm volatile("mov.b64 %0, %1;" : "=d"(c[j]) : "d"(c_svr_exp[j]));
    }
};

__device__ __forceinline__ double svr_exp_neg(double y, const double* tab, const SvrExpK& K) {
    const unsigned long long v = (unsigned long long)__double_as_longlong(y);
    const double m = __fma_rn(-y, K.c[0], 0x1.8p52);
    const double kd = __dsub_rn(m, 0x1.8p52);
    double r = __fma_rn(-kd, K.c[1], -y);
    r = __fma_rn(-kd, K.c[2], r);
    double q = K.c[3];
    q = __fma_rn(q, r, K.c[4]);
    q = __fma_rn(q, r, K.c[5]);
    q = __fma_rn(q, r, 0.5);
    q = __fma_rn(q, r, 1.0);
    q = __fma_rn(q, r, 1.0);
    const int k = __double2loint(m);
    const double t = __dmul_rn(tab[k & 63], q);
    if (v <= 0x4086180000000000ull)  // bits(707.0)
        return __hiloint2double(__double2hiint(t) + ((k >> 6) << 20), __double2loint(t));
    return svr_exp_rare(v, t, k);
}

__device__ __forceinline__ double svr_exp_neg(double y, const double* tab) {
    const unsigned long long v = (unsigned long long)__double_as_longlong(y);
    const double m = __fma_rn(-y, c_svr_exp[0], 0x1.8p52);
    const double kd = __dsub_rn(m, 0x1.8p52);
    double r = __fma_rn(-kd, c_svr_exp[1], -y);
    r = __fma_rn(-kd, c_svr_exp[2], r);
    double q = c_svr_exp[3];
#pragma unroll
    for (int j = 4; j < 9; ++j) q = __fma_rn(q, r, c_svr_exp[j]);
    const int k = __double2loint(m);
    const double t = __dmul_rn(tab[k & 63], q);
    if (v <= 0x4086180000000000ull)  // bits(707.0)
        return __hiloint2double(__double2hiint(t) + ((k >> 6) << 20), __double2loint(t));
    return svr_exp_rare(v, t, k);
}

__device__ __forceinline__ double svr_exp(double x) { return svr_exp_neg(-x, g_svr_exp2); }

// A training kernel entry: exp(-gamma * ((d0*d0 + d1*d1) + d2*d2)) (the oracle's
// rbf(), each operation rounded once), stored as libsvm stores it: rounded to
// single precision (DESIGN Q31).
__device__ __forceinline__ double svr_rbf_train(const double* a, const double* b, double gamma) {
    const double d0 = __dsub_rn(a[0], b[0]), d1 = __dsub_rn(a[1], b[1]), d2 = __dsub_rn(a[2], b[2]);
    const double d = __dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2));
    return (double)__double2float_rn(svr_exp_neg(__dmul_rn(gamma, d), g_svr_exp2));
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
// the oracle's order (the exp aside, see the top of the file); what runs in
// parallel is only independent work (kernel entries, the elementwise gradient
// update) and the arg-extremum scans, whose results do not depend on the scan
// order under the last-index tie rule.
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
        K[q] = svr_rbf_train(z + 3 * a, z + 3 * b, gamma);
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

// svr_forecast_kernel's dynamic shared memory (doubles): z[3n] | coef[n] | zs[T] | zc[T]
// (plus the static 2^(j/64) table)
__host__ __device__ inline int svr_fc_smem_doubles(int L, int T) { return 4 * (L - 1) + 2 * T; }
constexpr int kSvrFcThreads = 128, kSvrFcPer = 8;  // 128 threads x 8 periods per block

// One block per (trace, 1024 decision periods): the trace's support vectors,
// coefficients and the z-scored phase features of every phase are staged in
// shared memory once; one thread per period runs the recursive horizon of
// oracle_plan_trace (prediction k is the lag of prediction k+1, from the last
// observed value) and writes its mean to every window of the period.  P = 1 is
// the one-step forecast with the observed lag.  Each prediction follows
// oracle_svr_predict: f = sum_t coef_t K(z_t, zq) (in t order) - rho,
// mu_y + sigma_y f clamped at 0, with the squared distance and the sum fused
// (fma) and this library's exp, so within ~1e-13 of the oracle's (not bit
// for bit); two kernel terms are evaluated per loop step (independent exp
// chains) and accumulated in order.
template <typename E>
__global__ void __launch_bounds__(kSvrFcThreads) svr_forecast_kernel(const __grid_constant__ SvrParams p) {
    extern __shared__ __align__(16) double vsm[];
    const int64_t i = blockIdx.x;
    if (p.records[i * kRecDoubles + 5] != 0.0) return;  // bad history: no model (the sweep reports it)
    const double* M = p.models + i * kSvrDoubles;
    const int n = (int)M[kSvrN], T = p.T;
    __shared__ double e2[64];  // static: addressed as shared memory directly in the term loop
    double* z = vsm;
    double* cf = z + 3 * n;
    double* zs = cf + n;
    double* zc = zs + T;
    const bool constant = M[kSvrKind] != 0.0;
    const double mu0 = M[kSvrMu], mu1 = M[kSvrMu + 1], mu2 = M[kSvrMu + 2], mu3 = M[kSvrMu + 3];
    const double sg0 = M[kSvrSigma], sg1 = M[kSvrSigma + 1], sg2 = M[kSvrSigma + 2], sg3 = M[kSvrSigma + 3];
    const bool k0 = M[kSvrKeep] != 0.0, k1 = M[kSvrKeep + 1] != 0.0, k2 = M[kSvrKeep + 2] != 0.0;
    const double gamma = M[kSvrGamma], rho = M[kSvrRho];
    if (!constant) {
        for (int q = threadIdx.x; q < 64; q += blockDim.x) e2[q] = g_svr_exp2[q];
        for (int q = threadIdx.x; q < 3 * n; q += blockDim.x) z[q] = M[kSvrZ + q];
        for (int q = threadIdx.x; q < n; q += blockDim.x) cf[q] = M[kSvrCoef + q];
        for (int q = threadIdx.x; q < T; q += blockDim.x) {
            zs[q] = k0 ? __ddiv_rn(__dsub_rn(p.phase[q], mu0), sg0) : 0.0;
            zc[q] = k1 ? __ddiv_rn(__dsub_rn(p.phase[T + q], mu1), sg1) : 0.0;
        }
    }
    __syncthreads();
    const SvrExpK EK;
    const int W = p.N - p.L, P = p.P;
    const E* row = reinterpret_cast<const E*>(p.traces) + i * p.ld;
    const int per_end = min(p.n_per, (int)(blockIdx.y + 1) * kSvrFcThreads * kSvrFcPer);
    for (int per = blockIdx.y * kSvrFcThreads * kSvrFcPer + threadIdx.x; per < per_end; per += kSvrFcThreads) {
        const int b = per * P;
        const int nw = W - b < P ? W - b : P;
        double prev = (double)row[p.L + b - 1], sum = 0.0;
        int ph = (int)(((int64_t)p.phase0 + p.L + b) % T);
        for (int k = 0; k < nw; ++k) {
            double pr;
            if (constant) {
                pr = mu3;
            } else {
                const double q0 = zs[ph], q1 = zc[ph];
                const double q2 = k2 ? __ddiv_rn(__dsub_rn(prev, mu2), sg2) : 0.0;
                double f = 0.0;
                int t = 0;
                for (; t + 1 < n; t += 2) {
                    const double a0 = __dsub_rn(z[3 * t], q0), a1 = __dsub_rn(z[3 * t + 1], q1),
                                 a2 = __dsub_rn(z[3 * t + 2], q2);
                    const double b0 = __dsub_rn(z[3 * t + 3], q0), b1 = __dsub_rn(z[3 * t + 4], q1),
                                 b2 = __dsub_rn(z[3 * t + 5], q2);
                    const double da = __fma_rn(a2, a2, __fma_rn(a1, a1, __dmul_rn(a0, a0)));
                    const double db = __fma_rn(b2, b2, __fma_rn(b1, b1, __dmul_rn(b0, b0)));
                    const double Ka = svr_exp_neg(__dmul_rn(gamma, da), e2, EK);
                    const double Kb = svr_exp_neg(__dmul_rn(gamma, db), e2, EK);
                    f = __fma_rn(cf[t], Ka, f);
                    f = __fma_rn(cf[t + 1], Kb, f);
                }
                if (t < n) {
                    const double a0 = __dsub_rn(z[3 * t], q0), a1 = __dsub_rn(z[3 * t + 1], q1),
                                 a2 = __dsub_rn(z[3 * t + 2], q2);
                    const double da = __fma_rn(a2, a2, __fma_rn(a1, a1, __dmul_rn(a0, a0)));
                    f = __fma_rn(cf[t], svr_exp_neg(__dmul_rn(gamma, da), e2, EK), f);
                }
                f = __dsub_rn(f, rho);
                pr = __dadd_rn(mu3, __dmul_rn(sg3, f));
            }
            const double fk = pr > 0.0 ? pr : 0.0;
            sum = __dadd_rn(sum, fk);
            prev = fk;
            ph = ph + 1 == T ? 0 : ph + 1;
        }
        const double chat = __ddiv_rn(sum, (double)nw);
        double* out = p.forecast + i * p.ld_f + b;
        for (int k = 0; k < nw; ++k) out[k] = chat;
    }
}
