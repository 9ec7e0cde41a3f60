// k2_roll.cuh — the rolling refit fused into the sweep (SURVEY §8(a) a3,
// §8(c) tolerance contract): refit_stride R >= 1, fp32 traces
// with an aligned job start, one eta, no forecast output.  Included by
// kernels.cu inside its anonymous namespace.
//
// Window w is forecast by the least-squares model fitted on the L points
// before its origin r = s0 + R floor((w - s0)/R) (P:67 applied at every
// origin; Q1).  Instead of oracle_fit's two-pass sequence per origin
// (rolling_forecast_kernel, bit-identical, FP64-bound at ~1e3 flops per
// origin), this kernel keeps the raw moments of the origin's L-1 rows in
// registers and slides them one row per origin (add the new row, remove the
// oldest), then solves the centred normal equations in closed form:
//   D_ab = n S_ab - S_a S_b                    (n-scaled centred moments)
//   P = [[D_ss, D_sc], [D_sc, D_cc]]           (phase block: per origin phase, a table)
//   q = P^-1 (D_sl, D_cl),  u = P^-1 (D_sy, D_cy)
//   s_ll = D_ll - q.(D_sl, D_cl),  r_y = D_ly - q.(D_sy, D_cy)
//   b_l = r_y / s_ll,  (b_s, b_c) = u - b_l q   (Schur complement)
//   chat = mu_y + b_s (S[phi] - mu_s) + b_c (C[phi] - mu_c) + b_l (c[w-1] - mu_l)
// -- the same least-squares solution (the OLS prediction does not depend on
// the z-scoring, Q5), in a different rounding order: forecasts agree with the
// oracle's to ~1e-13 relative, within the 1e-9 bar; a choice may differ only
// at a certified near-tie (tests: assert_parity_tol).  Windows whose fit is
// near-degenerate -- a (near-)constant target or lag column, s_ll/D_ll below
// 1e-8 (the oracle's ridge fallback fires at 1e-12), a phase block without
// both columns -- take oracle_fit's exact sequence (fit_one, cold).
//
// Decomposition: a warp owns one trace at a time and streams it in chunks of
// 1024 windows (32 lanes x 32 consecutive windows) through a two-slot TMA ring
// that carries the chunk's history halo; each lane computes its run's first
// origin's moments directly (L-1 rows), then slides.  Eq. 6 by the envelope
// table (canonical rule in a band), replay sums per lane, completion and
// baseline as the headline kernels .

// The completion walk of a run of windows in window order, 32 at a time per
// round (lane = window), from the samples done before the run: the window
// where the samples reach J, its fraction f and the sums before it.  Cold,
// once per trace.
struct LCompletion {
    double f, Ep, Cp, Pk, cw;
    int w;       // completion window within the slot, -1: none
};
__device__ __noinline__ LCompletion run_completion(const float* sv, const uint8_t* crow, int nwin, double before,
                                                    double J, const ProfileTable* pf, int lane) {
    LCompletion r{1.0, 0.0, 0.0, 0.0, 0.0, -1};
    double carry = before;
    for (int r0 = 0; r0 < nwin; r0 += 32) {
        const int j = r0 + lane;
        const bool valid = j < nwin;
        const uint32_t k = valid ? crow[j] : 0u;
        const double2 ln = valid ? pf->line[k] : make_double2(0.0, 0.0);
        const double cw = valid ? (double)sv[j] : 0.0;
        const double incl = __dadd_rn(carry, warp_incl_scan(ln.x, lane));
        const double prev = __shfl_up_sync(kFull, incl, 1);
        const double before_w = lane == 0 ? carry : prev;
        const unsigned hits = __ballot_sync(kFull, valid && incl >= J);
        const int wl_ = hits ? __ffs(hits) - 1 : 32;
        const bool pre = valid && lane < wl_;
        r.Ep = __dadd_rn(r.Ep, warp_sum(pre ? ln.y : 0.0));
        r.Cp = __dadd_rn(r.Cp, warp_sum(pre ? __dmul_rn(ln.y, cw) : 0.0));
        if (wl_ < 32) {
            const double bw = __shfl_sync(kFull, before_w, wl_);
            const double sk = __shfl_sync(kFull, ln.x, wl_);
            r.w = r0 + wl_;
            r.f = __ddiv_rn(__dsub_rn(J, bw), sk);  // pro-rata last window
            r.Pk = __shfl_sync(kFull, ln.y, wl_);
            r.cw = __shfl_sync(kFull, cw, wl_);
            return r;
        }
        carry = __shfl_sync(kFull, incl, 31);
    }
    return r;
}

#ifndef CHASE_R_WARPS
#define CHASE_R_WARPS 8
#endif
#ifndef CHASE_R_GROUP
#define CHASE_R_GROUP 4  // windows per unrolled group of the R = 1 path (overlapping solve chains)
#endif
constexpr int kRWarps = CHASE_R_WARPS;
constexpr int kRThreads = 32 * kRWarps;
constexpr int kRRun = 32;                 // windows per lane per chunk
constexpr int kRChunk = 32 * kRRun;       // 1024 windows per chunk
constexpr int kRMaxL = 64;                // history lengths the fused kernel takes (L <= 64)
constexpr int kRHalo = kRMaxL + 32;       // values before the chunk kept in the slot (L + R - 1 <= 96 for R <= 33)
constexpr int kRSlotF = kRHalo + kRChunk; // floats per slot
constexpr int kRPhase = 12;               // per-origin-phase table: Ss, Sc, i11, i12, i22, ok, S[rho], C[rho],
                                          // S[rho - n], C[rho - n] (the window's own phase and the leaving row's),
                                          // mu_s = Ss/n, mu_c = Sc/n

struct RLayout {
    int tables, ptab, warp_bytes, total;
    int slot, rec, chb, mbar;  // offsets inside a warp block
};

__host__ __device__ inline RLayout make_rlayout(int T, int tables_bytes) {
    RLayout R;
    R.slot = 0;
    R.rec = 2 * kRSlotF * 4;
    R.chb = R.rec + 2 * kRecBytes;
    R.mbar = R.chb + kRChunk;
    R.warp_bytes = (R.mbar + 16 + 127) & ~127;
    R.tables = kRWarps * R.warp_bytes;
    R.ptab = R.tables + round16(tables_bytes);
    R.total = R.ptab + round16(T * kRPhase * 8);
    return R;
}

// Raw moments of one origin's L-1 rows t (y_t = c[t], l_t = c[t-1], s_t, k_t
// the phase columns of the target's time).
struct RMom {
    double Sy, Syy, Sly, Ssy, Sky, Ssl, Skl;
};

// The trace's values, from the slot when the index is in it, else from HBM
// (rows of a large refit stride's origin before the chunk: cold).
struct RVals {
    const float* sb;     // slot floats: sb[q] = c[a0 + q]
    const float* row;    // the trace row in HBM
    int a0, a1;          // [a0, a1): absolute indices held by the slot
    __device__ __forceinline__ double operator()(int a) const {
        CHASE_CHECK(a >= 0);
        return (double)(a >= a0 && a < a1 ? sb[a - a0] : __ldg(row + a));
    }
};

__device__ __forceinline__ void mom_row(RMom& m, double y, double l, double s, double k, double sg) {
    // sg = +1 adds the row, -1 removes it
    m.Sy = __fma_rn(sg, y, m.Sy);
    const double ys = __dmul_rn(sg, y), ls = __dmul_rn(sg, l);
    m.Syy = __fma_rn(ys, y, m.Syy);
    m.Sly = __fma_rn(ls, y, m.Sly);
    m.Ssy = __fma_rn(ys, s, m.Ssy);
    m.Sky = __fma_rn(ys, k, m.Sky);
    m.Ssl = __fma_rn(ls, s, m.Ssl);
    m.Skl = __fma_rn(ls, k, m.Skl);
}

// Moments of origin r directly from its rows t = r-n .. r-1.
__device__ __noinline__ RMom mom_direct(const RVals& v, int r, int n, int phase0, int T, const double* S,
                                        const double* C) {
    RMom m{0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    int ph = (int)(((int64_t)phase0 + r - n) % T);
    double l = v(r - n - 1);
    for (int t = r - n; t < r; ++t) {
        const double y = v(t);
        mom_row(m, y, l, S[ph], C[ph], 1.0);
        l = y;
        ph = ph + 1 == T ? 0 : ph + 1;
    }
    return m;
}

// The model of an origin: chat(w) = mu_y + b_s (S[phi_w] - mu_s) + b_c (C[phi_w] - mu_c) + b_l (lag - mu_l);
// exact = true: (c0, w) from oracle_fit's sequence, chat = (c0 + w_s S) + w_c C + w_l lag (Q24).
struct RModel {
    double a, bs, bc, bl;   // closed form: a = mu_y - b_s mu_s - b_c mu_c - b_l mu_l (per origin)
    bool exact;
    int status;             // exact fit: CHASE_ERR_FIT when it failed
};

// Closed-form solve; returns false for a near-degenerate fit (the caller takes the exact path).
__device__ __forceinline__ bool mom_solve(const RMom& m, double cy_last, double cy_first_lag, double dn, double inv_n,
                                          const double* pt, RModel& md) {
    if (pt[5] == 0.0) return false;  // the phase block lacks a column (e.g. T <= 2)
    const double Ss = pt[0], Sc = pt[1], i11 = pt[2], i12 = pt[3], i22 = pt[4];
    // lag moments from the target ones: Sl = Sy - c[r-1] + c[r-n-1], Sll likewise
    const double Sl = __dadd_rn(__dsub_rn(m.Sy, cy_last), cy_first_lag);
    const double Sll = __fma_rn(cy_first_lag, cy_first_lag, __fma_rn(-cy_last, cy_last, m.Syy));
    const double Dyy = __fma_rn(dn, m.Syy, -__dmul_rn(m.Sy, m.Sy));
    const double Dll = __fma_rn(dn, Sll, -__dmul_rn(Sl, Sl));
    const double Dly = __fma_rn(dn, m.Sly, -__dmul_rn(Sl, m.Sy));
    const double Dsl = __fma_rn(dn, m.Ssl, -__dmul_rn(Ss, Sl));
    const double Dcl = __fma_rn(dn, m.Skl, -__dmul_rn(Sc, Sl));
    const double Dsy = __fma_rn(dn, m.Ssy, -__dmul_rn(Ss, m.Sy));
    const double Dcy = __fma_rn(dn, m.Sky, -__dmul_rn(Sc, m.Sy));
    // a (near-)constant target or lag column: the oracle's F2 / zero-variance branches
    if (!(Dyy > __dmul_rn(1e-10, __dmul_rn(dn, m.Syy)))) return false;
    if (!(Dll > __dmul_rn(1e-10, __dmul_rn(dn, Sll)))) return false;
    const double q1 = __fma_rn(i11, Dsl, __dmul_rn(i12, Dcl));
    const double q2 = __fma_rn(i12, Dsl, __dmul_rn(i22, Dcl));
    const double sll = __dsub_rn(Dll, __fma_rn(q1, Dsl, __dmul_rn(q2, Dcl)));
    // 1 - R^2 of the lag on the phase columns: the oracle's ridge branch fires at <= 1e-12
    if (!(sll > __dmul_rn(1e-8, Dll))) return false;
    const double u1 = __fma_rn(i11, Dsy, __dmul_rn(i12, Dcy));
    const double u2 = __fma_rn(i12, Dsy, __dmul_rn(i22, Dcy));
    const double ry = __dsub_rn(Dly, __fma_rn(q1, Dsy, __dmul_rn(q2, Dcy)));
    const double bl = __ddiv_rn(ry, sll);
    const double bs = __fma_rn(-bl, q1, u1), bc = __fma_rn(-bl, q2, u2);
    const double mu_y = __dmul_rn(m.Sy, inv_n), mu_l = __dmul_rn(Sl, inv_n);
    const double mu_s = __dmul_rn(Ss, inv_n), mu_c = __dmul_rn(Sc, inv_n);
    md.a = __fma_rn(-bl, mu_l, __fma_rn(-bc, mu_c, __fma_rn(-bs, mu_s, mu_y)));
    md.bs = bs;
    md.bc = bc;
    md.bl = bl;
    md.exact = false;
    md.status = 0;
    return isfinite(md.a) && isfinite(bl) && isfinite(bs) && isfinite(bc);
}

// oracle_fit's exact sequence for origin r (near-degenerate windows; cold).
__device__ __noinline__ RModel exact_model(const RVals& v, int r, int L, int T, int phase0, const double* S,
                                           const double* C, double ridge, double tol) {
    float h[kRMaxL];
    for (int q = 0; q < L; ++q) h[q] = (float)v(r - L + q);
    double rec[kRecDoubles];
    fit_one<float>(h, L, T, (int)(((int64_t)phase0 + r - L) % T), S, C, ridge, tol, rec);
    RModel md;
    md.a = rec[0];
    md.bs = rec[1];
    md.bc = rec[2];
    md.bl = rec[3];
    md.exact = true;
    md.status = (int)rec[5] == CHASE_ERR_FIT ? CHASE_ERR_FIT : 0;
    return md;
}

// 1/x to ~1 ulp: the SFU seed and two Newton steps (the closed form's one
// division; the tolerance contract allows it).
__device__ __forceinline__ double rcp_nr2(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    r = __fma_rn(r, __fma_rn(-x, r, 1.0), r);
    r = __fma_rn(r, __fma_rn(-x, r, 1.0), r);
    return r;
}

// mom_solve with the reciprocal in place of the IEEE division (the R = 1 path).
__device__ __forceinline__ bool mom_solve_fast(const RMom& m, double cy_last, double cy_first_lag, double dn,
                                               double inv_n, const double* pt, RModel& md) {
    if (pt[5] == 0.0) return false;
    const double Ss = pt[0], Sc = pt[1], i11 = pt[2], i12 = pt[3], i22 = pt[4];
    const double Sl = __dadd_rn(__dsub_rn(m.Sy, cy_last), cy_first_lag);
    const double Sll = __fma_rn(cy_first_lag, cy_first_lag, __fma_rn(-cy_last, cy_last, m.Syy));
    const double Dyy = __fma_rn(dn, m.Syy, -__dmul_rn(m.Sy, m.Sy));
    const double Dll = __fma_rn(dn, Sll, -__dmul_rn(Sl, Sl));
    const double Dly = __fma_rn(dn, m.Sly, -__dmul_rn(Sl, m.Sy));
    const double Dsl = __fma_rn(dn, m.Ssl, -__dmul_rn(Ss, Sl));
    const double Dcl = __fma_rn(dn, m.Skl, -__dmul_rn(Sc, Sl));
    const double Dsy = __fma_rn(dn, m.Ssy, -__dmul_rn(Ss, m.Sy));
    const double Dcy = __fma_rn(dn, m.Sky, -__dmul_rn(Sc, m.Sy));
    const double q1 = __fma_rn(i11, Dsl, __dmul_rn(i12, Dcl));
    const double q2 = __fma_rn(i12, Dsl, __dmul_rn(i22, Dcl));
    const double sll = __dsub_rn(Dll, __fma_rn(q1, Dsl, __dmul_rn(q2, Dcl)));
    const double u1 = __fma_rn(i11, Dsy, __dmul_rn(i12, Dcy));
    const double u2 = __fma_rn(i12, Dsy, __dmul_rn(i22, Dcy));
    const double ry = __dsub_rn(Dly, __fma_rn(q1, Dsy, __dmul_rn(q2, Dcy)));
    const double bl = __dmul_rn(ry, rcp_nr2(sll));
    const double bs = __fma_rn(-bl, q1, u1), bc = __fma_rn(-bl, q2, u2);
    const double mu_y = __dmul_rn(m.Sy, inv_n), mu_l = __dmul_rn(Sl, inv_n);
    md.a = __fma_rn(-bl, mu_l, __fma_rn(-bc, pt[11], __fma_rn(-bs, pt[10], mu_y)));  // pt[10..11]: mu_s, mu_c
    md.bs = bs;
    md.bc = bc;
    md.bl = bl;
    md.exact = false;
    md.status = 0;
    // near-degenerate (the oracle's F2 / zero-variance / ridge branches): the exact path.  A
    // non-finite value makes the trace invalid whatever its forecasts.
    const double tn = __dmul_rn(1e-10, dn);
    return Dyy > __dmul_rn(tn, m.Syy) && Dll > __dmul_rn(tn, Sll) && sll > __dmul_rn(1e-8, Dll);
}

// One row in and one out of the moments, values from the slot (R = 1 path):
// add row t (y = c[t], l = c[t-1], phase pt_), remove row t - n (phase po).
__device__ __forceinline__ void mom_slide(RMom& m, const float* sv, int t, int n, const double* S, const double* C,
                                          int pa, int po) {
    mom_row(m, (double)sv[t], (double)sv[t - 1], S[pa], C[pa], 1.0);
    mom_row(m, (double)sv[t - n], (double)sv[t - n - 1], S[po], C[po], -1.0);
}

// The exact prediction of window a (origin a, R = 1) from oracle_fit's
// sequence: the near-degenerate windows of the closed form (cold).
__device__ __noinline__ double roll_exact_predict(const RVals& v, int a, int L, int T, int phase0, const double* S,
                                                  const double* C, double ridge, double tol, int& fit_bad) {
    float h[kRMaxL];
    for (int q = 0; q < L; ++q) h[q] = (float)v(a - L + q);
    double rec[kRecDoubles];
    fit_one<float>(h, L, T, (int)(((int64_t)phase0 + a - L) % T), S, C, ridge, tol, rec);
    if ((int)rec[5] == CHASE_ERR_FIT) fit_bad |= CHASE_ERR_FIT;
    const int ph = (int)(((int64_t)phase0 + a) % T);
    return __dadd_rn(__dadd_rn(__dadd_rn(rec[0], __dmul_rn(rec[1], S[ph])), __dmul_rn(rec[2], C[ph])),
                     __dmul_rn(rec[3], v(a - 1)));
}

__device__ __forceinline__ double roll_predict(const RModel& md, double Sph, double Cph, double lag) {
    if (md.exact)  // Q24: ((c0 + w_s S) + w_c C) + w_l lag
        return __dadd_rn(__dadd_rn(__dadd_rn(md.a, __dmul_rn(md.bs, Sph)), __dmul_rn(md.bc, Cph)),
                         __dmul_rn(md.bl, lag));
    return __fma_rn(md.bl, lag, __fma_rn(md.bc, Cph, __fma_rn(md.bs, Sph, md.a)));
}

// Per-origin-phase table (rho = phase of the origin r): the phase columns' sums
// over the rows t = r-n .. r-1 and the inverse of their centred block.
__device__ void roll_phase_table(const double* S, const double* C, int T, int n, double* out) {
    for (int rho = threadIdx.x; rho < T; rho += blockDim.x) {
        double Ss = 0.0, Sc = 0.0, Sss = 0.0, Scc = 0.0, Ssc = 0.0;
        int ph = ((rho - n) % T + T) % T;
        for (int i = 0; i < n; ++i) {
            Ss = __dadd_rn(Ss, S[ph]);
            Sc = __dadd_rn(Sc, C[ph]);
            Sss = __fma_rn(S[ph], S[ph], Sss);
            Scc = __fma_rn(C[ph], C[ph], Scc);
            Ssc = __fma_rn(S[ph], C[ph], Ssc);
            ph = ph + 1 == T ? 0 : ph + 1;
        }
        const double dn = (double)n;
        const double Dss = __fma_rn(dn, Sss, -__dmul_rn(Ss, Ss));
        const double Dcc = __fma_rn(dn, Scc, -__dmul_rn(Sc, Sc));
        const double Dsc = __fma_rn(dn, Ssc, -__dmul_rn(Ss, Sc));
        const double det = __fma_rn(Dss, Dcc, -__dmul_rn(Dsc, Dsc));
        const bool ok = Dss > 1e-9 * dn * Sss && Dcc > 1e-9 * dn * Scc && det > 1e-6 * Dss * Dcc;
        double* o = out + rho * kRPhase;
        o[0] = Ss;
        o[1] = Sc;
        o[2] = ok ? __ddiv_rn(Dcc, det) : 0.0;
        o[3] = ok ? -__ddiv_rn(Dsc, det) : 0.0;
        o[4] = ok ? __ddiv_rn(Dss, det) : 0.0;
        o[5] = ok ? 1.0 : 0.0;
        const int pl = ((rho - n) % T + T) % T;
        o[6] = S[rho];
        o[7] = C[rho];
        o[8] = S[pl];
        o[9] = C[pl];
        o[10] = __dmul_rn(Ss, 1.0 / dn);
        o[11] = __dmul_rn(Sc, 1.0 / dn);
    }
}

#ifndef CHASE_R_MINB
#define CHASE_R_MINB 1
#endif
__global__ void __launch_bounds__(kRThreads, CHASE_R_MINB) roll_fused_kernel(const __grid_constant__ SweepParams P) {
    mark_path(P.diag, CHASE_PATH_ROLL_FUSED);
    extern __shared__ __align__(128) uint8_t sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const RLayout RL = make_rlayout(P.T, P.tables_bytes);
    uint8_t* wbase = sm + warp * RL.warp_bytes;
    float* slots = reinterpret_cast<float*>(wbase + RL.slot);
    uint8_t* chb = wbase + RL.chb;
    uint64_t* mbar = reinterpret_cast<uint64_t*>(wbase + RL.mbar);
    const int T = P.T, L = P.L, n = L - 1, W = P.W, R = P.refit;
    {
        const uint4* src = reinterpret_cast<const uint4*>(P.tables);
        uint4* dst = reinterpret_cast<uint4*>(sm + RL.tables);
        for (int q = tid; q < P.tables_bytes / 16; q += kRThreads) dst[q] = src[q];
    }
    __syncthreads();
    const uint8_t* tabs = sm + RL.tables;
    const TablesHeader* H = reinterpret_cast<const TablesHeader*>(tabs);
    const double* S = reinterpret_cast<const double*>(tabs + H->off_phase);
    const double* C = S + T;
    const ProfileTable* profs = reinterpret_cast<const ProfileTable*>(tabs + H->off_prof);
    const PairTable* pairs = reinterpret_cast<const PairTable*>(tabs + H->off_pair);
    double* ptab = reinterpret_cast<double*>(sm + RL.ptab);
    roll_phase_table(S, C, T, n, ptab);
    if (lane == 0) {
        mbar_init(mbar, 1);
        mbar_init(mbar + 1, 1);
        fence_mbar_init();
    }
    __syncthreads();

    const float* traces = reinterpret_cast<const float*>(P.traces);
    const int64_t GW = (int64_t)gridDim.x * kRWarps;
    const int64_t gw = (int64_t)blockIdx.x * kRWarps + warp;
    const int s0 = L;
    const int n_chunks = (W + kRChunk - 1) / kRChunk;
    const double dn = (double)n, inv_n = 1.0 / dn;
    const bool store_choice = P.choice != nullptr;

    // producer (lane 0): unit = (trace, chunk), the slot holds c[a0, a0 + kRSlotF), a0 = s0 + 1024 ch - kRHalo
    int64_t pi = gw;
    int pc = 0, pq = 0;
    auto issue = [&]() {
        if (pi >= P.n_traces) return;
        if (lane == 0) {
            const uint64_t policy = evict_first_policy();
            const int slot_id = (pc + pq * n_chunks) & 1;
            const int a0 = s0 + pc * kRChunk - kRHalo;      // may be < 0: start at 0 (the halo's front is unused)
            const int lo = max(a0, 0);
            const int hi = min(s0 + (pc + 1) * kRChunk, P.N);
            const uint32_t bytes = (uint32_t)(((hi - lo) * 4 + 15) & ~15);
            uint64_t* bar = mbar + slot_id;
            float* dst = slots + slot_id * kRSlotF + (lo - a0);
            if (pc == 0) {
                mbar_arrive_expect_tx(bar, bytes + (uint32_t)kRecBytes);
                bulk_g2s(wbase + RL.rec + (pq & 1) * kRecBytes, P.records + pi * kRecDoubles, kRecBytes, bar, policy);
            } else {
                mbar_arrive_expect_tx(bar, bytes);
            }
            bulk_g2s(dst, traces + pi * P.ld + lo, bytes, bar, policy);
        }
        if (++pc == n_chunks) {
            pc = 0;
            pi += GW;
            ++pq;
        }
    };
    issue();
    issue();

    unsigned n_slow = 0;
    uint32_t unit = 0;
    int q = 0;
    for (int64_t i = gw; i < P.n_traces; i += GW, ++q) {
        int status = 0, c_may = n_chunks, mb = W, prof = 0;
        double J = 0.0, Kc = 0.0, invK = 0.0;
        double Sl = 0.0, El = 0.0, Cl = 0.0, Cbl = 0.0;
        bool done = false;
        const float* row = traces + i * P.ld;
        for (int ch = 0; ch < n_chunks; ++ch, ++unit) {
            const int slot_id = unit & 1;
            mbar_wait(mbar + slot_id, (unit >> 1) & 1u);
            const float* sb = slots + slot_id * kRSlotF;
            const int a0 = s0 + ch * kRChunk - kRHalo;
            const RVals V{sb, row, a0, min(s0 + (ch + 1) * kRChunk, P.N)};
            const double* rec = reinterpret_cast<const double*>(wbase + RL.rec + (q & 1) * kRecBytes);
            if (ch == 0) {
                prof = (int)rec[13];
                J = rec[12];
                status = (int)rec[5];
                if (status == 0 && !(rec[15] > 0.0)) status = CHASE_ERR_MAXCI;
                const int m = (int)rec[8];
                mb = (J > 0.0 && m >= 1 && m <= W) ? m - 1 : W;
                Kc = rec[10];
                invK = rec[11];
                c_may = J > 0.0 ? (rec[14] >= (double)W ? n_chunks - 1
                                                        : (int)(fmax(rec[14] - 1.0, 0.0) * (1.0 / kRChunk)))
                                : n_chunks;
            }
            const ProfileTable* pf = profs + prof;
            const PairTable* pt = pairs + prof;
            const int cs = ch * kRChunk;
            const int nw = min(kRChunk, W - cs);
            const int j0 = kRRun * lane;
            const int nl = max(0, min(kRRun, nw - j0));  // this lane's windows
            double aS = 0.0, aE = 0.0, aC = 0.0, aCs = 0.0;
            float vmin = FLT_MAX;
            // are all of the slot's values positive normal floats (the R = 1 path's integer conversion)?
            bool fast_vals = false;
            if (R == 1) {
                uint32_t bm = 0u;
                const int lo = max(a0, 0), hi = min(s0 + cs + kRChunk, P.N);
                for (int q = lo + lane; q < hi; q += 32) bm = max(bm, __float_as_uint(sb[q - a0]) - 0x00800000u);
                fast_vals = !__any_sync(kFull, bm >= 0x7f000000u);
            }
            int bad = 0, fit_bad = 0;
            if (status == 0 || status == CHASE_ERR_MAXCI || status == CHASE_ERR_FIT) {
                // ---- the lane's run: windows w = cs + j0 + jj (absolute a = s0 + w)
                if (R == 1 && nl > 0 && fast_vals) {
                    // every window refits.  Window a's moments M(a) slide to M(a + 1) by adding row a
                    // (y = c[a], l = c[a-1]) and removing row a - n (y = c[a-n], l = c[a-n-1]); each
                    // window's closed-form solve and prediction depend only on M(a), so the unrolled
                    // group of 4 windows overlaps four solve chains with the cheap slide chain.  The
                    // slot's values are positive normal floats (checked above): fp64 on the FMA pipe.
                    const float* sv = sb - a0;  // sv[a] = c[a] for a in the slot
                    const int ab = s0 + cs + j0;
                    RMom m = mom_direct(V, ab, n, P.phase0, T, S, C);
                    int ph = (int)(((int64_t)P.phase0 + ab) % T);  // phase of window a (= of its origin)
                    double c_prev = f32bits_to_f64(__float_as_uint(sv[ab - 1]));        // c[a-1]
                    double o_prev = f32bits_to_f64(__float_as_uint(sv[ab - n - 1]));    // c[a-n-1]
                    constexpr int G = CHASE_R_GROUP;
                    for (int g = 0; g < nl; g += G) {
                        double pu[G], cu[G];
#pragma unroll
                        for (int u = 0; u < G; ++u) {
                            const int a = ab + g + u;
                            const double* rp = ptab + ph * kRPhase;
                            const double cwv = f32bits_to_f64(__float_as_uint(sv[a]));      // c[a]
                            const double ov = f32bits_to_f64(__float_as_uint(sv[a - n]));  // c[a-n]
                            RModel md;
                            const bool ok = mom_solve_fast(m, c_prev, o_prev, dn, inv_n, rp, md);
                            pu[u] = ok ? __fma_rn(md.bl, c_prev, __fma_rn(md.bc, rp[7], __fma_rn(md.bs, rp[6], md.a)))
                                       : roll_exact_predict(V, a, L, T, P.phase0, S, C, P.ridge, P.tol, fit_bad);
                            cu[u] = cwv;
                            // slide to a + 1: row a in, row a - n out
                            m.Sy = __dadd_rn(__dsub_rn(m.Sy, ov), cwv);
                            m.Syy = __fma_rn(-ov, ov, __fma_rn(cwv, cwv, m.Syy));
                            m.Sly = __fma_rn(-o_prev, ov, __fma_rn(c_prev, cwv, m.Sly));
                            m.Ssy = __fma_rn(-rp[8], ov, __fma_rn(rp[6], cwv, m.Ssy));
                            m.Sky = __fma_rn(-rp[9], ov, __fma_rn(rp[7], cwv, m.Sky));
                            m.Ssl = __fma_rn(-rp[8], o_prev, __fma_rn(rp[6], c_prev, m.Ssl));
                            m.Skl = __fma_rn(-rp[9], o_prev, __fma_rn(rp[7], c_prev, m.Skl));
                            c_prev = cwv;
                            o_prev = ov;
                            ph = ph + 1 == T ? 0 : ph + 1;
                        }
#pragma unroll
                        for (int u = 0; u < G; ++u) {
                            if (g + u >= nl) break;
                            const double p = pu[u];
                            uint32_t k;
                            if (invK != 0.0) {
                                k = plan_lookup(__dmul_rn(p, invK), pt);
                                if (k == (uint32_t)kZeroLine) {
                                    k = canonical_choose(p > 0.0 ? p : 0.0, Kc, pt->a, pf->thr, pf->K);
                                    ++n_slow;
                                }
                            } else {
                                k = canonical_choose(p > 0.0 ? p : 0.0, Kc, pt->a, pf->thr, pf->K);
                                ++n_slow;
                            }
                            const double2 ln = pf->line[k];
                            aS = __dadd_rn(aS, ln.x);
                            aE = __dadd_rn(aE, ln.y);
                            aC = __fma_rn(ln.y, cu[u], aC);
                            aCs = __dadd_rn(aCs, cu[u]);
                            chb[j0 + g + u] = (uint8_t)k;
                        }
                    }
                    vmin = FLT_MIN;  // (every value checked positive normal)
                } else {
                RModel md{0.0, 0.0, 0.0, 0.0, false, 0};
                RMom m{0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
                int r_cur = -1;
                int pw = 0, pn = 0, po = 0;  // phases: window a, the next row to add, the next row to remove
                if (nl > 0) pw = (int)(((int64_t)P.phase0 + s0 + cs + j0) % T);
                uint32_t word = 0u;
                for (int jj = 0; jj < nl; ++jj) {
                    const int w = cs + j0 + jj, a = s0 + w;
                    const int r = s0 + R * (w / R);
                    if (r != r_cur) {  // a new origin: moments (slide by the stride or direct), then the fit
                        if (r_cur >= 0 && r - r_cur <= 8) {
                            for (int t = r_cur; t < r; ++t) {  // slide one row per step: add t, remove t - n
                                mom_row(m, V(t), V(t - 1), S[pn], C[pn], 1.0);
                                mom_row(m, V(t - n), V(t - n - 1), S[po], C[po], -1.0);
                                pn = pn + 1 == T ? 0 : pn + 1;
                                po = po + 1 == T ? 0 : po + 1;
                            }
                        } else {
                            m = mom_direct(V, r, n, P.phase0, T, S, C);
                            pn = (int)(((int64_t)P.phase0 + r) % T);
                            po = (int)(((int64_t)P.phase0 + r - n) % T);
                        }
                        r_cur = r;
                        // the origin's phase is pn (the next row to add is t = r)
                        if (!mom_solve(m, V(r - 1), V(r - n - 1), dn, inv_n, ptab + pn * kRPhase, md)) {
                            md = exact_model(V, r, L, T, P.phase0, S, C, P.ridge, P.tol);
                            fit_bad |= md.status;
                        }
                    }
                    const float raw = sb[a - a0];
                    const double cw = (double)raw;
                    const double p = roll_predict(md, S[pw], C[pw], V(a - 1));  // unclamped forecast
                    pw = pw + 1 == T ? 0 : pw + 1;
                    uint32_t k;
                    if (invK != 0.0) {
                        k = plan_lookup(__dmul_rn(p, invK), pt);
                        if (k == (uint32_t)kZeroLine) {
                            k = canonical_choose(p > 0.0 ? p : 0.0, Kc, pt->a, pf->thr, pf->K);
                            ++n_slow;
                        }
                    } else {
                        k = canonical_choose(p > 0.0 ? p : 0.0, Kc, pt->a, pf->thr, pf->K);
                        ++n_slow;
                    }
                    const double2 ln = pf->line[k];
                    aS = __dadd_rn(aS, ln.x);
                    aE = __dadd_rn(aE, ln.y);
                    aC = __fma_rn(ln.y, cw, aC);
                    aCs = __dadd_rn(aCs, cw);
                    vmin = fminf(vmin, raw);
                    word |= k << (8 * (jj & 3));
                    if ((jj & 3) == 3 || jj == nl - 1) {
                        *reinterpret_cast<uint32_t*>(chb + j0 + (jj & ~3)) = word;
                        word = 0u;
                    }
                }
                }
            }
            __syncwarp();
            if (store_choice && nl > 0) {  // the lane's 32 choice bytes (16-byte aligned): two 16-byte stores
                uint8_t* dst = P.choice + i * P.ld_c + cs + j0;
                const uint4* src = reinterpret_cast<const uint4*>(chb + j0);
                reinterpret_cast<uint4*>(dst)[0] = src[0];  // (cs + j0 + 16 <= round_up(W, 16) <= ld_c)
                if (nl > 16) {
                    if (cs + j0 + 32 <= P.ld_c) reinterpret_cast<uint4*>(dst)[1] = src[1];
                    else for (int jj = 16; jj < nl; ++jj) dst[jj] = chb[j0 + jj];
                }
            }
            bad |= (vmin < 0.0f || !(aCs <= DBL_MAX)) ? 1 : 0;
            const bool any_bad = __any_sync(kFull, bad != 0);
            const bool any_fit = __any_sync(kFull, fit_bad != 0);
            if (any_bad) status = CHASE_ERR_DATA;
            else if (any_fit && status == 0) status = CHASE_ERR_FIT;
            if (status == 0) {
                // baseline: sum of c over the windows before mb
                double Cbt = 0.0;
                if (cs + nw <= mb) Cbt = aCs;
                else if (cs < mb) Cbt = (j0 + nl <= mb - cs) ? aCs : 0.0;  // lanes wholly before mb
                if (cs < mb && mb < cs + nw) {  // the lane holding mb: its partial sum (cold)
                    const int src = (mb - cs) / kRRun;
                    if (lane == src) {
                        double s = 0.0;
                        for (int jj = 0; jj < mb - cs - j0; ++jj) s = __dadd_rn(s, (double)sb[s0 + cs + j0 + jj - a0]);
                        Cbt = s;
                    }
                }
                Cbl = __dadd_rn(Cbl, Cbt);
                bool completes = false;
                if (!done && ch >= c_may) completes = warp_sum(__dadd_rn(Sl, aS)) >= J;
                if (completes) {
                    // the lane holding the completion window: warp scan of the lanes' sums
                    const double S_prev = warp_sum(Sl);
                    const double incl = warp_incl_scan(aS, lane);
                    const double ex = __shfl_up_sync(kFull, incl, 1);
                    const double before = __dadd_rn(S_prev, lane == 0 ? 0.0 : ex);
                    const unsigned who = __ballot_sync(kFull, nl > 0 && before < J && __dadd_rn(before, aS) >= J);
                    if (who != 0) {
                        const int src = __ffs(who) - 1;
                        const bool full = lane < src;
                        const double Eb = warp_sum(full ? __dadd_rn(El, aE) : El);
                        const double Cb = warp_sum(full ? __dadd_rn(Cl, aC) : Cl);
                        const int nsrc = max(0, min(kRRun, nw - kRRun * src));
                        const LCompletion cp = run_completion(sb + (s0 + cs + kRRun * src - a0), chb + kRRun * src,
                                                               nsrc, __shfl_sync(kFull, before, src), J, pf, lane);
                        if (cp.w >= 0 && lane == 0) {
                            double* o = P.raw + i * kRawDoubles;
                            o[0] = __dadd_rn(Eb, cp.Ep);
                            o[1] = __dadd_rn(Cb, cp.Cp);
                            o[2] = J;
                            o[3] = cp.f;
                            o[4] = (double)((int64_t)L + cs + kRRun * src + cp.w);
                            o[5] = cp.Pk;
                            o[6] = cp.cw;
                            o[7] = 1.0;
                        }
                        if (__shfl_sync(kFull, cp.w, 0) >= 0) done = true;
                    }
                }
                if (!done) {
                    Sl = __dadd_rn(Sl, aS);
                    El = __dadd_rn(El, aE);
                    Cl = __dadd_rn(Cl, aC);
                }
            }
            __syncwarp();
            issue();  // this slot is free again
            if (ch == n_chunks - 1) {  // ---- end of trace
                if (status == 0) {
                    const double t4 = warp_sum4(Sl, El, Cl, Cbl, lane);
                    const double Ex = __shfl_sync(kFull, t4, 8), Cx = __shfl_sync(kFull, t4, 16);
                    const double Cb = __shfl_sync(kFull, t4, 24);
                    if (lane == 0) {
                        P.records[i * kRecDoubles + 9] = Cb;
                        if (!done) {
                            double* o = P.raw + i * kRawDoubles;
                            o[0] = Ex;
                            o[1] = Cx;
                            o[2] = t4;
                            o[3] = 0.0;
                            o[4] = -1.0;
                            o[5] = o[6] = o[7] = 0.0;
                        }
                    }
                }
                if (lane == 0) {
                    P.status[i] = (uint8_t)status;
                    if (status != 0) {
                        const unsigned long long slot =
                            atomicAdd(reinterpret_cast<unsigned long long*>(&P.diag->n_bad), 1ull);
                        P.bad_list[slot] = i;
                        atomicMin(reinterpret_cast<unsigned long long*>(&P.diag->first_bad_trace),
                                  (unsigned long long)i);
                    }
                }
            }
        }
    }
    n_slow = __reduce_add_sync(kFull, n_slow);
    if (lane == 0 && n_slow)
        atomicAdd(reinterpret_cast<unsigned long long*>(&P.diag->n_slow_windows), (unsigned long long)n_slow);
}
