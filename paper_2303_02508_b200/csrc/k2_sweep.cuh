// sweep.cuh — the fused planner kernel (K2), included by kernels.cu inside its
// anonymous namespace.
//
// Warp-per-trace streaming.  Every warp of a persistent CTA owns whole traces
// (trace i -> global warp i mod #warps) and streams each one in chunks of
// kWarpW = 32 x 36 windows through its own 2-stage TMA ring (cp.async.bulk +
// mbarrier, issued by lane 0), so there is no CTA-wide barrier in the steady
// state.  Lane l plans windows [36 l, 36 l + 36) of a chunk:
//   predict (Eq. 1) -> Eq. 6 argmin via the exact envelope bucket table
//   (canonical K-way path deferred for windows in a rounding band) ->
//   fixed-work replay partials (sum Thr*Delta, sum P, sum P*c; sum c)
// then one transposed warp reduction per chunk and eta.  The chunk that
// completes the job (once per trace and eta) runs a warp scan and the lane
// holding the completion window re-walks its 36 windows.  Choices are staged
// per warp in smem and bulk-stored (cp.async.bulk.global.shared).

struct Acc {
    double S, E, C, Cs;  // sum s_k, sum P_k, sum P_k*c, sum c (every window: validation + baseline)
    float vmin;          // min raw value (fast path validation; NaN/inf show up in Cs)
    uint32_t slow;       // OR of staged choice words: bit 5 of a byte = kZeroLine (deferred window)
    int bad;             // generic path validation (1) / REPLAY bad choice (2)
    int bad_pad;         // canonical-path window count (diagnostic)
};

// Full 16-byte-aligned fp32 groups of 4 windows: the hot loop.
// tv[jj] = c[w0 + jj] (tv[-1] = lag of the first window), Ap[jj] = A(phi0+jj).
template <bool FIRST, bool FC>
__device__ __forceinline__ void fused_full(const float* __restrict__ tv, int ngroups, const double* __restrict__ Ap,
                                           double wl, double invK, const PairTable* __restrict__ pt,
                                           const double2* __restrict__ lines, uint32_t* __restrict__ words,
                                           double* __restrict__ fout, Acc& a) {
    double lag = (double)tv[-1];
    // the A terms (or, FIN, the forecasts in global memory) of group g+1 load during group g
    double2 A01n = ngroups > 0 ? *reinterpret_cast<const double2*>(Ap) : make_double2(0.0, 0.0);
    double2 A23n = ngroups > 0 ? *reinterpret_cast<const double2*>(Ap + 2) : make_double2(0.0, 0.0);
#pragma unroll 1
    for (int g = 0; g < ngroups; ++g) {
        const float4 v = *reinterpret_cast<const float4*>(tv + 4 * g);
        if (FIRST) a.vmin = fminf(fminf(fminf(a.vmin, v.x), v.y), fminf(v.z, v.w));  // FMNMX3 x2
        const double2 A01 = A01n, A23 = A23n;
        if (g + 1 < ngroups) {
            A01n = *reinterpret_cast<const double2*>(Ap + 4 * g + 4);
            A23n = *reinterpret_cast<const double2*>(Ap + 4 * g + 6);
        }
        const float vv[4] = {v.x, v.y, v.z, v.w};
        const double AA[4] = {A01.x, A01.y, A23.x, A23.y};
        uint32_t word = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double cw = (double)vv[u];
            const double p = __dadd_rn(AA[u], __dmul_rn(wl, lag));  // Eq. 1, unclamped for the lookup
            if (FC) fout[4 * g + u] = p > 0.0 ? p : 0.0;
            const uint32_t k = plan_lookup(__dmul_rn(p, invK), pt);
            word |= k << (8 * u);
            const double2 ln = lines[k];  // (Thr_k * Delta, P_k)
            a.S = __dadd_rn(a.S, ln.x);
            a.E = __dadd_rn(a.E, ln.y);
            a.C = __dadd_rn(a.C, __dmul_rn(ln.y, cw));
            if (FIRST) a.Cs = __dadd_rn(a.Cs, cw);
            lag = cw;
        }
        words[g] = word;
        a.slow |= word;
    }
}

// Any element type / alignment / window count (odd L, f64, ragged tails).
// Out of line (cold); returns its partial sums by value so the caller's
// accumulators stay in registers.
template <bool FIRST, bool FC, typename E, bool CANON = false>
__device__ __noinline__ Acc fused_generic(const E* tv, int j_begin, int nwin, const double* Ap, double wl, double invK,
                                          const PairTable* pt, const double2* lines, uint8_t* bytes, double* fout,
                                          double Kc = 0.0, const ProfileTable* pf = nullptr) {
    Acc a{0.0, 0.0, 0.0, 0.0, FLT_MAX, 0u, 0, 0};
    double lag = (double)tv[j_begin - 1];
    for (int jj = j_begin; jj < nwin; ++jj) {
        const E raw = tv[jj];
        const double cw = (double)raw;
        const double p = __dadd_rn(Ap[jj], __dmul_rn(wl, lag));
        if (FC) fout[jj] = p > 0.0 ? p : 0.0;
        uint32_t k;
        if (CANON) {
            k = canonical_choose(p > 0.0 ? p : 0.0, Kc, pt->a, pf->thr, pf->K);
            ++a.bad_pad;
        } else {
            k = plan_lookup(__dmul_rn(p, invK), pt);
            if (k == (uint32_t)kZeroLine) a.slow |= 0x20u;
        }
        bytes[jj] = (uint8_t)k;
        const double2 ln = lines[k];
        a.S = __dadd_rn(a.S, ln.x);
        a.E = __dadd_rn(a.E, ln.y);
        a.C = __dadd_rn(a.C, __dmul_rn(ln.y, cw));
        if (FIRST) {
            a.Cs = __dadd_rn(a.Cs, cw);
            a.bad |= bad_value(raw) ? 1 : 0;
        }
        lag = cw;
    }
    return a;
}

__device__ __forceinline__ void acc_merge(Acc& a, const Acc& b) {
    a.S = __dadd_rn(a.S, b.S);
    a.E = __dadd_rn(a.E, b.E);
    a.C = __dadd_rn(a.C, b.C);
    a.Cs = __dadd_rn(a.Cs, b.Cs);
    a.slow |= b.slow;
    a.bad |= b.bad;
    a.bad_pad += b.bad_pad;
}

// The deferred windows (kZeroLine): canonical K-way Eq. 6, then their replay
// contributions (exact for dyadic inputs in any order).  Returns
// the corrections by value so the accumulators stay in registers.
struct SlowFix {
    double S, E, C;
    int n;
};
template <typename E>
__device__ __noinline__ SlowFix fix_slow(const E* tv, int nwin, const double* Ap, double wl, double Kc,
                                         const PairTable* pt, const ProfileTable* pf, uint8_t* bytes) {
    SlowFix r{0.0, 0.0, 0.0, 0};
    for (int jj = 0; jj < nwin; ++jj) {
        if (bytes[jj] != (uint8_t)kZeroLine) continue;
        const double x = predict(Ap[jj], wl, (double)tv[jj - 1]);
        const uint32_t k = canonical_choose(x, Kc, pt->a, pf->thr, pf->K);
        bytes[jj] = (uint8_t)k;
        const double2 ln = pf->line[k];
        const double cw = (double)tv[jj];
        r.S = __dadd_rn(r.S, ln.x);
        r.E = __dadd_rn(r.E, ln.y);
        r.C = __dadd_rn(r.C, __dmul_rn(ln.y, cw));
        ++r.n;
    }
    return r;
}

template <typename E>
__device__ void predict_chunk(const E* tv, int nwin, const double* Ap, double wl, double* fout, Acc& a) {
    double lag = nwin > 0 ? (double)tv[-1] : 0.0;
    for (int jj = 0; jj < nwin; ++jj) {
        const E raw = tv[jj];
        fout[jj] = predict(Ap[jj], wl, lag);
        a.bad |= bad_value(raw) ? 1 : 0;
        lag = (double)raw;
    }
}

template <bool FIRST, typename E>
__device__ void replay_chunk(const E* tv, int nwin, const uint8_t* cin, int K, const double2* lines, uint8_t* bytes,
                             Acc& a) {
    for (int jj = 0; jj < nwin; ++jj) {
        uint32_t k = cin[jj];
        if (k >= (uint32_t)K) {
            a.bad |= 2;
            k = 0;
        }
        bytes[jj] = (uint8_t)k;
        const E raw = tv[jj];
        const double cw = (double)raw;
        const double2 ln = lines[k];
        a.S = __dadd_rn(a.S, ln.x);
        a.E = __dadd_rn(a.E, ln.y);
        a.C = __dadd_rn(a.C, __dmul_rn(ln.y, cw));
        if (FIRST) {
            a.Cs = __dadd_rn(a.Cs, cw);
            a.bad |= bad_value(raw) ? 1 : 0;
        }
    }
}

template <typename E>
__device__ bool chunk_has_bad(const E* tv, int nwin) {
    bool b = false;
    for (int jj = 0; jj < nwin; ++jj) b |= bad_value(tv[jj]);
    return b;
}

// ---- shared-memory plan: tables | per warp {A tables, 2 stages, 2 choice buffers, state, mbarriers}
__host__ __device__ inline int aext_len(int T) { return T + kChunk + 4; }

// per eta (warp-uniform): Kc, 1/Kc, done, S_run, E_run, C_run, Cb_run, -
// (the running sums are used by the multi-eta path; the single-eta path keeps
// per-lane running sums in registers and reduces only when it must)
constexpr int kEtaState = 8;
#ifndef CHASE_STAGES
#define CHASE_STAGES 2  // 3 before: 2 is faster on the FIN paths (C4 SVR step 46.3 -> 43.6 ms, rolling R=24 16.7 -> 14.0 ms)
#endif
constexpr int kStages = CHASE_STAGES;  // per-warp TMA ring depth

struct WarpLayout {
    int aext, stage, chb, eta, ctx, mbar, bytes;
};

// Producer cursor and counters, kept in smem (lane 0 reads/writes them once
// per chunk) so they do not occupy registers across the hot loop.
struct WarpCtx {
    const void* psrc;       // next chunk's first element
    int64_t pi;             // next trace to load
    int32_t pc;             // next chunk index
    uint32_t issued;        // loads issued so far (stage parity)
    unsigned long long slow;  // deferred-window count
    int64_t reserved;
};

__host__ __device__ inline WarpLayout make_warp_layout(int T, int stage_bytes, int n_eta) {
    WarpLayout L;
    int o = 0;
    L.aext = o; o += 2 * round16(aext_len(T) * 8);
    L.stage = o; o += kStages * stage_bytes;
    L.chb = o; o += kWarpW;
    L.eta = o; o += n_eta * kEtaState * 8;
    L.ctx = o; o += (int)sizeof(WarpCtx);
    L.mbar = o; o += 8 * kStages;
    L.bytes = round16(o);
    return L;
}

__host__ __device__ inline int sweep_smem_total(int tables_bytes, int T, int stage_bytes, int n_eta) {
    return round16(tables_bytes) + kWarpsPerCta * make_warp_layout(T, stage_bytes, n_eta).bytes;
}

// Warp-parallel search for the completion window inside lane `src`'s
// windows: 32 windows per round, inclusive scan of s_k = Thr_k*Delta from
// `before` (the samples done before them).  Returns the window (relative to
// the lane's first), f, and E/C of the windows before it.
struct Completion {
    double f, Ep, Cp, Pk, cw;
    int w;
};
template <typename E>
__device__ __noinline__ Completion find_completion(const E* tv_src, const uint8_t* bytes_src, int nwin_src,
                                                   double before, double J, const double2* lines, int lane) {
    Completion r{1.0, 0.0, 0.0, 0.0, 0.0, nwin_src - 1};
    double carry = before;
    for (int r0 = 0; r0 < nwin_src; r0 += 32) {
        const int jj = r0 + lane;
        const bool valid = jj < nwin_src;
        const uint32_t k = valid ? bytes_src[jj] : 0u;
        const double2 ln = valid ? lines[k] : make_double2(0.0, 0.0);
        const double cw = valid ? (double)tv_src[jj] : 0.0;
        const double incl = __dadd_rn(carry, warp_incl_scan(ln.x, lane));
        const double prev = __shfl_up_sync(kFull, incl, 1);
        const double before_w = lane == 0 ? carry : prev;
        const unsigned hits = __ballot_sync(kFull, valid && incl >= J);
        const bool is_last = r0 + 32 >= nwin_src;
        const int wl_ = hits ? __ffs(hits) - 1 : (is_last ? min(31, nwin_src - 1 - r0) : 32);
        const bool pre = valid && lane < wl_;  // windows strictly before the completion window
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

// FIN (rolling refit): the forecasts come from P.fc_in (rolling_forecast_kernel)
// instead of the per-trace folded table: Ap = that row, w_lag = 0, so p = fc + 0*lag = fc.
template <int MODE, typename E, bool AL, bool MULTI, bool FIN = false>
#ifndef CHASE_SWEEP_MINB
#define CHASE_SWEEP_MINB 2
#endif
__global__ void __launch_bounds__(kThreads, CHASE_SWEEP_MINB) sweep_kernel(const __grid_constant__ SweepParams P) {
    mark_path(P.diag, FIN ? (CHASE_PATH_GENERAL | CHASE_PATH_FC_IN) : CHASE_PATH_GENERAL);
    extern __shared__ __align__(128) uint8_t sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const WarpLayout WL = make_warp_layout(P.T, P.stage_bytes, P.n_eta);
    uint8_t* wbase = sm + round16(P.tables_bytes) + warp * WL.bytes;
    const int alen = round16(aext_len(P.T) * 8) / 8;
    double* A_even = reinterpret_cast<double*>(wbase + WL.aext);
    double* A_odd = A_even + alen;
    uint8_t* stage0 = wbase + WL.stage;
    uint8_t* chb0 = wbase + WL.chb;
    double* eta_st = reinterpret_cast<double*>(wbase + WL.eta);
    WarpCtx* ctx = reinterpret_cast<WarpCtx*>(wbase + WL.ctx);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(wbase + WL.mbar);

    {   // constant tables -> smem (16-byte vectors), once per CTA
        const uint4* src = reinterpret_cast<const uint4*>(P.tables);
        uint4* dst = reinterpret_cast<uint4*>(sm);
        for (int q = tid; q < P.tables_bytes / 16; q += kThreads) dst[q] = src[q];
    }
    if (lane == 0) {
        for (int q0 = 0; q0 < kStages; ++q0) mbar_init(&mbar[q0], 1);
        fence_mbar_init();
    }
    __syncthreads();  // the only CTA-wide barrier

    const TablesHeader* H = reinterpret_cast<const TablesHeader*>(sm);
    const double* phS = reinterpret_cast<const double*>(sm + H->off_phase);
    const double* phC = phS + P.T;
    const ProfileTable* profs = reinterpret_cast<const ProfileTable*>(sm + H->off_prof);
    const PairTable* pairs = reinterpret_cast<const PairTable*>(sm + H->off_pair);

    const int64_t GW = (int64_t)gridDim.x * kWarpsPerCta;
    const int64_t gw = (int64_t)blockIdx.x * kWarpsPerCta + warp;
    const int n_pass = MODE == MODE_PREDICT ? 1 : P.n_eta;
    const E* traces = reinterpret_cast<const E*>(P.traces);
    const int nc = P.n_chunks;
    const int T = P.T;
    const int W_last = P.W_last;  // windows of the last chunk
    const int a0 = P.a0;          // chunk c loads elements [a0 + c*kWarpW, ...), 16-byte aligned
    const int off0 = P.off0;      // tv = stage + off0 elements

    // producer (lane 0): next (trace, chunk) to load; cursor lives in smem
    auto issue_next = [&]() {
        const int64_t pi = ctx->pi;
        if (pi >= P.n_traces) return;
        const int pc = ctx->pc;
        const uint32_t issued = ctx->issued;
        const E* psrc = reinterpret_cast<const E*>(ctx->psrc);
        const uint64_t policy = evict_first_policy();
        const int st = (int)(issued % kStages);
        uint8_t* dst = stage0 + st * P.stage_bytes;
        const uint32_t bytes = pc == nc - 1 ? P.bytes_last : P.bytes_full;
        if (pc == 0) {
            mbar_arrive_expect_tx(&mbar[st], bytes + (uint32_t)kRecBytes);
            bulk_g2s(dst + P.stage_bytes - kRecBytes, P.records + pi * kRecDoubles, kRecBytes, &mbar[st], policy);
        } else {
            mbar_arrive_expect_tx(&mbar[st], bytes);
        }
        CHASE_CHECK(bytes + (P.stage_bytes > kRecBytes ? kRecBytes : 0) <= (uint32_t)P.stage_bytes);
        bulk_g2s(dst, psrc, bytes, &mbar[st], policy);
        ctx->issued = issued + 1;
        if (pc + 1 == nc) {
            ctx->pc = 0;
            ctx->pi = pi + GW;
            ctx->psrc = traces + (pi + GW) * P.ld + a0;
        } else {
            ctx->pc = pc + 1;
            ctx->psrc = psrc + kWarpW;
        }
    };
    if (lane == 0) {
        ctx->pi = gw;
        ctx->pc = 0;
        ctx->issued = 0;
        ctx->psrc = traces + gw * P.ld + a0;
        ctx->slow = 0ull;
        for (int q0 = 0; q0 < kStages; ++q0) issue_next();
    }

    const int lane_phase = (kChunk * lane) % T;
    const int j0 = kChunk * lane;
    uint32_t q = 0;

    double Sl = 0.0, El = 0.0, Cl = 0.0, Cbl = 0.0;  // single-eta path: per-lane running sums
    for (int64_t i = gw; i < P.n_traces; i += GW) {
        int status = 0, prof = 0;
        double wl = 0.0, J = 0.0, smax = 0.0;
        int64_t mb = P.W;
        int phase_c = P.phase_start;
        for (int c = 0; c < nc; ++c, ++q) {
            const int st = (int)(q % kStages);
            uint8_t* stage = stage0 + st * P.stage_bytes;
            mbar_wait(&mbar[st], (q / kStages) & 1);
            if (c == 0) {  // ---- per-trace setup (warp-uniform)
                const double* rec = reinterpret_cast<const double*>(stage + P.stage_bytes - kRecBytes);
                prof = P.profile_id ? (int)P.profile_id[i] : 0;
                if (prof >= P.n_prof) prof = 0;
                smax = profs[prof].smax;
                J = P.job ? P.job[i] : 0.0;
                status = (int)rec[5];
                wl = FIN ? 0.0 : rec[3];
                const double maxci = P.max_ci_fixed > 0.0 ? P.max_ci_fixed : rec[4];
                if (status == 0 && MODE == MODE_FUSED && !(maxci > 0.0)) status = CHASE_ERR_MAXCI;
                const int64_t m = (int64_t)rec[8];
                mb = (J > 0.0 && m >= 1 && m <= P.W) ? m - 1 : P.W;
                if (status == 0 && MODE != MODE_REPLAY && !FIN) {
                    const double c0 = rec[0], wsn = rec[1], wcs = rec[2];
                    const int n_a = aext_len(T);
                    int ph = lane % T;
                    for (int j = lane; j < n_a; j += 32) {
                        // A(phi) = (c0 + w_sin*S[phi]) + w_cos*C[phi]  (canonical fold of Eq. 1)
                        const int ph1 = ph + 1 == T ? 0 : ph + 1;
                        A_even[j] = __dadd_rn(__dadd_rn(c0, __dmul_rn(wsn, phS[ph])), __dmul_rn(wcs, phC[ph]));
                        A_odd[j] = __dadd_rn(__dadd_rn(c0, __dmul_rn(wsn, phS[ph1])), __dmul_rn(wcs, phC[ph1]));
                        ph += 32;
                        while (ph >= T) ph -= T;
                    }
                }
                if (lane < n_pass) {  // Kc and 1/Kc once per trace and eta
                    const PairTable* pt = pairs + prof * P.n_eta + lane;
                    const double Kc = __dmul_rn(pt->kbase, maxci);
                    double* es = eta_st + lane * kEtaState;
                    es[0] = Kc;
                    es[1] = per_trace_invK(pt, Kc);
                    es[2] = es[3] = es[4] = es[5] = es[6] = 0.0;
                }
                Sl = El = Cl = Cbl = 0.0;
                __syncwarp();
            } else {
                phase_c += P.phase_step;
                if (phase_c >= T) phase_c -= T;
            }

            const int nwin = c < nc - 1 ? kChunk : max(0, min(kChunk, W_last - j0));
            const E* tv = reinterpret_cast<const E*>(stage) + off0 + j0;  // tv[jj] = c[w0 + jj]
            int phi0 = phase_c + lane_phase;                              // phase of my first window
            if (phi0 >= T) phi0 -= T;
            const int64_t jb = (int64_t)c * kWarpW + j0;                  // my first window, from s0
            const double* Ap = FIN ? P.fc_in + i * P.ld_fin + jb
                                   : ((phi0 & 1) ? A_odd + (phi0 - 1) : A_even + phi0);  // 16-byte aligned
            // samples cannot reach J before this many windows: skip the completion test until then
            const int64_t w_through = min((int64_t)P.W, (int64_t)(c + 1) * kWarpW);
            const bool may_complete = J > 0.0 && __dmul_rn(__dmul_rn((double)w_through, smax), 1.000001) >= J;

            if (status == CHASE_ERR_MAXCI || status == CHASE_ERR_FIT) {
                // S:29 precedence: a bad value anywhere makes the trace status 4
                if (__any_sync(kFull, chunk_has_bad(tv, nwin))) status = CHASE_ERR_DATA;
            }

            for (int e = 0; e < n_pass && status == 0; ++e) {
                uint8_t* chb = chb0;
                if (MODE != MODE_PREDICT) __syncwarp();  // every lane finished reading the choice buffer
                double* es = eta_st + e * kEtaState;
                const double Kc = es[0], invK = es[1];
                const bool done = es[2] != 0.0;
                const PairTable* pt = pairs + prof * P.n_eta + e;
                const ProfileTable* pf = profs + prof;

                Acc a{0.0, 0.0, 0.0, 0.0, FLT_MAX, 0u, 0, 0};
                int fast_groups = 0;
                if (MODE == MODE_FUSED) {
                    double* fout = (P.forecast && e == 0) ? P.forecast + i * P.ld_f + jb : nullptr;
                    if (invK == 0.0) {
                        // Kc outside [2^-900, 2^900]: every window on the canonical rule (cold)
                        Acc b;
                        if (e == 0 && fout) b = fused_generic<true, true, E, true>(tv, 0, nwin, Ap, wl, invK, pt, pf->line, chb + j0, fout, Kc, pf);
                        else if (e == 0) b = fused_generic<true, false, E, true>(tv, 0, nwin, Ap, wl, invK, pt, pf->line, chb + j0, fout, Kc, pf);
                        else b = fused_generic<false, false, E, true>(tv, 0, nwin, Ap, wl, invK, pt, pf->line, chb + j0, fout, Kc, pf);
                        acc_merge(a, b);
                        if (b.bad_pad) atomicAdd(&ctx->slow, (unsigned long long)b.bad_pad);
                    } else {
                    if (AL && sizeof(E) == 4) {
                        fast_groups = nwin >> 2;
                        const float* tf = reinterpret_cast<const float*>(tv);
                        uint32_t* words = reinterpret_cast<uint32_t*>(chb + j0);
                        if (e == 0) {
                            if (fout) fused_full<true, true>(tf, fast_groups, Ap, wl, invK, pt, pf->line, words, fout, a);
                            else fused_full<true, false>(tf, fast_groups, Ap, wl, invK, pt, pf->line, words, fout, a);
                        } else {
                            fused_full<false, false>(tf, fast_groups, Ap, wl, invK, pt, pf->line, words, fout, a);
                        }
                    }
                    if (4 * fast_groups < nwin) {
                        Acc b;
                        if (e == 0) {
                            if (fout) b = fused_generic<true, true, E>(tv, 4 * fast_groups, nwin, Ap, wl, invK, pt, pf->line, chb + j0, fout);
                            else b = fused_generic<true, false, E>(tv, 4 * fast_groups, nwin, Ap, wl, invK, pt, pf->line, chb + j0, fout);
                        } else {
                            b = fused_generic<false, false, E>(tv, 4 * fast_groups, nwin, Ap, wl, invK, pt, pf->line, chb + j0, fout);
                        }
                        acc_merge(a, b);
                    }
                    if (a.slow & 0x20202020u) {
                        const SlowFix fx = fix_slow<E>(tv, nwin, Ap, wl, Kc, pt, pf, chb + j0);
                        a.S = __dadd_rn(a.S, fx.S);
                        a.E = __dadd_rn(a.E, fx.E);
                        a.C = __dadd_rn(a.C, fx.C);
                        atomicAdd(&ctx->slow, (unsigned long long)fx.n);
                    }
                    }
                } else if (MODE == MODE_PREDICT) {
                    if (FIN) a.bad |= chunk_has_bad(tv, nwin) ? 1 : 0;  // rolling: forecasts already written
                    else predict_chunk<E>(tv, nwin, Ap, wl, P.forecast + i * P.ld_f + jb, a);
                } else {
                    const uint8_t* cin = P.choice_in + ((int64_t)e * P.n_traces + i) * P.ld_c + jb;
                    if (e == 0) replay_chunk<true, E>(tv, nwin, cin, pf->K, pf->line, chb + j0, a);
                    else replay_chunk<false, E>(tv, nwin, cin, pf->K, pf->line, chb + j0, a);
                }

                int flag = a.bad;
                if (e == 0 && fast_groups > 0 && (!(a.vmin >= 0.0f) || !(a.Cs <= DBL_MAX))) flag |= 1;
                flag = (int)__reduce_or_sync(kFull, (unsigned)flag);
                if (flag) {
                    status = (flag & 1) ? CHASE_ERR_DATA : CHASE_ERR_CHOICE;
                    break;
                }
                if (MODE == MODE_FUSED && P.choice) {
                    // coalesced 16-byte copies of the staged choices (bytes [W, round16(W)) are scratch)
                    __syncwarp();
                    uint4* dst = reinterpret_cast<uint4*>(P.choice + ((int64_t)e * P.n_traces + i) * P.ld_c +
                                                          (int64_t)c * kWarpW);
                    const uint4* srcv = reinterpret_cast<const uint4*>(chb);
                    const int n16 = (c < nc - 1 ? kWarpW : W_last + 15) >> 4;
                    for (int q16 = lane; q16 < n16; q16 += 32) st_na_v4(dst + q16, srcv[q16]);
                }
                if (MODE == MODE_PREDICT) continue;

                double Cbt = 0.0;  // baseline: sum of c over the windows before w*_b
                if (e == 0) {
                    if (jb + nwin <= mb) Cbt = a.Cs;
                    else if (jb < mb)
                        for (int jj = 0; jj < (int)(mb - jb); ++jj) Cbt = __dadd_rn(Cbt, (double)tv[jj]);
                }
                if constexpr (!MULTI) {
                    // ---- one eta: per-lane running sums; warp sums only where the job can complete
                    Cbl = __dadd_rn(Cbl, Cbt);
                    if (!done && may_complete) {
                        const double S_prev = warp_sum(Sl);
                        if (__dadd_rn(S_prev, warp_sum(a.S)) >= J) {
                            const double incl = warp_incl_scan(a.S, lane);
                            const double ex = __shfl_up_sync(kFull, incl, 1);
                            const double before = __dadd_rn(S_prev, lane == 0 ? 0.0 : ex);
                            const bool full = __dadd_rn(before, a.S) < J;
                            const unsigned who = __ballot_sync(kFull, !full && before < J && nwin > 0);
                            if (who != 0) {
                                const double Eb = warp_sum(full ? __dadd_rn(El, a.E) : El);
                                const double Cb = warp_sum(full ? __dadd_rn(Cl, a.C) : Cl);
                                const int src = __ffs(who) - 1;
                                const int nw_src = c < nc - 1 ? kChunk : max(0, min(kChunk, W_last - kChunk * src));
                                const Completion cp = find_completion<E>(tv + kChunk * (src - lane), chb + kChunk * src,
                                                                         nw_src, __shfl_sync(kFull, before, src), J,
                                                                         pf->line, lane);
                                const int wrel = cp.w;
                                const double f = cp.f, Ep = cp.Ep, Cp = cp.Cp, Pk = cp.Pk, cst = cp.cw;
                                if (lane == 0) {
                                    double* r = P.raw + ((int64_t)e * P.n_traces + i) * kRawDoubles;
                                    r[0] = __dadd_rn(Eb, Ep);
                                    r[1] = __dadd_rn(Cb, Cp);
                                    r[2] = J;
                                    r[3] = f;
                                    r[4] = (double)((int64_t)P.L + (int64_t)c * kWarpW + kChunk * src + wrel);
                                    r[5] = Pk;
                                    r[6] = cst;
                                    r[7] = 1.0;
                                    es[2] = 1.0;
                                }
                                __syncwarp();
                                continue;
                            }
                            // no window reached J in the scan order (non-dyadic rounding): carry on
                        }
                    }
                    if (!done) {
                        Sl = __dadd_rn(Sl, a.S);
                        El = __dadd_rn(El, a.E);
                        Cl = __dadd_rn(Cl, a.C);
                    }
                } else {
                    // ---- several etas: per-chunk warp totals into the warp-uniform state
                    const double tot = warp_sum4(a.S, a.E, a.C, Cbt, lane);  // lanes 0, 8, 16, 24
                    const double S_tile = __shfl_sync(kFull, tot, 0);
                    const double S_run = es[3];
                    if (e == 0 && lane == 24) es[6] = __dadd_rn(es[6], tot);
                    bool carried = false;
                    if (!done && J > 0.0 && __dadd_rn(S_run, S_tile) >= J) {
                        const double incl = warp_incl_scan(a.S, lane);
                        const double ex = __shfl_up_sync(kFull, incl, 1);
                        const double before = __dadd_rn(S_run, lane == 0 ? 0.0 : ex);
                        const bool full = __dadd_rn(before, a.S) < J;
                        const unsigned who = __ballot_sync(kFull, !full && before < J && nwin > 0);
                        if (who != 0) {
                            const double Em = warp_sum(full ? a.E : 0.0), Cm = warp_sum(full ? a.C : 0.0);
                            const int src = __ffs(who) - 1;
                            const int nw_src = c < nc - 1 ? kChunk : max(0, min(kChunk, W_last - kChunk * src));
                            const Completion cp = find_completion<E>(tv + kChunk * (src - lane), chb + kChunk * src,
                                                                     nw_src, __shfl_sync(kFull, before, src), J,
                                                                     pf->line, lane);
                            const int wrel = cp.w;
                            const double f = cp.f, Ep = cp.Ep, Cp = cp.Cp, Pk = cp.Pk, cst = cp.cw;
                            if (lane == 0) {
                                double* r = P.raw + ((int64_t)e * P.n_traces + i) * kRawDoubles;
                                r[0] = __dadd_rn(__dadd_rn(es[4], Em), Ep);
                                r[1] = __dadd_rn(__dadd_rn(es[5], Cm), Cp);
                                r[2] = J;
                                r[3] = f;
                                r[4] = (double)((int64_t)P.L + (int64_t)c * kWarpW + kChunk * src + wrel);
                                r[5] = Pk;
                                r[6] = cst;
                                r[7] = 1.0;
                                es[2] = 1.0;
                            }
                            carried = true;
                        }
                    }
                    if (!done && !carried) {
                        if (lane == 0) es[3] = __dadd_rn(S_run, S_tile);
                        if (lane == 8) es[4] = __dadd_rn(es[4], tot);
                        if (lane == 16) es[5] = __dadd_rn(es[5], tot);
                    }
                    __syncwarp();
                }
            }

            if (c == nc - 1) {  // ---- end of trace: totals of the jobs that did not complete
                if (MODE != MODE_PREDICT && status == 0) {
                    if constexpr (!MULTI) {
                        const double Cb = warp_sum(Cbl);
                        const bool done = eta_st[2] != 0.0;
                        const double Sx = warp_sum(Sl), Ex = warp_sum(El), Cx = warp_sum(Cl);
                        if (lane == 0) {
                            P.records[i * kRecDoubles + 9] = Cb;
                            if (!done) {
                                double* r = P.raw + i * kRawDoubles;
                                r[0] = Ex;
                                r[1] = Cx;
                                r[2] = Sx;
                                r[3] = 0.0;
                                r[4] = -1.0;
                                r[5] = r[6] = r[7] = 0.0;
                            }
                        }
                    } else if (lane == 0) {
                        P.records[i * kRecDoubles + 9] = eta_st[6];
                        for (int e = 0; e < n_pass; ++e) {
                            const double* es = eta_st + e * kEtaState;
                            if (es[2] != 0.0) continue;
                            double* r = P.raw + ((int64_t)e * P.n_traces + i) * kRawDoubles;
                            r[0] = es[4];
                            r[1] = es[5];
                            r[2] = es[3];
                            r[3] = 0.0;
                            r[4] = -1.0;
                            r[5] = r[6] = r[7] = 0.0;
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
            __syncwarp();  // every lane is done with stage `st`
            if (lane == 0) issue_next();
        }
    }

    if (lane == 0) {
        if (ctx->slow) atomicAdd(reinterpret_cast<unsigned long long*>(&P.diag->n_slow_windows), ctx->slow);
    }
}
