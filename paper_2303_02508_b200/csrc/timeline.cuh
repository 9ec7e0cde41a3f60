// timeline.cuh — timeline / audit rows of a planned replay,
// included by kernels.cu inside its anonymous namespace.
//
// SPEC emit_timeline (Figure 1/2 rows): one row per
// decision period {period_start, forecast_ci, actual_mean_ci, chosen_limit_w,
// avg_power_w, samples_done, energy_j, carbon_g}, the fixed-work replay of
// oracle_replay split by period (full windows count in full, the completion
// window by its fraction, later windows not at all).  One warp per selected
// trace, one lane per period, 32 periods per round: each lane sums its
// period's windows in order, a warp scan gives the samples done before every
// period, and the lane whose period holds the completion window re-walks it
// with the pro-rata rule.  oracle_timeline's per-period operation order.
struct TimelineParams {
    const void* traces;
    int64_t ld, n_traces;
    int32_t N, L, P, n_prof;
    double delta;
    const uint8_t* choice;   // [n][ld_c] (one eta) or null: the max-limit baseline
    int64_t ld_c;
    const double* forecast;  // [n][ld_f] or null
    int64_t ld_f;
    const uint8_t* tables;   // profiles (ProfileTable[n_prof] at H->off_prof)
    const uint8_t* profile_id;
    const double* job;
    const int64_t* ids;      // [m] or null: traces 0..m-1
    int64_t m;
    double* rows;            // [m][n_per][8]
    double* summary;         // [m][4] or null: {stepwise carbon g, Eq. 3 carbon g, AvgPower W, AvgCI g/kWh}
};

// Rows of a round are staged per warp in shared memory and leave as one TMA
// bulk store (32 rows = 2 KB, contiguous in the output), not as 8 strided
// 8-byte stores per lane.
template <typename E>
#ifndef CHASE_TL_MINB
#define CHASE_TL_MINB 8  // <= 64 registers: 8 CTAs per SM (C4 P=1: 19.4 -> 16.0 ms on one box)
#endif
__global__ void __launch_bounds__(128, CHASE_TL_MINB) timeline_kernel(const __grid_constant__ TimelineParams p) {
    __shared__ __align__(128) double tl_rows[4][32 * 8];
    const int lane = threadIdx.x & 31;
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (r >= p.m) return;
    double* st = tl_rows[threadIdx.x >> 5];
    const int64_t i = p.ids ? p.ids[r] : r;
    const int s0 = p.L, W = p.N - p.L, Pp = p.P;
    const int n_per = (W + Pp - 1) / Pp;
    if (i < 0 || i >= p.n_traces) {  // a trace id outside [0, n_traces): NaN rows (chase.h)
        double* o = p.rows + r * (int64_t)n_per * 8;
        for (int64_t q = lane; q < (int64_t)n_per * 8; q += 32) o[q] = CUDART_NAN;
        if (p.summary && lane < 4) p.summary[r * 4 + lane] = CUDART_NAN;
        return;
    }
    int prof = p.profile_id ? (int)p.profile_id[i] : 0;
    if (prof >= p.n_prof) prof = 0;
    const ProfileTable* pf = blob_profiles(p.tables) + prof;
    const E* row = reinterpret_cast<const E*>(p.traces) + i * p.ld;
    const uint8_t* ch = p.choice ? p.choice + i * p.ld_c : nullptr;
    const double J = p.job ? p.job[i] : 0.0;
    double S = 0.0;      // samples done before the current round (warp-uniform)
    bool done = false;
    double tE = 0.0, tC = 0.0, tcj = 0.0, ttw = 0.0;  // this lane's job totals (Eq. 3 summary)
    double* out = p.rows + r * (int64_t)n_per * 8;
    for (int j0 = 0; j0 < n_per; j0 += 32) {
        const int j = j0 + lane;
        const bool valid = j < n_per;
        const int b = j * Pp;
        const int n = valid ? min(Pp, W - b) : 0;
        double csum = 0.0, ssum = 0.0, esum = 0.0, psum = 0.0;  // full-window sums of the period
        for (int q = 0; q < n; ++q) {
            const double cw = (double)row[s0 + b + q];
            const int kw = ch ? ch[b + q] : pf->K - 1;
            const double2 ln = pf->line[kw];
            csum = __dadd_rn(csum, cw);
            ssum = __dadd_rn(ssum, ln.x);
            esum = __dadd_rn(esum, ln.y);
            psum = __dadd_rn(psum, __dmul_rn(ln.y, cw));
        }
        const double incl = warp_incl_scan(ssum, lane);
        const double ex = __shfl_up_sync(kFull, incl, 1);
        const double before = __dadd_rn(S, lane == 0 ? 0.0 : ex);  // samples done before period j
        // the period in which the running samples first reach J
        const bool hit = !done && valid && J > 0.0 && __dadd_rn(before, ssum) >= J;
        const unsigned hits = __ballot_sync(kFull, hit);
        const int first = hits ? __ffs(hits) - 1 : 32;
        double samples = ssum, E = esum, C = psum, cj = csum, tw = (double)n;
        if (done || lane > first) {
            samples = E = C = cj = tw = 0.0;
        } else if (lane == first) {  // re-walk the completion period window by window
            double Sr = before;
            samples = E = C = cj = tw = 0.0;
            for (int q = 0; q < n; ++q) {
                const double cw = (double)row[s0 + b + q];
                const int kw = ch ? ch[b + q] : pf->K - 1;
                const double2 ln = pf->line[kw];
                const double prevS = Sr;
                Sr = __dadd_rn(Sr, ln.x);
                if (Sr >= J) {
                    const double f = __ddiv_rn(__dsub_rn(J, prevS), ln.x);
                    samples = __dadd_rn(samples, __dsub_rn(J, prevS));
                    E = __dadd_rn(E, __dmul_rn(f, ln.y));
                    C = __dadd_rn(C, __dmul_rn(f, __dmul_rn(ln.y, cw)));
                    cj = __dadd_rn(cj, __dmul_rn(f, cw));
                    tw = __dadd_rn(tw, f);
                    break;
                }
                samples = __dadd_rn(samples, ln.x);
                E = __dadd_rn(E, ln.y);
                C = __dadd_rn(C, __dmul_rn(ln.y, cw));
                cj = __dadd_rn(cj, cw);
                tw = __dadd_rn(tw, 1.0);
            }
        }
        if (valid) {
            tE = __dadd_rn(tE, E);
            tC = __dadd_rn(tC, C);
            tcj = __dadd_rn(tcj, cj);
            ttw = __dadd_rn(ttw, tw);
        }
        if (j0 > 0 && lane == 0) bulk_wait_read0();  // the previous round's store has read the staging rows
        __syncwarp();
        if (valid) {
            const int k = ch ? ch[b] : pf->K - 1;
            double* o = st + lane * 8;
            o[0] = (double)(s0 + b);
            o[1] = p.forecast ? p.forecast[i * p.ld_f + b] : CUDART_NAN;
            o[2] = n == 1 ? csum : __ddiv_rn(csum, (double)n);  // x/1 = x exactly
            o[3] = (double)pf->limit_w[k];
            o[4] = pf->line[k].y;
            o[5] = samples;
            o[6] = __dmul_rn(E, p.delta);
            o[7] = __ddiv_rn(__dmul_rn(C, p.delta), 3.6e6);
        }
        __syncwarp();
        if (lane == 0) {
            fence_proxy_async();
            bulk_s2g(out + (int64_t)j0 * 8, st, (uint32_t)(min(32, n_per - j0) * 64));
            bulk_commit();
        }
        done = done || hits != 0;
        S = __dadd_rn(S, __shfl_sync(kFull, incl, 31));
    }
    if (p.summary) {  // Eq. 3 next to the stepwise carbon (oracle_job_summary; sums in warp order, <= 1e-9)
        tE = warp_sum(tE);
        tC = warp_sum(tC);
        tcj = warp_sum(tcj);
        ttw = warp_sum(ttw);
        if (lane == 0) {
            const double avg_ci = __ddiv_rn(tcj, ttw);
            double* o = p.summary + r * 4;
            o[0] = __ddiv_rn(__dmul_rn(tC, p.delta), 3.6e6);
            o[1] = __ddiv_rn(__dmul_rn(__dmul_rn(tE, p.delta), avg_ci), 3.6e6);
            o[2] = __ddiv_rn(tE, ttw);
            o[3] = avg_ci;
        }
    }
    if (lane == 0) bulk_wait_read0();  // the staging rows stay valid until the last store has read them
}

// Per-limit cost vectors behind the decisions (SPEC PeriodDecision S:296-297,
// Eq. 6), audit output: for selected trace r and period j,
// cost_k = ((a_k * chat) + Kc) / Thr_k with chat the period's decision value,
// a_k = eta P_k and Kc = ((1 - eta) Pmax) MaxCI -- the canonical rule's
// operations, so the chosen limit is the first minimum of its row.  One
// thread per (trace, period, k); rows padded to ld_k with NaN.
struct CostParams {
    const double* forecast;
    int64_t ld_f, n_traces;
    int32_t W, P, n_per, ld_k, n_prof;
    const uint8_t* tables;    // blob: profiles + one pair table per profile (eta[0])
    const uint8_t* profile_id;
    const double* max_ci;     // [n] or null (max_ci_fixed > 0)
    double max_ci_fixed;
    const int64_t* ids;
    int64_t m;
    double* costs;            // [m][n_per][ld_k]
};

__global__ void __launch_bounds__(256) period_cost_kernel(const __grid_constant__ CostParams p) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t per_row = (int64_t)p.n_per * p.ld_k;
    if (t >= p.m * per_row) return;
    const int64_t r = t / per_row;
    const int j = (int)((t - r * per_row) / p.ld_k);
    const int k = (int)(t - r * per_row - (int64_t)j * p.ld_k);
    const int64_t i = p.ids ? p.ids[r] : r;
    if (i < 0 || i >= p.n_traces) {  // a trace id outside [0, n_traces): NaN costs (chase.h)
        p.costs[t] = CUDART_NAN;
        return;
    }
    int prof = p.profile_id ? (int)p.profile_id[i] : 0;
    if (prof >= p.n_prof) prof = 0;
    const ProfileTable* pf = blob_profiles(p.tables) + prof;
    const TablesHeader* H = reinterpret_cast<const TablesHeader*>(p.tables);
    const PairTable* pt = reinterpret_cast<const PairTable*>(p.tables + H->off_pair) + prof;
    double v = CUDART_NAN;
    if (k < pf->K) {
        const double chat = p.forecast[i * p.ld_f + (int64_t)j * p.P];
        const double maxci = p.max_ci_fixed > 0.0 ? p.max_ci_fixed : p.max_ci[i];
        const double Kc = __dmul_rn(pt->kbase, maxci);
        v = __ddiv_rn(__dadd_rn(__dmul_rn(pt->a[k], chat), Kc), pf->thr[k]);
    }
    p.costs[t] = v;
}

// SPEC --count-profiling (DESIGN Q33): the profiling run before the job,
// one trace step per limit in increasing order over steps L-K .. L-1, each at
// the limit's average power.  One thread per trace: {time s, energy J,
// carbon g} in oracle_profiling_overhead's operation order.
template <typename E>
__global__ void __launch_bounds__(256) profiling_kernel(const void* traces, int64_t ld, int64_t n, int L,
                                                        double delta, const uint8_t* tables, int n_prof,
                                                        const uint8_t* profile_id, double* out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int prof = profile_id ? (int)profile_id[i] : 0;
    if (prof >= n_prof) prof = 0;
    const ProfileTable* pf = blob_profiles(tables) + prof;
    const E* row = reinterpret_cast<const E*>(traces) + i * ld;
    const int K = pf->K;
    double Ep = 0.0, Cp = 0.0;
    for (int k = 0; k < K; ++k) {
        const double P = pf->line[k].y;
        Ep = __dadd_rn(Ep, P);
        Cp = __dadd_rn(Cp, __dmul_rn(P, (double)row[L - K + k]));
    }
    out[3 * i] = __dmul_rn((double)K, delta);
    out[3 * i + 1] = __dmul_rn(Ep, delta);
    out[3 * i + 2] = __ddiv_rn(__dmul_rn(Cp, delta), 3.6e6);
}
