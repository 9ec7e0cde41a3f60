/*
 * oracle.c — plain CPU oracle for the Chase batched trace-replay planner.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Built with
 *   gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC
 * Every function follows the paper (P:n) / SPEC (S:n) step by step, in fp64,
 * one rounding per written operation, no blocking or reordering.
 *
 * Pins (tests/test_oracle_*.py) tie each function to something other than
 * itself: exact rational least squares (fractions), numpy lstsq, the SPEC
 * worked examples, closed forms, an exact-rational argmin away from ties,
 * brute-force replay in rationals, and invariants.  See DESIGN.md §4.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------- Eq. 2 */
/* sin_time(t) = sin(2*pi*t/T), cos_time(t) = cos(2*pi*t/T); the
 * phase of step t is anchored to UTC midnight (DESIGN Q3), so the
 * table is indexed by phi = (phase0 + t) mod T. */
void oracle_phase_table(int32_t T, double* S, double* Cc) {
    for (int32_t phi = 0; phi < T; ++phi) {
        double theta = (2.0 * M_PI * (double)phi) / (double)T;
        S[phi] = sin(theta);
        Cc[phi] = cos(theta);
    }
}

/* ---------------------------------------------------------------- Eq. 1 fit */
/* Cholesky of the m x m SPD matrix G (row-major 3x3 storage) into Lc;
 * returns 0 when some pivot d <= tol ("singularity"; DESIGN Q6). */
static int cholesky3(int m, const double G[3][3], double tol, double Lc[3][3]) {
    for (int j = 0; j < m; ++j) {
        double d = G[j][j];
        for (int k = 0; k < j; ++k) d = d - Lc[j][k] * Lc[j][k];
        if (!(d > tol)) return 0;
        Lc[j][j] = sqrt(d);
        for (int i = j + 1; i < m; ++i) {
            double v = G[i][j];
            for (int k = 0; k < j; ++k) v = v - Lc[i][k] * Lc[j][k];
            Lc[i][j] = v / Lc[j][j];
        }
    }
    return 1;
}

/* S:131-139 fit_linear: ordinary least squares on z-scored features via the
 * normal equations (S:196 standardisation, population sigma, DESIGN Q5),
 * ridge lambda = 1e-8 on singularity, constant target -> intercept
 * only, zero-variance columns dropped (DESIGN Q7). */
int32_t oracle_fit(const double* hist, int32_t L, int32_t T, int32_t phi0,
                   const double* S, const double* Cc,
                   double ridge_lambda, double singular_tol, oracle_model_t* m) {
    memset(m, 0, sizeof(*m));
    const int32_t n = L - 1;           /* L points give L-1 lagged rows (Q2) */
    const double dn = (double)n;

    /* F2: constant target */
    int constant = 1;
    for (int32_t i = 2; i <= n; ++i)
        if (hist[i] != hist[1]) { constant = 0; break; }
    if (constant) {
        m->kind = 1;
        m->c0 = hist[1];
        m->mu[3] = hist[1];
        return 0;
    }

    /* Row i (1..n): x = (S[phi], Cc[phi], hist[i-1]), y = hist[i]. */
    #define XS(i) S[((phi0) + (i)) % T]
    #define XC(i) Cc[((phi0) + (i)) % T]
    #define XL(i) hist[(i) - 1]
    #define Y(i)  hist[(i)]

    /* F3: sequential means ... */
    double sum[4] = {0.0, 0.0, 0.0, 0.0};
    for (int32_t i = 1; i <= n; ++i) {
        sum[0] = sum[0] + XS(i);
        sum[1] = sum[1] + XC(i);
        sum[2] = sum[2] + XL(i);
        sum[3] = sum[3] + Y(i);
    }
    double mu[4];
    for (int j = 0; j < 4; ++j) mu[j] = sum[j] / dn;
    /* ... and two-pass population standard deviations */
    double ss[4] = {0.0, 0.0, 0.0, 0.0};
    for (int32_t i = 1; i <= n; ++i) {
        double d0 = XS(i) - mu[0];
        double d1 = XC(i) - mu[1];
        double d2 = XL(i) - mu[2];
        double d3 = Y(i) - mu[3];
        ss[0] = ss[0] + d0 * d0;
        ss[1] = ss[1] + d1 * d1;
        ss[2] = ss[2] + d2 * d2;
        ss[3] = ss[3] + d3 * d3;
    }
    double sg[4];
    for (int j = 0; j < 4; ++j) sg[j] = sqrt(ss[j] / dn);
    for (int j = 0; j < 4; ++j) { m->mu[j] = mu[j]; m->sigma[j] = sg[j]; }
    if (!(sg[3] > 0.0)) {              /* numerically constant target */
        m->kind = 1;
        m->c0 = mu[3];
        return 0;
    }

    int cols[3], mcols = 0;
    for (int j = 0; j < 3; ++j)
        if (sg[j] > 0.0) cols[mcols++] = j;
    m->n_cols = mcols;

    /* F4: G = Z^T Z, h = Z^T u, sequential over rows */
    double G[3][3] = {{0}}, h[3] = {0};
    for (int32_t i = 1; i <= n; ++i) {
        double x[3] = {XS(i), XC(i), XL(i)};
        double z[3];
        for (int a = 0; a < mcols; ++a) z[a] = (x[cols[a]] - mu[cols[a]]) / sg[cols[a]];
        double u = (Y(i) - mu[3]) / sg[3];
        for (int a = 0; a < mcols; ++a) {
            for (int b = 0; b <= a; ++b) G[a][b] = G[a][b] + z[a] * z[b];
            h[a] = h[a] + z[a] * u;
        }
    }
    for (int a = 0; a < mcols; ++a)
        for (int b = 0; b < a; ++b) G[b][a] = G[a][b];
    #undef XS
    #undef XC
    #undef XL
    #undef Y

    /* F5: Cholesky, ridge fallback */
    double Lc[3][3] = {{0}};
    const double tol = singular_tol * dn;
    if (mcols > 0 && !cholesky3(mcols, G, tol, Lc)) {
        for (int a = 0; a < mcols; ++a) G[a][a] = G[a][a] + ridge_lambda;
        m->ridge = 1;
        memset(Lc, 0, sizeof(Lc));
        if (!cholesky3(mcols, G, tol, Lc)) { m->status = 6; return 6; }
    }

    /* F6: beta = G^-1 h  (L z = h, then L^T beta = z) */
    double zt[3] = {0}, beta[3] = {0};
    for (int a = 0; a < mcols; ++a) {
        double v = h[a];
        for (int b = 0; b < a; ++b) v = v - Lc[a][b] * zt[b];
        zt[a] = v / Lc[a][a];
    }
    for (int a = mcols - 1; a >= 0; --a) {
        double v = zt[a];
        for (int b = a + 1; b < mcols; ++b) v = v - Lc[b][a] * beta[b];
        beta[a] = v / Lc[a][a];
    }

    /* Un-standardise: w_j = (sigma_y*beta_j)/sigma_j,
     * c0 = ((mu_y - w_s*mu_s) - w_c*mu_c) - w_l*mu_l (kept columns only). */
    double w[3] = {0.0, 0.0, 0.0};
    for (int a = 0; a < mcols; ++a) w[cols[a]] = (sg[3] * beta[a]) / sg[cols[a]];
    double c0 = mu[3];
    for (int a = 0; a < mcols; ++a) c0 = c0 - w[cols[a]] * mu[cols[a]];
    m->c0 = c0;
    m->ws = w[0];
    m->wc = w[1];
    m->wl = w[2];
    m->kind = 0;
    return 0;
}

/* Eq. 1 predict_one, clamp below at 0 (Q8). */
double oracle_predict(const oracle_model_t* m, double s, double c, double lag) {
    double A = (m->c0 + m->ws * s) + m->wc * c;
    double p = A + m->wl * lag;
    return p > 0.0 ? p : 0.0;
}

/* ---------------------------------------------------------------- Eq. 6 */
double oracle_cost(double eta, double avg_power, double thr, double pmax,
                   double maxci, double chat) {
    double a = eta * avg_power;
    double Kc = ((1.0 - eta) * pmax) * maxci;
    return ((a * chat) + Kc) / thr;
}

/* P:120-124 min over p in P; ties -> lowest limit. */
int32_t oracle_choose(int32_t K, const double* avg_power, const double* thr,
                      double eta, double pmax, double maxci, double chat) {
    int32_t best = 0;
    double best_cost = oracle_cost(eta, avg_power[0], thr[0], pmax, maxci, chat);
    for (int32_t k = 1; k < K; ++k) {
        double ck = oracle_cost(eta, avg_power[k], thr[k], pmax, maxci, chat);
        if (ck < best_cost) { best_cost = ck; best = k; }
    }
    return best;
}

/* S:300-308 cta = tta*avg_power*avg_ci / 3.6e6 (W*s*(g/kWh) -> g). */
double oracle_cta(double tta_s, double avg_power_w, double avg_ci) {
    return ((tta_s * avg_power_w) * avg_ci) / 3.6e6;
}

/* S:309-317 / Eq. 5. */
double oracle_total_cost(double tta_s, double avg_power_w, double avg_ci,
                         double eta, double pmax, double maxci) {
    double inner = (eta * (avg_power_w * avg_ci)) + ((1.0 - eta) * (pmax * maxci));
    return (tta_s * inner) / 3.6e6;
}

/* ---------------------------------------------------------------- replay */
/* DESIGN R1-R2: fixed work ("does not change the number of samples"),
 * stepwise carbon (Q14), pro-rata last window, trace
 * exhaustion is an error. */
int32_t oracle_replay(const double* c, int32_t N, int32_t s0,
                      const uint8_t* choice, const double* avg_power,
                      const double* thr, double delta, double J,
                      double* out4, int32_t* completion_window) {
    double S = 0.0, E = 0.0, C = 0.0;
    for (int32_t w = s0; w < N; ++w) {
        int k = choice[w - s0];
        double sk = thr[k] * delta;
        double prevS = S;
        S = S + sk;
        if (J > 0.0 && S >= J) {
            double f = (J - prevS) / sk;
            out4[0] = ((double)(w - s0) + f) * delta;
            out4[1] = (E + f * avg_power[k]) * delta;
            out4[2] = ((C + f * (avg_power[k] * c[w])) * delta) / 3.6e6;
            out4[3] = J;
            *completion_window = w;
            return 0;
        }
        E = E + avg_power[k];
        C = C + avg_power[k] * c[w];
    }
    out4[0] = (double)(N - s0) * delta;
    out4[1] = E * delta;
    out4[2] = (C * delta) / 3.6e6;
    out4[3] = S;
    *completion_window = -1;
    return J > 0.0 ? 3 : 0;
}

/* ---------------------------------------------------------------- planner */
int32_t oracle_plan_trace(const double* c, int32_t N, int32_t L, int32_t T,
                          int32_t phase0, int32_t refit_stride, int32_t period, const double* svr,
                          double ridge_lambda, double singular_tol,
                          const double* S, const double* Cc,
                          int32_t K, const double* avg_power, const double* thr,
                          int32_t n_eta, const double* eta,
                          double pmax, double max_ci_cfg,
                          double delta, double J,
                          double* forecast, uint8_t* choice,
                          oracle_totals_t* totals) {
    const int32_t s0 = L, W = N - L;
    memset(totals, 0, sizeof(oracle_totals_t) * (size_t)n_eta);
    for (int e = 0; e < n_eta; ++e) totals[e].completion_window = -1;

    int32_t status = 0;
    for (int32_t t = 0; t < N; ++t)          /* values >= 0, finite */
        if (!(c[t] >= 0.0) || !isfinite(c[t])) { status = 4; break; }
    double maxci = max_ci_cfg;
    if (status == 0 && !(max_ci_cfg > 0.0)) {  /* P:184, S:73 window_max */
        maxci = c[0];
        for (int32_t t = 1; t < L; ++t) if (c[t] > maxci) maxci = c[t];
        if (!(maxci > 0.0)) status = 5;
    }

    uint8_t* own = NULL;
    if (!choice) { own = (uint8_t*)malloc((size_t)n_eta * (size_t)W); choice = own; }

    oracle_model_t m;
    static __thread oracle_svr_t sv;   /* f2: the epsilon-SVR forecaster when svr != NULL */
    int32_t origin = -1;
    /* One decision per period of `period` trace steps ("the
     * period between forecasts and power limit adjustments"; <= 1: one step).
     * At the period start w the forecaster runs recursively over the horizon
     * n = min(period, N - w) from the last OBSERVED value (S:158-166
     * forecast_horizon: prediction k feeds the lag of prediction k+1), and
     * Eq. 6 takes the mean of the horizon forecasts.  The period's
     * windows all get that decision; forecast[] holds the decision value. */
    const int32_t P = period > 1 ? period : 1;
    for (int32_t w = s0; status == 0 && w < N; w += P) {
        int32_t r = refit_stride > 0 ? s0 + refit_stride * ((w - s0) / refit_stride) : s0;
        if (r != origin) {
            origin = r;
            int32_t phi0 = (int32_t)(((int64_t)phase0 + r - L) % T);
            if (svr) {
                if (oracle_svr_fit(c + (r - L), L, T, phi0, S, Cc, svr[0], svr[1], svr[2], svr[3],
                                   (int32_t)svr[4], &sv) != 0) { status = 6; break; }
            } else if (oracle_fit(c + (r - L), L, T, phi0, S, Cc, ridge_lambda,
                                  singular_tol, &m) != 0) { status = 6; break; }
        }
        const int32_t n = N - w < P ? N - w : P;
        double prev = c[w - 1], sum = 0.0;
        for (int32_t k = 0; k < n; ++k) {
            int32_t phi = (int32_t)(((int64_t)phase0 + w + k) % T);
            double f = svr ? oracle_svr_predict(&sv, S[phi], Cc[phi], prev) : oracle_predict(&m, S[phi], Cc[phi], prev);
            sum = sum + f;
            prev = f;
        }
        double chat = sum / (double)n;
        for (int32_t k = 0; k < n; ++k) {
            if (forecast) forecast[w - s0 + k] = chat;
            for (int e = 0; e < n_eta; ++e)
                choice[(size_t)e * W + (w - s0 + k)] =
                    (uint8_t)oracle_choose(K, avg_power, thr, eta[e], pmax, maxci, chat);
        }
    }

    if (status != 0) {
        if (forecast) for (int32_t j = 0; j < W; ++j) forecast[j] = NAN;
        memset(choice, 0xFF, (size_t)n_eta * W);
        for (int e = 0; e < n_eta; ++e) totals[e].status = status;
        free(own);
        return status;
    }

    /* baseline: constant max limit */
    uint8_t* base = (uint8_t*)malloc((size_t)W);
    memset(base, K - 1, (size_t)W);
    double b4[4];
    int32_t bw;
    int32_t bst = oracle_replay(c, N, s0, base, avg_power, thr, delta, J, b4, &bw);
    free(base);

    int32_t worst = bst;
    for (int e = 0; e < n_eta; ++e) {
        double a4[4];
        int32_t aw;
        int32_t ast = oracle_replay(c, N, s0, choice + (size_t)e * W, avg_power,
                                    thr, delta, J, a4, &aw);
        totals[e].time_s = a4[0];
        totals[e].energy_j = a4[1];
        totals[e].carbon_g = a4[2];
        totals[e].samples = a4[3];
        totals[e].base_time_s = b4[0];
        totals[e].base_energy_j = b4[1];
        totals[e].base_carbon_g = b4[2];
        totals[e].completion_window = aw;
        totals[e].status = ast ? ast : bst;
        if (totals[e].status > worst) worst = totals[e].status;
    }
    free(own);
    return worst;
}

int32_t oracle_plan_batch_f32(const float* traces, int64_t n_traces, int64_t N,
                              int64_t ld, int32_t L, int32_t T, int32_t phase0,
                              int32_t refit_stride, int32_t period, const double* svr, double ridge_lambda,
                              double singular_tol, int32_t n_profiles,
                              const int32_t* prof_K, const int32_t* prof_off,
                              const double* avg_power, const double* thr,
                              const double* prof_pmax,
                              const uint8_t* profile_id, int32_t n_eta,
                              const double* eta, double pmax_cfg,
                              double max_ci_cfg, double delta,
                              const double* job_samples, double* forecast,
                              uint8_t* choice, oracle_totals_t* totals,
                              double* sums, int32_t threads) {
    const int64_t W = N - L;
    double* S = (double*)malloc(sizeof(double) * (size_t)T);
    double* Cc = (double*)malloc(sizeof(double) * (size_t)T);
    oracle_phase_table(T, S, Cc);
    (void)n_profiles;
    int32_t used = 1;
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
    #pragma omp parallel num_threads(threads)
    {
        #pragma omp single
        used = omp_get_num_threads();
    }
#else
    threads = 1;
#endif

    #pragma omp parallel num_threads(threads)
    {
        double* c = (double*)malloc(sizeof(double) * (size_t)N);
        uint8_t* ch = (uint8_t*)malloc((size_t)n_eta * (size_t)W);
        oracle_totals_t* tt = (oracle_totals_t*)malloc(sizeof(oracle_totals_t) * (size_t)n_eta);
        #pragma omp for schedule(dynamic, 16)
        for (int64_t i = 0; i < n_traces; ++i) {
            for (int64_t t = 0; t < N; ++t) c[t] = (double)traces[i * ld + t];
            int p = profile_id ? profile_id[i] : 0;
            int K = prof_K[p];
            const double* P = avg_power + prof_off[p];
            const double* Th = thr + prof_off[p];
            /* MaxPower defaults to the highest power limit */
            double pmax = pmax_cfg > 0.0 ? pmax_cfg : prof_pmax[p];
            double J = job_samples ? job_samples[i] : 0.0;
            oracle_plan_trace(c, (int32_t)N, L, T, phase0, refit_stride, period, svr,
                              ridge_lambda, singular_tol, S, Cc, K, P, Th,
                              n_eta, eta, pmax, max_ci_cfg, delta, J,
                              forecast ? forecast + i * W : NULL, ch, tt);
            for (int e = 0; e < n_eta; ++e) {
                if (choice) memcpy(choice + ((size_t)e * n_traces + i) * W, ch + (size_t)e * W, (size_t)W);
                totals[(size_t)e * n_traces + i] = tt[e];
            }
        }
        free(c); free(ch); free(tt);
    }

    if (sums) {
        memset(sums, 0, sizeof(double) * 8 * (size_t)n_eta);
        for (int e = 0; e < n_eta; ++e) {
            double* s = sums + 8 * e;
            for (int64_t i = 0; i < n_traces; ++i) {
                const oracle_totals_t* t = &totals[(size_t)e * n_traces + i];
                if (t->status != 0) continue;
                s[0] = s[0] + t->time_s;
                s[1] = s[1] + t->energy_j;
                s[2] = s[2] + t->carbon_g;
                s[3] = s[3] + t->samples;
                s[4] = s[4] + t->base_time_s;
                s[5] = s[5] + t->base_energy_j;
                s[6] = s[6] + t->base_carbon_g;
                s[7] = s[7] + 1.0;
            }
        }
    }
    free(S); free(Cc);
    return used;
}


/* ---------------------------------------------------------------- forecast evaluation */
/* SPEC mape: 100/n * sum |a_i - p_i| / |a_i|, sequential sum. */
double oracle_mape(const double* actual, const double* predicted, int64_t n) {
    if (n < 1) return NAN;
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        if (actual[i] == 0.0) return NAN;
        s = s + fabs(actual[i] - predicted[i]) / fabs(actual[i]);
    }
    return (100.0 / (double)n) * s;
}

/* SPEC evaluate_models: fit once on the first L points, walk
 * forward with the true lag; linear vs persistence. */
int32_t oracle_evaluate(const double* c, int32_t N, int32_t L, int32_t T, int32_t phase0,
                        double ridge_lambda, double singular_tol, const double* S,
                        const double* Cc, const double* svr, double* out2) {
    out2[0] = out2[1] = NAN;
    for (int32_t t = 0; t < N; ++t)
        if (!(c[t] >= 0.0) || !isfinite(c[t])) return 4;
    oracle_model_t m;
    static __thread oracle_svr_t sv;
    if (svr) {
        if (oracle_svr_fit(c, L, T, phase0 % T, S, Cc, svr[0], svr[1], svr[2], svr[3], (int32_t)svr[4], &sv) != 0)
            return 6;
    } else if (oracle_fit(c, L, T, phase0 % T, S, Cc, ridge_lambda, singular_tol, &m) != 0) {
        return 6;
    }
    const int32_t n = N - L;
    double* pl = (double*)malloc(sizeof(double) * (size_t)n);
    for (int32_t w = L; w < N; ++w) {
        int32_t phi = (int32_t)(((int64_t)phase0 + w) % T);
        pl[w - L] = svr ? oracle_svr_predict(&sv, S[phi], Cc[phi], c[w - 1]) : oracle_predict(&m, S[phi], Cc[phi], c[w - 1]);
    }
    out2[0] = oracle_mape(c + L, pl, n);
    out2[1] = oracle_mape(c + L, c + L - 1, n);   /* persistence: p(w) = c[w-1] */
    free(pl);
    return isnan(out2[0]) ? 8 : 0;
}

int32_t oracle_evaluate_batch_f32(const float* traces, int64_t n_traces, int64_t N, int64_t ld,
                                  int32_t L, int32_t T, int32_t phase0, double ridge_lambda,
                                  double singular_tol, const double* svr, double* out, int32_t* status,
                                  int32_t threads) {
    double* S = (double*)malloc(sizeof(double) * (size_t)T);
    double* Cc = (double*)malloc(sizeof(double) * (size_t)T);
    oracle_phase_table(T, S, Cc);
    int32_t used = 1;
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
    used = threads;
#else
    threads = 1;
#endif
    #pragma omp parallel num_threads(threads)
    {
        double* c = (double*)malloc(sizeof(double) * (size_t)N);
        #pragma omp for schedule(dynamic, 16)
        for (int64_t i = 0; i < n_traces; ++i) {
            for (int64_t t = 0; t < N; ++t) c[t] = (double)traces[i * ld + t];
            status[i] = oracle_evaluate(c, (int32_t)N, L, T, phase0, ridge_lambda, singular_tol, S, Cc, svr,
                                        out + 2 * i);
        }
        free(c);
    }
    free(S); free(Cc);
    return used;
}


/* ---------------------------------------------------------------- timeline */
/* SPEC emit_timeline: per-period rows of a planned replay. */
int32_t oracle_timeline(const double* c, int32_t N, int32_t L, int32_t period, const uint8_t* choice,
                        const double* forecast, int32_t K, const int32_t* limit_w, const double* avg_power,
                        const double* thr, double delta, double J, double* rows) {
    const int32_t s0 = L, W = N - L, P = period > 1 ? period : 1;
    double S = 0.0;
    int done = 0, np = 0;
    for (int32_t b = 0; b < W; b += P, ++np) {
        const int32_t n = W - b < P ? W - b : P;
        double* r = rows + 8 * (size_t)np;
        int k = choice ? choice[b] : K - 1;
        double csum = 0.0, samples = 0.0, E = 0.0, C = 0.0;
        for (int32_t q = 0; q < n; ++q) {
            const int32_t w = s0 + b + q;
            csum = csum + c[w];
            if (done) continue;
            int kw = choice ? choice[b + q] : K - 1;
            double sk = thr[kw] * delta;
            double prevS = S;
            S = S + sk;
            if (J > 0.0 && S >= J) {
                double f = (J - prevS) / sk;
                samples = samples + (J - prevS);
                E = E + f * avg_power[kw];
                C = C + f * (avg_power[kw] * c[w]);
                done = 1;
                continue;
            }
            samples = samples + sk;
            E = E + avg_power[kw];
            C = C + avg_power[kw] * c[w];
        }
        r[0] = (double)(s0 + b);
        r[1] = forecast ? forecast[b] : NAN;
        r[2] = csum / (double)n;
        r[3] = (double)limit_w[k];
        r[4] = avg_power[k];
        r[5] = samples;
        r[6] = E * delta;
        r[7] = (C * delta) / 3.6e6;
    }
    return np;
}


/* Eq. 3 next to the stepwise integration (SPEC optimizer DESIGN
 * DECISION S:432): over the job's run (the fixed-work replay of
 * oracle_replay, the completion window pro rata), TTA = (windows + f) Delta,
 * AvgPower = energy / TTA, AvgCI = the time-weighted mean intensity, and
 * CTA_eq3 = TTA * AvgPower * AvgCI = energy * AvgCI; the stepwise carbon is
 * sum P_k c_w (pro rata).  out4 = {stepwise carbon g, Eq. 3 carbon g,
 * AvgPower W, AvgCI g/kWh}.  choice NULL: the max-limit baseline. */
void oracle_job_summary(const double* c, int32_t N, int32_t L, const uint8_t* choice, int32_t K,
                        const double* avg_power, const double* thr, double delta, double J, double* out4) {
    double S = 0.0, E = 0.0, C = 0.0, cj = 0.0, tw = 0.0;
    for (int32_t w = L; w < N; ++w) {
        const int k = choice ? choice[w - L] : K - 1;
        const double sk = thr[k] * delta;
        const double prevS = S;
        S = S + sk;
        if (J > 0.0 && S >= J) {
            const double f = (J - prevS) / sk;
            E = E + f * avg_power[k];
            C = C + f * (avg_power[k] * c[w]);
            cj = cj + f * c[w];
            tw = tw + f;
            break;
        }
        E = E + avg_power[k];
        C = C + avg_power[k] * c[w];
        cj = cj + c[w];
        tw = tw + 1.0;
    }
    const double avg_ci = cj / tw;
    out4[0] = (C * delta) / 3.6e6;
    out4[1] = ((E * delta) * avg_ci) / 3.6e6;
    out4[2] = E / tw;
    out4[3] = avg_ci;
}


/* SPEC --count-profiling (DESIGN Q33): profiling runs one trace step
 * per limit, in increasing limit order, over the K steps just before the job
 * start (steps L-K .. L-1), each at that limit's average power.  out3 =
 * {time s, energy J, carbon g} to add to a replay's totals; needs L >= K. */
int32_t oracle_profiling_overhead(const double* c, int32_t L, int32_t K, const double* avg_power, double delta,
                                  double* out3) {
    if (L < K) return 2;
    double E = 0.0, C = 0.0;
    for (int32_t k = 0; k < K; ++k) {
        E = E + avg_power[k];
        C = C + avg_power[k] * c[L - K + k];
    }
    out3[0] = (double)K * delta;
    out3[1] = E * delta;
    out3[2] = (C * delta) / 3.6e6;
    return 0;
}


/* ---------------------------------------------------------------- epsilon-SVR (f2) */
/* The RBF kernel's exp is libm's exp (DESIGN Q31): the plain definition.  The
 * paper names scikit-learn's SVR, whose libsvm kernel evaluates
 * exp(-gamma*||a-b||^2) with the C library's exp; no faster or differently
 * rounded exp enters the oracle.  x > 0 (never a kernel argument) gives NaN. */
double oracle_rbf_exp(double x) {
    if (!(x <= 0.0)) return NAN;
    return exp(x);
}

/* K(a, b) = exp(-gamma * ||a - b||^2), the squared distance summed left to
 * right: ((d0*d0) + (d1*d1)) + (d2*d2), each operation rounded once. */
static double rbf(const double* a, const double* b, double gamma) {
    const double d0 = a[0] - b[0], d1 = a[1] - b[1], d2 = a[2] - b[2];
    const double d = ((d0 * d0) + (d1 * d1)) + (d2 * d2);
    return oracle_rbf_exp(-(gamma * d));
}

int32_t oracle_svr_fit(const double* hist, int32_t L, int32_t T, int32_t phi0, const double* S, const double* Cc,
                       double C, double eps, double gamma, double tol, int32_t max_iter, oracle_svr_t* m) {
    memset(m, 0, sizeof(*m));
    const int32_t n = L - 1;
    m->n = n;
    if (n < 2 || n > ORACLE_SVR_MAXN) { m->status = 2; return 2; }
    for (int32_t t = 0; t < L; ++t)
        if (!(hist[t] >= 0.0) || !isfinite(hist[t])) { m->status = 4; return 4; }
    const double dn = (double)n;
    /* features and moments exactly as oracle_fit (rows i = 1..n) */
    double x[ORACLE_SVR_MAXN][3], y[ORACLE_SVR_MAXN];
    for (int32_t i = 1; i <= n; ++i) {
        int32_t ph = (phi0 + i) % T;
        x[i - 1][0] = S[ph];
        x[i - 1][1] = Cc[ph];
        x[i - 1][2] = hist[i - 1];
        y[i - 1] = hist[i];
    }
    double sum[4] = {0.0, 0.0, 0.0, 0.0};
    for (int32_t i = 0; i < n; ++i) {
        for (int j = 0; j < 3; ++j) sum[j] = sum[j] + x[i][j];
        sum[3] = sum[3] + y[i];
    }
    for (int j = 0; j < 4; ++j) m->mu[j] = sum[j] / dn;
    double ss[4] = {0.0, 0.0, 0.0, 0.0};
    for (int32_t i = 0; i < n; ++i) {
        for (int j = 0; j < 3; ++j) { double d = x[i][j] - m->mu[j]; ss[j] = ss[j] + d * d; }
        double d = y[i] - m->mu[3];
        ss[3] = ss[3] + d * d;
    }
    for (int j = 0; j < 4; ++j) m->sigma[j] = sqrt(ss[j] / dn);
    if (!(m->sigma[3] > 0.0)) { m->kind = 1; m->converged = 1; return 0; }   /* constant target */
    int kept = 0;
    for (int j = 0; j < 3; ++j) { m->keep[j] = m->sigma[j] > 0.0; kept += m->keep[j]; }
    double u[ORACLE_SVR_MAXN];
    for (int32_t i = 0; i < n; ++i) {
        for (int j = 0; j < 3; ++j) m->z[i][j] = m->keep[j] ? (x[i][j] - m->mu[j]) / m->sigma[j] : 0.0;
        u[i] = (y[i] - m->mu[3]) / m->sigma[3];
    }
    /* SPEC default gamma = 1/(3 * mean feature variance); standardised kept columns have variance 1 */
    m->gamma = gamma > 0.0 ? gamma : (kept > 0 ? 1.0 / (double)kept : 1.0);
    /* kernel matrix */
    static __thread double K[ORACLE_SVR_MAXN][ORACLE_SVR_MAXN];
    for (int32_t i = 0; i < n; ++i)
        for (int32_t j = 0; j < n; ++j) K[i][j] = (double)(float)rbf(m->z[i], m->z[j], m->gamma);
    /* SMO on 2n variables: t < n -> y = +1 (alpha), t >= n -> y = -1 (alpha*) */
    const int32_t l = 2 * n;
    double a[2 * ORACLE_SVR_MAXN], G[2 * ORACLE_SVR_MAXN];
    for (int32_t t = 0; t < l; ++t) {
        a[t] = 0.0;
        G[t] = t < n ? eps - u[t] : eps + u[t - n];      /* G = Q a + p, a = 0 */
    }
    const double TAU = 1e-12;
    int32_t it = 0;
    m->converged = 0;
    for (;;) {
        /* second-order working-set selection */
        double Gmax = -INFINITY, Gmax2 = -INFINITY, obj_min = INFINITY;
        int32_t i = -1, j = -1;
        for (int32_t t = 0; t < l; ++t) {
            if (t < n) { if (a[t] < C && -G[t] >= Gmax) { Gmax = -G[t]; i = t; } }
            else { if (a[t] > 0.0 && G[t] >= Gmax) { Gmax = G[t]; i = t; } }
        }
        if (i >= 0) {
            const double yi = i < n ? 1.0 : -1.0;
            for (int32_t t = 0; t < l; ++t) {
                const double yt = t < n ? 1.0 : -1.0;
                const double Qit = (yi * yt) * K[i % n][t % n];
                if (t < n) {
                    if (a[t] > 0.0) {
                        const double gd = Gmax + G[t];
                        if (G[t] >= Gmax2) Gmax2 = G[t];
                        if (gd > 0.0) {
                            const double qc = (K[i % n][i % n] + K[t % n][t % n]) - (2.0 * yi) * Qit;
                            const double od = -(gd * gd) / (qc > 0.0 ? qc : TAU);
                            if (od <= obj_min) { j = t; obj_min = od; }
                        }
                    }
                } else {
                    if (a[t] < C) {
                        const double gd = Gmax - G[t];
                        if (-G[t] >= Gmax2) Gmax2 = -G[t];
                        if (gd > 0.0) {
                            const double qc = (K[i % n][i % n] + K[t % n][t % n]) + (2.0 * yi) * Qit;
                            const double od = -(gd * gd) / (qc > 0.0 ? qc : TAU);
                            if (od <= obj_min) { j = t; obj_min = od; }
                        }
                    }
                }
            }
        }
        if (Gmax + Gmax2 < tol || j < 0) { m->converged = 1; break; }
        if (it >= max_iter) break;
        ++it;
        /* analytic pair update with clipping to [0, C] */
        const double yi = i < n ? 1.0 : -1.0, yj = j < n ? 1.0 : -1.0;
        const double Qij = (yi * yj) * K[i % n][j % n];
        const double ai = a[i], aj = a[j];
        if (yi != yj) {
            double qc = (K[i % n][i % n] + K[j % n][j % n]) + 2.0 * Qij;
            if (qc <= 0.0) qc = TAU;
            const double delta = (-G[i] - G[j]) / qc;
            const double diff = a[i] - a[j];
            a[i] = a[i] + delta;
            a[j] = a[j] + delta;
            if (diff > 0.0) { if (a[j] < 0.0) { a[j] = 0.0; a[i] = diff; } }
            else { if (a[i] < 0.0) { a[i] = 0.0; a[j] = -diff; } }
            if (diff > 0.0) { if (a[i] > C) { a[i] = C; a[j] = C - diff; } }
            else { if (a[j] > C) { a[j] = C; a[i] = C + diff; } }
        } else {
            double qc = (K[i % n][i % n] + K[j % n][j % n]) - 2.0 * Qij;
            if (qc <= 0.0) qc = TAU;
            const double delta = (G[i] - G[j]) / qc;
            const double sm = a[i] + a[j];
            a[i] = a[i] - delta;
            a[j] = a[j] + delta;
            if (sm > C) { if (a[i] > C) { a[i] = C; a[j] = sm - C; } }
            else { if (a[j] < 0.0) { a[j] = 0.0; a[i] = sm; } }
            if (sm > C) { if (a[j] > C) { a[j] = C; a[i] = sm - C; } }
            else { if (a[i] < 0.0) { a[i] = 0.0; a[j] = sm; } }
        }
        const double dai = a[i] - ai, daj = a[j] - aj;
        for (int32_t t = 0; t < l; ++t) {
            const double yt = t < n ? 1.0 : -1.0;
            const double Qti = (yt * yi) * K[t % n][i % n];
            const double Qtj = (yt * yj) * K[t % n][j % n];
            G[t] = G[t] + (Qti * dai + Qtj * daj);
        }
    }
    m->iters = it;
    /* bias: mean y*G over free variables, else the midpoint of the bounds */
    double ub = INFINITY, lb = -INFINITY, sfree = 0.0;
    int32_t nfree = 0;
    for (int32_t t = 0; t < l; ++t) {
        const double yt = t < n ? 1.0 : -1.0;
        const double yG = yt * G[t];
        if (a[t] >= C) { if (yt < 0.0) ub = fmin(ub, yG); else lb = fmax(lb, yG); }
        else if (a[t] <= 0.0) { if (yt > 0.0) ub = fmin(ub, yG); else lb = fmax(lb, yG); }
        else { ++nfree; sfree = sfree + yG; }
    }
    m->rho = nfree > 0 ? sfree / (double)nfree : (ub + lb) / 2.0;
    for (int32_t t = 0; t < n; ++t) m->coef[t] = a[t] - a[t + n];
    return 0;
}

double oracle_svr_predict(const oracle_svr_t* m, double s, double c, double lag) {
    if (m->kind == 1) return m->mu[3] > 0.0 ? m->mu[3] : 0.0;
    const double xv[3] = {s, c, lag};
    double zq[3];
    for (int j = 0; j < 3; ++j) zq[j] = m->keep[j] ? (xv[j] - m->mu[j]) / m->sigma[j] : 0.0;
    double f = 0.0;
    for (int32_t t = 0; t < m->n; ++t) f = f + m->coef[t] * rbf(m->z[t], zq, m->gamma);   /* sum of coef*K, in order */
    f = f - m->rho;
    const double p = m->mu[3] + m->sigma[3] * f;
    return p > 0.0 ? p : 0.0;
}
