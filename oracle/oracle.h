/*
 * oracle.h — plain, slow, obviously-correct CPU oracle for the Chase planner.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load liboracle.so.
 * The product path (paper_2303_02508_b200/, include/chase.h) never includes,
 * links or calls anything in this directory, and this directory never
 * includes anything from the product (no shared headers, tables or helpers).
 *
 * Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n
 * (the section/equation/operation is named beside each).  Readings of the
 * paper where it is silent or garbled are listed in DESIGN.md §3 (Q-numbers).
 *
 * Arithmetic contract: IEEE fp64, every operation rounded once, evaluated in
 * the written order, built with -O2 -ffp-contract=off (never -ffast-math).
 */
#ifndef CHASE_ORACLE_H
#define CHASE_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Fitted one-lag model of Eq. 1 in un-standardised form:
 *   chat = max(0, ((c0 + ws*sin) + wc*cos) + wl*lag)
 * kind 0 = least squares (Table 1 "Linear Regression")
 * kind 1 = constant target, intercept only (DESIGN Q7). */
typedef struct {
    double c0, ws, wc, wl;
    double mu[4];     /* means of sin, cos, lag, target (diagnostic) */
    double sigma[4];  /* population std devs (diagnostic)           */
    int32_t kind;
    int32_t ridge;    /* 1 when the lambda = 1e-8 fallback fired */
    int32_t status;   /* 0 ok, 6 fit failed after ridge               */
    int32_t n_cols;   /* features kept (sigma > 0)                    */
} oracle_model_t;

/* Per (trace, eta) replay result, S:373-383 SimReport totals. */
typedef struct {
    double time_s, energy_j, carbon_g, samples;
    double base_time_s, base_energy_j, base_carbon_g;
    int32_t completion_window;   /* w* (absolute step index) or -1 */
    int32_t status;              /* 0 ok, 3 exhausted, 4 bad value, 5 MaxCI<=0, 6 fit failed */
} oracle_totals_t;

/* Eq. 2: S[phi] = sin((2.0*pi*phi)/T), Cc[phi] = cos(...). */
void oracle_phase_table(int32_t T, double* S, double* Cc);

/* Fit Eq. 1 on L history points hist[0..L) ("one day prior", P:158;
 * S:122-139).  Row i = 1..L-1: x = (S[phi_i], Cc[phi_i], hist[i-1]),
 * y = hist[i], phi_i = (phi0 + i) mod T.  Returns m->status. */
int32_t oracle_fit(const double* hist, int32_t L, int32_t T, int32_t phi0,
                   const double* S, const double* Cc,
                   double ridge_lambda, double singular_tol, oracle_model_t* m);

/* Eq. 1 prediction with the clamp of S:152 (DESIGN Q8). */
double oracle_predict(const oracle_model_t* m, double s, double c, double lag);

/* Eq. 6 numerator/throughput without the 3.6e6 divisor (Q12):
 * cost_k = ((a_k*chat) + Kc)/Thr_k, a_k = eta*P_k, Kc = ((1-eta)*Pmax)*MaxCI */
double oracle_cost(double eta, double avg_power, double thr, double pmax,
                   double maxci, double chat);

/* argmin_k of oracle_cost, first minimum (lowest limit). */
int32_t oracle_choose(int32_t K, const double* avg_power, const double* thr,
                      double eta, double pmax, double maxci, double chat);

/* Eq. 3 CTA and Eq. 4-5 total cost, in g (divided by 3.6e6). */
double oracle_cta(double tta_s, double avg_power_w, double avg_ci);
double oracle_total_cost(double tta_s, double avg_power_w, double avg_ci,
                         double eta, double pmax, double maxci);

/* Fixed-work replay (DESIGN Q13/Q14).
 * c = full trace (N steps), windows w = s0..N-1, choice[w-s0] = limit index.
 * J > 0: run until J samples; J <= 0: run to the trace end.
 * out4 = {time_s, energy_j, carbon_g, samples}; returns status 0 / 3. */
int32_t oracle_replay(const double* c, int32_t N, int32_t s0,
                      const uint8_t* choice, const double* avg_power,
                      const double* thr, double delta, double J,
                      double* out4, int32_t* completion_window);

/* Whole planner for one trace: fit (once, or rolling with refit_stride R),
 * svr != NULL: the epsilon-SVR forecaster {C, eps, gamma, tol, max_iter} (f2)
 * instead of least squares,
 * predict every window, choose for every eta, replay aware + baseline.
 * period > 1: one decision per period of that many steps, on the mean of the
 * recursive horizon forecast; forecast[]
 * then holds each window's decision value (the period mean).
 *   c[N]            trace (g/kWh)
 *   forecast[W]     out, may be NULL
 *   choice[n_eta*W] out, may be NULL (then an internal buffer is used)
 *   totals[n_eta]   out
 * max_ci_cfg <= 0 -> MaxCI = max(c[0..L));
   pmax: the resolved MaxPower (> 0; the batch driver applies the P:183 default). */
int32_t oracle_plan_trace(const double* c, int32_t N, int32_t L, int32_t T,
                          int32_t phase0, int32_t refit_stride, int32_t period, const double* svr,
                          double ridge_lambda, double singular_tol,
                          const double* S, const double* Cc,
                          int32_t K, const double* avg_power, const double* thr,
                          int32_t n_eta, const double* eta,
                          double pmax_cfg, double max_ci_cfg,
                          double delta, double J,
                          double* forecast, uint8_t* choice,
                          oracle_totals_t* totals);

/* Batch driver over fp32 traces [n_traces][ld] with OpenMP across traces
 * (threads <= 0: library default).  profile_id may be NULL (all profile 0).
 * Profiles are packed: prof_K[p] rows starting at prof_off[p]; prof_pmax[p]
 * is the profile's largest limit (the P:183 default for pmax_cfg <= 0).
 * job_samples may be NULL (J <= 0 for all traces).
 * sums[n_eta][8] = {time, energy, carbon, samples, base_time, base_energy,
 * base_carbon, n_ok} accumulated in trace order over status-0 traces.
 * Returns the number of threads used. */
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
                              double* sums, int32_t threads);

/* ---- epsilon-SVR forecaster (Table 1's best model; SPEC fit_svr
 * S:140-148).  RBF kernel on the z-scored features of Eq. 1
 * (fit-window statistics, population sigma, zero-variance columns dropped),
 * target z-scored too; the dual is solved by sequential minimal optimisation
 * with second-order working-set selection (Fan, Chen & Lin 2005, the solver
 * of LIBSVM: 2n variables, y = +1 / -1, p = eps -/+ u), stopping when the
 * maximal KKT violation is below tol or after max_iter pair updates; the bias
 * is the mean y*G over free variables (else the midpoint of the bounds).
 * f(x) = sum_t (a_t - a*_t) K(z_t, z(x)) - rho;  chat = max(0, mu_y + sigma_y f).
 * exp() of the kernel is libm's exp (oracle_rbf_exp), as in scikit-learn's
 * libsvm: the plain definition.  The GPU kernel evaluates its own faster exp,
 * so the two agree to a tolerance, not bit for bit (DESIGN Q31). */
#define ORACLE_SVR_MAXN 63
typedef struct {
    double z[ORACLE_SVR_MAXN][3];  /* standardised training features */
    double coef[ORACLE_SVR_MAXN];  /* a_t - a*_t                      */
    double mu[4], sigma[4];        /* sin, cos, lag, target           */
    double gamma, rho;
    int32_t n, kind;               /* kind 0 SVR, 1 constant target    */
    int32_t iters, converged;      /* SMO pair updates; 1 if KKT <= tol */
    int32_t keep[3];               /* feature kept (sigma > 0)         */
    int32_t status;                /* 0 ok, 4 bad value                */
} oracle_svr_t;

/* libm exp(x) for x <= 0 (the RBF kernel's argument); NaN for x > 0. */
double oracle_rbf_exp(double x);

/* Fit on the L history points hist[0..L) (rows as oracle_fit).  gamma <= 0:
 * 1/(3 * mean variance of the standardised features) (SPEC default). */
int32_t oracle_svr_fit(const double* hist, int32_t L, int32_t T, int32_t phi0, const double* S, const double* Cc,
                       double C, double eps, double gamma, double tol, int32_t max_iter, oracle_svr_t* m);
double oracle_svr_predict(const oracle_svr_t* m, double s, double c, double lag);

/* SPEC emit_timeline (Figure 1/2 rows) for one trace:
 * one row per decision period of `period` steps (<= 1: per window) starting
 * at the job start s0 = L, from the planned choices (choice[W]; NULL: the
 * max-limit baseline) and the decision forecasts (forecast[W] or
 * NULL: NaN):
 *   {period_start (absolute step), forecast_ci, actual_mean_ci (mean of c
 *    over the period's windows), chosen_limit_w, avg_power_w, samples_done,
 *    energy_j, carbon_g}
 * with the fixed-work replay of oracle_replay split by period: full windows
 * count s_k, P_k*Delta and P_k*Delta*c/3.6e6; the completion window its
 * fraction f (samples J - S_before, so they sum to J exactly); later windows
 * nothing.  rows[n_periods][8]; returns n_periods. */
int32_t oracle_timeline(const double* c, int32_t N, int32_t L, int32_t period, const uint8_t* choice,
                        const double* forecast, int32_t K, const int32_t* limit_w, const double* avg_power,
                        const double* thr, double delta, double J, double* rows);

/* SPEC --count-profiling (DESIGN Q33): one trace step per limit over
 * steps L-K .. L-1 at each limit's average power; out3 = {time s, energy J,
 * carbon g}.  Returns 2 when L < K. */
int32_t oracle_profiling_overhead(const double* c, int32_t L, int32_t K, const double* avg_power, double delta,
                                  double* out3);

/* Eq. 3 product-form carbon next to the stepwise one for one
 * planned replay: out4 = {stepwise carbon g, TTA*AvgPower*AvgCI
 * carbon g, AvgPower W, time-weighted AvgCI g/kWh} over the job's run. */
void oracle_job_summary(const double* c, int32_t N, int32_t L, const uint8_t* choice, int32_t K,
                        const double* avg_power, const double* thr, double delta, double J, double* out4);

/* SPEC mape (Table 1 metric P:159-161): 100/n * sum |a_i - p_i| / |a_i|.
 * Returns NaN when n < 1 or some a_i == 0 ("errors: zero actual"). */
double oracle_mape(const double* actual, const double* predicted, int64_t n);

/* SPEC evaluate_models (P:159-161 walk-forward, Table 1) for one
 * trace: fit Eq. 1 once on c[0..L), then one-step predictions of every
 * window w = L..N-1 with the TRUE lag c[w-1] (the first seeded by the last
 * fit point: N - L predictions, Open Question S:211-212), next to the
 * persistence baseline p(w) = c[w-1].  out2 = {MAPE linear, MAPE persistence}
 * (percent; NaN if undefined).  Returns 0, 4 (negative / non-finite value),
 * 6 (fit failed) or 8 (a zero actual: MAPE undefined). */
int32_t oracle_evaluate(const double* c, int32_t N, int32_t L, int32_t T, int32_t phase0,
                        double ridge_lambda, double singular_tol, const double* S,
                        const double* Cc, const double* svr, double* out2);

/* Batch of fp32 traces [n][ld] (OpenMP across traces): out[n][2], status[n]. */
int32_t oracle_evaluate_batch_f32(const float* traces, int64_t n_traces, int64_t N, int64_t ld,
                                  int32_t L, int32_t T, int32_t phase0, double ridge_lambda,
                                  double singular_tol, const double* svr, double* out, int32_t* status,
                                  int32_t threads);

#ifdef __cplusplus
}
#endif
#endif
