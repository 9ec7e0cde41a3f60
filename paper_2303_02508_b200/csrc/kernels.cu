// kernels.cu — sm_100a kernels of the Chase batched trace-replay planner.
//
//   fit_kernel        §3.1 Eq. 1-2 fit on the L history points, lane = trace,
//                     canonical sequential order (bit-identical to the oracle),
//                     plus the per-trace baseline completion count.
//   sweep_kernel      persistent CTAs of independent warps; each warp streams
//                     whole traces in 1152-window chunks through its own TMA
//                     bulk-copy ring: predict (Eq. 1) -> Eq. 6 argmin by the
//                     exact envelope bucket table (canonical K-way path
//                     deferred for the rare windows in a rounding band) ->
//                     replay partials -> warp reductions; choices staged in
//                     smem and bulk-stored (sweep.cuh).
//   finalize_kernel   per-trace totals (Eq. 3 stepwise carbon, pro-rata last
//                     window, max-power baseline) + fixed-order per-GPU sums.
//   plan_kernel       Eq. 6 argmin from given forecasts (split path).
//   rolling_*_kernel  rolling refit (refit_stride >= 1): one thread per
//                     (trace, origin), oracle_fit's exact operation order
//                     (rolling.cuh); the sweep then reads those forecasts.
//
// Arithmetic contract: every fp64 step that decides an output is written with
// explicit round-to-nearest intrinsics (and the file is built -fmad=false),
// in the same order as the oracle (DESIGN.md §3 Q9), so forecasts and choices
// are bit-identical and dyadic replay totals are exact.
#include <cfloat>
#include <math_constants.h>
#include <cstdlib>
#include <cstring>

#include "kernels.h"

namespace chase {
namespace {

#include "device_common.cuh"
#include "fit.cuh"
#include "k2_sweep.cuh"
#include "k2_headline.cuh"
#include "k2_roll.cuh"
#include "k2_roll_lane.cuh"
#include "finalize.cuh"
#include "rolling.cuh"
#include "mape.cuh"
#include "timeline.cuh"
#include "svr.cuh"

int num_sms() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms > 0 ? sms : 148;
}

template <int MODE, typename E, bool AL, bool MULTI, bool FIN = false>
cudaError_t launch_sweep_t(const SweepParams& p, cudaStream_t s) {
    const int smem = sweep_smem_total(p.tables_bytes, p.T, p.stage_bytes, p.n_eta);
    auto kern = sweep_kernel<MODE, E, AL, MULTI, FIN>;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (err != cudaSuccess) return err;
    int per_sm = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
    if (err != cudaSuccess) return err;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    int64_t grid = (int64_t)num_sms() * per_sm;
    const int64_t need = (p.n_traces + kWarpsPerCta - 1) / kWarpsPerCta;  // one trace per warp at least
    if (grid > need) grid = need;
    kern<<<(unsigned)grid, kThreads, smem, s>>>(p);
    ++g_launches;
    return cudaGetLastError();
}

}  // namespace

// ------------------------------------------------------------------ host launchers
uint64_t kernel_launches() { return g_launches; }

int sweep_stage_bytes(int elem_size) { return round16((kWarpW + 8) * elem_size) + kRecBytes; }

size_t sweep_smem_bytes(int tables_bytes, int T, int elem_size, int mode) {  // mode: n_eta
    return (size_t)sweep_smem_total(tables_bytes, T, sweep_stage_bytes(elem_size), mode);
}

int64_t finalize_grid(int64_t n_traces) { return (n_traces + kFinThreads - 1) / kFinThreads; }

cudaError_t launch_upload(const void* host, size_t bytes, void* dst, cudaStream_t s, chase_diag_t* reset) {
    const uint8_t* h = static_cast<const uint8_t*>(host);
    for (size_t off = 0; off < bytes; off += sizeof(UploadChunk)) {
        UploadChunk c;
        const size_t n = bytes - off < sizeof(UploadChunk) ? bytes - off : sizeof(UploadChunk);
        memcpy(c.bytes, h + off, n);
        upload_kernel<<<1, 256, 0, s>>>(c, (int)n, static_cast<uint8_t*>(dst) + off, off == 0 ? reset : nullptr);
        ++g_launches;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_fit(const FitParams& p, cudaStream_t s) {
    if (p.n_traces <= 0) return cudaSuccess;
    const unsigned grid = (unsigned)((p.n_traces + 127) / 128);
    if (!p.baseline_only && p.L <= 64 && grid > 1) {  // (one CTA computes the record itself)
        fit_phase_kernel<<<1, 1, 0, s>>>(p.tables, p.T, p.L, p.phase0, p.prec);
        ++g_launches;
    }
    const int esz = p.is_f64 ? 8 : 4;
    const int smem = round16(128 * 65 * esz) + 2 * p.T * 8 + (p.L <= 64 ? phase_stride(p.L) * 8 : 0);
    if (p.is_f64) {
        cudaFuncSetAttribute(fit_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        fit_kernel<double><<<grid, 128, smem, s>>>(p);
    } else {
        cudaFuncSetAttribute(fit_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        fit_kernel<float><<<grid, 128, smem, s>>>(p);
    }
    ++g_launches;
    return cudaGetLastError();
}

// Dynamic shared memory the headline kernel needs for T and n_prof: the layout
// depends on the CTA's shared-window base, so plan for the worst candidate.
int headline_smem(int T, int n_prof, int k0len) {
    // blob bytes before the pair tables (header, phase, profiles): see make_hlayout
    const int head_bytes = (int)sizeof(TablesHeader) + ((2 * T * 8) + 15) / 16 * 16 + n_prof * (int)sizeof(ProfileTable);
    int smem = 0;
    for (int base = 0; base <= 8192; base += 16) {
        const int t = make_hlayout(T, head_bytes, n_prof, base, k0len).total;
        smem = t > smem ? t : smem;
    }
    return smem;
}

int max_smem_optin() {
    static int v = -1;
    if (v < 0) {
        int dev = 0, x = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&x, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || x <= 0) {
            cudaGetLastError();
            x = 232448;  // sm_100: 227 KB per block
        }
        v = x;
    }
    return v;
}

bool headline_eligible(int mode, bool f64, bool aligned, const SweepParams& p) {
    // the per-warp blocks (A tables, stage, staged choices) and the per-profile bucket
    // entries must fit one CTA's shared memory: large T (e.g. 5-minute data) or many
    // profiles take the general sweep (forecast-first for decision periods)
    return mode == MODE_FUSED && !f64 && aligned && p.n_eta == 1 && !p.forecast && !p.fc_in &&
           !getenv("CHASE_FORCE_GENERAL") && headline_smem(p.T, p.n_prof, 0) <= max_smem_optin();
}

cudaError_t launch_sweep(int mode, bool f64, bool aligned, const SweepParams& p, cudaStream_t s) {
    if (p.n_traces <= 0) return cudaSuccess;
    if (mode == MODE_PREDICT && p.fc_in) {  // rolling chase_fit_forecast: validation pass only
        if (f64) return aligned ? launch_sweep_t<MODE_PREDICT, double, true, false, true>(p, s)
                                : launch_sweep_t<MODE_PREDICT, double, false, false, true>(p, s);
        return aligned ? launch_sweep_t<MODE_PREDICT, float, true, false, true>(p, s)
                       : launch_sweep_t<MODE_PREDICT, float, false, false, true>(p, s);
    }
    if (mode == MODE_FUSED && p.fc_in) {  // rolling refit: forecasts precomputed by rolling_forecast_kernel
        const bool multi = p.n_eta > 1;
        if (f64) {
            if (multi) return aligned ? launch_sweep_t<MODE_FUSED, double, true, true, true>(p, s)
                                      : launch_sweep_t<MODE_FUSED, double, false, true, true>(p, s);
            return aligned ? launch_sweep_t<MODE_FUSED, double, true, false, true>(p, s)
                           : launch_sweep_t<MODE_FUSED, double, false, false, true>(p, s);
        }
        if (multi) return aligned ? launch_sweep_t<MODE_FUSED, float, true, true, true>(p, s)
                                  : launch_sweep_t<MODE_FUSED, float, false, true, true>(p, s);
        return aligned ? launch_sweep_t<MODE_FUSED, float, true, false, true>(p, s)
                       : launch_sweep_t<MODE_FUSED, float, false, false, true>(p, s);
    }
    if (headline_eligible(mode, f64, aligned, p)) {
        // the headline shape: lean specialised kernel (k2_headline.cuh), with its own chunk geometry
        SweepParams q = p;
        {
            const int64_t L = p.L, W = p.W, vec = 4;
            q.n_chunks = (int32_t)((W + kHWarpW - 1) / kHWarpW);
            q.a0 = (int32_t)(L - vec);
            q.off0 = (int32_t)vec;
            q.W_last = (int32_t)(W - (int64_t)(q.n_chunks - 1) * kHWarpW);
            q.bytes_full = (uint32_t)((kHWarpW + vec) * 4);
            int64_t last_end = (L + (int64_t)(q.n_chunks - 1) * kHWarpW + q.W_last + vec - 1) / vec * vec;
            if (last_end > p.ld) last_end = p.ld;
            q.bytes_last = (uint32_t)((last_end - (q.a0 + (int64_t)(q.n_chunks - 1) * kHWarpW)) * 4);
            q.phase_step = kHWarpW % p.T;
            q.stage_bytes = hstage_bytes();
            // last chunk: the fewest windows per lane (4 mod 8: conflict-free LDS.128) covering W_last
            int k = (q.W_last + 31) / 32;
            k = k < 4 ? 4 : k;
            while (k % 8 != 4) ++k;
            q.kc_last = k > kHChunk ? kHChunk : k;
        }
        // decision periods: the closed-form horizon table ({K0, x0min} for haext_len(T)
        // phases, then {h', -r Kc}, {-A_b, 0}) for every P > 1 when it fits;
        // else every period runs its horizon (§6.5)
        q.k0len = 0;
        const int k0len = 2 * (haext_len(p.T) + 2);
        if (p.period > (CHASE_P2_CF ? 1 : 2) && (CHASE_LONG_CF || p.period * 30 < kHWarpW) && !getenv("CHASE_NO_CFH") &&
            headline_smem(p.T, p.n_prof, k0len) <= max_smem_optin())
            q.k0len = k0len;
        const int smem = headline_smem(p.T, p.n_prof, q.k0len);
        q.smem_total = smem;
        // decision periods: long ones (at most 31 per warp chunk) in 32-period batches
        // (lane-direct for them measured slower: P = 168 14.3 vs 12.9 ms, P = 720 16.2 vs 11.6)
        auto kern = p.period <= 1                 ? sweep_fast_kernel<0>
                    : p.period * 30 >= kHWarpW     ? sweep_fast_kernel<2>
                    : p.period == 24 && q.k0len > 0 ? sweep_fast_kernel<26>  // daily: lane-direct, P fixed
                    : kHChunk % p.period != 0      ? sweep_fast_kernel<1>
                    : p.period == 2                ? sweep_fast_kernel<4>
                    : p.period == 3                ? sweep_fast_kernel<5>
                    : p.period == 4                ? sweep_fast_kernel<6>
                    : p.period == 5                ? sweep_fast_kernel<7>
                    : p.period == 6                ? sweep_fast_kernel<8>
                    : p.period == 10               ? sweep_fast_kernel<12>
                    : p.period == 12               ? sweep_fast_kernel<14>
                    : p.period == 15               ? sweep_fast_kernel<17>
                                                   : sweep_fast_kernel<3>;
        cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (err != cudaSuccess) return err;
        int per_sm = 0;
        err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kHThreads, smem);
        if (err != cudaSuccess) return err;
        if (per_sm < 1) return cudaErrorInvalidConfiguration;
        int64_t grid = (int64_t)num_sms() * per_sm;
        const int64_t need = (p.n_traces + kHWarps - 1) / kHWarps;  // one trace per warp at least
        if (grid > need) grid = need;
        kern<<<(unsigned)grid, kHThreads, smem, s>>>(q);
        ++g_launches;
        return cudaGetLastError();
    }
#define CHASE_SWEEP_CASE(M, MU)                                                                        \
    if (mode == M && multi == MU) {                                                                    \
        if (f64) return aligned ? launch_sweep_t<M, double, true, MU>(p, s) : launch_sweep_t<M, double, false, MU>(p, s); \
        return aligned ? launch_sweep_t<M, float, true, MU>(p, s) : launch_sweep_t<M, float, false, MU>(p, s); \
    }
    const bool multi = mode != MODE_PREDICT && p.n_eta > 1;
    CHASE_SWEEP_CASE(MODE_FUSED, false)
    CHASE_SWEEP_CASE(MODE_FUSED, true)
    CHASE_SWEEP_CASE(MODE_PREDICT, false)
    CHASE_SWEEP_CASE(MODE_REPLAY, false)
    CHASE_SWEEP_CASE(MODE_REPLAY, true)
#undef CHASE_SWEEP_CASE
    return cudaErrorInvalidValue;
}

// Does a one-eta sweep of this shape without forecast output run in place (periods in
// the headline kernel, or the fused rolling refit), i.e. need no forecast scratch?
bool sweep_in_place(bool f64, bool aligned, int L, int T, int n_prof, int n_eta, bool rolling, bool periods,
                    int tables_bytes) {
    if (f64 || !aligned || n_eta != 1) return false;
    SweepParams p;
    memset(&p, 0, sizeof(p));
    p.L = L;
    p.T = T;
    p.n_eta = 1;
    p.n_prof = n_prof;
    p.tables_bytes = tables_bytes;
    if (periods) return headline_eligible(MODE_FUSED, false, true, p);
    if (rolling) {
        p.refit = 1;
        return roll_fused_eligible(p);
    }
    return false;
}

bool roll_fused_eligible(const SweepParams& p) {
    return p.refit >= 1 && p.n_eta == 1 && !p.forecast && !p.fc_in && p.L <= kRMaxL && p.L % 4 == 0 &&
           p.T <= 2048 && !getenv("CHASE_ROLL_EXACT") &&
           make_rlayout(p.T, p.tables_bytes).total <= max_smem_optin();
}

cudaError_t launch_roll_fused(const SweepParams& p, cudaStream_t s) {
    if (p.n_traces <= 0) return cudaSuccess;
    if (!getenv("CHASE_ROLL_RUNS") && make_rllayout(p.T, p.L, p.tables_bytes).total <= max_smem_optin()) {
        // lane = trace (k2_roll_lane.cuh), the default where its tiles fit
        const int smem = make_rllayout(p.T, p.L, p.tables_bytes).total;
        // R > 1: the moments slide every window and each origin fits them (mode 1), or each
        // origin's moments come from its rows (mode 2, CHASE_RL_DIRECT)
        auto kern = p.refit == 1 ? roll_lane_kernel<0> : getenv("CHASE_RL_DIRECT") ? roll_lane_kernel<2> : roll_lane_kernel<1>;
        cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (err != cudaSuccess) return err;
        int per_sm = 0;
        err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRLThreads, smem);
        if (err != cudaSuccess) return err;
        if (per_sm < 1) return cudaErrorInvalidConfiguration;
        int64_t grid = (int64_t)num_sms() * per_sm;
        const int64_t need = ((p.n_traces + 31) / 32 + kRLWarps - 1) / kRLWarps;
        if (grid > need) grid = need;
        kern<<<(unsigned)grid, kRLThreads, smem, s>>>(p);
        ++g_launches;
        return cudaGetLastError();
    }
    const int smem = make_rlayout(p.T, p.tables_bytes).total;
    cudaError_t err = cudaFuncSetAttribute(roll_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (err != cudaSuccess) return err;
    int per_sm = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, roll_fused_kernel, kRThreads, smem);
    if (err != cudaSuccess) return err;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    int64_t grid = (int64_t)num_sms() * per_sm;
    const int64_t need = (p.n_traces + kRWarps - 1) / kRWarps;
    if (grid > need) grid = need;
    roll_fused_kernel<<<(unsigned)grid, kRThreads, smem, s>>>(p);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_plan(const PlanParams& p, cudaStream_t s) {
    if (p.n_traces <= 0 || p.W <= 0) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, p.tables_bytes);
    if (e != cudaSuccess) return e;
    const int64_t groups = p.n_traces * ((p.W + 3) / 4);
    int64_t grid = (groups + 255) / 256;
    if (grid > (int64_t)num_sms() * 8) grid = (int64_t)num_sms() * 8;
    plan_kernel<<<(unsigned)grid, 256, p.tables_bytes, s>>>(p);
    ++g_launches;
    return cudaGetLastError();
}

int roll_phase_doubles(int T, int L) { return T * roll_phase_stride(L); }

cudaError_t launch_rolling(const void* traces, bool f64, int64_t ld, int64_t n_traces, int N, int L, int T, int phase0,
                           int R, double ridge, double tol, const double* phase, double* ptab, double* records,
                           double max_ci_fixed, double* forecast, int64_t ld_f, cudaStream_t s) {
    if (n_traces <= 0) return cudaSuccess;
    rolling_phase_kernel<<<(T + 127) / 128, 128, 0, s>>>(phase, phase + T, T, L, ptab);
    ++g_launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    RollParams p;
    p.traces = traces;
    p.ld = ld;
    p.n_traces = n_traces;
    p.N = N;
    p.L = L;
    p.T = T;
    p.phase0 = phase0;
    p.R = R;
    p.n_orig = (N - L + R - 1) / R;
    p.ridge = ridge;
    p.tol = tol;
    p.phase = phase;
    p.ptab = ptab;
    p.records = records;
    p.max_ci_fixed = max_ci_fixed;
    p.forecast = forecast;
    p.ld_f = ld_f;
    const int64_t total = n_traces * (int64_t)p.n_orig;
    const int64_t grid = (total + 127) / 128;
    if (grid > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    if (f64) rolling_forecast_kernel<double><<<(unsigned)grid, 128, 0, s>>>(p);
    else rolling_forecast_kernel<float><<<(unsigned)grid, 128, 0, s>>>(p);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_periods(const void* traces, bool f64, int64_t ld, int64_t n_traces, int N, int L, int T, int phase0,
                           int P, const double* phase, const double* records, double* forecast, int64_t ld_f,
                           cudaStream_t s) {
    if (n_traces <= 0) return cudaSuccess;
    PeriodParams p;
    p.traces = traces;
    p.ld = ld;
    p.n_traces = n_traces;
    p.N = N;
    p.L = L;
    p.T = T;
    p.phase0 = phase0;
    p.P = P;
    p.n_per = (N - L + P - 1) / P;
    p.phase = phase;
    p.records = records;
    p.forecast = forecast;
    p.ld_f = ld_f;
    const int64_t warps = n_traces * (int64_t)((p.n_per + 31) / 32);
    const int64_t grid = (warps + 3) / 4;
    if (grid > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    if (f64) period_forecast_kernel<double><<<(unsigned)grid, 128, 0, s>>>(p);
    else period_forecast_kernel<float><<<(unsigned)grid, 128, 0, s>>>(p);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_mape(const void* traces, bool f64, int64_t ld, int64_t n_traces, int N, int L, int T, int phase0,
                        const double* phase, const double* records, const double* fc_in, int64_t ld_fin, double* out,
                        int32_t* status, cudaStream_t s) {
    if (n_traces <= 0) return cudaSuccess;
    MapeParams p;
    p.traces = traces;
    p.ld = ld;
    p.n_traces = n_traces;
    p.N = N;
    p.L = L;
    p.T = T;
    p.phase0 = phase0;
    p.phase = phase;
    p.records = records;
    p.fc_in = fc_in;
    p.ld_fin = ld_fin;
    p.out = out;
    p.status = status;
    int64_t grid = (n_traces + 7) / 8;
    const int64_t cap = (int64_t)num_sms() * 8;
    if (grid > cap) grid = cap;
    const int smem = mape_smem_bytes(T);
    auto kern = f64 ? (fc_in ? mape_kernel<double, true> : mape_kernel<double, false>)
                    : (fc_in ? mape_kernel<float, true> : mape_kernel<float, false>);
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<(unsigned)grid, 256, smem, s>>>(p);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_svr(const void* traces, bool f64, int64_t ld, int64_t n_traces, int N, int L, int T, int phase0,
                       int P, double C, double eps, double gamma, double tol, int max_iter, const double* phase,
                       double* records, double* models, double* forecast, int64_t ld_f, cudaStream_t s) {
    static_assert(kSvrModelDoubles == kSvrDoubles, "model record size");
    if (n_traces <= 0) return cudaSuccess;
    if (L - 1 > kSvrMaxN || L < 3) return cudaErrorInvalidValue;
    SvrParams p;
    p.traces = traces;
    p.ld = ld;
    p.n_traces = n_traces;
    p.N = N;
    p.L = L;
    p.T = T;
    p.phase0 = phase0;
    p.max_iter = max_iter;
    p.P = P < 1 ? 1 : P;
    p.n_per = (N - L + p.P - 1) / p.P;
    p.C = C;
    p.eps = eps;
    p.gamma = gamma;
    p.tol = tol;
    p.phase = phase;
    p.models = models;
    p.records = records;
    p.forecast = forecast;
    p.ld_f = ld_f;
    const int smem = kSvrWarps * svr_smem_doubles(L) * 8;
    const int64_t grid = (n_traces + kSvrWarps - 1) / kSvrWarps;
    if (grid > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    if (f64) {
        cudaFuncSetAttribute(svr_fit_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        svr_fit_kernel<double><<<(unsigned)grid, 32 * kSvrWarps, smem, s>>>(p);
    } else {
        cudaFuncSetAttribute(svr_fit_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        svr_fit_kernel<float><<<(unsigned)grid, 32 * kSvrWarps, smem, s>>>(p);
    }
    ++g_launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int64_t chunks = (p.n_per + kSvrFcThreads * kSvrFcPer - 1) / (kSvrFcThreads * kSvrFcPer);
    if (n_traces > 0x7fffffffLL || chunks > 65535) return cudaErrorInvalidConfiguration;
    const dim3 g2((unsigned)n_traces, (unsigned)chunks);
    const int smem2 = svr_fc_smem_doubles(L, T) * 8;
    if (smem2 > 48 * 1024) {
        cudaFuncSetAttribute(svr_forecast_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
        cudaFuncSetAttribute(svr_forecast_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
    }
    if (f64) svr_forecast_kernel<double><<<g2, kSvrFcThreads, smem2, s>>>(p);
    else svr_forecast_kernel<float><<<g2, kSvrFcThreads, smem2, s>>>(p);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_timeline(const void* traces, bool f64, int64_t ld, int64_t n_traces, int N, int L, int P,
                            int n_prof, double delta, const uint8_t* choice, int64_t ld_c, const double* forecast,
                            int64_t ld_f, const uint8_t* tables, const uint8_t* profile_id, const double* job,
                            const int64_t* ids, int64_t m, double* rows, double* summary, cudaStream_t s) {
    if (m <= 0) return cudaSuccess;
    TimelineParams p;
    p.traces = traces;
    p.ld = ld;
    p.n_traces = n_traces;
    p.N = N;
    p.L = L;
    p.P = P;
    p.n_prof = n_prof;
    p.delta = delta;
    p.choice = choice;
    p.ld_c = ld_c;
    p.forecast = forecast;
    p.ld_f = ld_f;
    p.tables = tables;
    p.profile_id = profile_id;
    p.job = job;
    p.ids = ids;
    p.m = m;
    p.rows = rows;
    p.summary = summary;
    const int64_t grid = (m + 3) / 4;
    if (f64) timeline_kernel<double><<<(unsigned)grid, 128, 0, s>>>(p);
    else timeline_kernel<float><<<(unsigned)grid, 128, 0, s>>>(p);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_profiling(const void* traces, bool f64, int64_t ld, int64_t n, int L, double delta,
                             const uint8_t* tables, int n_prof, const uint8_t* profile_id, double* out, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const int64_t grid = (n + 255) / 256;
    if (grid > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    if (f64) profiling_kernel<double><<<(unsigned)grid, 256, 0, s>>>(traces, ld, n, L, delta, tables, n_prof, profile_id, out);
    else profiling_kernel<float><<<(unsigned)grid, 256, 0, s>>>(traces, ld, n, L, delta, tables, n_prof, profile_id, out);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_period_costs(const double* forecast, int64_t ld_f, int64_t n_traces, int W, int P, int ld_k,
                                int n_prof, const uint8_t* tables, const uint8_t* profile_id, const double* max_ci,
                                double max_ci_fixed, const int64_t* ids, int64_t m, double* costs, cudaStream_t s) {
    if (m <= 0) return cudaSuccess;
    CostParams p;
    p.forecast = forecast;
    p.ld_f = ld_f;
    p.n_traces = n_traces;
    p.W = W;
    p.P = P;
    p.n_per = (W + P - 1) / P;
    p.ld_k = ld_k;
    p.n_prof = n_prof;
    p.tables = tables;
    p.profile_id = profile_id;
    p.max_ci = max_ci;
    p.max_ci_fixed = max_ci_fixed;
    p.ids = ids;
    p.m = m;
    p.costs = costs;
    const int64_t total = m * (int64_t)p.n_per * ld_k;
    const int64_t grid = (total + 255) / 256;
    if (grid > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    period_cost_kernel<<<(unsigned)grid, 256, 0, s>>>(p);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_fixup(const uint8_t* status, const int64_t* bad_list, int64_t n_traces, uint8_t* choice,
                         int64_t ld_c, int64_t W, int n_eta_choice, double* forecast, int64_t ld_f,
                         chase_diag_t* diag, cudaStream_t s) {
    if (n_traces <= 0) return cudaSuccess;
    if (choice || forecast) {  // (with the first-bad status)
        fixup_kernel<<<(unsigned)(2 * num_sms()), 256, 0, s>>>(bad_list, diag, n_traces, choice, ld_c, W, n_eta_choice,
                                                                forecast, ld_f, status);
    } else {
        diag_status_kernel<<<1, 32, 0, s>>>(status, n_traces, diag);
    }
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_finalize(const FinalizeParams& p, const int64_t* bad_list, chase_sum_t* sum, uint8_t* choice,
                            int64_t ld_c, int n_eta_choice, double* forecast, int64_t ld_f, chase_diag_t* diag,
                            cudaStream_t s) {
    if (p.n_traces > 0) {
        const int64_t grid = finalize_grid(p.n_traces);
        FinalizeParams q = p;
        q.sum_direct = grid == 1 ? sum : nullptr;  // one block writes the sums itself
        if (p.is_f64) finalize_kernel<double><<<(unsigned)grid, kFinThreads, 0, s>>>(q);
        else finalize_kernel<float><<<(unsigned)grid, kFinThreads, 0, s>>>(q);
        ++g_launches;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        if (sum && grid > 1) {
            finalize_sums_kernel<<<p.n_eta, 256, 0, s>>>(p.block_sums, grid, p.n_eta, sum);
            ++g_launches;
        }
    } else if (sum) {
        cudaError_t e = cudaMemsetAsync(sum, 0, sizeof(chase_sum_t) * (size_t)p.n_eta, s);
        if (e != cudaSuccess) return e;
    }
    return launch_fixup(p.status, bad_list, p.n_traces, choice, ld_c, p.W, n_eta_choice, forecast, ld_f, diag, s);
}

cudaError_t launch_diag_reset(chase_diag_t* diag, cudaStream_t s) {
    diag_reset_kernel<<<1, 32, 0, s>>>(diag);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_diag_merge(chase_diag_t* acc, chase_diag_t* chunk, int64_t c0, cudaStream_t s) {
    if (c0 == 0) diag_reset_kernel<<<1, 32, 0, s>>>(acc);
    if (c0 == 0) ++g_launches;
    diag_merge_kernel<<<1, 32, 0, s>>>(acc, chunk, c0);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_diag_merge_eta(chase_diag_t* acc, const uint8_t* ws, size_t slice, size_t diag_off,
                                  size_t status_off, int n_eta, int64_t n, cudaStream_t s) {
    diag_merge_eta_kernel<<<1, 256, 0, s>>>(acc, ws, slice, diag_off, status_off, n_eta, n);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_accumulate(double* acc, const double* add, int n, cudaStream_t s) {
    accumulate_sums_kernel<<<1, 128, 0, s>>>(acc, add, n);
    ++g_launches;
    return cudaGetLastError();
}

}  // namespace chase
