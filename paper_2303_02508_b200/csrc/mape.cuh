// mape.cuh — forecast-evaluation sweep, included by
// kernels.cu inside its anonymous namespace.
//
// SPEC evaluate_models (the walk-forward Table 1 experiment of
// P:159-161): the fit-once model (fit_kernel's record) predicts every window
// w = L..N-1 from the TRUE lag c[w-1], and the MAPE of those
// predictions and of persistence p(w) = c[w-1] is reported per trace.  One
// warp per trace, lanes on consecutive windows (coalesced loads); per-lane
// fp64 partial sums of |a - p| * (1/a), then a fixed warp tree (≤ 1e-9 of the
// oracle's sequential sum; the predictions themselves are bit-identical).
struct MapeParams {
    const void* traces;
    int64_t ld, n_traces;
    int32_t N, L, T, phase0;
    const double* phase;    // S[T], C[T]
    const double* records;  // fit-once models [n][16]
    const double* fc_in;    // [n][ld_fin] predictions (the SVR's) or null: Eq. 1 from the record
    int64_t ld_fin;
    double* out;            // [n][2]: MAPE linear, MAPE persistence (percent; NaN if undefined)
    int32_t* status;        // [n] or null: 0, 4 bad value, 6 fit failed, 8 zero actual
};

template <typename E>
__global__ void __launch_bounds__(256) mape_kernel(const __grid_constant__ MapeParams p) {
    extern __shared__ double ph_sm[];
    const int T = p.T;
    for (int q = threadIdx.x; q < 2 * T; q += blockDim.x) ph_sm[q] = p.phase[q];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t GW = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int s0 = p.L;
    const int64_t n = p.N - s0;
    for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < p.n_traces; i += GW) {
        const double* rec = p.records + i * kRecDoubles;
        int st = (int)rec[5];
        const double c0 = rec[0], ws = rec[1], wc = rec[2], wl = rec[3];
        const E* row = reinterpret_cast<const E*>(p.traces) + i * p.ld;
        double el = 0.0, ep = 0.0;
        int bad = 0, zero = 0;
        // 4 windows per lane per iteration (w = base + lane + 32u): 8 independent loads in flight
        int ph = (int)(((int64_t)p.phase0 + s0 + lane) % T);
        const int step32 = 32 % T;
        for (int base = s0; base < p.N; base += 128) {
            E raw[4], lagr[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int w = base + lane + 32 * u;
                raw[u] = w < p.N ? row[w] : (E)1;
                lagr[u] = w < p.N ? row[w - 1] : (E)1;
            }
            int phu = ph;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int w = base + lane + 32 * u;
                if (w < p.N) {
                    const double cw = (double)raw[u], lag = (double)lagr[u];
                    bad |= bad_value(raw[u]) ? 1 : 0;
                    zero |= cw == 0.0 ? 1 : 0;
                    double pred;
                    if (p.fc_in) {
                        pred = p.fc_in[i * p.ld_fin + (w - s0)];
                    } else {  // Eq. 1 prediction, oracle_predict's rounding order
                        const double A =
                            __dadd_rn(__dadd_rn(c0, __dmul_rn(ws, ph_sm[phu])), __dmul_rn(wc, ph_sm[T + phu]));
                        const double pr = __dadd_rn(A, __dmul_rn(wl, lag));
                        pred = pr > 0.0 ? pr : 0.0;
                    }
                    const double r = __drcp_rn(cw);
                    el = __dadd_rn(el, __dmul_rn(fabs(__dsub_rn(cw, pred)), r));
                    ep = __dadd_rn(ep, __dmul_rn(fabs(__dsub_rn(cw, lag)), r));
                }
                phu += step32;
                if (phu >= T) phu -= T;
            }
            ph = phu;
        }
        el = warp_sum(el);
        ep = warp_sum(ep);
        bad = (int)__reduce_or_sync(kFull, (unsigned)bad);
        zero = (int)__reduce_or_sync(kFull, (unsigned)zero);
        if (lane == 0) {
            if (st == 0 && bad) st = CHASE_ERR_DATA;
            if (st == 0 && zero) st = CHASE_ERR_ZERO_ACTUAL;
            const double k = __ddiv_rn(100.0, (double)n);
            p.out[2 * i] = st == 0 ? __dmul_rn(k, el) : CUDART_NAN;
            p.out[2 * i + 1] = (st == 0 || st == CHASE_ERR_ZERO_ACTUAL) && !zero ? __dmul_rn(k, ep) : CUDART_NAN;
            if (p.status) p.status[i] = st;
        }
    }
}
