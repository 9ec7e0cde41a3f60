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

#ifndef CHASE_MAPE_KV
#define CHASE_MAPE_KV 2
#endif

// 1/c to ~1e-13 relative: the MUFU seed (~2^-22) and one Newton step in fp64
// (a MAPE term needs <= 1e-9; the reciprocal seed runs on the SFU pipe).
__device__ __forceinline__ double rcp_nr(double c) {
    double r0;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r0) : "d"(c));
    const double e = __fma_rn(-c, r0, 1.0);
    return __fma_rn(r0, e, r0);
}

// Exact float -> double for a positive normal float, on the integer pipe
// (F2F.F64.F32 runs at ~1/3 of the DADD rate, profiles/fp64_probe.json).
__device__ __forceinline__ double f2d_normal(uint32_t u) {
    return __hiloint2double((int)((u >> 3) + 0x38000000u), (int)(u << 29));
}
// u is a positive normal finite float (the fast path's precondition)
__device__ __forceinline__ bool f32_normal_pos(uint32_t u) { return u - 0x00800000u < 0x7f000000u; }

// One trace, the plain per-window order (cold: f64 traces, subnormal floats, the SVR forecasts).
template <typename E>
__device__ __noinline__ void mape_trace_exact(const MapeParams& p, const double* ph_sm, int64_t i, double c0,
                                              double ws, double wc, double wl, int lane, double& el, double& ep,
                                              int& bad, int& zero) {
    const int T = p.T, s0 = p.L;
    const E* row = reinterpret_cast<const E*>(p.traces) + i * p.ld;
    for (int w = s0 + lane; w < p.N; w += 32) {
        const E raw = row[w];
        const double cw = (double)raw, lag = (double)row[w - 1];
        bad |= bad_value(raw) ? 1 : 0;
        zero |= cw == 0.0 ? 1 : 0;
        double pred;
        if (p.fc_in) {
            pred = p.fc_in[i * p.ld_fin + (w - s0)];
        } else {
            const int ph = (int)(((int64_t)p.phase0 + w) % T);
            const double A = __dadd_rn(__dadd_rn(c0, __dmul_rn(ws, ph_sm[ph])), __dmul_rn(wc, ph_sm[T + ph]));
            const double pr = __dadd_rn(A, __dmul_rn(wl, lag));
            pred = pr > 0.0 ? pr : 0.0;
        }
        const double r = __drcp_rn(cw);
        el = __dadd_rn(el, __dmul_rn(fabs(__dsub_rn(cw, pred)), r));
        ep = __dadd_rn(ep, __dmul_rn(fabs(__dsub_rn(cw, lag)), r));
    }
}

// Per warp shared memory: A_ext[T + 4], A(phi) = (c0 + w_s S[phi]) + w_c C[phi] (oracle_predict's fold).
__host__ __device__ inline int mape_smem_bytes(int T) { return (2 * T + 8 * (T + 4)) * 8; }

// Fast path (fp32 traces, Eq. 1 forecasts): each lane takes 4 consecutive
// windows per step (one 16-byte load, the lag of the first from the lane
// below by a shuffle), 128 windows per warp step, four steps' loads in flight.
#ifndef CHASE_MAPE_MINB
#define CHASE_MAPE_MINB 4  // <= 64 registers (uncapped: 108-112 with the FIN variant; 9.84 vs 10.27 ms)
#endif
template <typename E, bool FIN>
__global__ void __launch_bounds__(256, CHASE_MAPE_MINB) mape_kernel(const __grid_constant__ MapeParams p) {
    extern __shared__ double ph_sm[];
    const int T = p.T;
    for (int q = threadIdx.x; q < 2 * T; q += blockDim.x) ph_sm[q] = p.phase[q];
    __syncthreads();
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    double* Aw = ph_sm + 2 * T + wib * (T + 4);
    const int64_t GW = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int s0 = p.L;
    const int64_t n = p.N - s0;
    for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib; i < p.n_traces; i += GW) {
        const double* rec = p.records + i * kRecDoubles;
        int st = (int)rec[5];
        const double c0 = rec[0], ws = rec[1], wc = rec[2], wl = rec[3];
        double el = 0.0, ep = 0.0;
        int bad = 0, zero = 0;
        bool exact = sizeof(E) != 4;
        const double* fcrow = FIN ? p.fc_in + i * p.ld_fin - s0 : nullptr;  // fcrow[w]: window w's forecast
        if (!exact) {
            for (int q = lane; q < T + 4; q += 32) {
                const int ph = q < T ? q : q - T;
                Aw[q] = __dadd_rn(__dadd_rn(c0, __dmul_rn(ws, ph_sm[ph])), __dmul_rn(wc, ph_sm[T + ph]));
            }
            __syncwarp();
            const uint32_t* row = reinterpret_cast<const uint32_t*>(p.traces) + i * p.ld;
            const int a0 = s0 & ~3;                       // 16-byte aligned start (row starts are aligned)
            uint32_t carry = __ldg(row + a0 - 1);         // c[a0 - 1]: the lag of lane 0's first window
            // every value in [s0 - 1, N) must be a positive normal float for the fast path; anything
            // else (zero, negative, inf / NaN, subnormal) sends the trace to the exact path
            uint32_t umin = __ldg(row + s0 - 1), umax = umin;
            int ph = (int)(((int64_t)p.phase0 + a0 + 4 * lane) % T);
            const int step_ph = 128 % T;
            constexpr int kV = CHASE_MAPE_KV;             // 16-byte loads per lane per step
            // one 4-window vector: windows w0..w0+3 (check: some outside [s0, N))
            auto vec = [&](const uint4 v, const uint32_t lagbits, const int w0, const bool check) {
                const uint32_t uu[4] = {v.x, v.y, v.z, v.w};
                double lag = f2d_normal(lagbits);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int w = w0 + u;
                    const uint32_t b = uu[u];
                    if (check && w < s0) {  // a history value: only the next window's lag
                        lag = f2d_normal(b);
                        continue;
                    }
                    if (check && w >= p.N) continue;
                    umin = min(umin, b);
                    umax = max(umax, b);
                    const double cw = f2d_normal(b);
                    double pred;
                    if (FIN) {  // the SVR's forecast (already clamped)
                        pred = fcrow[w];
                    } else {
                        const double pr = __dadd_rn(Aw[ph + u], __dmul_rn(wl, lag));
                        const long long pb = __double_as_longlong(pr);
                        pred = __longlong_as_double(pb & ~(pb >> 63));  // max(pr, 0)
                    }
                    const double r = rcp_nr(cw);
                    el = __dadd_rn(el, __dmul_rn(fabs(__dsub_rn(cw, pred)), r));
                    ep = __dadd_rn(ep, __dmul_rn(fabs(__dsub_rn(cw, lag)), r));
                    lag = cw;
                }
            };
            // software pipeline: the next step's kV vectors load while this step's compute
            auto load = [&](uint4* v, const int base) {
                if (base + 128 * kV <= p.N) {  // whole step inside the row (uniform): no bounds checks
#pragma unroll
                    for (int q = 0; q < kV; ++q) v[q] = __ldg(reinterpret_cast<const uint4*>(row + base + 128 * q + 4 * lane));
                    return;
                }
#pragma unroll
                for (int q = 0; q < kV; ++q) {
                    const int w0 = base + 128 * q + 4 * lane;
                    if (w0 + 4 <= p.N) {
                        v[q] = __ldg(reinterpret_cast<const uint4*>(row + w0));
                    } else {
                        v[q].x = w0 < p.N ? __ldg(row + w0) : 0x3f800000u;
                        v[q].y = w0 + 1 < p.N ? __ldg(row + w0 + 1) : 0x3f800000u;
                        v[q].z = w0 + 2 < p.N ? __ldg(row + w0 + 2) : 0x3f800000u;
                        v[q].w = 0x3f800000u;
                    }
                }
            };
            uint4 vc[kV];
            load(vc, a0);
            for (int base = a0; base < p.N; base += 128 * kV) {
                uint4 vn[kV];
                if (base + 128 * kV < p.N) load(vn, base + 128 * kV);
                const bool interior = base >= s0 && base + 128 * kV <= p.N;
#pragma unroll
                for (int q = 0; q < kV; ++q) {
                    const uint32_t up = __shfl_up_sync(kFull, vc[q].w, 1);
                    const uint32_t lag0 = lane == 0 ? carry : up;
                    carry = __shfl_sync(kFull, vc[q].w, 31);
                    const int w0 = base + 128 * q + 4 * lane;
                    if (interior) vec(vc[q], lag0, w0, false);
                    else vec(vc[q], lag0, w0, true);
                    ph += step_ph;
                    if (ph >= T) ph -= T;
                }
#pragma unroll
                for (int q = 0; q < kV; ++q) vc[q] = vn[q];
            }
            exact = __any_sync(kFull, umin < 0x00800000u || umax > 0x7f7fffffu);
            if (exact) el = ep = 0.0;
        }
        if (exact) mape_trace_exact<E>(p, ph_sm, i, c0, ws, wc, wl, lane, el, ep, bad, zero);
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
        __syncwarp();
    }
}
