// finalize.cuh — per-trace totals, fixed-order sums, fix-up, plan-from-forecast
// and upload kernels (included by kernels.cu).

// ------------------------------------------------------------------ finalize (K3)
// Per trace: the replay totals of DESIGN R2 (stepwise carbon S:432, pro-rata
// last window S:433, exhaustion S:436) and the max-power baseline,
// in the oracle's operation order; then fixed-order block sums.
template <typename E>
__global__ void __launch_bounds__(kFinThreads) finalize_kernel(const __grid_constant__ FinalizeParams p) {
    __shared__ double red[kFinThreads][8];
    const int64_t i = (int64_t)blockIdx.x * kFinThreads + threadIdx.x;
    const bool valid = i < p.n_traces;
    const E* traces = reinterpret_cast<const E*>(p.traces);
    int st = valid ? (int)p.status[i] : 1;
    double bt = 0.0, be = 0.0, bc = 0.0;
    int bstat = 0, worst = st;
    double J = 0.0;
    int prof = 0;
    const ProfileTable* pf = nullptr;
    if (valid && st == 0) {
        prof = p.profile_id ? (int)p.profile_id[i] : 0;
        if (prof >= p.n_prof) prof = 0;
        pf = blob_profiles(p.tables) + prof;
        J = p.job ? p.job[i] : 0.0;
        const double* rec = p.records + i * kRecDoubles;
        const double sbv = pf->line[pf->K - 1].x, Pb = pf->line[pf->K - 1].y, Cb = rec[9];
        const int64_t m = (int64_t)rec[8];
        if (J > 0.0 && m >= 1 && m <= p.W) {
            const double prevS = __dmul_rn((double)(m - 1), sbv);
            const double f = __ddiv_rn(__dsub_rn(J, prevS), sbv);
            const double Eb = __dmul_rn((double)(m - 1), Pb);
            const double Cbp = __dmul_rn(Pb, Cb);
            const double cst = (double)traces[i * p.ld + p.L + (m - 1)];
            bt = __dmul_rn(__dadd_rn((double)(m - 1), f), p.delta);
            be = __dmul_rn(__dadd_rn(Eb, __dmul_rn(f, Pb)), p.delta);
            bc = __ddiv_rn(__dmul_rn(__dadd_rn(Cbp, __dmul_rn(f, __dmul_rn(Pb, cst))), p.delta), 3.6e6);
        } else {
            bt = __dmul_rn((double)p.W, p.delta);
            be = __dmul_rn(__dmul_rn((double)p.W, Pb), p.delta);
            bc = __ddiv_rn(__dmul_rn(__dmul_rn(Pb, Cb), p.delta), 3.6e6);
            if (J > 0.0) bstat = CHASE_ERR_TRACE_EXHAUSTED;
        }
    }
    for (int e = 0; e < p.n_eta; ++e) {
        double v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (valid) {
            chase_totals_t t;
            t.time_s = t.energy_j = t.carbon_g = t.samples = 0.0;
            t.base_time_s = t.base_energy_j = t.base_carbon_g = 0.0;
            t.completion_window = -1;
            t.status = st;
            if (st == 0) {
                const double* r = p.raw + ((int64_t)e * p.n_traces + i) * kRawDoubles;
                int ste = 0;
                if (r[7] != 0.0) {
                    const double f = r[3], Pk = r[5];
                    const int64_t wstar = (int64_t)r[4];
                    t.time_s = __dmul_rn(__dadd_rn((double)(wstar - p.L), f), p.delta);
                    t.energy_j = __dmul_rn(__dadd_rn(r[0], __dmul_rn(f, Pk)), p.delta);
                    t.carbon_g = __ddiv_rn(__dmul_rn(__dadd_rn(r[1], __dmul_rn(f, __dmul_rn(Pk, r[6]))), p.delta), 3.6e6);
                    t.samples = J;
                    t.completion_window = (int32_t)wstar;
                } else {
                    t.time_s = __dmul_rn((double)p.W, p.delta);
                    t.energy_j = __dmul_rn(r[0], p.delta);
                    t.carbon_g = __ddiv_rn(__dmul_rn(r[1], p.delta), 3.6e6);
                    t.samples = r[2];
                    if (J > 0.0) ste = CHASE_ERR_TRACE_EXHAUSTED;
                }
                t.base_time_s = bt;
                t.base_energy_j = be;
                t.base_carbon_g = bc;
                t.status = ste ? ste : bstat;
                if (t.status > worst) worst = t.status;
                if (t.status == 0) {
                    v[0] = t.time_s; v[1] = t.energy_j; v[2] = t.carbon_g; v[3] = t.samples;
                    v[4] = bt; v[5] = be; v[6] = bc; v[7] = 1.0;
                }
            }
            if (p.per_trace) p.per_trace[(int64_t)e * p.n_traces + i] = t;
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) red[threadIdx.x][r] = v[r];
        __syncthreads();
        if (threadIdx.x < 8) {
            double acc = 0.0;
            for (int t = 0; t < kFinThreads; ++t) acc = __dadd_rn(acc, red[t][threadIdx.x]);
            p.block_sums[((int64_t)blockIdx.x * p.n_eta + e) * 8 + threadIdx.x] = acc;
            // one block: finalize_sums_kernel would fold exactly this value (0 + acc, + 0s)
            if (p.sum_direct) reinterpret_cast<double*>(p.sum_direct + e)[threadIdx.x] = acc;
        }
        __syncthreads();
    }
    if (valid) p.status[i] = (uint8_t)worst;
    const unsigned ex = __ballot_sync(0xffffffffu, valid && worst == CHASE_ERR_TRACE_EXHAUSTED);
    if ((threadIdx.x & 31) == 0 && ex)
        atomicAdd(reinterpret_cast<unsigned long long*>(&p.diag->n_exhausted), (unsigned long long)__popc(ex));
}

// Per-GPU sums of the finalize blocks' partials: thread t folds the blocks
// b = t, t + 256, ... in order, then a fixed smem tree (deterministic).
__global__ void __launch_bounds__(256) finalize_sums_kernel(const double* block_sums, int64_t grid, int n_eta,
                                                            chase_sum_t* sum) {
    __shared__ double red[256][8];
    const int e = blockIdx.x, t = threadIdx.x;
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t b = t; b < grid; b += 256) {
        const double* src = block_sums + (b * n_eta + e) * 8;
#pragma unroll
        for (int r = 0; r < 8; ++r) acc[r] = __dadd_rn(acc[r], src[r]);
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) red[t][r] = acc[r];
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (t < w)
#pragma unroll
            for (int r = 0; r < 8; ++r) red[t][r] = __dadd_rn(red[t][r], red[t + w][r]);
        __syncthreads();
    }
    if (t < 8) reinterpret_cast<double*>(sum + e)[t] = red[0][t];
}

// Invalid traces (status 4..7; listed by the sweep kernels as they finish a
// trace): choices 0xFF, forecasts NaN.
__global__ void fixup_kernel(const int64_t* bad_list, chase_diag_t* diag, int64_t n, uint8_t* choice,
                             int64_t ld_c, int64_t W, int n_eta, double* forecast, int64_t ld_f,
                             const uint8_t* status) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // (diag_status_kernel's work, one launch fewer)
        const uint64_t fb = (uint64_t)diag->first_bad_trace;
        if (fb < (uint64_t)n) diag->first_bad_status = status[fb];
    }
    const int64_t n_bad = (int64_t)diag->n_bad;
    for (int64_t b = blockIdx.x; b < n_bad; b += gridDim.x) {
        const int64_t i = bad_list[b];
        if (choice)
            for (int e = 0; e < n_eta; ++e)
                for (int64_t w = threadIdx.x; w < W; w += blockDim.x) choice[((int64_t)e * n + i) * ld_c + w] = 0xff;
        if (forecast)
            for (int64_t w = threadIdx.x; w < W; w += blockDim.x)
                forecast[i * ld_f + w] = __longlong_as_double(0x7ff8000000000000ll);
    }
}

__global__ void diag_status_kernel(const uint8_t* status, int64_t n, chase_diag_t* diag) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        const uint64_t fb = (uint64_t)diag->first_bad_trace;
        if (fb < (uint64_t)n) diag->first_bad_status = status[fb];
    }
}

__global__ void diag_reset_kernel(chase_diag_t* d) {
    if (threadIdx.x == 0) {
        d->first_bad_trace = -1;  // all ones: atomicMin (unsigned) finds the lowest index
        d->first_bad_status = 0;
        d->n_bad = d->n_exhausted = d->n_slow_windows = d->kernel_path = d->n_seq_periods = 0;
    }
}

// chase_sweep_host: fold one chunk's diagnostics (trace indices local to the
// chunk, offset by its first trace c0) into the call's accumulated ones; with
// c0 < 0 copy the accumulated diagnostics back into the workspace.
__global__ void diag_merge_kernel(chase_diag_t* acc, chase_diag_t* chunk, int64_t c0) {
    if (threadIdx.x != 0) return;
    if (c0 < 0) {
        *chunk = *acc;
        return;
    }
    const uint64_t fb = (uint64_t)chunk->first_bad_trace;
    if (fb != ~0ull && (uint64_t)(fb + c0) < (uint64_t)acc->first_bad_trace) {
        acc->first_bad_trace = (int64_t)(fb + c0);
        acc->first_bad_status = chunk->first_bad_status;
    }
    acc->n_bad += chunk->n_bad;
    acc->n_exhausted += chunk->n_exhausted;
    acc->n_slow_windows += chunk->n_slow_windows;
    acc->n_seq_periods += chunk->n_seq_periods;
    acc->kernel_path |= chunk->kernel_path;
}

// chase_sweep's eta split: fold the one-eta slices' diagnostics
// into slice 0's (in place).  Every slice validates the same traces, so n_bad
// and first_bad stay slice 0's; n_exhausted is recounted per trace from the
// slices' status bytes (a trace counts once, at its worst status over the
// eta, as finalize_kernel counts it); the rest add up.
__global__ void diag_merge_eta_kernel(chase_diag_t* acc, const uint8_t* ws, size_t slice, size_t diag_off,
                                      size_t status_off, int n_eta, int64_t n) {
    __shared__ unsigned long long ex;
    if (threadIdx.x == 0) ex = 0;
    __syncthreads();
    unsigned long long mine = 0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        uint8_t worst = 0;
        for (int e = 0; e < n_eta; ++e) worst = max(worst, ws[(size_t)e * slice + status_off + i]);
        mine += worst == CHASE_ERR_TRACE_EXHAUSTED ? 1ull : 0ull;
    }
    atomicAdd(&ex, mine);
    __syncthreads();
    if (threadIdx.x == 0) {
        acc->n_exhausted = ex;
        for (int e = 1; e < n_eta; ++e) {
            const chase_diag_t* d = reinterpret_cast<const chase_diag_t*>(ws + (size_t)e * slice + diag_off);
            acc->n_slow_windows += d->n_slow_windows;
            acc->n_seq_periods += d->n_seq_periods;
            acc->kernel_path |= d->kernel_path;
        }
    }
}

__global__ void accumulate_sums_kernel(double* acc, const double* add, int n) {
    const int q = threadIdx.x;
    if (q < n) acc[q] = __dadd_rn(acc[q], add[q]);
}

// ------------------------------------------------------------------ plan from forecasts
__global__ void __launch_bounds__(256) plan_kernel(const __grid_constant__ PlanParams p) {
    extern __shared__ __align__(16) uint8_t psm[];
    for (int q = threadIdx.x; q < p.tables_bytes / 16; q += blockDim.x)
        reinterpret_cast<uint4*>(psm)[q] = reinterpret_cast<const uint4*>(p.tables)[q];
    __syncthreads();
    const TablesHeader* H = reinterpret_cast<const TablesHeader*>(psm);
    const ProfileTable* profs = reinterpret_cast<const ProfileTable*>(psm + H->off_prof);
    const PairTable* pairs = reinterpret_cast<const PairTable*>(psm + H->off_pair);
    const int64_t groups = (p.W + 3) / 4;  // 4 windows per thread-step
    const int64_t total = p.n_traces * groups;
    int64_t slow_count = 0;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = g / groups, w0 = (g - i * groups) * 4;
        int prof = p.profile_id ? (int)p.profile_id[i] : 0;
        if (prof >= p.n_prof) prof = 0;
        const ProfileTable* pf = profs + prof;
        const double maxci = p.max_ci_fixed > 0.0 ? p.max_ci_fixed : p.max_ci[i];
        const bool trace_ok = maxci > 0.0;
        double x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) x[u] = w0 + u < p.W ? p.forecast[i * p.ld_f + w0 + u] : 0.0;
        for (int e = 0; e < p.n_eta; ++e) {
            const PairTable* pt = pairs + prof * p.n_eta + e;
            const double Kc = __dmul_rn(pt->kbase, maxci);
            const double invK = per_trace_invK(pt, Kc);
            uint32_t word = 0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                uint32_t k = 0xffu;
                if (w0 + u < p.W && trace_ok && x[u] >= 0.0 && x[u] <= DBL_MAX) {
                    k = plan_lookup(__dmul_rn(x[u], invK), pt);
                    if (k == (uint32_t)kZeroLine) {
                        k = canonical_choose(x[u], Kc, pt->a, pf->thr, pf->K);
                        ++slow_count;
                    }
                }
                word |= k << (8 * u);
            }
            *reinterpret_cast<uint32_t*>(p.choice + ((int64_t)e * p.n_traces + i) * p.ld_c + w0) = word;
        }
    }
    unsigned long long sc = (unsigned long long)slow_count;
    for (int o = 16; o > 0; o >>= 1) sc += __shfl_xor_sync(kFull, sc, o);
    if ((threadIdx.x & 31) == 0 && sc) atomicAdd(reinterpret_cast<unsigned long long*>(&p.diag->n_slow_windows), sc);
}

struct UploadChunk {
    uint8_t bytes[30720];
};
__global__ void upload_kernel(const __grid_constant__ UploadChunk c, int n, uint8_t* dst, chase_diag_t* reset) {
    if (reset && threadIdx.x == 0) {  // (diag_reset_kernel's work, one launch fewer)
        reset->first_bad_trace = -1;
        reset->first_bad_status = 0;
        reset->n_bad = reset->n_exhausted = reset->n_slow_windows = reset->kernel_path = reset->n_seq_periods = 0;
    }
    for (int q = threadIdx.x; q < n; q += blockDim.x) dst[q] = c.bytes[q];
}

