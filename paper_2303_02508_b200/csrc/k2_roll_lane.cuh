// k2_roll_lane.cuh — the rolling refit fused into the sweep, lane = trace
// (DESIGN §6.4).  Same method and tolerance contract as k2_roll.cuh (sliding
// raw moments, closed-form solve per origin, oracle_fit's exact sequence for
// near-degenerate fits), laid out for the FP64 work instead of for the stream:
//
//   - a warp plans 32 traces at once, lane l the trace 32 g + l, all lanes on
//     the same window index, so every phase-dependent quantity (S[phi],
//     C[phi], the origin phase's block inverse) is warp-uniform: broadcast
//     shared-memory reads;
//   - each lane slides its own trace's moments from job start to the end (one
//     direct sum per trace, then one row in and one out per window for R = 1;
//     R > 1: the direct sums of each origin's rows);
//   - the traces come in tiles of 64 windows (+ the L values before them) by
//     per-lane TMA bulk copies into a per-warp two-slot ring; a lane reads its
//     row with conflict-free 16-byte loads (odd row stride in 16-byte units);
//   - completion, baseline and validation are per lane: no warp collectives.
// Included by kernels.cu inside its anonymous namespace, after k2_roll.cuh.

#ifndef CHASE_RL_WARPS
#define CHASE_RL_WARPS 8
#endif
#ifndef CHASE_RL_GROUP
#define CHASE_RL_GROUP 4   // windows per unrolled group (overlapping solve chains)
#endif
constexpr int kRLWarps = CHASE_RL_WARPS;
constexpr int kRLThreads = 32 * kRLWarps;
#ifndef CHASE_RL_TILE
#define CHASE_RL_TILE 64
#endif
#ifndef CHASE_RL_ALIGN
#define CHASE_RL_ALIGN 1  // 1: tiles after the first start on 128-B boundaries
#endif
#ifndef CHASE_RL_HALO_COPY
#define CHASE_RL_HALO_COPY 1  // 1: tiles after a trace's first load only their own windows (4 B/window)
#endif
#ifndef CHASE_RL_MINB
#define CHASE_RL_MINB 1
#endif
constexpr int kRLTile = CHASE_RL_TILE;   // windows per tile (a multiple of 16)

// row stride (floats) of a tile: L + 64 values rounded to an odd number of 16-byte units
__host__ __device__ inline int rl_stride(int L) {
    int u = (L + kRLTile + 3) / 4;
    if ((u & 1) == 0) ++u;
    return 4 * u;
}

struct RLLayout {
    int tables, ptab, warp_bytes, total;
    int ring, chb, mbar;  // inside a warp block
    int stride;           // floats per row
};

__host__ __device__ inline RLLayout make_rllayout(int T, int L, int tables_bytes) {
    RLLayout R;
    R.stride = rl_stride(L);
    R.ring = 0;
    R.chb = 2 * 32 * R.stride * 4;                 // choice words: [32][kRLTile/4 + 1] u32 (odd stride)
    R.mbar = R.chb + 32 * (kRLTile / 4 + 1) * 4;
    R.warp_bytes = (R.mbar + 16 + 127) & ~127;
    R.tables = kRLWarps * R.warp_bytes;
    R.ptab = R.tables + round16(tables_bytes);
    R.total = R.ptab + round16(T * kRPhase * 8);
    return R;
}

// One lane's state over its trace (registers; the completion record is kept once).
struct RLState {
    RMom m;
    RModel md;
    double c_prev, o_prev;             // c[a-1], c[a-n-1] of the next window a
    double Sr, Er, Cr, Cb, Cs_all;     // replay sums, baseline c sum, validation sum
    double rE, rC, rf, rPk, rcw;       // the completion window's record
    int ph, rw, fit_bad;
    int to_origin;                     // R > 1: windows until the next refit origin (0: this one)
    unsigned n_slow;
    float vmin;
    bool done;
};

// The trace-level constants of a lane and of its current tile.
struct RLConst {
    const double* ptab;
    const double* S;
    const double* C;
    const PairTable* pt;
    const ProfileTable* pf;
    const float* row;       // this lane's tile row (row[q] = c[ab - L + q])
    const float* grow;      // the trace row in HBM
    double J, Kc, invK, dn, inv_n, ridge, tol;
    int L, T, n, phase0, R, mb, ab, nw, s0;
    bool live;
};

// Window a of a lane (cw = c[a], ov = c[a - n]): for R = 1 the closed-form fit of
// the current moments and their slide to a + 1, else (at an origin) the fit of
// the origin's rows; then the forecast, Eq. 6 and the replay in window order.
// MODE 0: R = 1 (a fit every window); 1: R > 1 with the moments slid every window
// and a fit at each origin; 2: R > 1 with each origin's moments from its rows.
template <int MODE>
__device__ __forceinline__ uint32_t rl_window(RLState& st, const RLConst& k, int a, double cw, double ov) {
    constexpr bool R1 = MODE == 0;
    const int w = a - k.s0;
    const double* rp = k.ptab + st.ph * kRPhase;
    if (MODE != 2) {
        if (MODE == 0 || st.to_origin == 0) {  // (MODE 1: an origin, w % R == 0; warp-uniform)
            if (!mom_solve_fast(st.m, st.c_prev, st.o_prev, k.dn, k.inv_n, rp, st.md)) {
                const RVals V{k.row, k.grow, k.ab - k.L, k.ab + k.nw};
                st.md = exact_model(V, a, k.L, k.T, k.phase0, k.S, k.C, k.ridge, k.tol);
                st.fit_bad |= st.md.status;
            }
        }
        // slide to a + 1: row a in, row a - n out (phase columns: the window's and the leaving row's)
        RMom& m = st.m;
        m.Sy = __dadd_rn(__dsub_rn(m.Sy, ov), cw);
        m.Syy = __fma_rn(-ov, ov, __fma_rn(cw, cw, m.Syy));
        m.Sly = __fma_rn(-st.o_prev, ov, __fma_rn(st.c_prev, cw, m.Sly));
        m.Ssy = __fma_rn(-rp[8], ov, __fma_rn(rp[6], cw, m.Ssy));
        m.Sky = __fma_rn(-rp[9], ov, __fma_rn(rp[7], cw, m.Sky));
        m.Ssl = __fma_rn(-rp[8], st.o_prev, __fma_rn(rp[6], st.c_prev, m.Ssl));
        m.Skl = __fma_rn(-rp[9], st.o_prev, __fma_rn(rp[7], st.c_prev, m.Skl));
    } else if (st.to_origin == 0) {  // an origin (w % R == 0; warp-uniform)
        const RVals V{k.row, k.grow, k.ab - k.L, k.ab + k.nw};
        const RMom mo = mom_direct(V, a, k.n, k.phase0, k.T, k.S, k.C);
        if (!mom_solve_fast(mo, st.c_prev, V(a - k.n - 1), k.dn, k.inv_n, rp, st.md)) {
            st.md = exact_model(V, a, k.L, k.T, k.phase0, k.S, k.C, k.ridge, k.tol);
            st.fit_bad |= st.md.status;
        }
    }
    const RModel& md = st.md;
    const double p = md.exact ? roll_predict(md, rp[6], rp[7], st.c_prev)
                              : __fma_rn(md.bl, st.c_prev, __fma_rn(md.bc, rp[7], __fma_rn(md.bs, rp[6], md.a)));
    st.c_prev = cw;
    st.o_prev = ov;
    st.ph = st.ph + 1 == k.T ? 0 : st.ph + 1;
    if (!R1) st.to_origin = st.to_origin == 0 ? k.R - 1 : st.to_origin - 1;
    // Eq. 6: the envelope lookup, the canonical rule in a band
    uint32_t kk = plan_lookup(__dmul_rn(p, k.invK), k.pt);
    if (kk == (uint32_t)kZeroLine || k.invK == 0.0) {
        kk = canonical_choose(p > 0.0 ? p : 0.0, k.Kc, k.pt->a, k.pf->thr, k.pf->K);
        st.n_slow += k.live ? 1u : 0u;
    }
    // replay in window order; the completion window once
    const double2 ln = k.pf->line[kk];
    const double Sn = __dadd_rn(st.Sr, ln.x);
    if (!st.done && k.J > 0.0 && Sn >= k.J) {
        st.rf = __ddiv_rn(__dsub_rn(k.J, st.Sr), ln.x);
        st.rE = st.Er;
        st.rC = st.Cr;
        st.rPk = ln.y;
        st.rcw = cw;
        st.rw = w;
        st.done = true;
    }
    st.Sr = Sn;
    st.Er = __dadd_rn(st.Er, ln.y);
    st.Cr = __fma_rn(ln.y, cw, st.Cr);
    if (w < k.mb) st.Cb = __dadd_rn(st.Cb, cw);
    st.Cs_all = __dadd_rn(st.Cs_all, cw);
    return kk;
}

template <int MODE>
__global__ void __launch_bounds__(kRLThreads, CHASE_RL_MINB) roll_lane_kernel(const __grid_constant__ SweepParams P) {
    mark_path(P.diag, CHASE_PATH_ROLL_FUSED);
    extern __shared__ __align__(128) uint8_t sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int T = P.T, L = P.L, n = L - 1, W = P.W, s0 = L;
    const RLLayout RL = make_rllayout(T, L, P.tables_bytes);
    uint8_t* wbase = sm + warp * RL.warp_bytes;
    float* ring = reinterpret_cast<float*>(wbase + RL.ring);
    uint32_t* chw = reinterpret_cast<uint32_t*>(wbase + RL.chb) + (kRLTile / 4 + 1) * lane;  // this lane's words
    uint64_t* mbar = reinterpret_cast<uint64_t*>(wbase + RL.mbar);
    const int stride = RL.stride;
    {
        const uint4* src = reinterpret_cast<const uint4*>(P.tables);
        uint4* dst = reinterpret_cast<uint4*>(sm + RL.tables);
        for (int q = tid; q < P.tables_bytes / 16; q += kRLThreads) dst[q] = src[q];
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
        mbar_init(mbar, 32);
        mbar_init(mbar + 1, 32);
        fence_mbar_init();
    }
    __syncthreads();

    const float* traces = reinterpret_cast<const float*>(P.traces);
    const int64_t n_groups = (P.n_traces + 31) / 32;
    const int64_t GW = (int64_t)gridDim.x * kRLWarps;
    // tiles: the first runs from the job start s0 to the next 128-B boundary past it plus
    // one tile, the rest start on 128-B boundaries (whole L2 lines: the per-lane loads
    // of 256 B then touch 2 lines, not 3)
    const int tbase = CHASE_RL_ALIGN ? (s0 & ~31) : s0;
    const int n_tiles = (P.N - tbase + kRLTile - 1) / kRLTile;
    auto tile_ab = [&](int t) { return t == 0 ? s0 : tbase + t * kRLTile; };
    auto tile_end = [&](int t) { return min(tbase + (t + 1) * kRLTile, P.N); };
    const bool store_choice = P.choice != nullptr;

    // producer: every lane loads its own trace's row of the tile (a unit = (group, tile))
    int64_t pg = (int64_t)blockIdx.x * kRLWarps + warp;
    int pt_ = 0;
    uint32_t produced = 0;
    auto issue = [&]() {
        if (pg >= n_groups) return;
        const int slot = produced & 1;
        const int64_t i = pg * 32 + lane;
        // a trace's first tile brings its L-value history; later tiles only their own
        // windows (their halo c[ab - L, ab) is copied from the previous tile's row)
        const int skip = pt_ == 0 || !CHASE_RL_HALO_COPY ? 0 : L;
        const int c0 = tile_ab(pt_) - L + skip;               // first column loaded
        const int c1 = tile_end(pt_);
        const uint32_t bytes = i < P.n_traces ? (uint32_t)(((c1 - c0) * 4 + 15) & ~15) : 0u;
        CHASE_CHECK(c1 - c0 + skip <= stride);
        uint64_t* bar = mbar + slot;
        mbar_arrive_expect_tx(bar, bytes);
        if (bytes)
            bulk_g2s(ring + (slot * 32 + lane) * stride + skip, traces + i * P.ld + c0, bytes, bar, evict_first_policy());
        ++produced;
        if (++pt_ == n_tiles) {
            pt_ = 0;
            pg += GW;
        }
    };
    issue();
    issue();

    unsigned n_slow = 0;
    uint32_t consumed = 0;
    for (int64_t g = (int64_t)blockIdx.x * kRLWarps + warp; g < n_groups; g += GW) {
        const int64_t i = g * 32 + lane;
        RLConst k;
        k.live = i < P.n_traces;
        const double* rec = P.records + (k.live ? i : 0) * kRecDoubles;
        int status = k.live ? (int)rec[5] : CHASE_ERR_DATA;
        if (status == 0 && !(rec[15] > 0.0)) status = CHASE_ERR_MAXCI;
        const int prof = k.live ? (int)rec[13] : 0;
        k.ptab = ptab;
        k.S = S;
        k.C = C;
        k.pf = profs + prof;
        k.pt = pairs + prof;
        k.grow = traces + (k.live ? i : 0) * P.ld;
        k.J = k.live ? rec[12] : 0.0;
        k.Kc = k.live ? rec[10] : 0.0;
        k.invK = k.live ? rec[11] : 1.0;  // (a dead lane takes the cheap lookup path)
        k.dn = (double)n;
        k.inv_n = 1.0 / k.dn;
        k.ridge = P.ridge;
        k.tol = P.tol;
        k.L = L;
        k.T = T;
        k.n = n;
        k.phase0 = P.phase0;
        k.R = P.refit;
        k.s0 = s0;
        const int mraw = k.live ? (int)rec[8] : 0;
        k.mb = (k.J > 0.0 && mraw >= 1 && mraw <= W) ? mraw - 1 : W;
        RLState st;
        st.m = RMom{0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        st.md = RModel{0.0, 0.0, 0.0, 0.0, false, 0};
        st.c_prev = st.o_prev = 0.0;
        st.Sr = st.Er = st.Cr = st.Cb = st.Cs_all = 0.0;
        st.rE = st.rC = st.rf = st.rPk = st.rcw = 0.0;
        st.ph = (int)(((int64_t)P.phase0 + s0) % T);  // phase of window 0 (= its origin's for R = 1)
        st.rw = -1;
        st.to_origin = 0;
        st.fit_bad = 0;
        st.n_slow = 0;
        st.vmin = FLT_MAX;
        st.done = false;
        for (int tl = 0; tl < n_tiles; ++tl, ++consumed) {
            const int slot = consumed & 1;
            mbar_wait(mbar + slot, (consumed >> 1) & 1u);
            k.row = ring + (slot * 32 + lane) * stride;  // row[q] = c[ab - L + q]
            k.ab = tile_ab(tl);                           // absolute index of the tile's window 0
            k.nw = tile_end(tl) - k.ab;
            const float* cv = k.row + L - k.ab;           // cv[a] = c[a] for a in [ab - L, ab + 64)
            CHASE_CHECK(L + k.nw <= stride);
            if (tl == 0) {
                // the job-start origin's moments from its rows (the history), the carried values
                const RVals V{k.row, k.grow, k.ab - L, k.ab + k.nw};
                st.m = mom_direct(V, k.ab, n, P.phase0, T, S, C);
                st.c_prev = (double)cv[k.ab - 1];
                st.o_prev = (double)cv[k.ab - n - 1];
            }
            const int nfull = k.nw & ~3;
            for (int j = 0; j < nfull; j += 4) {
                const float4 v4 = *reinterpret_cast<const float4*>(cv + k.ab + j);
                // c[a - n] for the group's windows a = ab + j + u: c[ab + j - L + 1 + u]
                // (ab + j - L is 16-byte aligned, L % 4 == 0)
                const float4 o4 = *reinterpret_cast<const float4*>(cv + k.ab + j - L);
                const float o5 = cv[k.ab + j - L + 4];
                st.vmin = fminf(fminf(fminf(st.vmin, v4.x), v4.y), fminf(v4.z, v4.w));
                const int a = k.ab + j;
                uint32_t word = rl_window<MODE>(st, k, a, (double)v4.x, (double)o4.y);
                word |= rl_window<MODE>(st, k, a + 1, (double)v4.y, (double)o4.z) << 8;
                word |= rl_window<MODE>(st, k, a + 2, (double)v4.z, (double)o4.w) << 16;
                word |= rl_window<MODE>(st, k, a + 3, (double)v4.w, (double)o5) << 24;
                chw[j >> 2] = word;
            }
            if (nfull < k.nw) {  // the trace's last windows (W % 4 != 0)
                uint32_t word = 0u;
                for (int j = nfull; j < k.nw; ++j) {
                    const float v = cv[k.ab + j];
                    st.vmin = fminf(st.vmin, v);
                    word |= rl_window<MODE>(st, k, k.ab + j, (double)v, (double)cv[k.ab + j - n]) << (8 * (j - nfull));
                }
                chw[nfull >> 2] = word;
            }
            __syncwarp();
            if (store_choice && k.live) {  // this lane's choice bytes of the tile
                uint8_t* dst = P.choice + i * P.ld_c + (k.ab - s0);  // (4-byte aligned: L % 4 == 0)
                for (int q = 0; q < (k.nw + 3) / 4; ++q) reinterpret_cast<uint32_t*>(dst)[q] = chw[q];
            }
            if (CHASE_RL_HALO_COPY && tl + 1 < n_tiles) {
                // the next tile's halo c[ab + 64 - L, ab + 64): this row's last L values, into
                // the head of the next slot's row (its TMA load writes only past the head)
                float* nrow = ring + (((consumed + 1) & 1) * 32 + lane) * stride;
                for (int q = 0; q < L; q += 4)
                    *reinterpret_cast<float4*>(nrow + q) = *reinterpret_cast<const float4*>(k.row + k.nw + q);
            }
            __syncwarp();
            issue();  // this slot is free again (every lane has read its row)
        }
        n_slow += st.n_slow;
        // ---- end of the trace group: per-lane results (S:29 validation, R2 inputs)
        if (k.live) {
            const bool bad = !(st.vmin >= 0.0f) || !(st.Cs_all <= DBL_MAX);
            if (status == 0 && bad) status = CHASE_ERR_DATA;
            if (status == 0 && st.fit_bad) status = CHASE_ERR_FIT;
            if ((status == CHASE_ERR_MAXCI || status == CHASE_ERR_FIT) && bad) status = CHASE_ERR_DATA;  // S:29 first
            if (status == 0) {
                P.records[i * kRecDoubles + 9] = st.Cb;
                double* o = P.raw + i * kRawDoubles;
                if (st.done) {
                    o[0] = st.rE;
                    o[1] = st.rC;
                    o[2] = k.J;
                    o[3] = st.rf;
                    o[4] = (double)((int64_t)L + st.rw);
                    o[5] = st.rPk;
                    o[6] = st.rcw;
                    o[7] = 1.0;
                } else {
                    o[0] = st.Er;
                    o[1] = st.Cr;
                    o[2] = st.Sr;
                    o[3] = 0.0;
                    o[4] = -1.0;
                    o[5] = o[6] = o[7] = 0.0;
                }
            }
            P.status[i] = (uint8_t)status;
            if (status != 0) {
                const unsigned long long slot = atomicAdd(reinterpret_cast<unsigned long long*>(&P.diag->n_bad), 1ull);
                P.bad_list[slot] = i;
                atomicMin(reinterpret_cast<unsigned long long*>(&P.diag->first_bad_trace), (unsigned long long)i);
            }
        }
    }
    n_slow = __reduce_add_sync(kFull, n_slow);
    if (lane == 0 && n_slow)
        atomicAdd(reinterpret_cast<unsigned long long*>(&P.diag->n_slow_windows), (unsigned long long)n_slow);
}
