// k2_lean.cuh — the headline planner kernel: one decision per
// window (P = 1), fp32 traces with an aligned job start, one eta, no forecast
// output.  Included by kernels.cu inside its anonymous namespace, after
// k2_headline.cuh (whose line-region layout and key helpers it shares).
//
// Decomposition.  A warp owns one trace at a time and streams it through a
// two-slot TMA ring (cp.async.bulk + mbarrier, lane 0 issues), 1024 windows
// per slot.  Inside a slot the windows go in blocks of 128: lane l takes the
// four consecutive windows 4l..4l+3 of a block (one conflict-free LDS.128 of
// the slot), so a block's 32 choice words are 128 contiguous bytes stored
// straight to HBM by the lanes (STG.32, coalesced) — no staging buffer, no
// per-chunk bulk store.  The lag of a lane's first window is the previous
// value in the slot (the slot carries the 4 values before its first window).
//
// Per window (hot loop):
//   c   = fp32 bits -> fp64 on the FMA pipe (f32bits_to_f64)
//   y   = fma(w_lag/Kc, c[w-1], A[phi]/Kc)           the one-fma Eq. 6 key
//   e   = ent8[clamp((hi32(y) >> 14) - base)]        bucket entry (LDS.64)
//   (s_k, P_k) = LDS.128 [PRMT(e, h vs T1)]          the line
//   S += s_k, E += P_k, C = fma(P_k, c, C), Cs += c  (group sums pairwise)
// The key's error bound needs |A| + |w_lag| c <= 85 y_min Kc: the trace's
// table bound Amax is checked once, every value of a slot is range-checked
// (bits in [FLT_MIN, c_lim]: one unsigned max per value), and a slot that
// fails is redone with the exact key (x = fl(A + fl(w_lag c)), y = fl(x/Kc
// rounded as x * fl(1/Kc))), which also validates.  Traces whose
// table fails the bound (or eta = 1: Kc = 0) run the exact key throughout;
// Kc outside [2^-900, 2^900] takes the canonical rule per window (Q27).
//
// Sums: per lane per slot (S, E, C, Cs), merged into per-lane running sums;
// from the first slot that can complete the job (a lower bound from J and
// max_k s_k) a warp sum of S tells whether the slot completes it, and then
// a cold walk of that slot finds the completion window w*, its fraction f
// and the partial sums, in window order (finalize_kernel applies R2).

#ifndef CHASE_L_WARPS
#define CHASE_L_WARPS 16
#endif
#ifndef CHASE_L_MINB
#define CHASE_L_MINB 1
#endif
constexpr int kLWarps = CHASE_L_WARPS;
constexpr int kLThreads = 32 * kLWarps;
constexpr int kLSlotW = 1024;                      // windows per ring slot (8 blocks of 128)
constexpr int kLSlotBytes = (kLSlotW + 4) * 4;     // + the 4 values before the slot's first window
static_assert(kLSlotBytes % 16 == 0, "slot bytes");

// B table length: phases [0, T + 4) (a lane's 4 windows never wrap)
__host__ __device__ inline int lean_btab_len(int T) { return (T + 4 + 1) & ~1; }

struct LLayout {
    int tables, heads, ent8, lines, warp_bytes, total;
    int n_before, after0;
    int ring, rec, btab, chs, mbar;  // offsets inside a warp block
    __host__ __device__ int warp_off(int w) const {
        return w < n_before ? w * warp_bytes : after0 + (w - n_before) * warp_bytes;
    }
};

__host__ __device__ inline LLayout make_llayout(int T, int head_bytes, int n_prof, int base) {
    LLayout L;
    L.ring = 0;
    L.rec = 2 * kLSlotBytes;
    L.btab = L.rec + 2 * kRecBytes;
    L.chs = L.btab + round16(lean_btab_len(T) * 8);
    L.mbar = L.chs + kLSlotW;
    L.warp_bytes = (L.mbar + 16 + 127) & ~127;
    L.lines = (int)kLineBase - base;
    HAlloc A{0, L.lines, L.lines + kLineRegion, L.lines + kLineRegion};
    L.n_before = L.lines > 0 ? L.lines / L.warp_bytes : 0;
    if (L.n_before > kLWarps) L.n_before = kLWarps;
    A.lo = L.n_before * L.warp_bytes;
    A.hi = (A.hi + 127) & ~127;
    L.after0 = A.hi;
    A.hi += (kLWarps - L.n_before) * L.warp_bytes;
    L.ent8 = A.take(n_prof * kNB * 8, 16);
    L.tables = A.take(round16(head_bytes), 16);
    L.heads = A.take(round16(n_prof * (int)sizeof(PairHead)), 16);
    L.total = A.hi;
    return L;
}

// Per-lane partial sums of a slot.
struct LAcc {
    double S, E, C, C2, Cs;
    uint32_t bmax;  // max over the slot's values of bits - bits(FLT_MIN) (unsigned; FAST only)
    uint32_t slow;  // OR of the choice words (bit 5 of a byte: a deferred window)
    float vmin;     // exact key: min value (validation)
    int bad;        // exact key: a bad value
};

// Four windows of a lane (values v, lag of the first, keys from Bq = the B
// (FAST) or A (exact) values at their phases).  Returns the choice word.
template <bool FAST>
__device__ __forceinline__ uint32_t lean_group(const float4 v, double lag, const double2 B01, const double2 B23,
                                               double wk, double invK, const uint2* __restrict__ ent8, int ebase,
                                               uint32_t ZB, double& C, LAcc& a) {
    const uint32_t vb[4] = {__float_as_uint(v.x), __float_as_uint(v.y), __float_as_uint(v.z), __float_as_uint(v.w)};
    const double BB[4] = {B01.x, B01.y, B23.x, B23.y};
    double cw4[4];
    if (FAST) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            a.bmax = max(a.bmax, vb[u] - 0x00800000u);
            cw4[u] = f32bits_to_f64(vb[u]);
        }
    } else {
        a.vmin = fminf(fminf(fminf(a.vmin, v.x), v.y), fminf(v.z, v.w));
        cw4[0] = (double)v.x;
        cw4[1] = (double)v.y;
        cw4[2] = (double)v.z;
        cw4[3] = (double)v.w;
    }
    uint32_t ad[4];
    double2 ln4[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        // FAST: y = fma(w_lag/Kc, lag, A/Kc); exact: y = fl(fl(A + fl(w_lag lag)) * fl(1/Kc)) (Q24)
        const double y = FAST ? __fma_rn(wk, lag, BB[u]) : __dmul_rn(__dadd_rn(BB[u], __dmul_rn(wk, lag)), invK);
        const int h = __double2hiint(y);
        const int idx = max(min((h >> kSH) - ebase, kNBUsed - 1), 0);
        ad[u] = line_addr(h, ent8[idx], ZB);
        ln4[u] = lds_line(ad[u]);  // (Thr_k * Delta, P_k)
        lag = cw4[u];
    }
    a.S = __dadd_rn(a.S, __dadd_rn(__dadd_rn(ln4[0].x, ln4[1].x), __dadd_rn(ln4[2].x, ln4[3].x)));
    a.E = __dadd_rn(a.E, __dadd_rn(__dadd_rn(ln4[0].y, ln4[1].y), __dadd_rn(ln4[2].y, ln4[3].y)));
    C = __fma_rn(ln4[3].y, cw4[3], __fma_rn(ln4[2].y, cw4[2], __fma_rn(ln4[1].y, cw4[1], __fma_rn(ln4[0].y, cw4[0], C))));
    a.Cs = __dadd_rn(a.Cs, __dadd_rn(__dadd_rn(cw4[0], cw4[1]), __dadd_rn(cw4[2], cw4[3])));
    const uint32_t word = __byte_perm(__byte_perm(ad[0], ad[1], 0x0051u), __byte_perm(ad[2], ad[3], 0x0051u), 0x5410u);
    a.slow |= word;
    return word;
}

// The trace-level constants a slot pass needs.
struct LTrace {
    const double* Bt;      // B (FAST) or A (exact) table, phases [0, T + 4)
    double wk, invK, Kc, wl;
    int ebase, T;
    uint32_t ZB;
    const uint2* e8;
    const PairTable* pt;
    const ProfileTable* pf;
    int prof;
};

// One slot, full blocks: nb blocks of 128 windows from slot values sv (sv[-1]:
// the lag of the first window), phases from ph0 (window 0 of the slot), choice
// words to crow (the slot's first choice byte, 16-byte aligned).
template <bool FAST>
__device__ __forceinline__ void lean_slot(const float* __restrict__ sv, int nb, int ph0, int d_ph, int off_l,
                                          const LTrace& t, uint8_t* __restrict__ crow, int lane, LAcc& a) {
    double C0 = 0.0, C1 = 0.0;
    int p = ph0 + off_l;
    if (p >= t.T) p -= t.T;
    int b = 0;
#pragma unroll 1
    for (; b + 1 < nb; b += 2) {
        const int j0 = 128 * b + 4 * lane;
        const float4 va = *reinterpret_cast<const float4*>(sv + j0);
        const float4 vb = *reinterpret_cast<const float4*>(sv + j0 + 128);
        const float la = sv[j0 - 1], lb = sv[j0 + 127];
        int pb = p + d_ph;
        if (pb >= t.T) pb -= t.T;
        const double2 A01 = *reinterpret_cast<const double2*>(t.Bt + p);
        const double2 A23 = *reinterpret_cast<const double2*>(t.Bt + p + 2);
        const double2 B01 = *reinterpret_cast<const double2*>(t.Bt + pb);
        const double2 B23 = *reinterpret_cast<const double2*>(t.Bt + pb + 2);
        if (FAST) {
            a.bmax = max(a.bmax, __float_as_uint(la) - 0x00800000u);
        }
        const double lad = FAST ? f32bits_to_f64(__float_as_uint(la)) : (double)la;
        const double lbd = FAST ? f32bits_to_f64(__float_as_uint(lb)) : (double)lb;
        const uint32_t wa = lean_group<FAST>(va, lad, A01, A23, t.wk, t.invK, t.e8, t.ebase, t.ZB, C0, a);
        const uint32_t wb = lean_group<FAST>(vb, lbd, B01, B23, t.wk, t.invK, t.e8, t.ebase, t.ZB, C1, a);
        *reinterpret_cast<uint32_t*>(crow + j0) = wa;
        *reinterpret_cast<uint32_t*>(crow + j0 + 128) = wb;
        p = pb + d_ph;
        if (p >= t.T) p -= t.T;
    }
    if (b < nb) {
        const int j0 = 128 * b + 4 * lane;
        const float4 va = *reinterpret_cast<const float4*>(sv + j0);
        const float la = sv[j0 - 1];
        const double2 A01 = *reinterpret_cast<const double2*>(t.Bt + p);
        const double2 A23 = *reinterpret_cast<const double2*>(t.Bt + p + 2);
        if (FAST) a.bmax = max(a.bmax, __float_as_uint(la) - 0x00800000u);
        const double lad = FAST ? f32bits_to_f64(__float_as_uint(la)) : (double)la;
        *reinterpret_cast<uint32_t*>(crow + j0) =
            lean_group<FAST>(va, lad, A01, A23, t.wk, t.invK, t.e8, t.ebase, t.ZB, C0, a);
    }
    a.C = __dadd_rn(a.C, __dadd_rn(C0, C1));
}

// The slot's last, partial block (the trace's last windows, nrem < 128): one
// window at a time with the exact key and the canonical rule where the key
// is in a band (cold).  Also the whole-slot path of the canonical-only traces
// (invK == 0).  Returns the lane's sums; writes its choice bytes.
__device__ __noinline__ LAcc lean_tail(const float* sv, int j_begin, int j_end, int ph0, const ExactModel& M,
                                       const LTrace& t, bool canon, uint8_t* crow, unsigned& n_slow) {
    LAcc a{0.0, 0.0, 0.0, 0.0, 0.0, 0u, 0u, FLT_MAX, 0};
    for (int j = j_begin; j < j_end; ++j) {
        const float raw = sv[j];
        const double cw = (double)raw;
        int phi = ph0 + j % t.T;
        if (phi >= t.T) phi -= t.T;
        const double p = __dadd_rn(M.A(phi), __dmul_rn(M.wl, (double)sv[j - 1]));
        uint32_t k = kZeroLine;
        if (!canon) {
            const int h = __double2hiint(__dmul_rn(p, M.invK));
            const int idx = max(min((h >> kSH) - t.ebase, kNBUsed - 1), 0);
            k = (line_addr(h, t.e8[idx], t.ZB) >> 8) & 0xffu;
        }
        if (k == (uint32_t)kZeroLine) {
            k = canonical_choose(p > 0.0 ? p : 0.0, M.Kc, t.pt->a, t.pf->thr, t.pf->K);
            ++n_slow;
        }
        crow[j] = (uint8_t)k;
        const double2 ln = t.pf->line[k];
        a.S = __dadd_rn(a.S, ln.x);
        a.E = __dadd_rn(a.E, ln.y);
        a.C = __dadd_rn(a.C, __dmul_rn(ln.y, cw));
        a.Cs = __dadd_rn(a.Cs, cw);
        a.vmin = fminf(a.vmin, raw);
        a.bad |= bad_value(raw) ? 1 : 0;
    }
    return a;
}

// The deferred (band) windows of a lane in one slot: the canonical rule on the
// exact forecast; fixes the choice bytes and returns the corrections (cold).
__device__ __noinline__ SlowFix lean_fix_slow(const float* sv, int nb, int ph0, int lane, const ExactModel& M,
                                              const LTrace& t, uint8_t* crow) {
    SlowFix r{0.0, 0.0, 0.0, 0};
    for (int b = 0; b < nb; ++b) {
        for (int u = 0; u < 4; ++u) {
            const int j = 128 * b + 4 * lane + u;
            if (crow[j] != (uint8_t)kZeroLine) continue;
            int phi = ph0 + j % t.T;
            if (phi >= t.T) phi -= t.T;
            const double x = predict(M.A(phi), M.wl, (double)sv[j - 1]);
            const uint32_t k = canonical_choose(x, M.Kc, t.pt->a, t.pf->thr, t.pf->K);
            crow[j] = (uint8_t)k;
            const double2 ln = t.pf->line[k];
            const double cw = (double)sv[j];
            r.S = __dadd_rn(r.S, ln.x);
            r.E = __dadd_rn(r.E, ln.y);
            r.C = __dadd_rn(r.C, __dmul_rn(ln.y, cw));
            ++r.n;
        }
    }
    return r;
}

// The completion walk of the slot that completes the job: windows in order
// (block, lane, 4 per lane), 32 at a time per round (lane = window), from the
// samples done before the slot.  Also the baseline's partial sum of c when
// its completion window mb falls in the slot.  Cold, once per trace.
struct LCompletion {
    double f, Ep, Cp, Pk, cw;
    int w;       // completion window within the slot, -1: none
};
__device__ __noinline__ LCompletion lean_completion(const float* sv, const uint8_t* crow, int nwin, double before,
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

// Sum of c over the slot's windows [0, m) (the baseline's completion chunk), in window order.
__device__ __noinline__ double lean_partial_cs(const float* sv, int m, int lane) {
    double s = 0.0;
    for (int j = lane; j < m; j += 32) s = __dadd_rn(s, (double)sv[j]);
    return warp_sum(s);
}

__global__ void __launch_bounds__(kLThreads, CHASE_L_MINB) lean_kernel(const __grid_constant__ SweepParams P) {
    mark_path(P.diag, CHASE_PATH_HEADLINE);
    extern __shared__ __align__(128) uint8_t sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t sbase = smem_u32(sm);
    const int head_bytes = reinterpret_cast<const TablesHeader*>(P.tables)->off_pair;
    const LLayout LL = make_llayout(P.T, head_bytes, P.n_prof, (int)sbase);
    if (LL.total > P.smem_total || LL.lines < 0) __trap();  // the host planned for another shared-window base
    uint2* ent8_all = reinterpret_cast<uint2*>(sm + LL.ent8);
    uint8_t* wbase = sm + LL.warp_off(warp);
    float* ring = reinterpret_cast<float*>(wbase + LL.ring);
    double* Bt = reinterpret_cast<double*>(wbase + LL.btab);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(wbase + LL.mbar);
    const int T = P.T;

    {   // constant tables -> smem, once per CTA (as sweep_fast_kernel)
        const uint4* src = reinterpret_cast<const uint4*>(P.tables);
        uint4* dst = reinterpret_cast<uint4*>(sm + LL.tables);
        for (int q = tid; q < head_bytes / 16; q += kLThreads) dst[q] = src[q];
        const int hw = (int)sizeof(PairHead) / 8;
        const double* ps = reinterpret_cast<const double*>(P.tables + head_bytes);
        double* hd = reinterpret_cast<double*>(sm + LL.heads);
        for (int q = tid; q < P.n_prof * hw; q += kLThreads)
            hd[q] = ps[(q / hw) * ((int)sizeof(PairTable) / 8) + q % hw];
    }
    __syncthreads();
    const TablesHeader* H = reinterpret_cast<const TablesHeader*>(sm + LL.tables);
    const double* phS = reinterpret_cast<const double*>(sm + LL.tables + H->off_phase);
    const double* phC = phS + T;
    const ProfileTable* profs = reinterpret_cast<const ProfileTable*>(sm + LL.tables + H->off_prof);
    const PairHead* heads = reinterpret_cast<const PairHead*>(sm + LL.heads);
    const PairTable* gpairs = reinterpret_cast<const PairTable*>(P.tables + head_bytes);
    {
        for (int q = tid; q < P.n_prof * (kMaxK + 1); q += kLThreads) {
            const int p = q / (kMaxK + 1), k = q % (kMaxK + 1);
            const double2 v = (k < profs[p].K) ? profs[p].line[k] : make_double2(0.0, 0.0);
            *reinterpret_cast<double2*>(sm + LL.lines + line_off(p, k)) = v;
        }
        for (int q = tid; q < P.n_prof * kNB; q += kLThreads) {
            const int p = q / kNB;
            const uint2 e = gpairs[p].ent[q % kNB];
            const uint32_t below = e.y & 0xffu;
            const uint32_t above = (e.y >> 16) ? (uint32_t)kZeroLine : ((e.y >> 8) & 0xffu);
            ent8_all[q] = make_uint2(e.x, (uint32_t)line_off(p, (int)below) | ((uint32_t)line_off(p, (int)above) << 16));
        }
    }
    if (lane == 0) {
        mbar_init(mbar, 1);
        mbar_init(mbar + 1, 1);
        fence_mbar_init();
    }
    __syncthreads();

    const float* traces = reinterpret_cast<const float*>(P.traces);
    const int64_t GW = (int64_t)gridDim.x * kLWarps;
    const int64_t gw = (int64_t)blockIdx.x * kLWarps + warp;
    const int W = P.W, L = P.L;
    const int n_slots = (W + kLSlotW - 1) / kLSlotW;
    const bool store_choice = P.choice != nullptr;
    const int off_l = (4 * lane) % T;          // phase offset of a lane's first window in a block
    const int d_ph = 128 % T;                  // phase advance per block
    const int d_slot = kLSlotW % T;            // per slot

    // producer (lane 0): unit = (trace, slot); two units in flight, the record with slot 0
    int64_t pi = gw;
    int ps = 0, pq = 0;  // next unit's trace, slot, and the trace's ordinal (record slot parity)
    auto issue = [&]() {
        if (pi >= P.n_traces) return;
        if (lane == 0) {
            const uint64_t policy = evict_first_policy();
            const int slot_id = (ps + pq * n_slots) & 1;  // units alternate slots
            const int nw = min(kLSlotW, W - ps * kLSlotW);
            const uint32_t bytes = (uint32_t)(((nw + 4) * 4 + 15) & ~15);
            uint64_t* bar = mbar + slot_id;
            if (ps == 0) {
                mbar_arrive_expect_tx(bar, bytes + (uint32_t)kRecBytes);
                bulk_g2s(wbase + LL.rec + (pq & 1) * kRecBytes, P.records + pi * kRecDoubles, kRecBytes, bar, policy);
            } else {
                mbar_arrive_expect_tx(bar, bytes);
            }
            bulk_g2s(ring + slot_id * (kLSlotBytes / 4), traces + pi * P.ld + L - 4 + (int64_t)ps * kLSlotW, bytes, bar,
                     policy);
        }
        if (++ps == n_slots) {
            ps = 0;
            pi += GW;
            ++pq;
        }
    };
    issue();
    issue();

    unsigned n_slow = 0;
    uint32_t unit = 0;  // units consumed (slot = unit & 1, mbarrier parity = (unit >> 1) & 1)
    int q = 0;          // trace ordinal of this warp
    for (int64_t i = gw; i < P.n_traces; i += GW, ++q) {
        int status = 0, s_may = n_slots, mb = W;
        double J = 0.0;
        double Sl = 0.0, El = 0.0, Cl = 0.0, Cbl = 0.0;  // per-lane running sums
        bool done = false;
        bool fast = false, canon = false;
        uint32_t blim = 0u;
        LTrace t;
        t.T = T;
        t.Bt = Bt;
        int ph_slot = (int)(((int64_t)P.phase0 + L) % T);  // phase of the slot's first window
        for (int s = 0; s < n_slots; ++s, ++unit) {
            const int slot_id = unit & 1;
            mbar_wait(mbar + slot_id, (unit >> 1) & 1u);
            const float* sv = ring + slot_id * (kLSlotBytes / 4) + 4;  // sv[j] = c[s0 + 1024 s + j], sv[-1] = lag
            const int nw = min(kLSlotW, W - s * kLSlotW);
            const double* rec = reinterpret_cast<const double*>(wbase + LL.rec + (q & 1) * kRecBytes);
            if (s == 0) {  // ---- per-trace setup from the record (fit_kernel, kernels.h)
                const int prof = (int)rec[13];
                t.prof = prof;
                t.pf = profs + prof;
                t.pt = reinterpret_cast<const PairTable*>(heads + prof);
                t.e8 = ent8_all + prof * kNB;
                t.ebase = t.pt->base;
                t.ZB = kLineBase | (uint32_t)line_off(prof, kZeroLine);
                J = rec[12];
                status = (int)rec[5];
                t.wl = rec[3];
                if (status == 0 && !(rec[15] > 0.0)) status = CHASE_ERR_MAXCI;
                const int m = (int)rec[8];
                mb = (J > 0.0 && m >= 1 && m <= W) ? m - 1 : W;
                t.Kc = rec[10];
                t.invK = rec[11];
                s_may = J > 0.0 ? (rec[14] >= (double)W ? n_slots - 1
                                                        : (int)(fmax(rec[14] - 1.0, 0.0) * (1.0 / kLSlotW)))
                                : n_slots;
                canon = t.invK == 0.0;
                if (status == 0) {
                    // the exact fold A(phi) = (c0 + w_sin S[phi]) + w_cos C[phi] (Q24) for phases [0, T + 4)
                    const double c0 = rec[0], wsn = rec[1], wcs = rec[2];
                    const int nb_t = lean_btab_len(T);
                    double amax = 0.0;
                    for (int j = lane; j < nb_t; j += 32) {
                        const int ph = j % T;
                        Bt[j] = __dadd_rn(__dadd_rn(c0, __dmul_rn(wsn, phS[ph])), __dmul_rn(wcs, phC[ph]));
                        amax = fmax(amax, fabs(Bt[j]));
                    }
                    amax = warp_max_d(amax);
                    // the one-fma key's bound (envelope.cpp's 512u shrink): |A| + |w_lag| c <= 85 y_min Kc
                    const double lam = __dmul_rn(__dmul_rn(85.0, t.pt->y_min), t.Kc);
                    if (!t.pt->k0 && !canon && amax < lam && fabs(t.wl) <= DBL_MAX) {
                        const double awl = fabs(t.wl);
                        const double cl = awl > 0.0 ? __ddiv_rd(__dsub_rd(lam, amax), awl) : (double)FLT_MAX;
                        const float clf = cl >= (double)FLT_MAX ? FLT_MAX : __double2float_rd(cl);
                        // the history's last value is the first window's lag
                        const float h_last = sv[-1];
                        if (clf >= FLT_MIN && h_last >= FLT_MIN && h_last <= clf) {
                            fast = true;
                            blim = __float_as_uint(clf) - 0x00800000u;
                            __syncwarp();
                            for (int j = lane; j < nb_t; j += 32) Bt[j] = __dmul_rn(Bt[j], t.invK);
                        }
                    }
                    t.wk = fast ? __dmul_rn(t.wl, t.invK) : t.wl;
                }
                __syncwarp();
            }

            // this slot's choice bytes: the caller's row (coalesced word stores), or, without a
            // choice output, a per-warp scratch in shared memory (the cold walks read them back)
            uint8_t* crow = store_choice ? P.choice + i * P.ld_c + (int64_t)s * kLSlotW : wbase + LL.chs;
            const int nbf = nw >> 7;  // full blocks
            bool issued = false;
            if (status == 0) {
                LAcc a{0.0, 0.0, 0.0, 0.0, 0.0, 0u, 0u, FLT_MAX, 0};
                const bool partial = (nw & 127) != 0;
                if (canon) {
                    const ExactModel M{rec[0], rec[1], rec[2], t.wl, t.Kc, t.invK, phS, phC};
                    for (int b = 0; b < (nw + 127) / 128; ++b) {
                        const int j0 = 128 * b + 4 * lane;
                        const LAcc r = lean_tail(sv, j0, min(j0 + 4, nw), ph_slot, M, t, true, crow, n_slow);
                        a.S = __dadd_rn(a.S, r.S); a.E = __dadd_rn(a.E, r.E); a.C = __dadd_rn(a.C, r.C);
                        a.Cs = __dadd_rn(a.Cs, r.Cs); a.vmin = fminf(a.vmin, r.vmin); a.bad |= r.bad;
                    }
                } else {
                    if (fast) lean_slot<true>(sv, nbf, ph_slot, d_ph, off_l, t, crow, lane, a);
                    else lean_slot<false>(sv, nbf, ph_slot, d_ph, off_l, t, crow, lane, a);
                    bool redo = fast && __any_sync(kFull, a.bmax > blim);
                    if (redo) {
                        // a value outside [FLT_MIN, c_lim]: the whole slot again with the exact key
                        const double c0 = rec[0], wsn = rec[1], wcs = rec[2];
                        __syncwarp();
                        for (int j = lane; j < lean_btab_len(T); j += 32) {
                            const int ph = j % T;
                            Bt[j] = __dadd_rn(__dadd_rn(c0, __dmul_rn(wsn, phS[ph])), __dmul_rn(wcs, phC[ph]));
                        }
                        __syncwarp();
                        LTrace te = t;
                        te.wk = t.wl;
                        a = LAcc{0.0, 0.0, 0.0, 0.0, 0.0, 0u, 0u, FLT_MAX, 0};
                        lean_slot<false>(sv, nbf, ph_slot, d_ph, off_l, te, crow, lane, a);
                        __syncwarp();
                        for (int j = lane; j < lean_btab_len(T); j += 32) Bt[j] = __dmul_rn(Bt[j], t.invK);
                        __syncwarp();
                    }
                    if (__any_sync(kFull, (a.slow & 0x20202020u) != 0u)) {  // deferred windows: canonical rule
                        __syncwarp();
                        if (a.slow & 0x20202020u) {
                            const ExactModel M{rec[0], rec[1], rec[2], t.wl, t.Kc, t.invK, phS, phC};
                            const SlowFix fx = lean_fix_slow(sv, nbf, ph_slot, lane, M, t, crow);
                            a.S = __dadd_rn(a.S, fx.S);
                            a.E = __dadd_rn(a.E, fx.E);
                            a.C = __dadd_rn(a.C, fx.C);
                            n_slow += (unsigned)fx.n;
                        }
                    }
                    if (partial) {  // the trace's last windows (cold)
                        __syncwarp();
                        const ExactModel M{rec[0], rec[1], rec[2], t.wl, t.Kc, t.invK, phS, phC};
                        const int j0 = 128 * nbf + 4 * lane;
                        const LAcc r = lean_tail(sv, j0, min(j0 + 4, nw), ph_slot, M, t, false, crow, n_slow);
                        a.S = __dadd_rn(a.S, r.S); a.E = __dadd_rn(a.E, r.E); a.C = __dadd_rn(a.C, r.C);
                        a.Cs = __dadd_rn(a.Cs, r.Cs); a.vmin = fminf(a.vmin, r.vmin); a.bad |= r.bad;
                    }
                }
                // validation: negatives via vmin (exact key), NaN/inf via the sum of c; the
                // one-fma key's range check already covers both
                const bool bad = __any_sync(kFull, !(a.vmin >= 0.0f) || !(a.Cs <= DBL_MAX) || a.bad);
                // baseline: sum of c over the windows before mb
                const int sw0 = s * kLSlotW;
                double Cbt = 0.0;
                if (sw0 + nw <= mb) Cbt = a.Cs;
                bool completes = false;
                if (!bad && !done && s >= s_may) completes = warp_sum(__dadd_rn(Sl, a.S)) >= J;
                if (!completes && !(sw0 < mb && mb < sw0 + nw)) {
                    __syncwarp();  // every lane is done with the slot (the choice bytes are in global memory)
                    issue();
                    issued = true;
                }
                if (bad) status = CHASE_ERR_DATA;
                if (status == 0) {
                    if (sw0 < mb && mb < sw0 + nw) {  // the baseline completes in this slot (cold)
                        __syncwarp();
                        const double part = lean_partial_cs(sv, mb - sw0, lane);
                        Cbt = lane == 0 ? part : 0.0;
                    }
                    Cbl = __dadd_rn(Cbl, Cbt);
                    if (completes) {  // the job completes in this slot: walk it in window order
                        __syncwarp();
                        const double S_prev = warp_sum(Sl);
                        const LCompletion cp = lean_completion(sv, crow, nw, S_prev, J, t.pf, lane);
                        if (cp.w >= 0) {
                            const double Eb = warp_sum(El), Cb = warp_sum(Cl);
                            if (lane == 0) {
                                double* r = P.raw + i * kRawDoubles;
                                r[0] = __dadd_rn(Eb, cp.Ep);
                                r[1] = __dadd_rn(Cb, cp.Cp);
                                r[2] = J;
                                r[3] = cp.f;
                                r[4] = (double)((int64_t)L + sw0 + cp.w);
                                r[5] = cp.Pk;
                                r[6] = cp.cw;
                                r[7] = 1.0;
                            }
                            done = true;
                        }
                        // else: no window reached J in window order (rounding): carry on
                    }
                    if (!done) {
                        Sl = __dadd_rn(Sl, a.S);
                        El = __dadd_rn(El, a.E);
                        Cl = __dadd_rn(Cl, a.C);
                    }
                }
            } else if (status == CHASE_ERR_MAXCI || status == CHASE_ERR_FIT) {
                // S:29 precedence: a bad value anywhere makes the trace status 4
                if (__any_sync(kFull, chunk_has_bad(sv + lane * 32, max(0, min(32, nw - lane * 32))))) status = CHASE_ERR_DATA;
            }
            if (s == n_slots - 1) {  // ---- end of trace
                if (status == 0) {
                    const double t4 = warp_sum4(Sl, El, Cl, Cbl, lane);  // totals in lanes 0, 8, 16, 24
                    const double Ex = __shfl_sync(kFull, t4, 8), Cx = __shfl_sync(kFull, t4, 16);
                    const double Cb = __shfl_sync(kFull, t4, 24);
                    if (lane == 0) {
                        P.records[i * kRecDoubles + 9] = Cb;
                        if (!done) {
                            double* r = P.raw + i * kRawDoubles;
                            r[0] = Ex;
                            r[1] = Cx;
                            r[2] = t4;
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
            if (!issued) {
                __syncwarp();
                issue();
            }
            ph_slot += d_slot;
            if (ph_slot >= T) ph_slot -= T;
        }
    }
    n_slow = __reduce_add_sync(kFull, n_slow);
    if (lane == 0 && n_slow)
        atomicAdd(reinterpret_cast<unsigned long long*>(&P.diag->n_slow_windows), (unsigned long long)n_slow);
}
