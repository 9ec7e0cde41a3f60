// k2_fast.cuh — the headline planner kernel, specialised for the common case
// (fused plan + replay, fp32 traces with a 16-byte aligned job start, one
// eta, no forecast output).  Same arithmetic, same decomposition as
// sweep_kernel (warp-per-trace streaming, TMA bulk-copy ring per warp), with
// all window bookkeeping in 32-bit registers, the per-lane replay sums in
// registers, and the choice words stored straight from registers (no smem
// round trip).  Included by kernels.cu inside its anonymous namespace.
//
// Everything the hot loop does per window (DESIGN §6/§7):
//   p = A[phi] + w_lag*c[w-1]            (Eq. 1, canonical order)
//   k = bucket(p / Kc)                   (Eq. 6 envelope; rare windows -> canonical)
//   S += Thr_k*Delta; E += P_k; C += P_k*c[w]; Cs += c[w]

#ifndef CHASE_H_WARPS
#define CHASE_H_WARPS 6
#endif
#ifndef CHASE_H_STAGES
#define CHASE_H_STAGES 2
#endif
#ifndef CHASE_H_MINB
#define CHASE_H_MINB 2
#endif
constexpr int kHWarps = CHASE_H_WARPS;    // independent warps per CTA
constexpr int kHThreads = 32 * kHWarps;
constexpr int kHStages = CHASE_H_STAGES;  // per-warp TMA ring depth

struct FastLayout {
    int aext, stage, chb, ctx, mbar, bytes;
};

__host__ __device__ inline FastLayout make_fast_layout(int T, int stage_bytes) {
    FastLayout L;
    int o = 0;
    L.aext = o; o += 2 * round16(aext_len(T) * 8);
    L.stage = o; o += kHStages * stage_bytes;
    L.chb = o; o += kWarpW;
    L.ctx = o; o += (int)sizeof(WarpCtx);
    L.mbar = o; o += 8 * kHStages;
    L.bytes = round16(o);
    return L;
}

__host__ __device__ inline int fast_ent4_bytes(int n_prof) { return n_prof * kNB * (int)sizeof(int4); }
__host__ __device__ inline int fast_smem_total(int tables_bytes, int T, int stage_bytes, int n_prof) {
    return round16(tables_bytes) + fast_ent4_bytes(n_prof) + kHWarps * make_fast_layout(T, stage_bytes).bytes;
}

// Headline lookup: 16-byte entries {T1, T2, below, above} expanded in smem at
// kernel start from the blob's 8-byte entries (one LDS.128, 2 ISETP, 2 SEL).
struct Ent4 {
    int T1, T2;
    uint32_t below, above;
};
__device__ __forceinline__ uint32_t plan_lookup4(double y, const Ent4* __restrict__ ent, int base) {
    const int h = __double2hiint(y);
    const int idx = max(min((h >> kSH) - base, kNBUsed - 1), 0);
    const int4 e = *reinterpret_cast<const int4*>(ent + idx);
    return h < e.x ? (uint32_t)e.z : (h > e.y ? (uint32_t)e.w : (uint32_t)kZeroLine);
}

// One full-aligned chunk of ngroups x 4 windows; choice words go to smem
// (for the completion search) and, when `cdst` is set, straight to global.
template <bool FIRST_STORE>
__device__ __forceinline__ void fast_groups(const float* __restrict__ tv, int ngroups, const double* __restrict__ Ap,
                                            double wl, double invK, const Ent4* __restrict__ ent4, int ebase,
                                            const double2* __restrict__ lines, uint32_t* __restrict__ words,
                                            uint32_t* __restrict__ cdst, Acc& a) {
    double lag = (double)tv[-1];
#pragma unroll 1
    for (int g = 0; g < ngroups; ++g) {
        const float4 v = *reinterpret_cast<const float4*>(tv + 4 * g);
        a.vmin = fminf(fminf(fminf(a.vmin, v.x), v.y), fminf(v.z, v.w));  // FMNMX3 x2
        const double2 A01 = *reinterpret_cast<const double2*>(Ap + 4 * g);
        const double2 A23 = *reinterpret_cast<const double2*>(Ap + 4 * g + 2);
        const float vv[4] = {v.x, v.y, v.z, v.w};
        const double AA[4] = {A01.x, A01.y, A23.x, A23.y};
        uint32_t word = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double cw = (double)vv[u];
            const double p = __dadd_rn(AA[u], __dmul_rn(wl, lag));  // Eq. 1, unclamped for the lookup
            const uint32_t k = plan_lookup4(__dmul_rn(p, invK), ent4, ebase);
            word |= k << (8 * u);
            const double2 ln = lines[k];  // (Thr_k * Delta, P_k)
            a.S = __dadd_rn(a.S, ln.x);
            a.E = __dadd_rn(a.E, ln.y);
            a.C = __dadd_rn(a.C, __dmul_rn(ln.y, cw));
            a.Cs = __dadd_rn(a.Cs, cw);
            lag = cw;
        }
        words[g] = word;
        if (FIRST_STORE) cdst[g] = word;
        a.slow |= word;
    }
}

__global__ void __launch_bounds__(kHThreads, CHASE_H_MINB) sweep_fast_kernel(const __grid_constant__ SweepParams P) {
    extern __shared__ __align__(128) uint8_t sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const FastLayout FL = make_fast_layout(P.T, P.stage_bytes);
    Ent4* ent4_all = reinterpret_cast<Ent4*>(sm + round16(P.tables_bytes));
    uint8_t* wbase = sm + round16(P.tables_bytes) + fast_ent4_bytes(P.n_prof) + warp * FL.bytes;
    const int alen = round16(aext_len(P.T) * 8) / 8;
    double* A_even = reinterpret_cast<double*>(wbase + FL.aext);
    double* A_odd = A_even + alen;
    uint8_t* stage0 = wbase + FL.stage;
    uint8_t* chb = wbase + FL.chb;
    WarpCtx* ctx = reinterpret_cast<WarpCtx*>(wbase + FL.ctx);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(wbase + FL.mbar);

    {   // constant tables -> smem, once per CTA
        const uint4* src = reinterpret_cast<const uint4*>(P.tables);
        uint4* dst = reinterpret_cast<uint4*>(sm);
        for (int q = tid; q < P.tables_bytes / 16; q += kHThreads) dst[q] = src[q];
    }
    __syncthreads();
    {   // expand the 8-byte bucket entries of each profile's (single-eta) pair table
        const TablesHeader* H0 = reinterpret_cast<const TablesHeader*>(sm);
        const PairTable* pr = reinterpret_cast<const PairTable*>(sm + H0->off_pair);
        for (int q = tid; q < P.n_prof * kNB; q += kHThreads) {
            const uint2 e = pr[q / kNB].ent[q % kNB];
            Ent4 x;
            x.T1 = (int)e.x;
            x.T2 = (int)e.x + (int)(e.y >> 16);
            x.below = e.y & 0xffu;
            x.above = (e.y >> 8) & 0xffu;
            ent4_all[q] = x;
        }
    }
    if (lane == 0)
        for (int q0 = 0; q0 < kHStages; ++q0) mbar_init(&mbar[q0], 1);
    if (lane == 0) fence_mbar_init();
    __syncthreads();

    const TablesHeader* H = reinterpret_cast<const TablesHeader*>(sm);
    const double* phS = reinterpret_cast<const double*>(sm + H->off_phase);
    const double* phC = phS + P.T;
    const ProfileTable* profs = reinterpret_cast<const ProfileTable*>(sm + H->off_prof);
    const PairTable* pairs = reinterpret_cast<const PairTable*>(sm + H->off_pair);
    const float* traces = reinterpret_cast<const float*>(P.traces);
    const int64_t GW = (int64_t)gridDim.x * kHWarps;
    const int64_t gw = (int64_t)blockIdx.x * kHWarps + warp;
    const int nc = P.n_chunks, T = P.T;

    auto issue_next = [&]() {  // lane 0: next (trace, chunk) load; cursor in smem
        const int64_t pi = ctx->pi;
        if (pi >= P.n_traces) return;
        const int pc = ctx->pc;
        const uint32_t st = ctx->issued;  // stage index (wraps at kStages)
        const float* psrc = reinterpret_cast<const float*>(ctx->psrc);
        uint8_t* dst = stage0 + st * P.stage_bytes;
        const uint32_t bytes = pc == nc - 1 ? P.bytes_last : P.bytes_full;
        const uint64_t policy = evict_first_policy();
        if (pc == 0) {
            mbar_arrive_expect_tx(&mbar[st], bytes + (uint32_t)kRecBytes);
            bulk_g2s(dst + P.stage_bytes - kRecBytes, P.records + pi * kRecDoubles, kRecBytes, &mbar[st], policy);
        } else {
            mbar_arrive_expect_tx(&mbar[st], bytes);
        }
        bulk_g2s(dst, psrc, bytes, &mbar[st], policy);
        ctx->issued = st + 1 == kHStages ? 0 : st + 1;
        if (pc + 1 == nc) {
            ctx->pc = 0;
            ctx->pi = pi + GW;
            ctx->psrc = traces + (pi + GW) * P.ld + P.a0;
        } else {
            ctx->pc = pc + 1;
            ctx->psrc = psrc + kWarpW;
        }
    };
    if (lane == 0) {
        ctx->pi = gw;
        ctx->pc = 0;
        ctx->issued = 0;
        ctx->psrc = traces + gw * P.ld + P.a0;
        ctx->slow = 0ull;
        for (int q0 = 0; q0 < kHStages; ++q0) issue_next();
    }

    const int j0 = kChunk * lane;
    const int lane_phase = j0 % T;
    int st = 0;          // stage of the next chunk
    uint32_t par = 0;    // its mbarrier phase parity

    for (int64_t i = gw; i < P.n_traces; i += GW) {
        int status = 0, prof = 0;
        double wl = 0.0, J = 0.0, smax = 0.0, Kc = 0.0, invK = 0.0;
        int mb = P.W;
        double Sl = 0.0, El = 0.0, Cl = 0.0, Cbl = 0.0;
        bool done = false;
        int phase_c = P.phase_start;
        uint32_t* crow = P.choice ? reinterpret_cast<uint32_t*>(P.choice + i * P.ld_c) + (j0 >> 2) : nullptr;
        int c_may = 0;   // first chunk in which S can reach J (S <= windows * max_k s_k)
        for (int c = 0, jb = j0; c < nc; ++c, jb += kWarpW) {
            uint8_t* stage = stage0 + st * P.stage_bytes;
            mbar_wait(&mbar[st], par);
            if (c == 0) {  // ---- per-trace setup
                const double* rec = reinterpret_cast<const double*>(stage + P.stage_bytes - kRecBytes);
                prof = P.profile_id ? (int)P.profile_id[i] : 0;
                if (prof >= P.n_prof) prof = 0;
                smax = profs[prof].smax;
                J = P.job ? P.job[i] : 0.0;
                status = (int)rec[5];
                wl = rec[3];
                const double maxci = P.max_ci_fixed > 0.0 ? P.max_ci_fixed : rec[4];
                if (status == 0 && !(maxci > 0.0)) status = CHASE_ERR_MAXCI;
                const int64_t m = (int64_t)rec[8];
                mb = (J > 0.0 && m >= 1 && m <= P.W) ? (int)(m - 1) : P.W;
                const PairTable* pt0 = pairs + prof;
                Kc = __dmul_rn(pt0->kbase, maxci);
                invK = per_trace_invK(pt0, Kc);
                if (J > 0.0) {
                    const double wmin = __ddiv_rn(J, __dmul_rn(smax, 1.000001));  // windows needed, rounded down
                    c_may = wmin >= (double)P.W ? nc - 1 : max(0, (int)(wmin / kWarpW) - 1);
                } else {
                    c_may = nc;  // fixed duration: never completes
                }
                if (status == 0) {
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
                __syncwarp();
            } else {
                phase_c += P.phase_step;
                if (phase_c >= T) phase_c -= T;
            }
            const int nwin = max(0, min(kChunk, P.W - jb));
            const float* tv = reinterpret_cast<const float*>(stage) + P.off0 + j0;  // tv[jj] = c[s0 + jb + jj]
            int phi0 = phase_c + lane_phase;
            if (phi0 >= T) phi0 -= T;
            const double* Ap = (phi0 & 1) ? A_odd + (phi0 - 1) : A_even + phi0;
            const PairTable* pt = pairs + prof;
            const ProfileTable* pf = profs + prof;

            if (status == 0) {
                Acc a{0.0, 0.0, 0.0, 0.0, FLT_MAX, 0u, 0, 0};
                uint32_t* words = reinterpret_cast<uint32_t*>(chb + j0);
                int ngr = nwin >> 2;
                if (invK == 0.0) {
                    ngr = 0;  // Kc outside [2^-900, 2^900]: every window on the canonical rule
                    acc_merge(a, fused_generic<true, false, float, true>(tv, 0, nwin, Ap, wl, invK, pt, pf->line,
                                                                         chb + j0, nullptr, Kc, pf));
                    if (a.bad_pad) atomicAdd(&ctx->slow, (unsigned long long)a.bad_pad);
                } else {
                    const Ent4* e4 = ent4_all + prof * kNB;
                    if (crow) fast_groups<true>(tv, ngr, Ap, wl, invK, e4, pt->base, pf->line, words, crow, a);
                    else fast_groups<false>(tv, ngr, Ap, wl, invK, e4, pt->base, pf->line, words, nullptr, a);
                    if (4 * ngr < nwin)
                        acc_merge(a, fused_generic<true, false, float>(tv, 4 * ngr, nwin, Ap, wl, invK, pt,
                                                                       pf->line, chb + j0, nullptr));
                    if (a.slow & 0x20202020u) {
                        const SlowFix fx = fix_slow<float>(tv, nwin, Ap, wl, Kc, pt, pf, chb + j0);
                        a.S = __dadd_rn(a.S, fx.S);
                        a.E = __dadd_rn(a.E, fx.E);
                        a.C = __dadd_rn(a.C, fx.C);
                        atomicAdd(&ctx->slow, (unsigned long long)fx.n);
                    }
                }
                // choice words not written from registers (canonical / tail / fixed windows)
                if (crow && (4 * ngr < nwin || (a.slow & 0x20202020u) || invK == 0.0))
                    for (int g = (a.slow & 0x20202020u) || invK == 0.0 ? 0 : ngr; 4 * g < nwin; ++g)
                        crow[g] = words[g];
                // validation: negatives via vmin, NaN/inf via the sum of c
                const int flag = (ngr > 0 && (!(a.vmin >= 0.0f) || !(a.Cs <= DBL_MAX))) ? 1 : a.bad;
                if (__any_sync(kFull, flag)) status = CHASE_ERR_DATA;
                if (status == 0) {
                    // baseline: sum of c over the windows before w*_b
                    double Cbt = 0.0;
                    if (jb + nwin <= mb) Cbt = a.Cs;
                    else if (jb < mb)
                        for (int jj = 0; jj < mb - jb; ++jj) Cbt = __dadd_rn(Cbt, (double)tv[jj]);
                    Cbl = __dadd_rn(Cbl, Cbt);
                    bool completed = false;
                    if (!done && c >= c_may) {
                        const double S_prev = warp_sum(Sl);
                        if (__dadd_rn(S_prev, warp_sum(a.S)) >= J) {
                            const double incl = warp_incl_scan(a.S, lane);
                            const double ex = __shfl_up_sync(kFull, incl, 1);
                            const double before = __dadd_rn(S_prev, lane == 0 ? 0.0 : ex);
                            const bool full = __dadd_rn(before, a.S) < J;
                            const unsigned who = __ballot_sync(kFull, !full && before < J && nwin > 0);
                            if (who != 0) {
                                __syncwarp();
                                const double Eb = warp_sum(full ? __dadd_rn(El, a.E) : El);
                                const double Cb = warp_sum(full ? __dadd_rn(Cl, a.C) : Cl);
                                const int src = __ffs(who) - 1;
                                const int nw_src = max(0, min(kChunk, P.W - (jb - j0) - kChunk * src));
                                const Completion cp = find_completion<float>(
                                    tv + kChunk * (src - lane), chb + kChunk * src, nw_src,
                                    __shfl_sync(kFull, before, src), J, pf->line, lane);
                                if (lane == 0) {
                                    double* r = P.raw + i * kRawDoubles;
                                    r[0] = __dadd_rn(Eb, cp.Ep);
                                    r[1] = __dadd_rn(Cb, cp.Cp);
                                    r[2] = J;
                                    r[3] = cp.f;
                                    r[4] = (double)((int64_t)P.L + (jb - j0) + kChunk * src + cp.w);
                                    r[5] = cp.Pk;
                                    r[6] = cp.cw;
                                    r[7] = 1.0;
                                }
                                done = completed = true;
                            }
                            // else: no window reached J in the scan order (non-dyadic rounding): carry on
                        }
                    }
                    if (!done && !completed) {
                        Sl = __dadd_rn(Sl, a.S);
                        El = __dadd_rn(El, a.E);
                        Cl = __dadd_rn(Cl, a.C);
                    }
                }
            } else if (status == CHASE_ERR_MAXCI || status == CHASE_ERR_FIT) {
                // S:29 precedence: a bad value anywhere makes the trace status 4
                if (__any_sync(kFull, chunk_has_bad(tv, nwin))) status = CHASE_ERR_DATA;
            }
            if (crow) crow += kWarpW / 4;

            if (c == nc - 1) {  // ---- end of trace
                if (status == 0) {
                    const double Cb = warp_sum(Cbl);
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
            __syncwarp();  // every lane is done with stage `st` and the choice buffer
            if (lane == 0) issue_next();
            if (++st == kHStages) {
                st = 0;
                par ^= 1u;
            }
        }
    }
    if (lane == 0 && ctx->slow)
        atomicAdd(reinterpret_cast<unsigned long long*>(&P.diag->n_slow_windows), ctx->slow);
}
