// kernels.cu — sm_100a kernels of the Chase batched trace-replay planner.
//
//   fit_kernel        §3.1 Eq. 1-2 fit on the L history points, lane = trace,
//                     canonical sequential order (bit-identical to the oracle),
//                     plus the per-trace baseline completion count.
//   sweep_kernel      persistent CTAs; per (trace, tile of 9216 windows): TMA
//                     bulk copy of the trace tile into a 2-stage smem ring,
//                     predict (Eq. 1) -> Eq. 6 argmin by the exact envelope
//                     bucket table (canonical K-way path deferred for the rare
//                     windows in a rounding band) -> replay partials -> warp /
//                     block reductions; choices staged in smem and bulk-stored.
//   finalize_kernel   per-trace totals (Eq. 3 stepwise carbon, pro-rata last
//                     window, max-power baseline) + fixed-order per-GPU sums.
//   plan_kernel       Eq. 6 argmin from given forecasts (split path).
//
// Arithmetic contract: every fp64 step that decides an output is written with
// explicit round-to-nearest intrinsics (and the file is built -fmad=false),
// in the same order as the oracle (DESIGN.md §3 Q9), so forecasts and choices
// are bit-identical and dyadic replay totals are exact.
#include <cfloat>
#include <cstring>

#include "kernels.h"

namespace chase {
namespace {

constexpr int kWarps = kThreads / 32;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kLeader = kThreads - 1;  // issues TMA copies / bulk stores, writes per-trace raw results
constexpr int kRecBytes = kRecDoubles * 8;

thread_local uint64_t g_launches = 0;

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// TMA bulk copy global -> shared, completion counted on `bar` (UBLKCP in SASS).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
        "%4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint32_t ldg_nc_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

__host__ __device__ inline int round16(int x) { return (x + 15) & ~15; }

// ------------------------------------------------------------------ Eq. 6
// Canonical rule: cost_k = ((a_k*x) + Kc)/Thr_k, each op rounded once, first
// minimum (lowest limit).  Taken by the windows in a rounding band.
__device__ __noinline__ uint32_t canonical_choose(double x, double Kc, const double* a, const double* thr,
                                                  int K) {
    uint32_t best = 0;
    double bc = __ddiv_rn(__dadd_rn(__dmul_rn(a[0], x), Kc), thr[0]);
    for (int k = 1; k < K; ++k) {
        double c = __ddiv_rn(__dadd_rn(__dmul_rn(a[k], x), Kc), thr[k]);
        if (c < bc) {
            bc = c;
            best = (uint32_t)k;
        }
    }
    return best;
}

// Envelope fast path: bucket of y = x * (1/Kc) by the high bits of
// its fp64 encoding, then at most one threshold pair.  Returns kZeroLine when
// y lies in a band where only the canonical rule is trusted.  Negative y (an
// unclamped forecast) lands in bucket 0 and decides exactly like x = 0.
__device__ __forceinline__ uint32_t plan_lookup(double y, const PairTable* pt) {
    const int hs = __double2hiint(y) >> kSH;
    const int idx = max(min(hs - pt->base, kNBUsed - 1), 0);
    const uint32_t e = pt->ent[idx];
    const double2 th = *reinterpret_cast<const double2*>(reinterpret_cast<const uint8_t*>(pt) + (e >> 16));
    const bool p1 = y <= th.x, p2 = y >= th.y;
    return p1 ? (e & 0xffu) : (p2 ? ((e >> 8) & 0xffu) : (uint32_t)kZeroLine);
}

__device__ __forceinline__ double per_trace_invK(const PairTable* pt, double Kc) {
    if (pt->k0) return 1.0;
    // Kc outside [2^-900, 2^900]: every window takes the canonical path (y = NaN).
    return (Kc >= 0x1p-900 && Kc <= 0x1p900) ? __ddiv_rn(1.0, Kc) : __longlong_as_double(0x7ff8000000000000ll);
}

template <typename E>
__device__ __forceinline__ bool bad_value(E v) {
    return !(v >= (E)0 && v <= (sizeof(E) == 4 ? (E)FLT_MAX : (E)DBL_MAX));
}

// Eq. 1 prediction with the clamp of S:152.
__device__ __forceinline__ double predict(double A, double wl, double lag) {
    const double p = __dadd_rn(A, __dmul_rn(wl, lag));
    return p > 0.0 ? p : 0.0;
}

// ------------------------------------------------------------------ warp collectives
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(kFull, v, o));
    return v;
}
__device__ __forceinline__ double warp_incl_scan(double v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        double n = __shfl_up_sync(kFull, v, o);
        if (lane >= o) v = __dadd_rn(n, v);
    }
    return v;
}
// Transposed butterfly: the warp totals of (v0, v1, v2, v3) end in lanes
// 0, 8, 16, 24 (12 fp64 shuffles instead of 20).  Fixed order -> deterministic.
__device__ __forceinline__ double warp_sum4(double v0, double v1, double v2, double v3, int lane) {
    const bool h4 = lane & 16;
    double r0 = __shfl_xor_sync(kFull, h4 ? v0 : v2, 16);
    double r1 = __shfl_xor_sync(kFull, h4 ? v1 : v3, 16);
    const double k0 = __dadd_rn(h4 ? v2 : v0, r0);
    const double k1 = __dadd_rn(h4 ? v3 : v1, r1);
    const bool h3 = lane & 8;
    double r = __shfl_xor_sync(kFull, h3 ? k0 : k1, 8);
    double s = __dadd_rn(h3 ? k1 : k0, r);
    s = __dadd_rn(s, __shfl_xor_sync(kFull, s, 4));
    s = __dadd_rn(s, __shfl_xor_sync(kFull, s, 2));
    s = __dadd_rn(s, __shfl_xor_sync(kFull, s, 1));
    return s;
}

struct SmemLayout {
    int tables, aext, stage, chb, part, part2, state, info, mbar, total;
};

__host__ __device__ inline int aext_len(int T) { return T + kChunk + 4; }

__host__ __device__ inline SmemLayout make_layout(int tables_bytes, int T, int stage_bytes) {
    SmemLayout L;
    int o = 0;
    L.tables = o; o += round16(tables_bytes);
    L.aext = o; o += 2 * round16(aext_len(T) * 8);
    L.stage = o; o += 2 * stage_bytes;
    L.chb = o; o += 2 * kTileW;
    L.part = o; o += 2 * kWarps * 4 * 8;
    L.part2 = o; o += kWarps * 2 * 8;
    L.state = o; o += kMaxEta * 4 * 8;
    L.info = o; o += 8 * 8;
    L.mbar = o; o += 16;
    L.total = round16(o);
    return L;
}

__device__ __forceinline__ const ProfileTable* blob_profiles(const uint8_t* blob) {
    const TablesHeader* H = reinterpret_cast<const TablesHeader*>(blob);
    return reinterpret_cast<const ProfileTable*>(blob + H->off_prof);
}

// ------------------------------------------------------------------ fit (K1)
// §3.1: the model is fitted once per trace on its L history points c[0..L)
// ("one day prior").  One lane per trace, the same
// sequential order and rounding as oracle_fit (bit-identical records).
template <typename E>
__device__ void fit_one(const E* h, int L, int T, int phi0, const double* S, const double* Cc, double ridge,
                        double tol_rel, double* rec) {
    const int n = L - 1;
    const double dn = (double)n;
    double maxci = (double)h[0];
    int bad = 0;
    for (int t = 0; t < L; ++t) {
        E v = h[t];
        bad |= bad_value(v);
        if ((double)v > maxci) maxci = (double)v;
    }
    double c0 = 0, w[3] = {0, 0, 0};
    int status = bad ? CHASE_ERR_DATA : 0, ridge_fired = 0, kind = 0;
    bool constant = true;
    for (int i = 2; i <= n; ++i)
        if ((double)h[i] != (double)h[1]) { constant = false; break; }
    if (status == 0 && constant) {
        kind = 1;
        c0 = (double)h[1];
    } else if (status == 0) {
        double sum[4] = {0, 0, 0, 0};
        for (int i = 1; i <= n; ++i) {
            int ph = (phi0 + i) % T;
            sum[0] = __dadd_rn(sum[0], S[ph]);
            sum[1] = __dadd_rn(sum[1], Cc[ph]);
            sum[2] = __dadd_rn(sum[2], (double)h[i - 1]);
            sum[3] = __dadd_rn(sum[3], (double)h[i]);
        }
        double mu[4], ss[4] = {0, 0, 0, 0}, sg[4];
        for (int j = 0; j < 4; ++j) mu[j] = __ddiv_rn(sum[j], dn);
        for (int i = 1; i <= n; ++i) {
            int ph = (phi0 + i) % T;
            double d0 = __dsub_rn(S[ph], mu[0]);
            double d1 = __dsub_rn(Cc[ph], mu[1]);
            double d2 = __dsub_rn((double)h[i - 1], mu[2]);
            double d3 = __dsub_rn((double)h[i], mu[3]);
            ss[0] = __dadd_rn(ss[0], __dmul_rn(d0, d0));
            ss[1] = __dadd_rn(ss[1], __dmul_rn(d1, d1));
            ss[2] = __dadd_rn(ss[2], __dmul_rn(d2, d2));
            ss[3] = __dadd_rn(ss[3], __dmul_rn(d3, d3));
        }
        for (int j = 0; j < 4; ++j) sg[j] = __dsqrt_rn(__ddiv_rn(ss[j], dn));
        if (!(sg[3] > 0.0)) {
            kind = 1;
            c0 = mu[3];
        } else {
            int cols[3], m = 0;
            for (int j = 0; j < 3; ++j)
                if (sg[j] > 0.0) cols[m++] = j;
            double G[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}}, hv[3] = {0, 0, 0};
            for (int i = 1; i <= n; ++i) {
                int ph = (phi0 + i) % T;
                double x[3] = {S[ph], Cc[ph], (double)h[i - 1]};
                double z[3];
                for (int a = 0; a < m; ++a) z[a] = __ddiv_rn(__dsub_rn(x[cols[a]], mu[cols[a]]), sg[cols[a]]);
                double u = __ddiv_rn(__dsub_rn((double)h[i], mu[3]), sg[3]);
                for (int a = 0; a < m; ++a) {
                    for (int b = 0; b <= a; ++b) G[a][b] = __dadd_rn(G[a][b], __dmul_rn(z[a], z[b]));
                    hv[a] = __dadd_rn(hv[a], __dmul_rn(z[a], u));
                }
            }
            for (int a = 0; a < m; ++a)
                for (int b = 0; b < a; ++b) G[b][a] = G[a][b];
            const double tol = __dmul_rn(tol_rel, dn);
            double Lc[3][3];
            bool ok = false;
            for (int attempt = 0; attempt < 2 && !ok; ++attempt) {
                if (attempt == 1) {
                    for (int a = 0; a < m; ++a) G[a][a] = __dadd_rn(G[a][a], ridge);
                    ridge_fired = 1;
                }
                for (int a = 0; a < 3; ++a)
                    for (int b = 0; b < 3; ++b) Lc[a][b] = 0.0;
                ok = true;
                for (int j = 0; j < m && ok; ++j) {
                    double d = G[j][j];
                    for (int k = 0; k < j; ++k) d = __dsub_rn(d, __dmul_rn(Lc[j][k], Lc[j][k]));
                    if (!(d > tol)) { ok = false; break; }
                    Lc[j][j] = __dsqrt_rn(d);
                    for (int i = j + 1; i < m; ++i) {
                        double v = G[i][j];
                        for (int k = 0; k < j; ++k) v = __dsub_rn(v, __dmul_rn(Lc[i][k], Lc[j][k]));
                        Lc[i][j] = __ddiv_rn(v, Lc[j][j]);
                    }
                }
                if (m == 0) ok = true;
            }
            if (!ok) {
                status = CHASE_ERR_FIT;
            } else {
                double zt[3] = {0, 0, 0}, beta[3] = {0, 0, 0};
                for (int a = 0; a < m; ++a) {
                    double v = hv[a];
                    for (int b = 0; b < a; ++b) v = __dsub_rn(v, __dmul_rn(Lc[a][b], zt[b]));
                    zt[a] = __ddiv_rn(v, Lc[a][a]);
                }
                for (int a = m - 1; a >= 0; --a) {
                    double v = zt[a];
                    for (int b = a + 1; b < m; ++b) v = __dsub_rn(v, __dmul_rn(Lc[b][a], beta[b]));
                    beta[a] = __ddiv_rn(v, Lc[a][a]);
                }
                for (int a = 0; a < m; ++a) w[cols[a]] = __ddiv_rn(__dmul_rn(sg[3], beta[a]), sg[cols[a]]);
                c0 = mu[3];
                for (int a = 0; a < m; ++a) c0 = __dsub_rn(c0, __dmul_rn(w[cols[a]], mu[cols[a]]));
            }
        }
    }
    rec[0] = c0;
    rec[1] = w[0];
    rec[2] = w[1];
    rec[3] = w[2];
    rec[4] = maxci;
    rec[5] = (double)status;
    rec[6] = (double)ridge_fired;
    rec[7] = (double)kind;
}

// Fit kernel: stage the CTA's 128 histories (L <= 64) into smem with coalesced
// loads (odd row stride), one lane per trace runs the canonical fit; also the
// max-power baseline's completion count m: the first m with
// m*s_b >= J, s_b = Thr_{K-1}*Delta (exact for the dyadic inputs; DESIGN R3).
template <typename E>
__global__ void __launch_bounds__(128) fit_kernel(const __grid_constant__ FitParams p) {
    extern __shared__ __align__(16) uint8_t fsm[];
    E* hs = reinterpret_cast<E*>(fsm);
    double* tab = reinterpret_cast<double*>(fsm + round16(128 * 65 * (int)sizeof(E)));
    const TablesHeader* H = reinterpret_cast<const TablesHeader*>(p.tables);
    const int L = p.L, T = p.T;
    const int64_t first = (int64_t)blockIdx.x * 128;
    const E* tr = reinterpret_cast<const E*>(p.traces);
    const bool staged = !p.baseline_only && L <= 64;
    if (!p.baseline_only) {
        const double* ph = reinterpret_cast<const double*>(p.tables + H->off_phase);
        for (int q = threadIdx.x; q < 2 * T; q += blockDim.x) tab[q] = ph[q];
    }
    if (staged) {
        const int stride = L | 1;
        for (int q = threadIdx.x; q < 128 * L; q += blockDim.x) {
            int r = q / L, t = q - r * L;
            int64_t i = first + r;
            if (i < p.n_traces) hs[r * stride + t] = tr[i * p.ld + t];
        }
    }
    __syncthreads();
    const int64_t i = first + threadIdx.x;
    if (i >= p.n_traces) return;
    double rec[kRecDoubles];
#pragma unroll
    for (int q = 0; q < kRecDoubles; ++q) rec[q] = 0.0;
    if (!p.baseline_only) {
        const E* h = staged ? hs + threadIdx.x * (L | 1) : tr + i * p.ld;
        fit_one<E>(h, L, T, p.phase0 % T, tab, tab + T, p.ridge, p.tol, rec);
    }
    const double J = p.job ? p.job[i] : 0.0;
    if (J > 0.0 && p.n_prof > 0) {
        int prof = p.profile_id ? (int)p.profile_id[i] : 0;
        if (prof >= p.n_prof) prof = 0;
        const ProfileTable* pf = blob_profiles(p.tables) + prof;
        const double sb = pf->line[pf->K - 1].x;
        const double qv = __ddiv_rn(J, sb);
        int64_t m = qv < 4.0e15 ? (int64_t)ceil(qv) : (int64_t)p.W + 2;
        if (m < 1) m = 1;
        while (m > 1 && __dmul_rn((double)(m - 1), sb) >= J) --m;
        while (m <= (int64_t)p.W && __dmul_rn((double)m, sb) < J) ++m;
        if (m > (int64_t)p.W) m = (int64_t)p.W + 1;
        rec[8] = (double)m;
    }
    double* out = p.records + i * kRecDoubles;
#pragma unroll
    for (int q = 0; q < kRecDoubles; ++q) out[q] = rec[q];
    if (p.models_out) {
#pragma unroll
        for (int q = 0; q < kModelDoubles; ++q) p.models_out[i * kModelDoubles + q] = rec[q];
    }
    if (p.max_ci_out) p.max_ci_out[i] = rec[4];
}

// ------------------------------------------------------------------ sweep (K2)
struct Acc {
    double S, E, C, Cs;  // sum s_k, sum P_k, sum P_k*c, sum c (every window: validation + baseline)
    float vmin;          // min raw value (fast path validation; NaN/inf show up in Cs)
    uint32_t slow;       // OR of staged choice words: bit 5 of a byte = kZeroLine (deferred window)
    int bad;             // generic path validation / REPLAY bad choice (2)
};

// Full, 16-byte-aligned fp32 chunk of kChunk windows: the hot loop.
// tv[jj] = c[w0 + jj] (tv[-1] = lag of the first window), Ap[jj] = A(phi0+jj).
template <bool FIRST, bool FC>
__device__ __forceinline__ void fused_full(const float* __restrict__ tv, const double* __restrict__ Ap, double wl,
                                           double invK, const PairTable* __restrict__ pt,
                                           const double2* __restrict__ lines, uint32_t* __restrict__ words,
                                           double* __restrict__ fout, Acc& a) {
    double lag = (double)tv[-1];
#pragma unroll 1
    for (int g = 0; g < kChunk / 4; ++g) {
        const float4 v = *reinterpret_cast<const float4*>(tv + 4 * g);
        const double2 A01 = *reinterpret_cast<const double2*>(Ap + 4 * g);
        const double2 A23 = *reinterpret_cast<const double2*>(Ap + 4 * g + 2);
        const float vv[4] = {v.x, v.y, v.z, v.w};
        const double AA[4] = {A01.x, A01.y, A23.x, A23.y};
        uint32_t word = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double cw = (double)vv[u];
            const double p = __dadd_rn(AA[u], __dmul_rn(wl, lag));  // Eq. 1, unclamped for the lookup
            if (FC) fout[4 * g + u] = p > 0.0 ? p : 0.0;
            const uint32_t k = plan_lookup(__dmul_rn(p, invK), pt);
            word |= k << (8 * u);
            const double2 ln = lines[k];                             // (Thr_k * Delta, P_k)
            a.S = __dadd_rn(a.S, ln.x);
            a.E = __dadd_rn(a.E, ln.y);
            a.C = __dadd_rn(a.C, __dmul_rn(ln.y, cw));
            if (FIRST) {
                a.Cs = __dadd_rn(a.Cs, cw);
                a.vmin = fminf(a.vmin, vv[u]);
            }
            lag = cw;
        }
        words[g] = word;
        a.slow |= word;
    }
}

// Any element type / alignment / partial chunk (tail threads, odd L, f64).
template <bool FIRST, bool FC, typename E>
__device__ void fused_generic(const E* tv, int nwin, int nwords, const double* Ap, double wl, double invK,
                              const PairTable* pt, const double2* lines, uint32_t* words, double* fout, Acc& a) {
    double lag = nwin > 0 ? (double)tv[-1] : 0.0;
    for (int g = 0; g < nwords; ++g) {
        uint32_t word = 0;
        for (int u = 0; u < 4; ++u) {
            const int jj = 4 * g + u;
            uint32_t k = 0xffu;
            if (jj < nwin) {
                const E raw = tv[jj];
                const double cw = (double)raw;
                const double p = __dadd_rn(Ap[jj], __dmul_rn(wl, lag));
                if (FC) fout[jj] = p > 0.0 ? p : 0.0;
                k = plan_lookup(__dmul_rn(p, invK), pt);
                if (k == (uint32_t)kZeroLine) a.slow |= 0x20u;
                const double2 ln = lines[k];
                a.S = __dadd_rn(a.S, ln.x);
                a.E = __dadd_rn(a.E, ln.y);
                a.C = __dadd_rn(a.C, __dmul_rn(ln.y, cw));
                if (FIRST) {
                    a.Cs = __dadd_rn(a.Cs, cw);
                    a.bad |= bad_value(raw) ? 1 : 0;
                }
                lag = cw;
            }
            word |= k << (8 * u);
        }
        words[g] = word;
    }
}

// The deferred windows (kZeroLine): canonical K-way Eq. 6, then their replay
// contributions (exact for dyadic inputs in any order).
template <typename E>
__device__ __noinline__ int fix_slow(const E* tv, int nwin, const double* Ap, double wl, double Kc, const PairTable* pt,
                                     const ProfileTable* pf, uint8_t* bytes, Acc& a) {
    int n = 0;
    for (int jj = 0; jj < nwin; ++jj) {
        if (bytes[jj] != (uint8_t)kZeroLine) continue;
        const double x = predict(Ap[jj], wl, (double)tv[jj - 1]);
        const uint32_t k = canonical_choose(x, Kc, pt->a, pf->thr, pf->K);
        bytes[jj] = (uint8_t)k;
        const double2 ln = pf->line[k];
        const double cw = (double)tv[jj];
        a.S = __dadd_rn(a.S, ln.x);
        a.E = __dadd_rn(a.E, ln.y);
        a.C = __dadd_rn(a.C, __dmul_rn(ln.y, cw));
        ++n;
    }
    return n;
}

template <typename E>
__device__ void predict_chunk(const E* tv, int nwin, const double* Ap, double wl, double* fout, Acc& a) {
    double lag = nwin > 0 ? (double)tv[-1] : 0.0;
    for (int jj = 0; jj < nwin; ++jj) {
        const E raw = tv[jj];
        fout[jj] = predict(Ap[jj], wl, lag);
        a.bad |= bad_value(raw) ? 1 : 0;
        lag = (double)raw;
    }
}

template <bool FIRST, typename E>
__device__ void replay_chunk(const E* tv, int nwin, int nwords, const uint32_t* cin, int K, const double2* lines,
                             uint32_t* words, Acc& a) {
    for (int g = 0; g < nwords; ++g) {
        const uint32_t w4 = 4 * g < nwin ? ldg_nc_u32(cin + g) : 0xffffffffu;
        for (int u = 0; u < 4; ++u) {
            const int jj = 4 * g + u;
            if (jj >= nwin) break;
            uint32_t k = (w4 >> (8 * u)) & 0xffu;
            if (k >= (uint32_t)K) {
                a.bad |= 2;
                k = 0;
            }
            const E raw = tv[jj];
            const double cw = (double)raw;
            const double2 ln = lines[k];
            a.S = __dadd_rn(a.S, ln.x);
            a.E = __dadd_rn(a.E, ln.y);
            a.C = __dadd_rn(a.C, __dmul_rn(ln.y, cw));
            if (FIRST) {
                a.Cs = __dadd_rn(a.Cs, cw);
                a.bad |= bad_value(raw) ? 1 : 0;
            }
        }
        words[g] = w4;
    }
}

template <typename E>
__device__ bool chunk_has_bad(const E* tv, int nwin) {
    bool b = false;
    for (int jj = 0; jj < nwin; ++jj) b |= bad_value(tv[jj]);
    return b;
}

template <int MODE, typename E, bool AL>
__global__ void __launch_bounds__(kThreads, 2) sweep_kernel(const __grid_constant__ SweepParams P) {
    extern __shared__ __align__(128) uint8_t sm[];
    constexpr int VEC = 16 / (int)sizeof(E);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const SmemLayout Ly = make_layout(P.tables_bytes, P.T, P.stage_bytes);
    const TablesHeader* H = reinterpret_cast<const TablesHeader*>(sm + Ly.tables);
    const int alen = round16(aext_len(P.T) * 8) / 8;
    double* A_even = reinterpret_cast<double*>(sm + Ly.aext);
    double* A_odd = A_even + alen;
    uint8_t* stage0 = sm + Ly.stage;
    uint8_t* chb0 = sm + Ly.chb;
    double* part = reinterpret_cast<double*>(sm + Ly.part);    // [2][kWarps][4]: S, E, C, Cb
    double* part2 = reinterpret_cast<double*>(sm + Ly.part2);  // [kWarps][2]
    double* state = reinterpret_cast<double*>(sm + Ly.state);  // [eta][4]: S_run, E_run, C_run, done
    double* info = reinterpret_cast<double*>(sm + Ly.info);    // completion window details
    uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + Ly.mbar);

    {   // constant tables -> smem (16-byte vectors)
        const uint4* src = reinterpret_cast<const uint4*>(P.tables);
        uint4* dst = reinterpret_cast<uint4*>(sm + Ly.tables);
        for (int q = tid; q < P.tables_bytes / 16; q += kThreads) dst[q] = src[q];
    }
    if (tid == kLeader) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();

    const double* phS = reinterpret_cast<const double*>(sm + Ly.tables + H->off_phase);
    const double* phC = phS + P.T;
    const ProfileTable* profs = reinterpret_cast<const ProfileTable*>(sm + Ly.tables + H->off_prof);
    const PairTable* pairs = reinterpret_cast<const PairTable*>(sm + Ly.tables + H->off_pair);

    const int64_t G = gridDim.x;
    const int64_t my_traces = P.n_traces > blockIdx.x ? (P.n_traces - blockIdx.x + G - 1) / G : 0;
    const int64_t n_items = my_traces * P.n_tiles;
    const int n_pass = MODE == MODE_PREDICT ? 1 : P.n_eta;
    const E* traces = reinterpret_cast<const E*>(P.traces);
    const uint64_t policy = evict_first_policy();

    // region [a, b) (elements) of trace row loaded for a tile
    auto tile_region = [&](int tile, int64_t& a, int64_t& b, int& Wt) {
        const int64_t ws = (int64_t)P.L + (int64_t)tile * kTileW;
        Wt = min(kTileW, P.W - tile * kTileW);
        a = AL ? ws - VEC : ((ws - 1) / VEC) * VEC;
        b = ((ws + Wt + VEC - 1) / VEC) * VEC;
        if (b > P.ld) b = P.ld;
    };
    auto issue = [&](int64_t item) {  // leader only
        if (item >= n_items) return;
        const int st = (int)(item & 1);
        const int64_t i = blockIdx.x + (item / P.n_tiles) * G;
        const int tile = (int)(item % P.n_tiles);
        int64_t a, b;
        int Wt;
        tile_region(tile, a, b, Wt);
        const uint32_t bytes = (uint32_t)((b - a) * (int64_t)sizeof(E));
        const bool rec = tile == 0;
        uint8_t* dst = stage0 + st * P.stage_bytes;
        mbar_arrive_expect_tx(&mbar[st], bytes + (rec ? (uint32_t)kRecBytes : 0u));
        bulk_g2s(dst, traces + i * P.ld + a, bytes, &mbar[st], policy);
        if (rec) bulk_g2s(dst + P.stage_bytes - kRecBytes, P.records + i * kRecDoubles, kRecBytes, &mbar[st], policy);
    };
    if (tid == kLeader) {
        issue(0);
        issue(1);
    }

    // per-trace uniform state (registers, all threads)
    int status = 0, prof = 0;
    double wl = 0.0, maxci = 0.0, J = 0.0;
    int64_t mb = 0;
    double Cb_run = 0.0;  // leader: baseline sum of c before w*_b
    int64_t slow_count = 0;
    int64_t gp = 0;       // pass counter (choice staging / partials parity)

    for (int64_t q = 0; q < n_items; ++q) {
        const int st = (int)(q & 1);
        const int64_t i = blockIdx.x + (q / P.n_tiles) * G;
        const int tile = (int)(q % P.n_tiles);
        int64_t a_abs, b_abs;
        int Wt;
        tile_region(tile, a_abs, b_abs, Wt);
        const int64_t ws_abs = (int64_t)P.L + (int64_t)tile * kTileW;
        uint8_t* stage = stage0 + st * P.stage_bytes;
        const E* tile_v = reinterpret_cast<const E*>(stage) + (ws_abs - a_abs);  // tile_v[j] = c[ws_abs + j]
        mbar_wait(&mbar[st], (uint32_t)((q >> 1) & 1));

        if (tile == 0) {
            const double* rec = reinterpret_cast<const double*>(stage + P.stage_bytes - kRecBytes);
            prof = P.profile_id ? (int)P.profile_id[i] : 0;
            if (prof >= P.n_prof) prof = 0;
            J = P.job ? P.job[i] : 0.0;
            status = (int)rec[5];
            wl = rec[3];
            maxci = P.max_ci_fixed > 0.0 ? P.max_ci_fixed : rec[4];
            if (status == 0 && MODE == MODE_FUSED && !(maxci > 0.0)) status = CHASE_ERR_MAXCI;
            const int64_t m = (int64_t)rec[8];
            mb = (J > 0.0 && m >= 1 && m <= P.W) ? m - 1 : P.W;
            if (status == 0 && MODE != MODE_REPLAY) {
                const double c0 = rec[0], wsn = rec[1], wcs = rec[2];
                const int n_a = aext_len(P.T);
                for (int qq = tid; qq < 2 * n_a; qq += kThreads) {
                    const int odd = qq >= n_a, j = qq - odd * n_a;
                    const int ph = (j + odd) % P.T;
                    // A(phi) = (c0 + w_sin*S[phi]) + w_cos*C[phi]  (canonical fold, Eq. 1)
                    (odd ? A_odd : A_even)[j] =
                        __dadd_rn(__dadd_rn(c0, __dmul_rn(wsn, phS[ph])), __dmul_rn(wcs, phC[ph]));
                }
            }
            if (tid == kLeader) {
                Cb_run = 0.0;
                for (int e = 0; e < n_pass; ++e) state[e * 4 + 0] = state[e * 4 + 1] = state[e * 4 + 2] = state[e * 4 + 3] = 0.0;
            }
        }
        __syncthreads();  // BA: A tables / state / landed stage visible

        const int j0 = kChunk * tid;
        const int nwin = max(0, min(kChunk, Wt - j0));
        const int nwords = j0 < ((Wt + 15) & ~15) ? kChunk / 4 : 0;
        const E* tv = tile_v + j0;
        const int phi0 = (int)(((int64_t)P.phase0 + ws_abs + j0) % P.T);
        const double* Ap = (phi0 & 1) ? A_odd + (phi0 - 1) : A_even + phi0;
        const int64_t jb = (int64_t)tile * kTileW + j0;  // my first window, counted from s0

        if (status == CHASE_ERR_MAXCI || status == CHASE_ERR_FIT) {
            // S:29 precedence: a bad value anywhere makes the trace status 4
            if (__syncthreads_or(chunk_has_bad(tv, nwin) ? 1 : 0)) status = CHASE_ERR_DATA;
        }

        for (int e = 0; e < n_pass && status == 0; ++e, ++gp) {
            const int sb = (int)(gp & 1);
            uint8_t* chb = chb0 + sb * kTileW;
            uint32_t* words = reinterpret_cast<uint32_t*>(chb) + (j0 >> 2);
            const double S_run = state[e * 4 + 0];
            const bool done = state[e * 4 + 3] != 0.0;
            const PairTable* pt = pairs + prof * P.n_eta + e;
            const ProfileTable* pf = profs + prof;
            const double Kc = __dmul_rn(pt->kbase, maxci);
            const double invK = per_trace_invK(pt, Kc);
            double* fout = (P.forecast && e == 0) ? P.forecast + i * P.ld_f + jb : nullptr;

            Acc a{0.0, 0.0, 0.0, 0.0, FLT_MAX, 0u, 0};
            bool fast = false;
            if (MODE == MODE_FUSED) {
                if (AL && sizeof(E) == 4 && nwin == kChunk) {
                    fast = true;
                    const float* tf = reinterpret_cast<const float*>(tv);
                    if (e == 0) {
                        if (fout) fused_full<true, true>(tf, Ap, wl, invK, pt, pf->line, words, fout, a);
                        else fused_full<true, false>(tf, Ap, wl, invK, pt, pf->line, words, fout, a);
                    } else {
                        fused_full<false, false>(tf, Ap, wl, invK, pt, pf->line, words, fout, a);
                    }
                } else if (nwords > 0) {
                    if (e == 0) {
                        if (fout) fused_generic<true, true, E>(tv, nwin, nwords, Ap, wl, invK, pt, pf->line, words, fout, a);
                        else fused_generic<true, false, E>(tv, nwin, nwords, Ap, wl, invK, pt, pf->line, words, fout, a);
                    } else {
                        fused_generic<false, false, E>(tv, nwin, nwords, Ap, wl, invK, pt, pf->line, words, fout, a);
                    }
                }
                if (a.slow & 0x20202020u) slow_count += fix_slow<E>(tv, nwin, Ap, wl, Kc, pt, pf, chb + j0, a);
            } else if (MODE == MODE_PREDICT) {
                predict_chunk<E>(tv, nwin, Ap, wl, P.forecast + i * P.ld_f + jb, a);
            } else {
                const uint32_t* cin = reinterpret_cast<const uint32_t*>(
                    P.choice_in + ((int64_t)e * P.n_traces + i) * P.ld_c + jb);
                if (e == 0) replay_chunk<true, E>(tv, nwin, nwords, cin, pf->K, pf->line, words, a);
                else replay_chunk<false, E>(tv, nwin, nwords, cin, pf->K, pf->line, words, a);
            }

            int flag = 0;
            double Cbt = 0.0;
            if (e == 0) {
                if (fast) flag |= (!(a.vmin >= 0.0f) || !(a.Cs <= DBL_MAX)) ? 1 : 0;
                flag |= a.bad;
                // baseline: sum of c over the windows before w*_b
                if (jb + nwin <= mb) Cbt = a.Cs;
                else if (jb < mb)
                    for (int jj = 0; jj < (int)(mb - jb); ++jj) Cbt = __dadd_rn(Cbt, (double)tv[jj]);
            } else {
                flag |= a.bad & 2;
            }
            const double tot = warp_sum4(a.S, a.E, a.C, Cbt, lane);
            double* pp = part + sb * kWarps * 4;
            if ((lane & 7) == 0) pp[warp * 4 + (lane >> 3)] = tot;
            if (MODE != MODE_PREDICT) fence_proxy_async();
            if (tid == kLeader) {
                bulk_wait_read0();  // the choice store of the previous pass left smem
                info[7] = 0.0;      // set by the thread that finds the completion window
            }
            const int bad_any = __syncthreads_or(flag);  // B1
            if (bad_any) {
                status = (bad_any & 1) ? CHASE_ERR_DATA : CHASE_ERR_CHOICE;
                break;
            }
            double S_tile = 0.0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) S_tile = __dadd_rn(S_tile, pp[w * 4 + 0]);
            if (tid == kLeader) {
                if (MODE == MODE_FUSED && P.choice) {
                    uint8_t* dst = P.choice + ((int64_t)e * P.n_traces + i) * P.ld_c + (int64_t)tile * kTileW;
                    bulk_s2g(dst, chb, (uint32_t)((Wt + 15) & ~15));
                    bulk_commit();
                }
                if (e == 0) {
                    double cb = 0.0;
                    for (int w = 0; w < kWarps; ++w) cb = __dadd_rn(cb, pp[w * 4 + 3]);
                    Cb_run = __dadd_rn(Cb_run, cb);
                }
            }
            if (MODE == MODE_PREDICT) continue;
            const bool completes = !done && J > 0.0 && __dadd_rn(S_run, S_tile) >= J;
            if (!completes) {
                if (tid == kLeader && !done) {
                    double et = 0.0, ct = 0.0;
                    for (int w = 0; w < kWarps; ++w) {
                        et = __dadd_rn(et, pp[w * 4 + 1]);
                        ct = __dadd_rn(ct, pp[w * 4 + 2]);
                    }
                    state[e * 4 + 0] = __dadd_rn(S_run, S_tile);
                    state[e * 4 + 1] = __dadd_rn(state[e * 4 + 1], et);
                    state[e * 4 + 2] = __dadd_rn(state[e * 4 + 2], ct);
                }
                continue;
            }
            // ---- the job completes inside this tile (once per trace and eta)
            const double incl = warp_incl_scan(a.S, lane);
            const double ex = __shfl_up_sync(kFull, incl, 1);
            double wpre = 0.0;
            for (int w = 0; w < warp; ++w) wpre = __dadd_rn(wpre, pp[w * 4 + 0]);
            const double before = __dadd_rn(__dadd_rn(S_run, wpre), lane == 0 ? 0.0 : ex);
            const double after = __dadd_rn(before, a.S);
            const bool full = after < J;
            const bool mine = !full && before < J && nwin > 0;
            const double Em = warp_sum(full ? a.E : 0.0), Cm = warp_sum(full ? a.C : 0.0);
            if (lane == 0) {
                part2[warp * 2 + 0] = Em;
                part2[warp * 2 + 1] = Cm;
            }
            if (mine) {
                double S = before, Ep = 0.0, Cp = 0.0, f = 1.0, cst = 0.0;
                int jj = 0;
                uint32_t k = 0;
                for (; jj < nwin; ++jj) {
                    k = chb[j0 + jj];
                    const double2 ln = pf->line[k];
                    const double cw = (double)tv[jj];
                    const double prev = S;
                    S = __dadd_rn(S, ln.x);
                    if (S >= J || jj == nwin - 1) {
                        f = __ddiv_rn(__dsub_rn(J, prev), ln.x);  // pro-rata last window
                        cst = cw;
                        break;
                    }
                    Ep = __dadd_rn(Ep, ln.y);
                    Cp = __dadd_rn(Cp, __dmul_rn(ln.y, cw));
                }
                info[0] = (double)(ws_abs + j0 + jj);
                info[1] = f;
                info[2] = Ep;
                info[3] = Cp;
                info[4] = pf->line[k].y;
                info[5] = cst;
                info[7] = 1.0;
            }
            __syncthreads();  // B2
            if (tid == kLeader && info[7] == 0.0) {
                // no window reached J in the scan order (non-dyadic rounding): carry on
                double et = 0.0, ct = 0.0;
                for (int w = 0; w < kWarps; ++w) {
                    et = __dadd_rn(et, pp[w * 4 + 1]);
                    ct = __dadd_rn(ct, pp[w * 4 + 2]);
                }
                state[e * 4 + 0] = __dadd_rn(S_run, S_tile);
                state[e * 4 + 1] = __dadd_rn(state[e * 4 + 1], et);
                state[e * 4 + 2] = __dadd_rn(state[e * 4 + 2], ct);
            } else if (tid == kLeader) {
                double em = 0.0, cm = 0.0;
                for (int w = 0; w < kWarps; ++w) {
                    em = __dadd_rn(em, part2[w * 2 + 0]);
                    cm = __dadd_rn(cm, part2[w * 2 + 1]);
                }
                double* r = P.raw + ((int64_t)e * P.n_traces + i) * kRawDoubles;
                r[0] = __dadd_rn(__dadd_rn(state[e * 4 + 1], em), info[2]);
                r[1] = __dadd_rn(__dadd_rn(state[e * 4 + 2], cm), info[3]);
                r[2] = J;
                r[3] = info[1];
                r[4] = info[0];
                r[5] = info[4];
                r[6] = info[5];
                r[7] = 1.0;
                state[e * 4 + 3] = 1.0;
            }
            __syncthreads();  // B3: info / part2 reusable, stage reads done
        }

        if (tile == P.n_tiles - 1 && tid == kLeader) {
            if (MODE != MODE_PREDICT && status == 0) {
                for (int e = 0; e < n_pass; ++e) {
                    if (state[e * 4 + 3] != 0.0) continue;
                    double* r = P.raw + ((int64_t)e * P.n_traces + i) * kRawDoubles;
                    r[0] = state[e * 4 + 1];
                    r[1] = state[e * 4 + 2];
                    r[2] = state[e * 4 + 0];
                    r[3] = 0.0;
                    r[4] = -1.0;
                    r[5] = r[6] = r[7] = 0.0;
                }
                P.records[i * kRecDoubles + 9] = Cb_run;
            }
            P.status[i] = (uint8_t)status;
            if (status != 0) {
                atomicAdd(reinterpret_cast<unsigned long long*>(&P.diag->n_bad), 1ull);
                atomicMin(reinterpret_cast<unsigned long long*>(&P.diag->first_bad_trace), (unsigned long long)i);
            }
        }
        if (tid == kLeader) issue(q + 2);  // stage `st` is free: every thread passed the last barrier
    }

    if (tid == kLeader) bulk_wait0();
    unsigned long long sc = (unsigned long long)slow_count;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sc += __shfl_xor_sync(kFull, sc, o);
    if (lane == 0 && sc) atomicAdd(reinterpret_cast<unsigned long long*>(&P.diag->n_slow_windows), sc);
}

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
        }
        __syncthreads();
    }
    if (valid) p.status[i] = (uint8_t)worst;
}

__global__ void finalize_sums_kernel(const double* block_sums, int64_t grid, int n_eta, chase_sum_t* sum) {
    const int e = blockIdx.x, r = threadIdx.x;
    if (e >= n_eta || r >= 8) return;
    double acc = 0.0;
    for (int64_t b = 0; b < grid; ++b) acc = __dadd_rn(acc, block_sums[(b * n_eta + e) * 8 + r]);
    reinterpret_cast<double*>(sum + e)[r] = acc;
}

// Invalid traces (status 4..7): choices 0xFF, forecasts NaN; count exhausted.
__global__ void fixup_kernel(const uint8_t* status, int64_t n, uint8_t* choice, int64_t ld_c, int64_t W, int n_eta,
                             double* forecast, int64_t ld_f, chase_diag_t* diag) {
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
        const int s = status[i];
        if (s == CHASE_ERR_TRACE_EXHAUSTED && threadIdx.x == 0)
            atomicAdd(reinterpret_cast<unsigned long long*>(&diag->n_exhausted), 1ull);
        if (s < CHASE_ERR_DATA) continue;
        if (threadIdx.x == 0)
            atomicMin(reinterpret_cast<unsigned long long*>(&diag->first_bad_trace), (unsigned long long)i);
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
        d->n_bad = d->n_exhausted = d->n_slow_windows = 0;
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
__global__ void upload_kernel(const __grid_constant__ UploadChunk c, int n, uint8_t* dst) {
    for (int q = threadIdx.x; q < n; q += blockDim.x) dst[q] = c.bytes[q];
}

int num_sms() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms > 0 ? sms : 148;
}

template <int MODE, typename E, bool AL>
cudaError_t launch_sweep_t(const SweepParams& p, cudaStream_t s) {
    const SmemLayout Ly = make_layout(p.tables_bytes, p.T, p.stage_bytes);
    auto kern = sweep_kernel<MODE, E, AL>;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Ly.total);
    if (err != cudaSuccess) return err;
    int per_sm = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, Ly.total);
    if (err != cudaSuccess) return err;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    int64_t grid = (int64_t)num_sms() * per_sm;
    if (grid > p.n_traces) grid = p.n_traces;
    kern<<<(unsigned)grid, kThreads, Ly.total, s>>>(p);
    ++g_launches;
    return cudaGetLastError();
}

}  // namespace

// ------------------------------------------------------------------ host launchers
uint64_t kernel_launches() { return g_launches; }

int sweep_stage_bytes(int elem_size) { return round16((kTileW + 8) * elem_size) + kRecBytes; }

size_t sweep_smem_bytes(int tables_bytes, int T, int elem_size, int mode) {
    (void)mode;
    return (size_t)make_layout(tables_bytes, T, sweep_stage_bytes(elem_size)).total;
}

int64_t finalize_grid(int64_t n_traces) { return (n_traces + kFinThreads - 1) / kFinThreads; }

cudaError_t launch_upload(const void* host, size_t bytes, void* dst, cudaStream_t s) {
    const uint8_t* h = static_cast<const uint8_t*>(host);
    for (size_t off = 0; off < bytes; off += sizeof(UploadChunk)) {
        UploadChunk c;
        const size_t n = bytes - off < sizeof(UploadChunk) ? bytes - off : sizeof(UploadChunk);
        memcpy(c.bytes, h + off, n);
        upload_kernel<<<1, 256, 0, s>>>(c, (int)n, static_cast<uint8_t*>(dst) + off);
        ++g_launches;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_fit(const FitParams& p, cudaStream_t s) {
    if (p.n_traces <= 0) return cudaSuccess;
    const int esz = p.is_f64 ? 8 : 4;
    const int smem = round16(128 * 65 * esz) + 2 * p.T * 8;
    const unsigned grid = (unsigned)((p.n_traces + 127) / 128);
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

cudaError_t launch_sweep(int mode, bool f64, bool aligned, const SweepParams& p, cudaStream_t s) {
    if (p.n_traces <= 0) return cudaSuccess;
#define CHASE_SWEEP_CASE(M)                                                                                 \
    if (mode == M) {                                                                                        \
        if (f64) return aligned ? launch_sweep_t<M, double, true>(p, s) : launch_sweep_t<M, double, false>(p, s); \
        return aligned ? launch_sweep_t<M, float, true>(p, s) : launch_sweep_t<M, float, false>(p, s);    \
    }
    CHASE_SWEEP_CASE(MODE_FUSED)
    CHASE_SWEEP_CASE(MODE_PREDICT)
    CHASE_SWEEP_CASE(MODE_REPLAY)
#undef CHASE_SWEEP_CASE
    return cudaErrorInvalidValue;
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

cudaError_t launch_fixup(const uint8_t* status, int64_t n_traces, uint8_t* choice, int64_t ld_c, int64_t W,
                         int n_eta_choice, double* forecast, int64_t ld_f, chase_diag_t* diag, cudaStream_t s) {
    if (n_traces <= 0) return cudaSuccess;
    const int64_t g = n_traces < (int64_t)num_sms() * 8 ? n_traces : (int64_t)num_sms() * 8;
    fixup_kernel<<<(unsigned)g, 128, 0, s>>>(status, n_traces, choice, ld_c, W, n_eta_choice, forecast, ld_f, diag);
    diag_status_kernel<<<1, 32, 0, s>>>(status, n_traces, diag);
    g_launches += 2;
    return cudaGetLastError();
}

cudaError_t launch_finalize(const FinalizeParams& p, chase_sum_t* sum, uint8_t* choice, int64_t ld_c,
                            int n_eta_choice, double* forecast, int64_t ld_f, chase_diag_t* diag, cudaStream_t s) {
    if (p.n_traces > 0) {
        const int64_t grid = finalize_grid(p.n_traces);
        if (p.is_f64) finalize_kernel<double><<<(unsigned)grid, kFinThreads, 0, s>>>(p);
        else finalize_kernel<float><<<(unsigned)grid, kFinThreads, 0, s>>>(p);
        ++g_launches;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        if (sum) {
            finalize_sums_kernel<<<p.n_eta, 32, 0, s>>>(p.block_sums, grid, p.n_eta, sum);
            ++g_launches;
        }
    } else if (sum) {
        cudaError_t e = cudaMemsetAsync(sum, 0, sizeof(chase_sum_t) * (size_t)p.n_eta, s);
        if (e != cudaSuccess) return e;
    }
    return launch_fixup(p.status, p.n_traces, choice, ld_c, p.W, n_eta_choice, forecast, ld_f, diag, s);
}

cudaError_t launch_diag_reset(chase_diag_t* diag, cudaStream_t s) {
    diag_reset_kernel<<<1, 32, 0, s>>>(diag);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_accumulate(double* acc, const double* add, int n, cudaStream_t s) {
    accumulate_sums_kernel<<<1, 128, 0, s>>>(acc, add, n);
    ++g_launches;
    return cudaGetLastError();
}

}  // namespace chase
