// kernels.cu — sm_100a kernels of the Chase batched trace-replay planner.
//
//   fit_once_kernel   §3.1 Eq. 1-2 fit on the L history points, lane = trace,
//                     canonical sequential order (bit-identical to the oracle).
//   sweep_kernel      persistent CTAs; per (trace, tile of 9216 windows): TMA
//                     bulk copy of the trace tile into a 2-stage smem ring,
//                     predict (Eq. 1) -> Eq. 6 argmin via the exact envelope
//                     bucket table (canonical K-way fallback) -> fixed-work
//                     replay partials -> block scan / reduce -> per-trace
//                     totals; choices staged in smem and bulk-stored.
//   plan_kernel       Eq. 6 argmin from given forecasts (split path).
//   finalize_kernel   fixed-order per-GPU sums, invalid-trace fix-up.
//
// Arithmetic contract: the fp64 steps that decide outputs are written with
// explicit round-to-nearest intrinsics (and the file is built -fmad=false),
// in the same order as the oracle (DESIGN.md §3 Q9), so forecasts and choices
// are bit-identical and dyadic replay totals are exact.
#include <cfloat>
#include <cstdio>

#include "kernels.h"

namespace chase {
namespace {

constexpr int kWarps = kThreads / 32;
constexpr unsigned kFull = 0xffffffffu;

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
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
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
// Canonical rule: cost_k = ((a_k*x) + Kc)/Thr_k, each op rounded once,
// first minimum (lowest limit).  Taken by < 1e-6 of windows.
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

// Envelope fast path: bucket of y = x * (1/Kc) by the high bits
// of its fp64 encoding, then at most one threshold pair.  `slow` is set when
// y falls in a band where only the canonical rule is trusted.
__device__ __forceinline__ uint32_t plan_fast(double x, double invK, const PairTable* pt, bool& slow) {
    double y = __dmul_rn(x, invK);
    int hi = __double2hiint(y);
    int idx = (hi >> kSH) - pt->base;
    idx = min(max(idx, 0), kNBUsed - 1);
    uint32_t e = pt->ent[idx];
    double2 th = pt->slots[e >> 10];
    bool p1 = y <= th.x;
    bool p2 = y >= th.y;
    slow = !(p1 || p2);
    return p1 ? (e & 31u) : ((e >> 5) & 31u);
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

struct SmemLayout {
    int tables, aext, stage, chb, scratch, scratch2, state, res, info, ctasum, mbar, total;
};

__host__ __device__ inline SmemLayout make_layout(int tables_bytes, int T, int stage_bytes) {
    SmemLayout L;
    int o = 0;
    L.tables = o; o += round16(tables_bytes);
    L.aext = o; o += round16((T + kChunk) * 8);
    L.stage = o; o += 2 * stage_bytes;
    L.chb = o; o += 2 * kTileW;
    L.scratch = o; o += 2 * kWarps * 4 * 8;
    L.scratch2 = o; o += kWarps * 2 * 8;
    L.state = o; o += kMaxEta * 4 * 8;
    L.res = o; o += kMaxEta * 8 * 8;
    L.info = o; o += 8 * 8;
    L.ctasum = o; o += kMaxEta * 8 * 8;
    L.mbar = o; o += 16;
    L.total = round16(o);
    return L;
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

template <typename E>
__global__ void __launch_bounds__(128) fit_once_kernel(const __grid_constant__ FitParams p) {
    // Stage the CTA's 128 histories (L <= 64) into smem with coalesced loads,
    // padded to an odd row stride; longer histories are read from global.
    extern __shared__ __align__(16) uint8_t fsm[];
    E* hs = reinterpret_cast<E*>(fsm);
    double* tab = reinterpret_cast<double*>(fsm + round16(128 * 65 * (int)sizeof(E)));
    const int L = p.L, T = p.T;
    const int64_t first = (int64_t)blockIdx.x * 128;
    const E* tr = reinterpret_cast<const E*>(p.traces);
    for (int q = threadIdx.x; q < 2 * T; q += blockDim.x) tab[q] = p.phase_tab[q];
    const bool staged = L <= 64;
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
    const E* h = staged ? hs + threadIdx.x * (L | 1) : tr + i * p.ld;
    double rec[kRecDoubles];
    fit_one<E>(h, L, T, p.phase0 % T, tab, tab + T, p.ridge, p.tol, rec);
    double* out = p.records + i * kRecDoubles;
#pragma unroll
    for (int q = 0; q < kRecDoubles; ++q) out[q] = rec[q];
    if (p.models_out) {
#pragma unroll
        for (int q = 0; q < kRecDoubles; ++q) p.models_out[i * kRecDoubles + q] = rec[q];
    }
    if (p.max_ci_out) p.max_ci_out[i] = rec[4];
}

// ------------------------------------------------------------------ sweep (K2)
template <int MODE, typename E, bool AL>
__global__ void __launch_bounds__(kThreads, 2) sweep_kernel(const __grid_constant__ SweepParams P) {
    extern __shared__ __align__(128) uint8_t sm[];
    constexpr int VEC = 16 / (int)sizeof(E);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const SmemLayout Ly = make_layout(P.tables_bytes, P.T, P.stage_bytes);

    const TablesHeader* H = reinterpret_cast<const TablesHeader*>(sm + Ly.tables);
    double* A_ext = reinterpret_cast<double*>(sm + Ly.aext);
    uint8_t* stage0 = sm + Ly.stage;
    uint8_t* chb0 = sm + Ly.chb;
    double* scratch = reinterpret_cast<double*>(sm + Ly.scratch);    // [2][kWarps][4]
    double* scratch2 = reinterpret_cast<double*>(sm + Ly.scratch2);  // [kWarps][2]
    double* state = reinterpret_cast<double*>(sm + Ly.state);        // [eta][4]: S, E, C, done
    double* res = reinterpret_cast<double*>(sm + Ly.res);            // [eta][8]
    double* info = reinterpret_cast<double*>(sm + Ly.info);          // completion info
    double* ctasum = reinterpret_cast<double*>(sm + Ly.ctasum);      // [eta][8]
    uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + Ly.mbar);

    // constant tables -> smem (16-byte vectors)
    {
        const uint4* src = reinterpret_cast<const uint4*>(P.tables);
        uint4* dst = reinterpret_cast<uint4*>(sm + Ly.tables);
        for (int q = tid; q < P.tables_bytes / 16; q += kThreads) dst[q] = src[q];
    }
    for (int q = tid; q < kMaxEta * 8; q += kThreads) ctasum[q] = 0.0;
    if (tid == 0) {
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

    // region of trace i loaded for tile t: [a, b) in elements
    auto tile_region = [&](int tile, int64_t& a, int64_t& b, int& Wt) {
        int64_t ws = (int64_t)P.L + (int64_t)tile * kTileW;
        Wt = min(kTileW, P.W - tile * kTileW);
        a = AL ? ws - VEC : ((ws - 1) / VEC) * VEC;
        b = ((ws + Wt + VEC - 1) / VEC) * VEC;
        if (b > P.ld) b = P.ld;
    };
    auto issue = [&](int64_t item) {  // thread 0 only
        if (item >= n_items) return;
        const int st = (int)(item & 1);
        const int64_t i = blockIdx.x + (item / P.n_tiles) * G;
        const int tile = (int)(item % P.n_tiles);
        int64_t a, b;
        int Wt;
        tile_region(tile, a, b, Wt);
        uint32_t bytes = (uint32_t)((b - a) * (int64_t)sizeof(E));
        const bool rec = MODE != MODE_REPLAY && tile == 0;
        uint8_t* dst = stage0 + st * P.stage_bytes;
        mbar_arrive_expect_tx(&mbar[st], bytes + (rec ? 64u : 0u));
        bulk_g2s(dst, traces + i * P.ld + a, bytes, &mbar[st], policy);
        if (rec) bulk_g2s(dst + P.stage_bytes - 64, P.records + i * kRecDoubles, 64, &mbar[st], policy);
    };
    if (tid == 0) {
        issue(0);
        issue(1);
    }

    // per-trace (uniform) state, kept in registers across the trace's tiles
    int status = 0, prof = 0, K = 0;
    double wl = 0.0, maxci = 0.0, J = 0.0;
    int64_t mb = 0, m_base = 0;
    bool base_exhausted = false;
    double Cb_run = 0.0;  // thread 0: baseline sum of c over windows before w*_b
    int64_t slow_count = 0;
    int64_t gp = 0;  // global pass counter (buffer parity)

    for (int64_t q = 0; q < n_items; ++q) {
        const int st = (int)(q & 1);
        const int64_t i = blockIdx.x + (q / P.n_tiles) * G;
        const int tile = (int)(q % P.n_tiles);
        int64_t a_abs, b_abs;
        int Wt;
        tile_region(tile, a_abs, b_abs, Wt);
        const int64_t ws_abs = (int64_t)P.L + (int64_t)tile * kTileW;
        uint8_t* stage = stage0 + st * P.stage_bytes;
        const E* tv = reinterpret_cast<const E*>(stage) + (ws_abs - a_abs);  // tv[j] = c[ws_abs + j]
        mbar_wait(&mbar[st], (uint32_t)((q >> 1) & 1));

        if (tile == 0) {
            prof = P.profile_id ? (int)P.profile_id[i] : 0;
            if (prof >= P.n_prof) prof = 0;
            K = profs[prof].K;
            J = P.job ? P.job[i] : 0.0;
            if (MODE != MODE_REPLAY) {
                const double* rec = reinterpret_cast<const double*>(stage + P.stage_bytes - 64);
                status = (int)rec[5];
                wl = rec[3];
                maxci = P.max_ci_fixed > 0.0 ? P.max_ci_fixed : rec[4];
                if (status == 0 && MODE == MODE_FUSED && !(maxci > 0.0)) status = CHASE_ERR_MAXCI;
                if (status == 0) {
                    const double c0 = rec[0], wsn = rec[1], wcs = rec[2];
                    for (int qq = tid; qq < P.T + kChunk; qq += kThreads) {
                        int ph = qq % P.T;
                        A_ext[qq] = __dadd_rn(__dadd_rn(c0, __dmul_rn(wsn, phS[ph])), __dmul_rn(wcs, phC[ph]));
                    }
                }
            } else {
                status = 0;
            }
            // baseline: constant largest limit; completion count m_base
            if (MODE != MODE_PREDICT) {
                const double sb = profs[prof].line[K - 1].x;
                mb = P.W;
                m_base = 0;
                base_exhausted = false;
                if (J > 0.0) {
                    double qv = __ddiv_rn(J, sb);
                    int64_t m = qv < 4.0e15 ? (int64_t)ceil(qv) : (int64_t)P.W + 2;
                    if (m < 1) m = 1;
                    while (m > 1 && __dmul_rn((double)(m - 1), sb) >= J) --m;
                    while (m <= (int64_t)P.W && __dmul_rn((double)m, sb) < J) ++m;
                    m_base = m;
                    if (m > P.W) base_exhausted = true;
                    else mb = m - 1;
                }
            }
            if (tid == 0) {
                Cb_run = 0.0;
                for (int e = 0; e < n_pass; ++e) {
                    state[e * 4 + 0] = state[e * 4 + 1] = state[e * 4 + 2] = state[e * 4 + 3] = 0.0;
                    for (int r = 0; r < 8; ++r) res[e * 8 + r] = 0.0;
                    res[e * 8 + 6] = -1.0;  // completion window
                }
            }
        }
        __syncthreads();  // BA: A_ext / state visible; stage landed for everyone

        const int j0 = kChunk * tid;
        const int nwin = max(0, min(kChunk, Wt - j0));
        const int nwords = j0 < ((Wt + 15) & ~15) ? kChunk / 4 : 0;  // words this thread stages

        for (int e = 0; e < n_pass && status == 0; ++e, ++gp) {
            const int sb = (int)(gp & 1);
            uint8_t* chb = chb0 + sb * kTileW;
            uint32_t* chb32 = reinterpret_cast<uint32_t*>(chb);
            const double S_run = state[e * 4 + 0];
            const bool done = state[e * 4 + 3] != 0.0;
            const bool replay = MODE != MODE_PREDICT && !done;
            const PairTable* pt = pairs + prof * P.n_eta + e;
            const double Kc = __dmul_rn(pt->kbase, maxci);
            const double invK = per_trace_invK(pt, Kc);
            const double2* lines = profs[prof].line;

            double St = 0.0, Et = 0.0, Ct = 0.0, Cbt = 0.0;
            int bad = 0;
            if (nwin > 0 || nwords > 0) {
                double lag = nwin > 0 ? (double)tv[j0 - 1] : 0.0;
                int phi0 = (int)(((int64_t)P.phase0 + ws_abs + j0) % P.T);
                const double* Ap = A_ext + phi0;
                const int64_t jbase = (int64_t)tile * kTileW + j0;  // window index from s0
                const uint32_t* cin = nullptr;
                if (MODE == MODE_REPLAY)
                    cin = reinterpret_cast<const uint32_t*>(P.choice_in + ((int64_t)e * P.n_traces + i) * P.ld_c +
                                                            (int64_t)tile * kTileW + j0);
                double* fout = nullptr;
                if (P.forecast && e == 0) fout = P.forecast + i * P.ld_f + (int64_t)tile * kTileW + j0;
#pragma unroll
                for (int g = 0; g < kChunk / 4; ++g) {
                    if (4 * g >= nwin) {
                        if (g < nwords && MODE != MODE_PREDICT) chb32[(j0 >> 2) + g] = 0xffffffffu;
                        continue;
                    }
                    E v[4];
                    if (AL && sizeof(E) == 4) {
                        float4 f4 = *reinterpret_cast<const float4*>(tv + j0 + 4 * g);
                        v[0] = (E)f4.x; v[1] = (E)f4.y; v[2] = (E)f4.z; v[3] = (E)f4.w;
                    } else {
#pragma unroll
                        for (int u = 0; u < 4; ++u) v[u] = tv[j0 + 4 * g + u];
                    }
                    uint32_t word = 0;
                    uint32_t cw_in = MODE == MODE_REPLAY ? ldg_nc_u32(cin + g) : 0u;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int jj = 4 * g + u;
                        uint32_t k = 0xffu;
                        if (jj < nwin) {
                            const double cw = (double)v[u];
                            if (e == 0) bad |= bad_value(v[u]);
                            if (MODE != MODE_REPLAY) {
                                double pr = __dadd_rn(Ap[jj], __dmul_rn(wl, lag));  // Eq. 1
                                double x = pr > 0.0 ? pr : 0.0;                     // clamp
                                if (fout) fout[jj] = x;
                                if (MODE == MODE_FUSED) {
                                    bool slow;
                                    k = plan_fast(x, invK, pt, slow);
                                    if (slow) {
                                        k = canonical_choose(x, Kc, pt->a, profs[prof].thr, K);
                                        ++slow_count;
                                    }
                                }
                            } else {
                                k = (cw_in >> (8 * u)) & 0xffu;
                                if (k >= (uint32_t)K) { bad |= 2; k = 0; }
                            }
                            if (MODE != MODE_PREDICT) {
                                if (replay) {
                                    const double2 ln = lines[k];  // (Thr_k * Delta, P_k)
                                    St = __dadd_rn(St, ln.x);
                                    Et = __dadd_rn(Et, ln.y);
                                    Ct = __dadd_rn(Ct, __dmul_rn(ln.y, cw));
                                }
                                if (e == 0 && jbase + jj < mb) Cbt = __dadd_rn(Cbt, cw);
                            }
                            lag = cw;
                        }
                        word |= k << (8 * u);
                    }
                    if (MODE != MODE_PREDICT) chb32[(j0 >> 2) + g] = word;
                }
            }
            // ---- block level: scan S, reduce E, C, Cb (fixed order)
            double Sincl = warp_incl_scan(St, lane);
            double Ew = warp_sum(Et), Cw = warp_sum(Ct), Cbw = warp_sum(Cbt);
            double* scr = scratch + sb * kWarps * 4;
            if (lane == 31) scr[warp * 4 + 0] = Sincl;
            if (lane == 0) {
                scr[warp * 4 + 1] = Ew;
                scr[warp * 4 + 2] = Cw;
                scr[warp * 4 + 3] = Cbw;
            }
            if (MODE != MODE_PREDICT) fence_proxy_async();
            if (tid == 0) bulk_wait_read0();  // previous pass's choice store has left smem
            const int bad_any = __syncthreads_or(bad);  // B1
            if (bad_any) {
                status = (bad_any & 2) ? CHASE_ERR_CHOICE : CHASE_ERR_DATA;
                break;
            }
            double S_tile = 0.0, E_tile = 0.0, C_tile = 0.0, Cb_tile = 0.0, S_wex = 0.0;
            for (int w = 0; w < kWarps; ++w) {
                if (w == warp) S_wex = S_tile;
                S_tile = __dadd_rn(S_tile, scr[w * 4 + 0]);
                E_tile = __dadd_rn(E_tile, scr[w * 4 + 1]);
                C_tile = __dadd_rn(C_tile, scr[w * 4 + 2]);
                Cb_tile = __dadd_rn(Cb_tile, scr[w * 4 + 3]);
            }
            if (tid == 0 && MODE == MODE_FUSED && P.choice) {
                uint8_t* dst = P.choice + ((int64_t)e * P.n_traces + i) * P.ld_c + (int64_t)tile * kTileW;
                bulk_s2g(dst, chb, (uint32_t)((Wt + 15) & ~15));
                bulk_commit();
            }
            if (tid == 0 && e == 0) Cb_run = __dadd_rn(Cb_run, Cb_tile);
            if (MODE == MODE_PREDICT) continue;
            const bool completes = !done && J > 0.0 && __dadd_rn(S_run, S_tile) >= J;
            if (!completes) {
                if (tid == 0 && !done) {
                    state[e * 4 + 0] = __dadd_rn(S_run, S_tile);
                    state[e * 4 + 1] = __dadd_rn(state[e * 4 + 1], E_tile);
                    state[e * 4 + 2] = __dadd_rn(state[e * 4 + 2], C_tile);
                }
                continue;
            }
            // ---- the job completes inside this tile (once per trace and eta)
            const double Sex = __shfl_up_sync(kFull, Sincl, 1);
            const double before = __dadd_rn(__dadd_rn(S_run, S_wex), lane == 0 ? 0.0 : Sex);
            const double after = __dadd_rn(before, St);
            const bool full = after < J;
            const bool mine = !full && before < J && nwin > 0;
            double Em = warp_sum(full ? Et : 0.0), Cm = warp_sum(full ? Ct : 0.0);
            if (lane == 0) {
                scratch2[warp * 2 + 0] = Em;
                scratch2[warp * 2 + 1] = Cm;
            }
            if (mine) {
                double S = before, Ep = 0.0, Cp = 0.0;
                int jj = 0;
                double f = 1.0;
                uint32_t k = 0;
                double cwst = 0.0;
                for (; jj < nwin; ++jj) {
                    k = chb[j0 + jj];
                    const double2 ln = lines[k];
                    const double cw = (double)tv[j0 + jj];
                    const double prev = S;
                    S = __dadd_rn(S, ln.x);
                    if (S >= J || jj == nwin - 1) {
                        f = __ddiv_rn(__dsub_rn(J, prev), ln.x);
                        cwst = cw;
                        break;
                    }
                    Ep = __dadd_rn(Ep, ln.y);
                    Cp = __dadd_rn(Cp, __dmul_rn(ln.y, cw));
                }
                info[0] = (double)(ws_abs + j0 + jj);
                info[1] = f;
                info[2] = Ep;
                info[3] = Cp;
                info[4] = lines[k].y;
                info[5] = cwst;
            }
            __syncthreads();  // B2
            if (tid == 0) {
                double Em_t = 0.0, Cm_t = 0.0;
                for (int w = 0; w < kWarps; ++w) {
                    Em_t = __dadd_rn(Em_t, scratch2[w * 2 + 0]);
                    Cm_t = __dadd_rn(Cm_t, scratch2[w * 2 + 1]);
                }
                const double Etot = __dadd_rn(__dadd_rn(state[e * 4 + 1], Em_t), info[2]);
                const double Ctot = __dadd_rn(__dadd_rn(state[e * 4 + 2], Cm_t), info[3]);
                const double f = info[1], Pk = info[4];
                const int64_t wstar = (int64_t)info[0];
                double* r = res + e * 8;
                r[0] = __dmul_rn(__dadd_rn((double)(wstar - P.L), f), P.delta);
                r[1] = __dmul_rn(__dadd_rn(Etot, __dmul_rn(f, Pk)), P.delta);
                r[2] = __ddiv_rn(__dmul_rn(__dadd_rn(Ctot, __dmul_rn(f, __dmul_rn(Pk, info[5]))), P.delta), 3.6e6);
                r[3] = J;
                r[6] = (double)wstar;
                state[e * 4 + 3] = 1.0;
            }
            __syncthreads();  // B3: info / scratch2 reusable, stage reads done
        }

        // ---- end of trace: totals, baseline, sums (thread 0)
        if (tile == P.n_tiles - 1 && tid == 0) {
            const ProfileTable& pf = profs[prof];
            if (MODE == MODE_PREDICT) {
                P.status[i] = (uint8_t)status;
            } else {
                double bt = 0.0, be = 0.0, bc = 0.0;
                int bstat = 0;
                if (status == 0) {
                    const double sbv = pf.line[K - 1].x, Pb = pf.line[K - 1].y;
                    if (J > 0.0 && !base_exhausted) {
                        const int64_t m = m_base;
                        const double prevS = __dmul_rn((double)(m - 1), sbv);
                        const double f = __ddiv_rn(__dsub_rn(J, prevS), sbv);
                        const double Eb = __dmul_rn((double)(m - 1), Pb);
                        const double Cb = __dmul_rn(Pb, Cb_run);
                        const double cst = (double)traces[i * P.ld + P.L + (m - 1)];
                        bt = __dmul_rn(__dadd_rn((double)(m - 1), f), P.delta);
                        be = __dmul_rn(__dadd_rn(Eb, __dmul_rn(f, Pb)), P.delta);
                        bc = __ddiv_rn(__dmul_rn(__dadd_rn(Cb, __dmul_rn(f, __dmul_rn(Pb, cst))), P.delta), 3.6e6);
                    } else {
                        bt = __dmul_rn((double)P.W, P.delta);
                        be = __dmul_rn(__dmul_rn((double)P.W, Pb), P.delta);
                        bc = __ddiv_rn(__dmul_rn(__dmul_rn(Pb, Cb_run), P.delta), 3.6e6);
                        if (J > 0.0) bstat = CHASE_ERR_TRACE_EXHAUSTED;
                    }
                }
                int worst = status;
                for (int e = 0; e < n_pass; ++e) {
                    double* r = res + e * 8;
                    int st_e = status;
                    if (status == 0 && state[e * 4 + 3] == 0.0) {  // no completion: fixed duration / exhausted
                        r[0] = __dmul_rn((double)P.W, P.delta);
                        r[1] = __dmul_rn(state[e * 4 + 1], P.delta);
                        r[2] = __ddiv_rn(__dmul_rn(state[e * 4 + 2], P.delta), 3.6e6);
                        r[3] = state[e * 4 + 0];
                        r[6] = -1.0;
                        if (J > 0.0) st_e = CHASE_ERR_TRACE_EXHAUSTED;
                    }
                    if (st_e == 0) st_e = bstat;
                    if (status != 0) {
                        for (int rr = 0; rr < 8; ++rr) r[rr] = 0.0;
                        r[6] = -1.0;
                    }
                    if (st_e > worst) worst = st_e;
                    if (P.per_trace) {
                        chase_totals_t t;
                        t.time_s = r[0];
                        t.energy_j = r[1];
                        t.carbon_g = r[2];
                        t.samples = r[3];
                        t.base_time_s = status ? 0.0 : bt;
                        t.base_energy_j = status ? 0.0 : be;
                        t.base_carbon_g = status ? 0.0 : bc;
                        t.completion_window = (int32_t)r[6];
                        t.status = st_e;
                        P.per_trace[(int64_t)e * P.n_traces + i] = t;
                    }
                    if (st_e == 0) {
                        double* cs = ctasum + e * 8;
                        cs[0] = __dadd_rn(cs[0], r[0]);
                        cs[1] = __dadd_rn(cs[1], r[1]);
                        cs[2] = __dadd_rn(cs[2], r[2]);
                        cs[3] = __dadd_rn(cs[3], r[3]);
                        cs[4] = __dadd_rn(cs[4], bt);
                        cs[5] = __dadd_rn(cs[5], be);
                        cs[6] = __dadd_rn(cs[6], bc);
                        cs[7] = __dadd_rn(cs[7], 1.0);
                    }
                }
                P.status[i] = (uint8_t)worst;
            }
            if (status != 0) {
                atomicAdd(reinterpret_cast<unsigned long long*>(&P.diag->n_bad), 1ull);
                atomicMin(reinterpret_cast<unsigned long long*>(&P.diag->first_bad_trace), (unsigned long long)i);
            }
        }
        // stage `st` is free once every thread passed the last barrier above
        if (tid == 0) issue(q + 2);
    }

    // per-CTA sums (fixed trace order) and diagnostics
    __syncthreads();
    if (tid == 0) {
        for (int e = 0; e < n_pass; ++e)
            for (int r = 0; r < 8; ++r)
                P.cta_sums[((int64_t)blockIdx.x * n_pass + e) * 8 + r] = ctasum[e * 8 + r];
        bulk_wait0();
    }
    unsigned long long sc = (unsigned long long)slow_count;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sc += __shfl_xor_sync(kFull, sc, o);
    if (lane == 0 && sc) atomicAdd(reinterpret_cast<unsigned long long*>(&P.diag->n_slow_windows), sc);
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
    const int64_t groups = (p.W + 3) / 4;               // 4 windows per thread-step
    const int64_t total = p.n_traces * groups;
    int64_t slow_count = 0;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = g / groups, w0 = (g - i * groups) * 4;
        int prof = p.profile_id ? (int)p.profile_id[i] : 0;
        if (prof >= p.n_prof) prof = 0;
        const int K = profs[prof].K;
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
                    bool slow;
                    k = plan_fast(x[u], invK, pt, slow);
                    if (slow) {
                        k = canonical_choose(x[u], Kc, pt->a, profs[prof].thr, K);
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

// ------------------------------------------------------------------ finalize / fix-up
__global__ void finalize_sums_kernel(const double* cta_sums, int grid, int n_eta, chase_sum_t* sum) {
    const int e = blockIdx.x, r = threadIdx.x;
    if (e >= n_eta || r >= 8) return;
    double acc = 0.0;
    for (int b = 0; b < grid; ++b) acc = __dadd_rn(acc, cta_sums[((int64_t)b * n_eta + e) * 8 + r]);
    reinterpret_cast<double*>(sum + e)[r] = acc;
}

// Invalid traces (status 4..7): choices 0xFF, forecasts NaN; count exhausted.
__global__ void fixup_kernel(const uint8_t* status, int64_t n, uint8_t* choice, int64_t ld_c, int64_t W,
                             int n_eta, double* forecast, int64_t ld_f, chase_diag_t* diag) {
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
        const int s = status[i];
        if (s == CHASE_ERR_TRACE_EXHAUSTED && threadIdx.x == 0)
            atomicAdd(reinterpret_cast<unsigned long long*>(&diag->n_exhausted), 1ull);
        if (s < CHASE_ERR_DATA) continue;
        if (threadIdx.x == 0) {
            unsigned long long old = atomicMin(reinterpret_cast<unsigned long long*>(&diag->first_bad_trace),
                                               (unsigned long long)i);
            (void)old;
        }
        if (choice)
            for (int e = 0; e < n_eta; ++e)
                for (int64_t w = threadIdx.x; w < W; w += blockDim.x) choice[((int64_t)e * n + i) * ld_c + w] = 0xff;
        if (forecast)
            for (int64_t w = threadIdx.x; w < W; w += blockDim.x)
                forecast[i * ld_f + w] = __longlong_as_double(0x7ff8000000000000ll);
    }
}

__global__ void diag_status_kernel(const uint8_t* status, int64_t n, chase_diag_t* diag) {
    // first_bad_status: status of the first bad trace (after fixup_kernel set the index)
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        uint64_t fb = (uint64_t)diag->first_bad_trace;
        if (fb < (uint64_t)n) diag->first_bad_status = status[fb];
    }
}

__global__ void diag_reset_kernel(chase_diag_t* d) {
    if (threadIdx.x == 0) {
        d->first_bad_trace = -1;  // as unsigned: max, so atomicMin works
        d->first_bad_status = 0;
        d->n_bad = d->n_exhausted = d->n_slow_windows = 0;
    }
}

struct UploadChunk {
    uint8_t bytes[30720];
};
__global__ void upload_kernel(const __grid_constant__ UploadChunk c, int n, uint8_t* dst) {
    for (int q = threadIdx.x; q < n; q += blockDim.x) dst[q] = c.bytes[q];
}

template <int MODE, typename E, bool AL>
cudaError_t launch_sweep_t(const SweepParams& p, int max_grid, int* grid_out, cudaStream_t s) {
    const SmemLayout Ly = make_layout(p.tables_bytes, p.T, p.stage_bytes);
    auto kern = sweep_kernel<MODE, E, AL>;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Ly.total);
    if (err != cudaSuccess) return err;
    int per_sm = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, Ly.total);
    if (err != cudaSuccess) return err;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    int64_t grid = (int64_t)sms * per_sm;
    if (grid > p.n_traces) grid = p.n_traces;
    if (grid > max_grid) grid = max_grid;
    if (grid < 1) grid = 1;
    *grid_out = (int)grid;
    kern<<<(unsigned)grid, kThreads, Ly.total, s>>>(p);
    return cudaGetLastError();
}

}  // namespace

// ------------------------------------------------------------------ host launchers
namespace {
thread_local uint64_t g_launches = 0;
}
uint64_t kernel_launches() { return g_launches; }

__global__ void accumulate_sums_kernel(double* acc, const double* add, int n) {
    int q = threadIdx.x;
    if (q < n) acc[q] = __dadd_rn(acc[q], add[q]);
}
cudaError_t launch_accumulate(double* acc, const double* add, int n, cudaStream_t s) {
    accumulate_sums_kernel<<<1, 128, 0, s>>>(acc, add, n);
    ++g_launches;
    return cudaGetLastError();
}

int sweep_stage_bytes(int elem_size) { return round16((kTileW + 8) * elem_size) + 64; }

size_t sweep_smem_bytes(int tables_bytes, int T, int elem_size, int mode) {
    (void)mode;
    return (size_t)make_layout(tables_bytes, T, sweep_stage_bytes(elem_size)).total;
}

cudaError_t launch_upload(const void* host, size_t bytes, void* dst, cudaStream_t s) {
    const uint8_t* h = static_cast<const uint8_t*>(host);
    for (size_t off = 0; off < bytes; off += sizeof(UploadChunk)) {
        UploadChunk c;
        size_t n = bytes - off < sizeof(UploadChunk) ? bytes - off : sizeof(UploadChunk);
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
        cudaFuncSetAttribute(fit_once_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        fit_once_kernel<double><<<grid, 128, smem, s>>>(p);
        ++g_launches;
    } else {
        cudaFuncSetAttribute(fit_once_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        fit_once_kernel<float><<<grid, 128, smem, s>>>(p);
        ++g_launches;
    }
    return cudaGetLastError();
}

cudaError_t launch_sweep(int mode, bool f64, bool aligned, const SweepParams& p, int max_grid, int* grid_out,
                         cudaStream_t s) {
    *grid_out = 0;
    if (p.n_traces <= 0) return cudaSuccess;
    ++g_launches;
#define CHASE_SWEEP_CASE(M)                                                                       \
    if (mode == M) {                                                                              \
        if (f64) return aligned ? launch_sweep_t<M, double, true>(p, max_grid, grid_out, s)       \
                                : launch_sweep_t<M, double, false>(p, max_grid, grid_out, s);     \
        return aligned ? launch_sweep_t<M, float, true>(p, max_grid, grid_out, s)                 \
                       : launch_sweep_t<M, float, false>(p, max_grid, grid_out, s);               \
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
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t groups = p.n_traces * ((p.W + 3) / 4);
    int64_t grid = (groups + 255) / 256;
    if (grid > (int64_t)sms * 8) grid = (int64_t)sms * 8;
    plan_kernel<<<(unsigned)grid, 256, p.tables_bytes, s>>>(p);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_finalize(const double* cta_sums, int grid, int n_eta, chase_sum_t* sum, const uint8_t* status,
                            int64_t n_traces, uint8_t* choice, int64_t ld_c, int64_t W, int n_eta_choice,
                            double* forecast, int64_t ld_f, chase_diag_t* diag, cudaStream_t s) {
    if (sum) {
        finalize_sums_kernel<<<n_eta, 32, 0, s>>>(cta_sums, grid, n_eta, sum);
        ++g_launches;
    }
    if (n_traces > 0) {
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        int64_t g = n_traces < (int64_t)sms * 8 ? n_traces : (int64_t)sms * 8;
        fixup_kernel<<<(unsigned)g, 128, 0, s>>>(status, n_traces, choice, ld_c, W, n_eta_choice, forecast, ld_f,
                                                 diag);
        diag_status_kernel<<<1, 32, 0, s>>>(status, n_traces, diag);
        g_launches += 2;
    }
    return cudaGetLastError();
}

cudaError_t launch_diag_reset(chase_diag_t* diag, cudaStream_t s) {
    diag_reset_kernel<<<1, 32, 0, s>>>(diag);
    ++g_launches;
    return cudaGetLastError();
}

}  // namespace chase
