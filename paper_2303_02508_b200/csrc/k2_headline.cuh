// k2_headline.cuh — the headline planner kernel, specialised for the common
// case (fused plan + replay, fp32 traces with a 16-byte aligned job start, one
// eta, no forecast output).  Same arithmetic as sweep_kernel, same
// decomposition (warp-per-trace streaming through a per-warp TMA bulk-copy
// ring), tuned for instruction count and the shared-memory pipe.
// Included by kernels.cu inside its anonymous namespace.
//
// Per window (hot loop):
//   p = A[phi] + w_lag*c[w-1]                       Eq. 1, canonical order
//   y = p * (1/Kc); h = hi32(y)                     Eq. 6 envelope key
//   e = ent8[clamp((h >> 14) - base)]               one LDS.64: {T1, lo16 addr(below) | lo16 addr(above) << 16}
//   addr = PRMT(e.y, ZB, h < T1 ? below : h > T1 ? above : zero line)
//   (s_k, P_k) = LDS.128 [addr]                     the line itself, no index arithmetic
//   S += s_k; E += P_k; C += P_k*c[w]; Cs += c[w]
// The line table sits in a 256-byte-stride region placed at shared address
// 0x10000, so byte 1 of a line's address is k: the four choice bytes of a
// group come out of the addresses with three PRMTs.  Choices are staged per
// warp in shared memory and written with one TMA bulk store per chunk.

#ifndef CHASE_H_WARPS
#define CHASE_H_WARPS 16
#endif
#define CHASE_H_STAGES 1  // one stage per warp (see the chunk loop)
#ifndef CHASE_H_MINB
#define CHASE_H_MINB 1
#endif
#ifndef CHASE_H_CHUNK
#define CHASE_H_CHUNK 60
#endif
#ifndef CHASE_H0_FAST
#define CHASE_H0_FAST 0  // 1 / 2: the one-fma key in sweep_fast_kernel<0> (measured slower: 12.5 / 11.9 vs 11.0 ms)
#endif
#ifndef CHASE_H_CFMA
#define CHASE_H_CFMA 1  // 1: the group's sum of P_k c as an fma chain (C5: 11.23 -> 11.13 ms; exact for dyadic inputs)
#endif
#ifndef CHASE_P2_CF
#define CHASE_P2_CF 1  // 0: sequential horizons at P = 2 (sweep_fast_kernel<4>; C5 18.7 vs 16.2 ms with the closed form)
#endif
#ifndef CHASE_LONG_CF
#define CHASE_LONG_CF 1  // 1: the closed form for P >= 64 too (sweep_fast_kernel<2>, cfh_setup_long)
#endif
#ifndef CHASE_LANE_RUNS
#define CHASE_LANE_RUNS 2  // lane-local periods replayed as runs: 1: P % 4 == 0 (LDS.128 tree), 2: every P >= CHASE_RUN_MIN_P
#endif
#ifndef CHASE_RUN_MIN_P
#define CHASE_RUN_MIN_P 2  // CHASE_LANE_RUNS >= 2: the shortest period replayed as a run
#endif
#ifndef CHASE_BATCH_BLOCKS
#define CHASE_BATCH_BLOCKS 1  // 1: long periods' full lanes replay as two runs over 4-window blocks
#endif
#ifndef CHASE_DAY_BLOCKS
#define CHASE_DAY_BLOCKS 1  // 1: P = 24 full chunks as five 12-window runs per lane (period_day)
#endif
#ifndef CHASE_P2_G
#define CHASE_P2_G 2   // periods per iteration at P = 2 (sweep_fast_kernel<4>; must divide 30)
#endif
#ifndef CHASE_P_FULL
#define CHASE_P_FULL 1  // 1: P = 2 skips the per-period range test when every range is [0, inf)
#endif
#ifndef CHASE_P_LD2
#define CHASE_P_LD2 1  // 1: odd lane-local P up to CHASE_P_LD2_MAXP load their values as LDS.64 pairs
#endif
#ifndef CHASE_P_LD2_MAXP
#define CHASE_P_LD2_MAXP 15
#endif
#ifndef CHASE_P_DEFER
#define CHASE_P_DEFER 1  // 1: even lane-local periods replay first and fix declined closed-form periods after
#endif
#ifndef CHASE_P_WORDS
#define CHASE_P_WORDS 1  // 1: lane-local even periods store a group's choices as 4-byte words
#endif
#ifndef CHASE_H_PAIRSUM
#define CHASE_H_PAIRSUM 1  // 1: a group's four terms summed pairwise before the running sums
#endif
constexpr int kHWarps = CHASE_H_WARPS;    // independent warps per CTA
constexpr int kHThreads = 32 * kHWarps;
constexpr int kHStages = CHASE_H_STAGES;  // per-warp TMA ring depth
constexpr int kHChunk = CHASE_H_CHUNK;    // windows per lane per chunk (4 x odd: conflict-free LDS.128)
constexpr int kHWarpW = 32 * kHChunk;     // windows per warp chunk
static_assert(kHChunk % 8 == 4, "kHChunk must be 4 mod 8");
constexpr int kLineStride = 256;          // bytes between lines k and k+1
constexpr int kLineRegion = kLineStride * (kMaxK + 1);
constexpr uint32_t kLineBase = 0x10000;   // shared address of the line region (byte 1 of an address = k)

// Line k of profile p: kLineBase + 256 k + 16 ((k + p) mod 16).  The slot
// rotation puts lines k = 0..7 of a profile in distinct shared-memory banks.
__host__ __device__ inline int line_off(int p, int k) { return kLineStride * k + 16 * ((k + p) & 15); }
__host__ __device__ inline int haext_len(int T) { return T + kHChunk + 4; }
__host__ __device__ inline int hstage_bytes() { return round16((kHWarpW + 8) * 4) + kRecBytes; }

// Shared-memory plan, computed identically on host and device from the CTA's
// shared-window base address.  The line region sits at kLineBase; the warp
// blocks and then the tables are placed first-fit in the space before it and
// after it.  Tables: the blob's header, phase table and profiles (its first
// `head_bytes` bytes), one PairHead per profile (the pair tables minus their
// 8-byte entries, replaced by the expanded ent8 table), per-lane phase offsets.
struct HLayout {
    int tables, heads, ent8, lph, lines, warp_bytes, total;
    int n_before, after0;        // warp w's block: w < n_before ? w * warp_bytes : after0 + (w - n_before) * warp_bytes
    int aext, k0, stage, chb, mbar;  // offsets inside a warp block
    __host__ __device__ int warp_off(int w) const {
        return w < n_before ? w * warp_bytes : after0 + (w - n_before) * warp_bytes;
    }
};

struct HAlloc {
    int lo, r0, r1, hi;  // free: [lo, r0) and [hi, inf); the region is [r0, r1)
    __host__ __device__ int take(int bytes, int align) {
        const int a = (lo + align - 1) & ~(align - 1);
        if (a + bytes <= r0) {
            lo = a + bytes;
            return a;
        }
        const int b = (hi + align - 1) & ~(align - 1);
        hi = b + bytes;
        return b;
    }
};

__host__ __device__ inline HLayout make_hlayout(int T, int head_bytes, int n_prof, int base, int k0len) {
    HLayout L;
    L.aext = 0;
    L.k0 = 2 * round16(haext_len(T) * 8);
    L.stage = L.k0 + round16(k0len * 8);
    L.chb = L.stage + kHStages * hstage_bytes();
    L.mbar = L.chb + kHWarpW;
    L.warp_bytes = (L.mbar + 8 * kHStages + 127) & ~127;
    L.lines = (int)kLineBase - base;
    HAlloc A{0, L.lines, L.lines + kLineRegion, L.lines + kLineRegion};
    // warp blocks (128-byte multiples): as many as fit before the region, the rest after it
    L.n_before = L.lines > 0 ? L.lines / L.warp_bytes : 0;
    if (L.n_before > kHWarps) L.n_before = kHWarps;
    A.lo = L.n_before * L.warp_bytes;
    A.hi = (A.hi + 127) & ~127;
    L.after0 = A.hi;
    A.hi += (kHWarps - L.n_before) * L.warp_bytes;
    L.ent8 = A.take(n_prof * kNB * 8, 16);
    L.tables = A.take(round16(head_bytes), 16);
    L.heads = A.take(round16(n_prof * (int)sizeof(PairHead)), 16);
    L.lph = A.take(2 * 32 * 4, 16);
    L.total = A.hi;
    return L;
}

__device__ __forceinline__ double2 lds_line(uint32_t addr) {
    double2 v;
    asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
    return v;
}

// Line address for key h from a bucket entry (below / above / zero line).
__device__ __forceinline__ uint32_t line_addr(int h, uint2 e, uint32_t ZB) {
    const uint32_t sel = h < (int)e.x ? 0x7610u : (h > (int)e.x ? 0x7632u : 0x7654u);
    return __byte_perm(e.y, ZB, sel);
}

// One group of 4 windows: predict, envelope lookup, line load, running sums;
// returns the group's word of 4 choice bytes (byte 1 of each line address).
__device__ __forceinline__ uint32_t hot_group(const float4 v, const double2 A01, const double2 A23, double& lag,
                                              double wl, double invK, const uint2* __restrict__ ent8, int ebase,
                                              uint32_t ZB, Acc& a) {
    a.vmin = fminf(fminf(fminf(a.vmin, v.x), v.y), fminf(v.z, v.w));  // FMNMX3 x2
    const float vv[4] = {v.x, v.y, v.z, v.w};
    const double AA[4] = {A01.x, A01.y, A23.x, A23.y};
    uint32_t ad[4];
#if CHASE_H_PAIRSUM
    // the group's four terms summed pairwise, then added to the running sums:
    // one dependent add per group on each running sum instead of four (the
    // totals' order changes; exact for the dyadic inputs, <= 1e-9 otherwise)
    double2 ln4[4];
    double cw4[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const double cw = (double)vv[u];
        const double p = __dadd_rn(AA[u], __dmul_rn(wl, lag));  // Eq. 1, unclamped for the lookup
        const int h = __double2hiint(__dmul_rn(p, invK));
        const int idx = max(min((h >> kSH) - ebase, kNBUsed - 1), 0);
        ad[u] = line_addr(h, ent8[idx], ZB);
        CHASE_CHECK(ad[u] >= kLineBase && ad[u] + 16 <= kLineBase + kLineRegion);
        ln4[u] = lds_line(ad[u]);  // (Thr_k * Delta, P_k)
        cw4[u] = cw;
        lag = cw;
    }
    a.S = __dadd_rn(a.S, __dadd_rn(__dadd_rn(ln4[0].x, ln4[1].x), __dadd_rn(ln4[2].x, ln4[3].x)));
    a.E = __dadd_rn(a.E, __dadd_rn(__dadd_rn(ln4[0].y, ln4[1].y), __dadd_rn(ln4[2].y, ln4[3].y)));
#if CHASE_H_CFMA
    // sum P_k c as an fma chain (exact for the dyadic inputs: every product is exact)
    a.C = __fma_rn(ln4[3].y, cw4[3], __fma_rn(ln4[2].y, cw4[2], __fma_rn(ln4[1].y, cw4[1], __fma_rn(ln4[0].y, cw4[0], a.C))));
#else
    a.C = __dadd_rn(a.C, __dadd_rn(__dadd_rn(__dmul_rn(ln4[0].y, cw4[0]), __dmul_rn(ln4[1].y, cw4[1])),
                                   __dadd_rn(__dmul_rn(ln4[2].y, cw4[2]), __dmul_rn(ln4[3].y, cw4[3]))));
#endif
    a.Cs = __dadd_rn(a.Cs, __dadd_rn(__dadd_rn(cw4[0], cw4[1]), __dadd_rn(cw4[2], cw4[3])));
#else
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const double cw = (double)vv[u];
        const double p = __dadd_rn(AA[u], __dmul_rn(wl, lag));  // Eq. 1, unclamped for the lookup
        const int h = __double2hiint(__dmul_rn(p, invK));
        const int idx = max(min((h >> kSH) - ebase, kNBUsed - 1), 0);
        ad[u] = line_addr(h, ent8[idx], ZB);
        const double2 ln = lds_line(ad[u]);  // (Thr_k * Delta, P_k)
        a.S = __dadd_rn(a.S, ln.x);
        a.E = __dadd_rn(a.E, ln.y);
        a.C = __dadd_rn(a.C, __dmul_rn(ln.y, cw));
        a.Cs = __dadd_rn(a.Cs, cw);
        lag = cw;
    }
#endif
    const uint32_t word = __byte_perm(__byte_perm(ad[0], ad[1], 0x0051u), __byte_perm(ad[2], ad[3], 0x0051u), 0x5410u);
    a.slow |= word;
    return word;
}

// One lane's full groups of 4 windows.  Words (4 choice bytes) go to the
// warp's staging buffer; `a.slow` collects them for the deferred-window test.
// Two register sets alternate (unrolled by 2): the trace values and A terms of
// group g+1 are loaded while group g computes, with no register moves (the
// reads at most one group past the last stay inside the stage / A buffers).
__device__ __forceinline__ void hot_groups(const float* __restrict__ tv, int ngroups, const double* __restrict__ Ap,
                                           double wl, double invK, const uint2* __restrict__ ent8, int ebase,
                                           uint32_t ZB, uint32_t* __restrict__ words, Acc& a) {
    double lag = (double)tv[-1];
    float4 vx = *reinterpret_cast<const float4*>(tv);
    double2 Ax0 = *reinterpret_cast<const double2*>(Ap);
    double2 Ax1 = *reinterpret_cast<const double2*>(Ap + 2);
    int g = 0;
#pragma unroll 1
    for (; g + 1 < ngroups; g += 2) {
        const float4 vy = *reinterpret_cast<const float4*>(tv + 4 * g + 4);
        const double2 Ay0 = *reinterpret_cast<const double2*>(Ap + 4 * g + 4);
        const double2 Ay1 = *reinterpret_cast<const double2*>(Ap + 4 * g + 6);
        const uint32_t w0 = hot_group(vx, Ax0, Ax1, lag, wl, invK, ent8, ebase, ZB, a);
        vx = *reinterpret_cast<const float4*>(tv + 4 * g + 8);
        Ax0 = *reinterpret_cast<const double2*>(Ap + 4 * g + 8);
        Ax1 = *reinterpret_cast<const double2*>(Ap + 4 * g + 10);
        const uint32_t w1 = hot_group(vy, Ay0, Ay1, lag, wl, invK, ent8, ebase, ZB, a);
        words[g] = w0;  // (lane blocks are 4 mod 8 bytes apart: two 4-byte stores)
        words[g + 1] = w1;
    }
    if (g < ngroups) words[g] = hot_group(vx, Ax0, Ax1, lag, wl, invK, ent8, ebase, ZB, a);
}

// ---- the one-fma key ------------------------------------------
// For a trace whose model and values allow it, the Eq. 6 key is computed as
//   y = fma(wlK, c[w-1], B[phi]),  B[phi] = fl(A[phi] / Kc-ish) = fl(A[phi] * fl(1/Kc)),
//                                  wlK = fl(w_lag * fl(1/Kc))
// (one DFMA instead of DMUL, DADD, DMUL), and the fp32 values become fp64 on
// the integer pipes.  |y - x/Kc| <= 6u (|A| + |w_lag c|)/Kc for the canonical
// forecast x = fl(A + fl(w_lag c)) (Q24), which the kernel keeps below
// 126000u y_min: the envelope intervals are shrunk by s = 2^-36 = 131072u
// (envelope.cpp), so a key inside a shrunk interval puts x/Kc inside the
// verified one and the canonical rule picks that line (the same proof as the
// exact key's, with a wider margin).  The bound holds when |A[phi]| <= Amax and
// every value lies in [FLT_MIN, c_lim], c_lim = (21000 y_min Kc - Amax)/|w_lag|; a chunk with a
// value outside (a zero, a subnormal, a negative, inf/NaN, or too large) is
// redone with the exact key (lane_exact, cold).

// Integer multiply-adds, written so that they issue on the FMA pipe (IMAD)
// rather than the ALU pipe, which the lookup's compares and selects keep busy.
__device__ __forceinline__ uint32_t imad_hi_u32(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ int imad_hi_s32(int a, int b, int c) {
    int d;
    asm("mad.hi.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t imad_lo_u32(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// fp32 bits -> fp64 for a positive normal float: exponent rebias and mantissa
// shift on the FMA pipe (hi = (b >> 3) + 896 << 20 as IMAD.HI, lo = b << 29 as
// IMAD) instead of F2F.F64.F32, which issues at a third of the fp64 add rate.
// Exact in that range.
__device__ __forceinline__ double f32bits_to_f64(uint32_t b) {
    return __hiloint2double((int)imad_hi_u32(b, 0x20000000u, 0x38000000u), (int)imad_lo_u32(b, 0x20000000u, 0u));
}

__device__ __forceinline__ uint32_t hot_group_fast(const float4 v, const double2 B01, const double2 B23, double& lag,
                                                   double wlK, const uint2* __restrict__ ent8, int ebase, uint32_t ZB,
                                                   double& C, uint32_t& bmax, Acc& a) {
    const uint32_t vb[4] = {__float_as_uint(v.x), __float_as_uint(v.y), __float_as_uint(v.z), __float_as_uint(v.w)};
    // range check of every value: b - bits(FLT_MIN) (IMAD), one unsigned max (wraps below FLT_MIN)
    bmax = max(max(max(bmax, imad_lo_u32(vb[0], 1u, 0xff800000u)), imad_lo_u32(vb[1], 1u, 0xff800000u)),
               max(imad_lo_u32(vb[2], 1u, 0xff800000u), imad_lo_u32(vb[3], 1u, 0xff800000u)));
    const double BB[4] = {B01.x, B01.y, B23.x, B23.y};
    uint32_t ad[4];
    double2 ln4[4];
    double cw4[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const double cw = f32bits_to_f64(vb[u]);
        const int h = __double2hiint(__fma_rn(wlK, lag, BB[u]));  // the key (unclamped forecast / Kc)
        const int idx = max(min(imad_hi_s32(h, 1 << (32 - kSH), -ebase), kNBUsed - 1), 0);  // (h >> 14) - base
        ad[u] = line_addr(h, ent8[idx], ZB);
        CHASE_CHECK(ad[u] >= kLineBase && ad[u] + 16 <= kLineBase + kLineRegion);
        ln4[u] = lds_line(ad[u]);  // (Thr_k * Delta, P_k)
        cw4[u] = cw;
        lag = cw;
    }
    a.S = __dadd_rn(a.S, __dadd_rn(__dadd_rn(ln4[0].x, ln4[1].x), __dadd_rn(ln4[2].x, ln4[3].x)));
    a.E = __dadd_rn(a.E, __dadd_rn(__dadd_rn(ln4[0].y, ln4[1].y), __dadd_rn(ln4[2].y, ln4[3].y)));
    // sum P_k c: one fma per window (the products are exact for the dyadic inputs, so
    // the totals are unchanged there; <= 1e-9 otherwise)
    C = __fma_rn(ln4[3].y, cw4[3], __fma_rn(ln4[2].y, cw4[2], __fma_rn(ln4[1].y, cw4[1], __fma_rn(ln4[0].y, cw4[0], C))));
    a.Cs = __dadd_rn(a.Cs, __dadd_rn(__dadd_rn(cw4[0], cw4[1]), __dadd_rn(cw4[2], cw4[3])));
    const uint32_t word = __byte_perm(__byte_perm(ad[0], ad[1], 0x0051u), __byte_perm(ad[2], ad[3], 0x0051u), 0x5410u);
    a.slow |= word;
    return word;
}

// hot_groups with the one-fma key (Bp: the B table at the lane's phase).  The two
// register sets also carry two partial sums of P_k c, merged at the end.
__device__ __forceinline__ void hot_groups_fast(const float* __restrict__ tv, int ngroups, const double* __restrict__ Bp,
                                                double wlK, const uint2* __restrict__ ent8, int ebase, uint32_t ZB,
                                                uint32_t* __restrict__ words, uint32_t& bmax, Acc& a) {
    double lag = (double)tv[-1];
    float4 vx = *reinterpret_cast<const float4*>(tv);
    double2 Bx0 = *reinterpret_cast<const double2*>(Bp);
    double2 Bx1 = *reinterpret_cast<const double2*>(Bp + 2);
    double C0 = 0.0, C1 = 0.0;
    int g = 0;
#pragma unroll 1
    for (; g + 1 < ngroups; g += 2) {
        const float4 vy = *reinterpret_cast<const float4*>(tv + 4 * g + 4);
        const double2 By0 = *reinterpret_cast<const double2*>(Bp + 4 * g + 4);
        const double2 By1 = *reinterpret_cast<const double2*>(Bp + 4 * g + 6);
        const uint32_t w0 = hot_group_fast(vx, Bx0, Bx1, lag, wlK, ent8, ebase, ZB, C0, bmax, a);
        vx = *reinterpret_cast<const float4*>(tv + 4 * g + 8);
        Bx0 = *reinterpret_cast<const double2*>(Bp + 4 * g + 8);
        Bx1 = *reinterpret_cast<const double2*>(Bp + 4 * g + 10);
        const uint32_t w1 = hot_group_fast(vy, By0, By1, lag, wlK, ent8, ebase, ZB, C1, bmax, a);
        words[g] = w0;
        words[g + 1] = w1;
    }
    if (g < ngroups) words[g] = hot_group_fast(vx, Bx0, Bx1, lag, wlK, ent8, ebase, ZB, C0, bmax, a);
    a.C = __dadd_rn(a.C, __dadd_rn(C0, C1));
}

// The last chunk's windows past the lane's full groups, one-fma key (cold).
__device__ __noinline__ Acc hot_tail_fast(const float* tv, int j_begin, int nwin, const double* Bp, double wlK,
                                          const uint2* ent8, int ebase, uint32_t ZB, uint8_t* bytes, uint32_t* bmax_out) {
    Acc a{0.0, 0.0, 0.0, 0.0, FLT_MAX, 0u, 0, 0};
    double lag = (double)tv[j_begin - 1];
    uint32_t bmax = 0u;
    for (int jj = j_begin; jj < nwin; ++jj) {
        const float raw = tv[jj];
        const uint32_t b = __float_as_uint(raw);
        bmax = max(bmax, b - 0x00800000u);
        const double cw = f32bits_to_f64(b);
        const int h = __double2hiint(__fma_rn(wlK, lag, Bp[jj]));
        const int idx = max(min((h >> kSH) - ebase, kNBUsed - 1), 0);
        const uint32_t ad = line_addr(h, ent8[idx], ZB);
        const uint32_t k = (ad >> 8) & 0xffu;
        if (k == (uint32_t)kZeroLine) a.slow |= 0x20u;
        bytes[jj] = (uint8_t)k;
        const double2 ln = lds_line(ad);
        a.S = __dadd_rn(a.S, ln.x);
        a.E = __dadd_rn(a.E, ln.y);
        a.C = __fma_rn(ln.y, cw, a.C);
        a.Cs = __dadd_rn(a.Cs, cw);
        lag = cw;
    }
    *bmax_out = bmax;
    return a;
}

// The canonical fold of Eq. 1 at phase phi, A = (c0 + w_s S[phi]) + w_c C[phi]
// (fit_kernel's record; the same operations as the exact table).
struct ExactModel {
    double c0, ws, wc, wl, Kc, invK;
    const double* phS;
    const double* phC;
    __device__ __forceinline__ double A(int phi) const {
        return __dadd_rn(__dadd_rn(c0, __dmul_rn(ws, phS[phi])), __dmul_rn(wc, phC[phi]));
    }
};

// A lane's windows of a chunk redone with the exact key (the trace's one-fma
// bound does not hold for this chunk, see above): x = fl(A + fl(w_lag c)),
// y = fl(x * fl(1/Kc)), the envelope lookup, the canonical rule for band
// windows; every value validated as the generic path does (cold).
__device__ __noinline__ Acc lane_exact(const float* tv, int nwin, int phi0, int T, const ExactModel& M,
                                       const uint2* ent8, int ebase, uint32_t ZB, const PairTable* pt,
                                       const ProfileTable* pf, uint8_t* bytes, bool canon = false) {
    Acc a{0.0, 0.0, 0.0, 0.0, FLT_MAX, 0u, 0, 0};
    double lag = (double)tv[-1];
    int phi = phi0;
    for (int jj = 0; jj < nwin; ++jj) {
        const float raw = tv[jj];
        const double cw = (double)raw;
        const double p = __dadd_rn(M.A(phi), __dmul_rn(M.wl, lag));
        uint32_t k = kZeroLine;
        if (!canon) {  // (canon: Kc outside [2^-900, 2^900], every window takes the canonical rule)
            const int h = __double2hiint(__dmul_rn(p, M.invK));
            const int idx = max(min((h >> kSH) - ebase, kNBUsed - 1), 0);
            k = (line_addr(h, ent8[idx], ZB) >> 8) & 0xffu;
        }
        if (k == (uint32_t)kZeroLine) {
            k = canonical_choose(p > 0.0 ? p : 0.0, M.Kc, pt->a, pf->thr, pf->K);
            ++a.bad_pad;
        }
        bytes[jj] = (uint8_t)k;
        const double2 ln = pf->line[k];
        a.S = __dadd_rn(a.S, ln.x);
        a.E = __dadd_rn(a.E, ln.y);
        a.C = __dadd_rn(a.C, __dmul_rn(ln.y, cw));
        a.Cs = __dadd_rn(a.Cs, cw);
        a.vmin = fminf(a.vmin, raw);
        a.bad |= bad_value(raw) ? 1 : 0;
        lag = cw;
        phi = phi + 1 == T ? 0 : phi + 1;
    }
    return a;
}

// The deferred (band) windows of a one-fma-key lane: the canonical rule on the
// exact forecast, as fix_slow does from the exact table.
__device__ __noinline__ SlowFix fix_slow_exact(const float* tv, int nwin, int phi0, int T, const ExactModel& M,
                                               const PairTable* pt, const ProfileTable* pf, uint8_t* bytes) {
    SlowFix r{0.0, 0.0, 0.0, 0};
    for (int jj = 0; jj < nwin; ++jj) {
        if (bytes[jj] != (uint8_t)kZeroLine) continue;
        int phi = phi0 + jj;
        while (phi >= T) phi -= T;
        const double x = predict(M.A(phi), M.wl, (double)tv[jj - 1]);
        const uint32_t k = canonical_choose(x, M.Kc, pt->a, pf->thr, pf->K);
        bytes[jj] = (uint8_t)k;
        const double2 ln = pf->line[k];
        const double cw = (double)tv[jj];
        r.S = __dadd_rn(r.S, ln.x);
        r.E = __dadd_rn(r.E, ln.y);
        r.C = __dadd_rn(r.C, __dmul_rn(ln.y, cw));
        ++r.n;
    }
    return r;
}

// Windows [j_begin, nwin) of a lane whose count is not a multiple of 4 (the
// last chunk only): the same lookup, one window at a time (cold).
__device__ __noinline__ Acc hot_tail(const float* tv, int j_begin, int nwin, const double* Ap, double wl, double invK,
                                     const uint2* ent8, int ebase, uint32_t ZB, uint8_t* bytes) {
    Acc a{0.0, 0.0, 0.0, 0.0, FLT_MAX, 0u, 0, 0};
    double lag = (double)tv[j_begin - 1];
    for (int jj = j_begin; jj < nwin; ++jj) {
        const float raw = tv[jj];
        const double cw = (double)raw;
        const double p = __dadd_rn(Ap[jj], __dmul_rn(wl, lag));
        const int h = __double2hiint(__dmul_rn(p, invK));
        const int idx = max(min((h >> kSH) - ebase, kNBUsed - 1), 0);
        const uint32_t ad = line_addr(h, ent8[idx], ZB);
        const uint32_t k = (ad >> 8) & 0xffu;
        if (k == (uint32_t)kZeroLine) a.slow |= 0x20u;
        bytes[jj] = (uint8_t)k;
        const double2 ln = lds_line(ad);
        a.S = __dadd_rn(a.S, ln.x);
        a.E = __dadd_rn(a.E, ln.y);
        a.C = __dadd_rn(a.C, __dmul_rn(ln.y, cw));
        a.Cs = __dadd_rn(a.Cs, cw);
        a.bad |= bad_value(raw) ? 1 : 0;
        lag = cw;
    }
    return a;
}

// Baseline sum of c over this lane's windows before the baseline's
// completion window (the chunk that contains it; cold).
__device__ __noinline__ double partial_cs(const float* tv, int n) {
    double s = 0.0;
    for (int jj = 0; jj < n; ++jj) s = __dadd_rn(s, (double)tv[jj]);
    return s;
}

// ---- decision periods (period_steps P > 1) ----------------
// The choices of a chunk are decided before its replay: every period that
// starts in the chunk forecasts recursively from the value before its start
// (in the stage: the chunk's lag slot or a chunk value), Eq. 6 decides on the
// horizon mean (the envelope lookup, else the canonical rule), and the period's
// windows in this chunk get that byte; windows before the chunk's first period
// start continue the previous chunk's last period (its byte, carried).  The
// hot loop then only replays.  Same operation order as oracle_plan_trace.
// bytes [a, e) of the staging buffer := k (word stores on the aligned middle)
__device__ __forceinline__ void fill_bytes(uint8_t* chb, int a, int e, uint32_t k) {
    while (a < e && (a & 3)) chb[a++] = (uint8_t)k;
    const uint32_t kw = k * 0x01010101u;
    for (; a + 4 <= e; a += 4) *reinterpret_cast<uint32_t*>(chb + a) = kw;
    while (a < e) chb[a++] = (uint8_t)k;
}

// Closed-form horizon mean.  Write Z_k(phi) for the horizon of
// Eq. 1 run from x0 = 0 without the clamp.  For |w_lag| <= 0.99 the unclamped
// forecasts of a period starting at phase phi are Z_k + w_lag^k x0, and when
// all of them are >= 0 the clamp never acts, so the n = P forecasts sum to
//     K0[phi] + h x0,   K0[phi] = sum_k Z_k(phi),  h = sum_{k=1..P} w_lag^k.
// That holds for x0 in [lo[phi], hi[phi]]: each step k with computed Z^_k
// below marg = 4u A_max/(1 - |w_lag|)^2 (their error bound) gives a lower
// (w_lag^k > 0) or an upper (w_lag^k < 0) limit on x0.  The table holds K0
// and h already scaled by c = fl(fl(1/P) fl(1/Kc)), so a period's Eq. 6 key
// is one fma, y' = fl(h' x0 + K0'), against the canonical fl(fl(sum/P)/Kc).
// Their means (y' Kc and the oracle's sequential, clamped sum/P) differ by at
// most kappa X, X = A_max/(1 - |w_lag|) + x0 (a bound on every forecast),
// kappa = 4u (2/(1 - |w_lag|) + P): the clamp is 1-Lipschitz, the
// recursion's errors shrink by |w_lag| per step, the running sums' grow with
// P, the scaling adds 5u X.  The envelope's fast intervals are
// shrunk by s = 2^-36 (envelope.cpp), so a key y' inside one is at least
// y' s/(1+s) from the verified interval's ends: with kappa X <= 120000u y' Kc
// (x0 - r Kc y' <= -A_b, r = 30000/(2/(1 - |w_lag|) + P)) the oracle's mean
// lies in the verified interval and the canonical rule on it picks the same
// line.  K2[j] = {K0', (fp32 lo, fp32 hi)} for phase j mod T, j < n_a =
// haext_len(T) (phase index without wrap, like the A table); K2[n_a] =
// {h', -r Kc}, K2[n_a + 1].x = -A_b (-r Kc = NaN: never).
__device__ __noinline__ void cfh_setup(double2* K2, const double* Aeven, int T, int n_a, int Pp, int phase_start,
                                       double wl, double invK, double Kc, double amax, int lane) {
    __syncwarp();  // the A table, written by every lane
    amax = warp_max_d(amax);
    const double aw = fabs(wl);
    const bool ok = aw <= 0.99 && amax <= DBL_MAX && invK != 0.0 && Kc > 0.0 && Kc <= DBL_MAX;
    const double inv = ok ? __ddiv_ru(1.0, __dsub_rd(1.0, aw)) : 1.0;  // >= 1/(1 - |w_lag|)
    const double marg = __dmul_ru(__dmul_ru(0x1p-51, amax), __dmul_ru(inv, inv));
    const double cs = __dmul_rn(1.0 / (double)Pp, invK);  // the key's scale c
    int g = Pp, t = T;  // period starts are phase_start + j P (mod T): one class mod gcd(P, T)
    while (t) {
        const int r = g % t;
        g = t;
        t = r;
    }
    const int nph = T / g;
    double h = 0.0;  // lane 0: h = sum_k w^k, accumulated beside its first horizon
    bool full = true;  // every phase's start-value range is [0, inf)
    for (int j = lane; j < nph; j += 32) {
        int p = (int)(((int64_t)phase_start + (int64_t)j * g) % T);
        const int phi = p;
        double x = 0.0, sum = 0.0, wk = 1.0, lo = 0.0, hi = INFINITY, hs = 0.0;
#pragma unroll 1
        for (int k = 0; k < Pp; ++k) {
            x = __dadd_rn(Aeven[p], __dmul_rn(wl, x));
            sum = __dadd_rn(sum, x);
            wk = __dmul_rn(wk, wl);
            hs = __dadd_rn(hs, wk);
            if (x < marg) {  // x0 w^k must lift step k clear of the clamp (w^k: k roundings, 2^-40 covers them)
                const double need = __dsub_ru(marg, x);
                if (wk > 0.0) lo = fmax(lo, __dmul_ru(__ddiv_ru(need, wk), 1.0 + 0x1p-40));
                else if (wk < 0.0) hi = fmin(hi, __dmul_rd(__ddiv_rd(need, wk), 1.0 + 0x1p-40));  // need/wk < 0
                else lo = INFINITY;
            }
            if (++p == T) p = 0;
        }
        const float lof = __double2float_ru(lo), hif = __double2float_rd(hi);
        K2[phi] = make_double2(__dmul_rn(sum, cs), __hiloint2double(__float_as_int(hif), __float_as_int(lof)));
        full = full && lof == 0.0f && hif == INFINITY;
        if (j == 0) h = hs;
    }
    full = __all_sync(kFull, full);
    for (int j = T + lane; j < n_a; j += 32) K2[j] = K2[j % T];
    if (lane == 0) {
        double nr = CUDART_NAN, nab = -INFINITY;
        if (ok) {
            // r Kc rounded down and A_b up by 2^-20 more: the fma test's own rounding stays inside
            const double r = __ddiv_rd(30000.0, __dadd_ru(__dmul_ru(2.0, inv), (double)Pp));
            nr = -__dmul_rd(__dmul_rd(r, Kc), 1.0 - 0x1p-20);
            nab = -__dmul_ru(__dmul_ru(amax, inv), 1.0 + 0x1p-20);
        }
        K2[n_a] = make_double2(__dmul_rn(h, cs), nr);
        K2[n_a + 1] = make_double2(nab, full ? 1.0 : 0.0);  // .y = 1: every range is [0, inf) (period_lane)
    }
    __syncwarp();
}

// The closed-form table for long periods (P >= 64, the 32-period batches of
// sweep_fast_kernel<2>), built by the whole warp instead of one
// P-step chain per phase:
//   K0(phi) = sum_{i<P} A(phi+i) H_{P-i},  H_m = sum_{j<m} w^j = (1 - w^m)/(1 - w),
// lane l taking the terms i = l (mod 32), then a warp sum; h = w H_P.  Each H
// carries a relative error <= 3u/(1 - |w|) and the sums add (P + 5)u, inside
// the same kappa.  The clamp-free start values come from one
// warp-wide condition instead of each step: for w >= 0 every unclamped x_k >=
// A_min > 0 once x0 >= 0; for w < 0, x_1 >= A_min - |w| x0 and x_k >= A_min -
// |w| A_max (k >= 2), so A_min > |w| A_max and x0 < A_min/|w| suffice.
__device__ __noinline__ void cfh_setup_long(double2* K2, const double* Aeven, int T, int n_a, int Pp, int phase_start,
                                            double wl, double invK, double Kc, double amax, double amin, int lane) {
    __syncwarp();  // the A table, written by every lane
    amax = warp_max_d(amax);
    amin = -warp_max_d(-amin);
    const double aw = fabs(wl);
    bool ok = aw <= 0.99 && amax <= DBL_MAX && invK != 0.0 && Kc > 0.0 && Kc <= DBL_MAX && amin > 0.0;
    double hi = INFINITY;
    if (wl < 0.0) {
        ok = ok && amin > __dmul_ru(__dmul_ru(aw, amax), 1.0 + 0x1p-40);
        hi = __dmul_rd(__ddiv_rd(amin, aw), 1.0 - 0x1p-40);
    }
    const double inv = ok ? __ddiv_ru(1.0, __dsub_rd(1.0, aw)) : 1.0;  // >= 1/(1 - |w|)
    const double cs = __dmul_rn(1.0 / (double)Pp, invK);
    const double onew = __dsub_rn(1.0, wl);
    auto powi = [](double b, int m) {  // b^m by squaring (m >= 0)
        double r = 1.0;
        while (m > 0) {
            if (m & 1) r = __dmul_rn(r, b);
            b = __dmul_rn(b, b);
            m >>= 1;
        }
        return r;
    };
    const double w32 = powi(wl, 32);
    const float lof = 0.0f, hif = __double2float_rd(hi);
    const double bounds = __hiloint2double(__float_as_int(hif), __float_as_int(lof));
    int g = Pp, t = T;
    while (t) {
        const int r = g % t;
        g = t;
        t = r;
    }
    const int nph = T / g;
    for (int j = 0; j < nph; ++j) {  // warp-uniform loop over the needed phases
        const int phi = (int)(((int64_t)phase_start + (int64_t)j * g) % T);
        double sum = 0.0;
        if (lane < Pp) {
            // terms i = lane + 32 q, q = qmax .. 0: m = P - i grows by 32 per step
            const int qmax = (Pp - 1 - lane) / 32;
            double wm = powi(wl, Pp - lane - 32 * qmax);
            int p = (int)(((int64_t)phi + lane + 32 * qmax) % T);
            const int back = 32 % T;
#pragma unroll 1
            for (int q = qmax; q >= 0; --q) {
                const double H = __ddiv_rn(__dsub_rn(1.0, wm), onew);
                sum = __fma_rn(Aeven[p], H, sum);
                wm = __dmul_rn(wm, w32);
                p -= back;
                if (p < 0) p += T;
            }
        }
        sum = warp_sum(sum);
        if (lane == 0) K2[phi] = make_double2(__dmul_rn(sum, cs), bounds);
    }
    __syncwarp();
    for (int j = T + lane; j < n_a; j += 32) K2[j] = K2[j % T];
    if (lane == 0) {
        double nr = CUDART_NAN, nab = -INFINITY;
        if (ok) {
            const double r = __ddiv_rd(30000.0, __dadd_ru(__dmul_ru(2.0, inv), (double)Pp));
            nr = -__dmul_rd(__dmul_rd(r, Kc), 1.0 - 0x1p-20);
            nab = -__dmul_ru(__dmul_ru(amax, inv), 1.0 + 0x1p-20);
        }
        const double h = __dmul_rn(wl, __ddiv_rn(__dsub_rn(1.0, powi(wl, Pp)), onew));
        K2[n_a] = make_double2(__dmul_rn(h, cs), nr);
        K2[n_a + 1] = make_double2(nab, 0.0);
    }
    __syncwarp();
}

// The closed-form decision for a full period from start value x0 (= x0f, an
// fp32 trace value) at entry kp (K2 + phase): the envelope's line, or
// kZeroLine when x0 is outside [lo, hi], the error bound fails or the key
// falls in a band; the caller then runs the sequential horizon (and counts it
// in n_seq).
__device__ __forceinline__ uint32_t cfh_choice(const double2* kp, double hc, double nr, double nab, float x0f,
                                               double x0, const uint2* ent8, int ebase, uint32_t ZB) {
    const double2 e = *kp;
    const double y = __fma_rn(hc, x0, e.x);
    const bool in = x0f >= __int_as_float(__double2loint(e.y)) && x0f <= __int_as_float(__double2hiint(e.y));
    // branch-free: the lookup runs either way, so the lookups of neighbouring
    // periods overlap their shared-memory latencies
    const int hk = __double2hiint(y);
    const int idx = max(min((hk >> kSH) - ebase, kNBUsed - 1), 0);
    const uint32_t k = (line_addr(hk, ent8[idx], ZB) >> 8) & 0xffu;
    return (in && __fma_rn(nr, y, x0) <= nab) ? k : (uint32_t)kZeroLine;
}

// The same decision as its line's shared address (the fused replay loads the
// line from it directly; the choice byte is its byte 1), ZB on decline.
// RANGE = false: every phase's range is [0, inf) (cfh_setup's flag), which every
// valid value is in; a chunk with an invalid value makes its trace status 4, whose
// choices and totals are replaced (Q25), so its decisions need no range test.
template <bool RANGE = true>
__device__ __forceinline__ uint32_t cfh_line(const double2* kp, double hc, double nr, double nab, float x0f, double x0,
                                             const uint2* ent8, int ebase, uint32_t ZB) {
    const double2 e = RANGE ? *kp : make_double2(kp->x, 0.0);
    const double y = __fma_rn(hc, x0, e.x);
    const bool in = !RANGE || (x0f >= __int_as_float(__double2loint(e.y)) && x0f <= __int_as_float(__double2hiint(e.y)));
    const int hk = __double2hiint(y);
    const int idx = max(min((hk >> kSH) - ebase, kNBUsed - 1), 0);
    const uint32_t la = line_addr(hk, ent8[idx], ZB);
    return (in && __fma_rn(nr, y, x0) <= nab) ? la : ZB;
}

__device__ __forceinline__ uint32_t line_of(int prof, uint32_t k) { return kLineBase + (uint32_t)line_off(prof, (int)k); }

// One period's decision from its horizon mean (the envelope lookup, else the canonical rule).
__device__ __forceinline__ uint32_t period_choice(double chat, double invK, double Kc, const uint2* ent8, int ebase,
                                                  uint32_t ZB, const PairTable* pt, const ProfileTable* pf,
                                                  unsigned& n_slow) {
    if (invK != 0.0) {
        const int h = __double2hiint(__dmul_rn(chat, invK));
        const int idx = max(min((h >> kSH) - ebase, kNBUsed - 1), 0);
        const uint32_t k = (line_addr(h, ent8[idx], ZB) >> 8) & 0xffu;
        if (k != (uint32_t)kZeroLine) return k;
    }
    ++n_slow;
    return canonical_choose(chat, Kc, pt->a, pf->thr, pf->K);
}

// max(pr, 0) as oracle_predict writes it (pr > 0 ? pr : 0): DSETP + two SELs
// (the compiler's fmax pattern costs twice that with its NaN fix-up)
__device__ __forceinline__ double relu_gt(double pr) {
    double f;
    asm("{\n\t.reg .pred p;\n\tsetp.gt.f64 p, %1, 0d0000000000000000;\n\t"
        "selp.f64 %0, %1, 0d0000000000000000, p;\n\t}"
        : "=d"(f) : "d"(pr));
    return f;
}

// One recursive-forecast step (Eq. 1, oracle_predict's order): prev := max(0, A + wl*prev); sum += prev
__device__ __forceinline__ void horizon_step(double A, double wl, double& prev, double& sum) {
    prev = relu_gt(__dadd_rn(A, __dmul_rn(wl, prev)));
    sum = __dadd_rn(sum, prev);
}

// M periods per lane decided side by side (periods j, j + 32, ..., j + 32(M-1)):
// M independent horizon chains interleaved step by step, so the fixed fp64
// latency of one chain is shared by M.  Chain k's phase is chain 0's plus
// k * (32 P mod T), read from the extended A table (needs T <= 64).  Every
// period here is a full one (n = P); lanes past the chunk's last period run
// masked chains and store nothing.
template <int M>
__device__ __forceinline__ void decide_multi(const float* stagev, int cs, int ce, int Pp, int j, int ph, int dph,
                                             int T, const double* Aeven, double wl, double invP, double invK, double Kc,
                                             const uint2* ent8, int ebase, uint32_t ZB, const PairTable* pt,
                                             const ProfileTable* pf, const double2* K0, double hcf, double cnr, double cnab,
                                             uint8_t* chb, unsigned& n_slow, unsigned& n_seq) {
    double prev[M], sum[M];
    int dk[M];
    uint32_t kk[M];
    bool need = false;
#pragma unroll
    for (int k = 0; k < M; ++k) {
        const int b = (j + 32 * k) * Pp;
        const float x0f = b < ce ? stagev[b - cs - 1] : 0.0f;
        prev[k] = (double)x0f;
        sum[k] = 0.0;
        dk[k] = (k * dph) % T;
        CHASE_CHECK(ph + dk[k] < haext_len(T));
        kk[k] = cfh_choice(K0 + ph + dk[k], hcf, cnr, cnab, x0f, prev[k], ent8, ebase, ZB);
        const bool nd = b < ce && kk[k] == (uint32_t)kZeroLine;
        n_seq += nd ? 1u : 0u;
        need |= nd;
    }
    int p = ph, s = 0;
    while (need && s < Pp) {
        const int seg = min(Pp - s, T - p);
        const double* Ap = Aeven + p;
#pragma unroll 1
        for (int q = 0; q < seg; ++q) {
#pragma unroll
            for (int k = 0; k < M; ++k) horizon_step(Ap[q + dk[k]], wl, prev[k], sum[k]);
        }
        s += seg;
        p += seg;
        if (p >= T) p -= T;
    }
    const bool pow2 = (Pp & (Pp - 1)) == 0;
#pragma unroll
    for (int k = 0; k < M; ++k) {
        const int b = (j + 32 * k) * Pp;
        if (b < ce) {
            if (kk[k] == (uint32_t)kZeroLine) {
                const double chat = pow2 ? __dmul_rn(sum[k], 1.0 / (double)Pp) : __ddiv_rn(sum[k], (double)Pp);
                kk[k] = period_choice(chat, invK, Kc, ent8, ebase, ZB, pt, pf, n_slow);
            }
            fill_bytes(chb, b - cs, min(b + Pp, ce) - cs, kk[k]);
        }
    }
}

__device__ __noinline__ void period_decisions(const float* stagev, int cs, int wc, int Wt, int Pp, int phase_start,
                                              int T, const double* Aeven, double wl, double invK, double Kc,
                                              const uint2* ent8, int ebase, uint32_t ZB, const PairTable* pt,
                                              const ProfileTable* pf, const double2* K0, double hcf, double cnr, double cnab,
                                              uint32_t k_carry, uint8_t* chb, int lane, unsigned& n_slow,
                                              unsigned& n_seq) {
    const int ce = cs + wc;
    const int jf = (cs + Pp - 1) / Pp;
    const int bf = min(jf * Pp, ce);
    if (lane == 0) fill_bytes(chb, 0, bf - cs, k_carry);
    {   // 33..128 full periods start in the chunk: 2-4 side-by-side chains per lane
        const int jl = (ce - 1) / Pp;
        const int m = (jl - jf + 32) / 32;
        if (T <= 64 && Pp >= 8 && m >= 2 && m <= 4 && (int64_t)jl * Pp + Pp <= Wt) {
            const int ph0 = (phase_start + (jf + lane) * Pp) % T, dph = (32 * Pp) % T;
            const int j = jf + lane;
            const double iP = 1.0 / (double)Pp;
#define CHASE_DM(M) decide_multi<M>(stagev, cs, ce, Pp, j, ph0, dph, T, Aeven, wl, iP, invK, Kc, ent8, ebase, ZB, pt, \
                                    pf, K0, hcf, cnr, cnab, chb, n_slow, n_seq)
            if (m == 2) CHASE_DM(2);
            else if (m == 3) CHASE_DM(3);
            else CHASE_DM(4);
#undef CHASE_DM
            return;
        }
    }
    // Aeven holds A[phi] for phi in [0, T + ext) (the table repeats past T): a
    // horizon runs without a wrap test for up to T + ext - phi steps
    const int tend = haext_len(T);
    const int ph_step = (32 * Pp) % T;  // phase advance between a lane's periods
    const bool pow2 = (Pp & (Pp - 1)) == 0;
    const double dP = (double)Pp, invP = 1.0 / dP;
    int ph = (phase_start + (jf + lane) * Pp) % T;
    for (int j = jf + lane; j * Pp < ce; j += 32) {
        const int b = j * Pp;
        const int n = min(Pp, Wt - b);
        const float x0f = stagev[b - cs - 1];
        double prev = (double)x0f, sum = 0.0;
        uint32_t kk = n == Pp ? cfh_choice(K0 + ph, hcf, cnr, cnab, x0f, prev, ent8, ebase, ZB)
                              : (uint32_t)kZeroLine;
        int p = ph, k = 0;
        n_seq += kk == (uint32_t)kZeroLine ? 1u : 0u;
        while (kk == (uint32_t)kZeroLine && k < n) {
            const int seg = min(n - k, tend - p);
            const double* Ap = Aeven + p;
            int q = 0;
#pragma unroll 1
            for (; q + 2 <= seg; q += 2) {
                const double a0 = Ap[q], a1 = Ap[q + 1];
                horizon_step(a0, wl, prev, sum);
                horizon_step(a1, wl, prev, sum);
            }
            if (q < seg) horizon_step(Ap[q], wl, prev, sum);
            k += seg;
            p += seg;
            while (p >= T) p -= T;
        }
        // sum/n; for a power-of-two n the product with 1/n is the same exact-then-rounded value
        if (kk == (uint32_t)kZeroLine) {
            double chat;
            if (n == Pp) chat = pow2 ? __dmul_rn(sum, invP) : __ddiv_rn(sum, dP);
            else chat = (n & (n - 1)) ? __ddiv_rn(sum, (double)n) : __dmul_rn(sum, 1.0 / (double)n);
            kk = period_choice(chat, invK, Kc, ent8, ebase, ZB, pt, pf, n_slow);
        }
        const int e = min(b + Pp, ce);
        if (Pp < 8) {
            for (int qq = b; qq < e; ++qq) chb[qq - cs] = (uint8_t)kk;
        } else {
            fill_bytes(chb, b - cs, e - cs, kk);
        }
        ph += ph_step;
        if (ph >= T) ph -= T;
    }
}

// Replay of a run of m windows at one line (the period's choice): the window
// sums collapse to S += m s_k, E += m P_k, C += P_k * sum c, Cs += sum c.  The
// order of the additions changes (exact for the dyadic inputs; within
// the 1e-9 bar otherwise, as the pairwise group sums of the per-window kernel).
__device__ __forceinline__ double run_csum(const float* __restrict__ tv, int q0, int q1, float& vmin) {
    double cs = 0.0;
    int q = q0;
    for (; q < q1 && (q & 3); ++q) {
        const float raw = tv[q];
        vmin = fminf(vmin, raw);
        cs = __dadd_rn(cs, (double)raw);
    }
    // 16 values per iteration: the four LDS.128 issue together (one shared-memory
    // latency per 16 windows, not per 4) and their sums form a tree
#pragma unroll 1
    for (; q + 16 <= q1; q += 16) {
        float4 v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = *reinterpret_cast<const float4*>(tv + q + 4 * i);
        double s[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            vmin = fminf(fminf(fminf(vmin, v[i].x), v[i].y), fminf(v[i].z, v[i].w));
            s[i] = __dadd_rn(__dadd_rn((double)v[i].x, (double)v[i].y), __dadd_rn((double)v[i].z, (double)v[i].w));
        }
        cs = __dadd_rn(cs, __dadd_rn(__dadd_rn(s[0], s[1]), __dadd_rn(s[2], s[3])));
    }
#pragma unroll 1
    for (; q + 4 <= q1; q += 4) {
        const float4 v = *reinterpret_cast<const float4*>(tv + q);
        vmin = fminf(fminf(fminf(vmin, v.x), v.y), fminf(v.z, v.w));
        cs = __dadd_rn(cs, __dadd_rn(__dadd_rn((double)v.x, (double)v.y), __dadd_rn((double)v.z, (double)v.w)));
    }
    for (; q < q1; ++q) {
        const float raw = tv[q];
        vmin = fminf(vmin, raw);
        cs = __dadd_rn(cs, (double)raw);
    }
    return cs;
}

__device__ __forceinline__ void replay_run(Acc& a, double2 ln, int m, double cs) {
    const double dm = (double)m;
    a.S = __dadd_rn(a.S, __dmul_rn(dm, ln.x));
    a.E = __dadd_rn(a.E, __dmul_rn(dm, ln.y));
    a.C = __dadd_rn(a.C, __dmul_rn(ln.y, cs));
    a.Cs = __dadd_rn(a.Cs, cs);
}

// Lane-local decision periods: when P divides the lane's share of a full chunk
// (kHChunk), every period of the lane's windows starts and ends in them and its
// start value c[b-1] is the lane's previous value (tv[-1]: the last of the
// previous lane's windows, or the chunk's lag slot).  Each lane then decides its
// own periods and replays them in one pass: horizon (Eq. 1, recursive), mean,
// Eq. 6 lookup, one line load per period, the running sums in window order
// (the same sequence replay_groups adds them in).  PC > 0: P known at compile time.
// The same replay from values already in registers (v[0, PC), PC < 16).
template <int PC, bool STORE = true>
__device__ __forceinline__ void lane_period_replay_v(const float* v, int q, uint32_t la, uint8_t* chl, Acc& a) {
    const double2 ln = lds_line(la);
    const uint8_t kk = (uint8_t)(la >> 8);  // the choice: byte 1 of the line address
#pragma unroll
    for (int k = 0; k < PC; ++k) {
        const float raw = v[k];
        const double cw = (double)raw;
        a.vmin = fminf(a.vmin, raw);
        a.S = __dadd_rn(a.S, ln.x);
        a.E = __dadd_rn(a.E, ln.y);
        a.C = __dadd_rn(a.C, __dmul_rn(ln.y, cw));
        a.Cs = __dadd_rn(a.Cs, cw);
        if (STORE) chl[q + k] = kk;
    }
}

// The same period as one run (the run form's contract): its PC values summed in
// a pairwise tree, then S += PC s_k, E += PC P_k, C += P_k sum c, Cs += sum c.
template <int PC, bool STORE = true>
__device__ __forceinline__ void lane_period_run_v(const float* v, int q, uint32_t la, uint8_t* chl, Acc& a) {
    double t[PC];
#pragma unroll
    for (int k = 0; k < PC; ++k) {
        a.vmin = fminf(a.vmin, v[k]);
        t[k] = (double)v[k];
    }
#pragma unroll
    for (int w = 1; w < PC; w *= 2)
#pragma unroll
        for (int i = 0; i + w < PC; i += 2 * w) t[i] = __dadd_rn(t[i], t[i + w]);
    replay_run(a, lds_line(la), PC, t[0]);
    if (STORE) {
        const uint8_t kk = (uint8_t)(la >> 8);
#pragma unroll
        for (int k = 0; k < PC; ++k) chl[q + k] = kk;
    }
}

// One period's replay at the line at shared address la (windows tv[q, q + Pn)).
template <int PC>
__device__ __forceinline__ void lane_period_replay(const float* __restrict__ tv, int q, int Pn, uint32_t la,
                                                   uint8_t* chl, Acc& a) {
    if constexpr (PC > 0 && PC % 4 == 0 && PC <= 16 && CHASE_LANE_RUNS) {
        // the period as one run (S += P s_k, E += P P_k, C += P_k sum c, Cs += sum c), its
        // values as LDS.128 summed in a tree: fewer dependent adds than per-window sums
        constexpr int NV = PC > 0 ? PC / 4 : 1;
        double s4[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            const float4 f = *reinterpret_cast<const float4*>(tv + q + 4 * i);
            a.vmin = fminf(fminf(fminf(a.vmin, f.x), f.y), fminf(f.z, f.w));
            s4[i] = __dadd_rn(__dadd_rn((double)f.x, (double)f.y), __dadd_rn((double)f.z, (double)f.w));
        }
#pragma unroll
        for (int w = 1; w < NV; w *= 2)
#pragma unroll
            for (int i = 0; i + w < NV; i += 2 * w) s4[i] = __dadd_rn(s4[i], s4[i + w]);
        replay_run(a, lds_line(la), PC > 0 ? PC : 4, s4[0]);
        const uint32_t kw = ((la >> 8) & 0xffu) * 0x01010101u;
#pragma unroll
        for (int i = 0; i < NV; ++i) *reinterpret_cast<uint32_t*>(chl + q + 4 * i) = kw;
        return;
    }
    if (PC > 0 && PC % 4 == 0 && PC < 16) {  // q % 4 == 0 too: LDS.128, conflict-free at the lane stride
        float v[PC > 0 ? PC : 4];
#pragma unroll
        for (int i = 0; i < (PC > 0 ? PC : 4) / 4; ++i) {
            const float4 f = *reinterpret_cast<const float4*>(tv + q + 4 * i);
            v[4 * i] = f.x; v[4 * i + 1] = f.y; v[4 * i + 2] = f.z; v[4 * i + 3] = f.w;
        }
        lane_period_replay_v<(PC > 0 ? PC : 4)>(v, q, la, chl, a);
        return;
    }
    const double2 ln = lds_line(la);
    const uint32_t kk = (la >> 8) & 0xffu;
    if (Pn < 16) {  // short runs: per-window sums (independent adds; the run form lengthens the chains)
#pragma unroll
        for (int k = 0; k < (PC > 0 ? PC : Pn); ++k) {
            const float raw = tv[q + k];
            const double cw = (double)raw;
            a.vmin = fminf(a.vmin, raw);
            a.S = __dadd_rn(a.S, ln.x);
            a.E = __dadd_rn(a.E, ln.y);
            a.C = __dadd_rn(a.C, __dmul_rn(ln.y, cw));
            a.Cs = __dadd_rn(a.Cs, cw);
            chl[q + k] = (uint8_t)kk;
        }
    } else {
        replay_run(a, ln, Pn, run_csum(tv, q, q + Pn, a.vmin));
        fill_bytes(chl, q, q + Pn, kk);
    }
}

// G consecutive periods of PN windows from tv[q] (q % 4 == 0, G*PN % 4 == 0): the
// G*PN values as LDS.128, G independent horizon chains interleaved, then the G
// replays in window order.  Returns the last value (the next group's start value).
template <int PN, int G, bool RANGE = true>
__device__ __forceinline__ float period_group(const float* __restrict__ tv, int q, float carry,
                                              const double* __restrict__ Ap, double wl, bool pow2, double dP,
                                              double invP, double invK, double Kc, const uint2* ent8, int ebase,
                                              uint32_t ZB, const PairTable* pt, const ProfileTable* pf, int prof,
                                              const double2* kq, double hcf, double cnr, double cnab, uint8_t* chl, Acc& a,
                                              unsigned& n_slow, unsigned& n_seq) {
    static_assert((G * PN) % 4 == 0, "group must be whole float4s");
    float v[G * PN];
#pragma unroll
    for (int i = 0; i < G * PN / 4; ++i) {
        const float4 f = *reinterpret_cast<const float4*>(tv + q + 4 * i);
        v[4 * i] = f.x; v[4 * i + 1] = f.y; v[4 * i + 2] = f.z; v[4 * i + 3] = f.w;
    }
    double pr[G], sm[G];
    float x0f[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        x0f[g] = g == 0 ? carry : v[g * PN - 1];
        pr[g] = (double)x0f[g];
        sm[g] = 0.0;
    }
    // (CHASE_P2_CF = 0: P = 2 keeps its two sequential steps)
    constexpr bool kCF = PN > 2 || CHASE_P2_CF;
    uint32_t la[G];  // the periods' line addresses (ZB: not decided yet)
    bool need = !kCF;
#pragma unroll
    for (int g = 0; g < G; ++g) {
        la[g] = kCF ? cfh_line<RANGE>(kq + q + g * PN, hcf, cnr, cnab, x0f[g], pr[g], ent8, ebase, ZB) : ZB;
        need |= la[g] == ZB;
    }
    // Deferred: the group replays first, a declined period on the zero line (no S, E,
    // C; its sum of c counts), and the cold block below adds its line's run afterwards
    // (S += PN s_k, E += PN P_k, C += P_k sum c) and rewrites its choice bytes.
    constexpr bool kDefer = CHASE_P_DEFER && kCF && CHASE_P_WORDS && CHASE_LANE_RUNS >= 2 && PN > CHASE_RUN_MIN_P - 1;
    if (!kDefer && need) {  // cold: the sequential horizon (Eq. 1) for the periods the closed form left
#pragma unroll
        for (int k = 0; k < PN; ++k)
#pragma unroll
            for (int g = 0; g < G; ++g) horizon_step(Ap[q + g * PN + k], wl, pr[g], sm[g]);
#pragma unroll
        for (int g = 0; g < G; ++g) {
            if (la[g] == ZB) {
                if (kCF) ++n_seq;
                const double ch = pow2 ? __dmul_rn(sm[g], invP) : __ddiv_rn(sm[g], dP);
                la[g] = line_of(prof, period_choice(ch, invK, Kc, ent8, ebase, ZB, pt, pf, n_slow));
            }
        }
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
        if constexpr (CHASE_LANE_RUNS >= 2 && PN > CHASE_RUN_MIN_P - 1)
            lane_period_run_v<PN, !CHASE_P_WORDS>(v + g * PN, q + g * PN, la[g], chl, a);
        else
            lane_period_replay_v<PN, !CHASE_P_WORDS>(v + g * PN, q + g * PN, la[g], chl, a);
    }
#if CHASE_P_WORDS
    // the group's choice bytes as 4-byte words (q % 4 == 0, chl 4-B aligned): byte 1 of
    // each period's line address; a word spans at most two periods (PN even)
#pragma unroll
    for (int w = 0; w < G * PN / 4; ++w) {
        const int pa = 4 * w / PN, pb = (4 * w + 3) / PN;
        uint32_t sel = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) sel |= (uint32_t)(((4 * w + i) / PN == pa) ? 1 : 5) << (4 * i);
        *reinterpret_cast<uint32_t*>(chl + q + 4 * w) = __byte_perm(la[pa], la[pb], sel);
    }
#endif
    if (kDefer && need) {  // cold: the declined periods' horizons, choices and runs
#pragma unroll
        for (int k = 0; k < PN; ++k)
#pragma unroll
            for (int g = 0; g < G; ++g) horizon_step(Ap[q + g * PN + k], wl, pr[g], sm[g]);
#pragma unroll
        for (int g = 0; g < G; ++g) {
            if (la[g] == ZB) {
                ++n_seq;
                const double ch = pow2 ? __dmul_rn(sm[g], invP) : __ddiv_rn(sm[g], dP);
                const uint32_t kk = period_choice(ch, invK, Kc, ent8, ebase, ZB, pt, pf, n_slow);
                double t[PN];
#pragma unroll
                for (int k = 0; k < PN; ++k) t[k] = (double)v[g * PN + k];
#pragma unroll
                for (int w = 1; w < PN; w *= 2)
#pragma unroll
                    for (int i = 0; i + w < PN; i += 2 * w) t[i] = __dadd_rn(t[i], t[i + w]);
                const double2 ln = lds_line(line_of(prof, kk));
                a.S = __dadd_rn(a.S, __dmul_rn((double)PN, ln.x));
                a.E = __dadd_rn(a.E, __dmul_rn((double)PN, ln.y));
                a.C = __dadd_rn(a.C, __dmul_rn(ln.y, t[0]));
#pragma unroll
                for (int k = 0; k < PN; ++k) chl[q + g * PN + k] = (uint8_t)kk;
            }
        }
    }
    return v[G * PN - 1];
}

template <int PC>
__device__ __forceinline__ void period_lane(const float* __restrict__ tv, int Pp, const double* __restrict__ Ap,
                                            double wl, double invK, double Kc, const uint2* ent8, int ebase,
                                            uint32_t ZB, const PairTable* pt, const ProfileTable* pf, int prof,
                                            const double2* kq, double hcf, double cnr, double cnab, uint8_t* chl, Acc& a,
                                            unsigned& n_slow, unsigned& n_seq, bool full = false) {
    const int Pn = PC > 0 ? PC : Pp;
    const bool pow2 = (Pn & (Pn - 1)) == 0;
    const double dP = (double)Pn, invP = 1.0 / dP;
    if (PC > 0 && PC % 2 == 0 && PC <= 6 && (kHChunk / (PC > 0 ? PC : 1)) % 2 == 0) {
        // even P: the 2P values of an iteration start 16-B aligned (tv is, and 2P % 4 == 0),
        // so they come in as LDS.128 (conflict-free at the 240-B lane stride; scalar loads
        // at that stride are 4-way bank conflicts) and the start values ride in registers.
        constexpr int PN = (PC > 0 && PC % 2 == 0) ? PC : 2;  // (odd PC never takes this branch)
        float carry = tv[-1];
        // (four periods per iteration at P = 2 measured slower: 17.7 -> 18.4 ms at C5, register spills)
        constexpr int GP = PN == 2 ? CHASE_P2_G : 2;  // periods per iteration
#if CHASE_P_FULL
        if (PN == 2 && full) {  // every start-value range is [0, inf): no range test per period (P = 6: slower)
#pragma unroll 1
            for (int q = 0; q < kHChunk; q += GP * PN)
                carry = period_group<PN, GP, false>(tv, q, carry, Ap, wl, pow2, dP, invP, invK, Kc, ent8, ebase, ZB, pt,
                                                    pf, prof, kq, hcf, cnr, cnab, chl, a, n_slow, n_seq);
            return;
        }
#endif
#pragma unroll 1
        for (int q = 0; q < kHChunk; q += GP * PN)
            carry = period_group<PN, GP>(tv, q, carry, Ap, wl, pow2, dP, invP, invK, Kc, ent8, ebase, ZB, pt, pf, prof,
                                         kq, hcf, cnr, cnab, chl, a, n_slow, n_seq);
        return;
    }
    if (PC > 0 && (kHChunk / (PC > 0 ? PC : 1)) % 2 == 0) {
        // two periods per iteration: their horizons are independent chains, interleaved
        // (odd P <= 5: the 2P values come in as LDS.64 pairs, 8-B aligned since 2P | q,
        // two-way bank conflicts at the 240-B lane stride instead of the scalar loads'
        // four-way; the start values ride in registers)
        constexpr int PR2 = PC > 0 ? PC : 1;
        constexpr bool kLd2 = CHASE_P_LD2 && PC > 0 && PC % 2 == 1 && PC <= CHASE_P_LD2_MAXP;
        float carry2 = tv[-1];
#pragma unroll 1
        for (int q = 0; q < kHChunk; q += 2 * Pn) {
            float w2[2 * PR2];
            if constexpr (kLd2) {
#pragma unroll
                for (int i = 0; i < PR2; ++i) {
                    const float2 f = *reinterpret_cast<const float2*>(tv + q + 2 * i);
                    w2[2 * i] = f.x;
                    w2[2 * i + 1] = f.y;
                }
            }
            const float fa = kLd2 ? carry2 : tv[q - 1], fb = kLd2 ? w2[PR2 - 1] : tv[q + Pn - 1];
            if constexpr (kLd2) carry2 = w2[2 * PR2 - 1];
            double pa = (double)fa, pb = (double)fb, sa = 0.0, sb = 0.0;
            uint32_t ka = cfh_line(kq + q, hcf, cnr, cnab, fa, pa, ent8, ebase, ZB);
            uint32_t kb = cfh_line(kq + q + Pn, hcf, cnr, cnab, fb, pb, ent8, ebase, ZB);
            // deferred (period_group's contract): both runs replay first, a declined one on
            // the zero line, and the cold block adds its line's run afterwards
            constexpr bool kDefer = CHASE_P_DEFER && CHASE_LANE_RUNS >= 2 && PC > CHASE_RUN_MIN_P - 1 && PC % 4 != 0;
            if constexpr (kDefer) {
                constexpr int PR = PC > 0 ? PC : 1;
                float va[PR], vb[PR];
#pragma unroll
                for (int k = 0; k < PR; ++k) {
                    va[k] = kLd2 ? w2[k] : tv[q + k];
                    vb[k] = kLd2 ? w2[PR + k] : tv[q + Pn + k];
                }
                lane_period_run_v<PR>(va, q, ka, chl, a);
                lane_period_run_v<PR>(vb, q + Pn, kb, chl, a);
                if (ka == ZB || kb == ZB) {  // cold: sequential horizons, then the declined runs
#pragma unroll
                    for (int k = 0; k < PR; ++k) {
                        horizon_step(Ap[q + k], wl, pa, sa);
                        horizon_step(Ap[q + Pn + k], wl, pb, sb);
                    }
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if ((h ? kb : ka) != ZB) continue;
                        ++n_seq;
                        const double sh = h ? sb : sa;
                        const double ch = pow2 ? __dmul_rn(sh, invP) : __ddiv_rn(sh, dP);
                        const uint32_t kk = period_choice(ch, invK, Kc, ent8, ebase, ZB, pt, pf, n_slow);
                        double t[PR];
#pragma unroll
                        for (int k = 0; k < PR; ++k) t[k] = (double)(h ? vb[k] : va[k]);
#pragma unroll
                        for (int w = 1; w < PR; w *= 2)
#pragma unroll
                            for (int i = 0; i + w < PR; i += 2 * w) t[i] = __dadd_rn(t[i], t[i + w]);
                        const double2 ln = lds_line(line_of(prof, kk));
                        a.S = __dadd_rn(a.S, __dmul_rn((double)PR, ln.x));
                        a.E = __dadd_rn(a.E, __dmul_rn((double)PR, ln.y));
                        a.C = __dadd_rn(a.C, __dmul_rn(ln.y, t[0]));
                        fill_bytes(chl, q + h * Pn, q + h * Pn + PR, kk);
                    }
                }
                continue;
            }
            n_seq += (ka == ZB ? 1u : 0u) + (kb == ZB ? 1u : 0u);
            if (ka == ZB || kb == ZB) {  // cold: sequential horizons
#pragma unroll
                for (int k = 0; k < (PC > 0 ? PC : 1); ++k) {
                    horizon_step(Ap[q + k], wl, pa, sa);
                    horizon_step(Ap[q + Pn + k], wl, pb, sb);
                }
                const double ca = pow2 ? __dmul_rn(sa, invP) : __ddiv_rn(sa, dP);
                const double cb = pow2 ? __dmul_rn(sb, invP) : __ddiv_rn(sb, dP);
                if (ka == ZB) ka = line_of(prof, period_choice(ca, invK, Kc, ent8, ebase, ZB, pt, pf, n_slow));
                if (kb == ZB) kb = line_of(prof, period_choice(cb, invK, Kc, ent8, ebase, ZB, pt, pf, n_slow));
            }
            if constexpr (CHASE_LANE_RUNS >= 2 && PC > CHASE_RUN_MIN_P - 1 && PC % 4 != 0) {
                float va[PC > 0 ? PC : 1], vb[PC > 0 ? PC : 1];
#pragma unroll
                for (int k = 0; k < (PC > 0 ? PC : 1); ++k) {
                    va[k] = tv[q + k];
                    vb[k] = tv[q + Pn + k];
                }
                lane_period_run_v<(PC > 0 ? PC : 1)>(va, q, ka, chl, a);
                lane_period_run_v<(PC > 0 ? PC : 1)>(vb, q + Pn, kb, chl, a);
            } else {
                lane_period_replay<PC>(tv, q, Pn, ka, chl, a);
                lane_period_replay<PC>(tv, q + Pn, Pn, kb, chl, a);
            }
        }
        return;
    }
#pragma unroll 1
    for (int q = 0; q < kHChunk; q += Pn) {
        const float x0f = tv[q - 1];
        double prev = (double)x0f, sum = 0.0;
        uint32_t la = cfh_line(kq + q, hcf, cnr, cnab, x0f, prev, ent8, ebase, ZB);
        // deferred (period_group's contract) for the LDS.128 run form: replay first, a
        // declined period on the zero line, its line's run added in the cold block
        constexpr bool kDefer = CHASE_P_DEFER && PC > 0 && PC % 4 == 0 && PC <= 16 && CHASE_LANE_RUNS;
        if (kDefer) lane_period_replay<PC>(tv, q, Pn, la, chl, a);
        if (la == ZB) {  // cold: the sequential horizon
            ++n_seq;
#pragma unroll
            for (int k = 0; k < Pn; ++k) horizon_step(Ap[q + k], wl, prev, sum);
            const double chat = pow2 ? __dmul_rn(sum, invP) : __ddiv_rn(sum, dP);
            const uint32_t kk = period_choice(chat, invK, Kc, ent8, ebase, ZB, pt, pf, n_slow);
            la = line_of(prof, kk);
            if constexpr (kDefer) {
                constexpr int NV = PC >= 4 ? PC / 4 : 1;
                double s4[NV];  // the run's sum of c, as lane_period_replay forms it
#pragma unroll
                for (int i = 0; i < NV; ++i) {
                    const float4 f = *reinterpret_cast<const float4*>(tv + q + 4 * i);
                    s4[i] = __dadd_rn(__dadd_rn((double)f.x, (double)f.y), __dadd_rn((double)f.z, (double)f.w));
                }
#pragma unroll
                for (int w = 1; w < NV; w *= 2)
#pragma unroll
                    for (int i = 0; i + w < NV; i += 2 * w) s4[i] = __dadd_rn(s4[i], s4[i + w]);
                const double2 ln = lds_line(la);
                a.S = __dadd_rn(a.S, __dmul_rn((double)(PC > 0 ? PC : 4), ln.x));
                a.E = __dadd_rn(a.E, __dmul_rn((double)(PC > 0 ? PC : 4), ln.y));
                a.C = __dadd_rn(a.C, __dmul_rn(ln.y, s4[0]));
                fill_bytes(chl, q, q + Pn, kk);
            }
        }
        if (!kDefer) lane_period_replay<PC>(tv, q, Pn, la, chl, a);
    }
}

// Sequential horizon (Eq. 1, oracle_predict's order) of n steps from phase ph
// and start value prev, reading the extended A table with wrap: the sum.
__device__ __forceinline__ double horizon_sum(const double* Aeven, int T, int ph, int n, double prev, double wl) {
    const int tend = haext_len(T);
    double sum = 0.0;
    int p = ph, k = 0;
    while (k < n) {
        const int seg = min(n - k, tend - p);
        const double* Ap = Aeven + p;
        int q = 0;
#pragma unroll 1
        for (; q + 2 <= seg; q += 2) {
            const double a0 = Ap[q], a1 = Ap[q + 1];
            horizon_step(a0, wl, prev, sum);
            horizon_step(a1, wl, prev, sum);
        }
        if (q < seg) horizon_step(Ap[q], wl, prev, sum);
        k += seg;
        p += seg;
        while (p >= T) p -= T;
    }
    return sum;
}

// Lane-direct decision periods (2 < P < 64 with the closed form):
// each lane decides every period that meets its own windows [w0, w0 + nwin)
// and replays them in the same pass, with no staged decisions and no warp
// barrier between the two.  A period needs only its start value c[b-1] (in the
// stage: tvs[b - cs - 1], the lag slot for b = cs) and its phase, so a period
// split between two lanes is decided by both (the same arithmetic; the lane
// holding its start counts it in n_slow / n_seq); one that began in an earlier
// chunk takes k_carry.  The closed form decides, else the sequential horizon.
template <int PC>
__device__ __forceinline__ void period_direct(const float* __restrict__ tvs, const float* __restrict__ tv, int nwin,
                                           int w0, int cs, int Wt, int Pr, int phi0, int T, const double* Aeven,
                                           double wl, double invK, double Kc, const uint2* ent8, int ebase,
                                           uint32_t ZB, const PairTable* pt, const ProfileTable* pf,
                                           const double2* K2, double hcf, double cnr, double cnab, uint32_t k_carry,
                                           int prof, uint8_t* chl, Acc& a, unsigned& n_slow, unsigned& n_seq) {
    if (nwin <= 0) return;
    const int Pp = PC > 0 ? PC : Pr;  // (PC > 0: P fixed at compile time)
    int b = (w0 / Pp) * Pp;
    int ph = (phi0 - (w0 - b)) % T;  // phase of b (w0 - b < P)
    if (ph < 0) ph += T;
    int q = 0;
    while (q < nwin) {
        CHASE_CHECK(ph >= 0 && ph < T);
        uint32_t kk = k_carry;
        if (b >= cs) {
            const int n = min(Pp, Wt - b);
            CHASE_CHECK(b - cs < kHWarpW);
            const float x0f = tvs[b - cs - 1];
            const double x0 = (double)x0f;
            kk = n == Pp ? cfh_choice(K2 + ph, hcf, cnr, cnab, x0f, x0, ent8, ebase, ZB)
                         : (uint32_t)kZeroLine;
            if (kk == (uint32_t)kZeroLine) {  // cold: the sequential horizon, then the lookup / canonical rule
                const bool own = b >= w0;
                if (own && n == Pp) ++n_seq;
                const double sum = horizon_sum(Aeven, T, ph, n, x0, wl);
                const double chat = (n & (n - 1)) ? __ddiv_rn(sum, (double)n) : __dmul_rn(sum, 1.0 / (double)n);
                unsigned ns = 0;
                kk = period_choice(chat, invK, Kc, ent8, ebase, ZB, pt, pf, ns);
                if (own) n_slow += ns;
            }
        }
        const int e = min(nwin, b + Pp - w0);
        if (Pp >= 16) {  // the run form for every piece (float4 sums once aligned; short pieces too)
            const double2 ln = lds_line(line_of(prof, kk));
            replay_run(a, ln, e - q, run_csum(tv, q, e, a.vmin));
            fill_bytes(chl, q, e, kk);
        } else {
            lane_period_replay<0>(tv, q, e - q, line_of(prof, kk), chl, a);
        }
        q = e;
        b += Pp;
        ph += Pp;
        while (ph >= T) ph -= T;
    }
}

// Daily periods (P = 24, PM 26) in a full chunk: a lane's 60 windows are five
// 12-window blocks, and with 1920 = 80 P and 60 = 2.5 P every period boundary
// is a block boundary (even lanes start on one, odd lanes 12 windows past one).
// The lane decides the three periods meeting its blocks (the first of an odd
// lane began in the previous lane's windows: decided by both, counted by the
// one holding its start) and replays each block as one run: S += 12 s_k,
// E += 12 P_k, C += P_k sum c, Cs += sum c (the run form's contract).
__device__ __forceinline__ uint32_t day_decide(const float* __restrict__ tv, int s, int b, int Wt, int ph, int T,
                                               const double* Aeven, double wl, double invK, double Kc,
                                               const uint2* ent8, int ebase, uint32_t ZB, const PairTable* pt,
                                               const ProfileTable* pf, const double2* K2, double hcf, double cnr,
                                               double cnab, int prof, bool own, unsigned& n_slow, unsigned& n_seq) {
    constexpr int Pp = 24;
    const int n = min(Pp, Wt - b);
    const float x0f = tv[s - 1];
    const double x0 = (double)x0f;
    uint32_t la = n == Pp ? cfh_line(K2 + ph, hcf, cnr, cnab, x0f, x0, ent8, ebase, ZB) : ZB;
    if (la == ZB) {  // cold: the sequential horizon, then the lookup / canonical rule
        if (own && n == Pp) ++n_seq;
        const double sum = horizon_sum(Aeven, T, ph, n, x0, wl);
        const double chat = (n & (n - 1)) ? __ddiv_rn(sum, (double)n) : __dmul_rn(sum, 1.0 / (double)n);
        unsigned ns = 0;
        la = line_of(prof, period_choice(chat, invK, Kc, ent8, ebase, ZB, pt, pf, ns));
        if (own) n_slow += ns;
    }
    return la;
}

__device__ __forceinline__ void day_block(const float* __restrict__ tv, int q, uint32_t la, uint8_t* chl, Acc& a) {
    float4 v[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) v[i] = *reinterpret_cast<const float4*>(tv + q + 4 * i);
    double s4[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        a.vmin = fminf(fminf(fminf(a.vmin, v[i].x), v[i].y), fminf(v[i].z, v[i].w));
        s4[i] = __dadd_rn(__dadd_rn((double)v[i].x, (double)v[i].y), __dadd_rn((double)v[i].z, (double)v[i].w));
    }
    const double cs = __dadd_rn(__dadd_rn(s4[0], s4[1]), s4[2]);
    replay_run(a, lds_line(la), 12, cs);
    const uint32_t kb = (la >> 8) & 0xffu;
    const uint32_t kw = kb * 0x01010101u;
#pragma unroll
    for (int i = 0; i < 3; ++i) *reinterpret_cast<uint32_t*>(chl + q + 4 * i) = kw;
}

static_assert(!CHASE_DAY_BLOCKS || (kHChunk == 60 && kHWarpW % 24 == 0), "period_day: five 12-window blocks per 60-window lane");
__device__ __forceinline__ void period_day(const float* __restrict__ tv, int w0, int Wt, int phi0, int T,
                                           const double* Aeven, double wl, double invK, double Kc, const uint2* ent8,
                                           int ebase, uint32_t ZB, const PairTable* pt, const ProfileTable* pf,
                                           const double2* K2, double hcf, double cnr, double cnab, int prof,
                                           uint8_t* chl, Acc& a, unsigned& n_slow, unsigned& n_seq) {
    const int odd = (w0 % 24) != 0;       // 12 windows past a period start
    const int sA = odd ? -12 : 0;         // the three periods' starts relative to the lane's first window
    int ph = phi0 + sA;
    if (ph < 0) ph += T;
    const uint32_t lA = day_decide(tv, sA, w0 + sA, Wt, ph, T, Aeven, wl, invK, Kc, ent8, ebase, ZB, pt, pf, K2,
                                   hcf, cnr, cnab, prof, !odd, n_slow, n_seq);
    ph = (ph + 24) % T;
    const uint32_t lB = day_decide(tv, sA + 24, w0 + sA + 24, Wt, ph, T, Aeven, wl, invK, Kc, ent8, ebase, ZB, pt, pf,
                                   K2, hcf, cnr, cnab, prof, true, n_slow, n_seq);
    ph = (ph + 24) % T;
    const uint32_t lC = day_decide(tv, sA + 48, w0 + sA + 48, Wt, ph, T, Aeven, wl, invK, Kc, ent8, ebase, ZB, pt, pf,
                                   K2, hcf, cnr, cnab, prof, true, n_slow, n_seq);
    // blocks 0..4: even lanes A A B B C, odd lanes A B B C C
    day_block(tv, 0, lA, chl, a);
    day_block(tv, 12, odd ? lB : lA, chl, a);
    day_block(tv, 24, lB, chl, a);
    day_block(tv, 36, odd ? lC : lB, chl, a);
    day_block(tv, 48, lC, chl, a);
}

// Long decision periods (P >= kHWarpW/30: at most 31 periods meet a chunk):
// the decisions are taken 32 periods at a time, one per lane, and kept in a
// register (lane l holds period jb + l).  A period's start value c[b-1] is read
// from global memory (one 4-byte load per period), so a batch spans chunks and
// every lane has a horizon to run (P = 168: 2 batches per year-long trace, not
// one 12-lane round per chunk).  Same per-period arithmetic as period_decisions.
template <bool CF>
__device__ __noinline__ uint32_t period_batch(const float* __restrict__ cg, int jb, int Wt, int Pp, int phase_start,
                                              int T, const double* Aeven, double wl, double invK, double Kc,
                                              const uint2* ent8, int ebase, uint32_t ZB, const PairTable* pt,
                                              const ProfileTable* pf, const double2* K0, double hcf, double cnr, double cnab,
                                              int lane, unsigned& n_slow, unsigned& n_seq) {
    const int b = (jb + lane) * Pp;
    if (b >= Wt) return 0u;
    const int n = min(Pp, Wt - b);
    const int tend = haext_len(T);
    const float x0f = __ldg(cg + b - 1);  // c[b-1]
    double prev = (double)x0f, sum = 0.0;
    int p = (int)(((int64_t)phase_start + b) % T), k = 0;
    if (CF && n == Pp) {
        const uint32_t kk = cfh_choice(K0 + p, hcf, cnr, cnab, x0f, prev, ent8, ebase, ZB);
        if (kk != (uint32_t)kZeroLine) return kk;
    }
    if (CF && n == Pp) ++n_seq;
    while (k < n) {
        const int seg = min(n - k, tend - p);
        const double* Ap = Aeven + p;
        int q = 0;
#pragma unroll 1
        for (; q + 2 <= seg; q += 2) {
            const double a0 = Ap[q], a1 = Ap[q + 1];
            horizon_step(a0, wl, prev, sum);
            horizon_step(a1, wl, prev, sum);
        }
        if (q < seg) horizon_step(Ap[q], wl, prev, sum);
        k += seg;
        p += seg;
        while (p >= T) p -= T;
    }
    const double chat = (n & (n - 1)) ? __ddiv_rn(sum, (double)n) : __dmul_rn(sum, 1.0 / (double)n);
    return period_choice(chat, invK, Kc, ent8, ebase, ZB, pt, pf, n_slow);
}

// Replay of one lane's windows [w0, w0 + nwin) from the batch decisions (lane l: period jb + l).
__device__ __forceinline__ void period_replay_batch(const float* __restrict__ tv, int nwin, int w0, int Pp, int jb,
                                                    uint32_t kb, int prof, uint8_t* chl, Acc& a) {
    int q = 0;
    const int jA = w0 / Pp;
    // a lane's windows meet at most two periods (P >= kHWarpW/30 > kHChunk); the
    // shuffles are warp-wide, so every lane fetches both
    const uint32_t k0 = __shfl_sync(kFull, kb, min(jA - jb, 31));
    const uint32_t k1 = __shfl_sync(kFull, kb, min(jA + 1 - jb, 31));
    const int split = min(nwin, max(0, (jA + 1) * Pp - w0));
    if (CHASE_BATCH_BLOCKS && nwin == kHChunk && (split & 3) == 0) {
        // a full lane, the period boundary on a 4-window block: 15 LDS.128 blocks summed
        // in trees into the two runs' value sums, one choice word per block
        double c0 = 0.0, c1 = 0.0;
        const uint32_t kw0 = k0 * 0x01010101u, kw1 = k1 * 0x01010101u;
#pragma unroll
        for (int i = 0; i < kHChunk / 4; ++i) {
            const float4 f = *reinterpret_cast<const float4*>(tv + 4 * i);
            a.vmin = fminf(fminf(fminf(a.vmin, f.x), f.y), fminf(f.z, f.w));
            const double sb = __dadd_rn(__dadd_rn((double)f.x, (double)f.y), __dadd_rn((double)f.z, (double)f.w));
            const bool first = 4 * i < split;
            if (first) c0 = __dadd_rn(c0, sb);
            else c1 = __dadd_rn(c1, sb);
            *reinterpret_cast<uint32_t*>(chl + 4 * i) = first ? kw0 : kw1;
        }
        if (split > 0) replay_run(a, lds_line(kLineBase + (uint32_t)line_off(prof, (int)k0)), split, c0);
        if (split < kHChunk) replay_run(a, lds_line(kLineBase + (uint32_t)line_off(prof, (int)k1)), kHChunk - split, c1);
        return;
    }
#pragma unroll 1
    for (int seg = 0; seg < 2; ++seg) {
        const uint32_t kk = seg == 0 ? k0 : k1;
        const int e = seg == 0 ? split : nwin;
        if (e > q) {
            const double2 ln = lds_line(kLineBase + (uint32_t)line_off(prof, (int)kk));
            replay_run(a, ln, e - q, run_csum(tv, q, e, a.vmin));
            fill_bytes(chl, q, e, kk);
            q = e;
        }
    }
}

// Replay of one lane's windows from the staged choice bytes (period mode).
__device__ __forceinline__ void replay_groups(const float* __restrict__ tv, int nwin, const uint8_t* __restrict__ bytes,
                                              int prof, Acc& a) {
    const int ngr = nwin >> 2;
    const uint32_t* words = reinterpret_cast<const uint32_t*>(bytes);
#pragma unroll 1
    for (int g = 0; g < ngr; ++g) {
        const float4 v = *reinterpret_cast<const float4*>(tv + 4 * g);
        a.vmin = fminf(fminf(fminf(a.vmin, v.x), v.y), fminf(v.z, v.w));
        const uint32_t word = words[g];
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int k = (int)((word >> (8 * u)) & 0xffu);
            const double cw = (double)vv[u];
            const double2 ln = lds_line(kLineBase + (uint32_t)line_off(prof, k));
            a.S = __dadd_rn(a.S, ln.x);
            a.E = __dadd_rn(a.E, ln.y);
            a.C = __dadd_rn(a.C, __dmul_rn(ln.y, cw));
            a.Cs = __dadd_rn(a.Cs, cw);
        }
    }
    for (int jj = 4 * ngr; jj < nwin; ++jj) {
        const float raw = tv[jj];
        const double cw = (double)raw;
        const double2 ln = lds_line(kLineBase + (uint32_t)line_off(prof, bytes[jj]));
        a.S = __dadd_rn(a.S, ln.x);
        a.E = __dadd_rn(a.E, ln.y);
        a.C = __dadd_rn(a.C, __dmul_rn(ln.y, cw));
        a.Cs = __dadd_rn(a.Cs, cw);
        a.bad |= bad_value(raw) ? 1 : 0;
    }
}

// PM: 0 = one decision per window (the headline), 1 = decision periods decided per
// chunk, 2 = long periods (P >= kHWarpW/30) decided in 32-period batches, 3 =
// lane-local periods (P | kHChunk, P known at run time; the last chunk as PM 1),
// PM >= 4 = the same with P = PM - 2 fixed at compile time (P = 2, 3, 4, 5, 6,
// 10, 12, 15), or lane-direct with P fixed when P does not divide a lane's
// chunk (PM 26: P = 24, with the closed-form table).  Separate instantiations
// keep each path's registers apart: one kernel holding all the compile-time P
// spilled more (P = 12: 14.6 vs 13.6 ms).
template <int PM>
#ifdef CHASE_H_MAXNREG
__global__ void __maxnreg__(CHASE_H_MAXNREG) sweep_fast_kernel(
#else
__global__ void __launch_bounds__(kHThreads, CHASE_H_MINB) sweep_fast_kernel(
#endif
    const __grid_constant__ SweepParams P) {
    constexpr bool PER = PM != 0;
    // PM >= 4: P = PM - 2 fixed at compile time, lane-local when it divides a lane's
    // chunk, else lane-direct (period_direct<P>, e.g. P = 24)
    constexpr bool kLaneLocal = PM == 3 || (PM >= 4 && kHChunk % (PM >= 4 ? PM - 2 : 1) == 0);
    constexpr int kDirectP = (PM >= 4 && !kLaneLocal) ? PM - 2 : 0;
    mark_path(P.diag, PER ? CHASE_PATH_H_PERIODS : CHASE_PATH_HEADLINE);
    extern __shared__ __align__(128) uint8_t sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t sbase = smem_u32(sm);
    const int head_bytes = reinterpret_cast<const TablesHeader*>(P.tables)->off_pair;
    const HLayout HL = make_hlayout(P.T, head_bytes, P.n_prof, (int)sbase, P.k0len);
    if (HL.total > P.smem_total || HL.lines < 0) __trap();  // the host planned for another shared-window base
    uint2* ent8_all = reinterpret_cast<uint2*>(sm + HL.ent8);
    int* lph = reinterpret_cast<int*>(sm + HL.lph);
    uint8_t* wbase = sm + HL.warp_off(warp);
    const int alen = round16(haext_len(P.T) * 8) / 8;
    double* A_even = reinterpret_cast<double*>(wbase + HL.aext);
    double* A_odd = A_even + alen;
    uint8_t* stage0 = wbase + HL.stage;
    uint8_t* chb = wbase + HL.chb;
    uint64_t* mbar = reinterpret_cast<uint64_t*>(wbase + HL.mbar);
    const int T = P.T;
    // periods: the closed-form horizon table (else any valid address: cnr = NaN declines every period)
    double2* K0w = reinterpret_cast<double2*>(P.k0len > 0 ? wbase + HL.k0 : wbase + HL.aext);

    {   // constant tables -> smem, once per CTA: header, phase, profiles; pair heads
        const uint4* src = reinterpret_cast<const uint4*>(P.tables);
        uint4* dst = reinterpret_cast<uint4*>(sm + HL.tables);
        for (int q = tid; q < head_bytes / 16; q += kHThreads) dst[q] = src[q];
        const int hw = (int)sizeof(PairHead) / 8;
        const double* ps = reinterpret_cast<const double*>(P.tables + head_bytes);
        double* hd = reinterpret_cast<double*>(sm + HL.heads);
        for (int q = tid; q < P.n_prof * hw; q += kHThreads)
            hd[q] = ps[(q / hw) * ((int)sizeof(PairTable) / 8) + q % hw];
        if (tid < 64) lph[tid] = ((tid < 32 ? kHChunk : P.kc_last) * (tid & 31)) % T;  // per-lane phase offsets
    }
    __syncthreads();
    const TablesHeader* H = reinterpret_cast<const TablesHeader*>(sm + HL.tables);
    const double* phS = reinterpret_cast<const double*>(sm + HL.tables + H->off_phase);
    const double* phC = phS + T;
    const ProfileTable* profs = reinterpret_cast<const ProfileTable*>(sm + HL.tables + H->off_prof);
    // pair heads: only the fields before `ent` are ever read through these pointers
    const PairHead* heads = reinterpret_cast<const PairHead*>(sm + HL.heads);
    const PairTable* gpairs = reinterpret_cast<const PairTable*>(P.tables + head_bytes);  // entries: setup only
    {   // line region: profile p, line k at kLineBase + line_off(p, k) (zero line at k = 32)
        for (int q = tid; q < P.n_prof * (kMaxK + 1); q += kHThreads) {
            const int p = q / (kMaxK + 1), k = q % (kMaxK + 1);
            const double2 v = (k < profs[p].K) ? profs[p].line[k] : make_double2(0.0, 0.0);
            *reinterpret_cast<double2*>(sm + HL.lines + line_off(p, k)) = v;
        }
        // 8-byte bucket entries {T1, lo16(addr below) | lo16(addr above) << 16}
        for (int q = tid; q < P.n_prof * kNB; q += kHThreads) {
            const int p = q / kNB;
            const uint2 e = gpairs[p].ent[q % kNB];
            const uint32_t below = e.y & 0xffu;
            const uint32_t above = (e.y >> 16) ? (uint32_t)kZeroLine : ((e.y >> 8) & 0xffu);  // band > 1 unit: slow
            ent8_all[q] = make_uint2(e.x, (uint32_t)line_off(p, (int)below) | ((uint32_t)line_off(p, (int)above) << 16));
        }
    }
    if (lane == 0) {
        mbar_init(mbar, 1);
        fence_mbar_init();
    }
    __syncthreads();

    const float* traces = reinterpret_cast<const float*>(P.traces);
    const int64_t GW = (int64_t)gridDim.x * kHWarps;
    const int64_t gw = (int64_t)blockIdx.x * kHWarps + warp;
    const int nc = P.n_chunks;
    const bool store_choice = P.choice != nullptr;
    const int lph_full = lph[lane], lph_last = lph[32 + lane];
    const int lane_mod_T = lane % T;

    // One stage per warp: the load of chunk c+1 (or of the next trace's first
    // chunk, with its record) is issued once chunk c is consumed (lane 0).
    auto issue = [&](int64_t ti, int tc) {
        if (ti >= P.n_traces || lane != 0) return;
        const uint64_t policy = evict_first_policy();
        const uint32_t bytes = tc == nc - 1 ? P.bytes_last : P.bytes_full;
        if (tc == 0) {
            mbar_arrive_expect_tx(mbar, bytes + (uint32_t)kRecBytes);
            bulk_g2s(stage0 + P.stage_bytes - kRecBytes, P.records + ti * kRecDoubles, kRecBytes, mbar, policy);
        } else {
            mbar_arrive_expect_tx(mbar, bytes);
        }
        CHASE_CHECK(bytes <= (uint32_t)(P.stage_bytes - kRecBytes) && P.a0 + (int64_t)tc * kHWarpW >= 0 &&
                    P.a0 + (int64_t)tc * kHWarpW + bytes / 4 <= P.ld);
        bulk_g2s(stage0, traces + ti * P.ld + P.a0 + (int64_t)tc * kHWarpW, bytes, mbar, policy);
    };
    issue(gw, 0);

    uint32_t par = 0;    // mbarrier phase parity of the next chunk
    unsigned n_slow = 0;
    unsigned n_seq = 0;  // periods: full periods whose horizon ran sequentially (the closed form declined)

    for (int64_t i = gw; i < P.n_traces; i += GW) {
        int status = 0, c_may = 0, mb = P.W, ebase = 0;
        double wl = 0.0, J = 0.0, Kc = 0.0, invK = 0.0;
        double Sl = 0.0, El = 0.0, Cl = 0.0, Cbl = 0.0;  // per-lane running sums
        bool done = false;
        int phase_c = P.phase_start;
        uint32_t ZB = 0;
        const uint2* e8 = ent8_all;
        const ProfileTable* pf = profs;
        const PairTable* pt = reinterpret_cast<const PairTable*>(heads);
        int prof_i = 0;
        bool fast = false;     // the one-fma key (PM 0)
        double wlK = 0.0;      // fl(w_lag * fl(1/Kc)) for the one-fma key
        uint32_t clim_bits = 0u;  // fp32 bits of c_lim: values above take the exact key
        uint32_t k_carry = 0;  // period mode: the decision of the period running into the next chunk
        int jb = 0;            // long periods: first period of the current batch
        uint32_t kb = 0;       // long periods: lane l's decision for period jb + l
        double hcf = 0.0, cnr = CUDART_NAN, cnab = -INFINITY;  // periods: the closed form's h, -r, -A_b (NaN: off)
        bool cfull = false;    // periods: every closed-form start-value range is [0, inf)
        for (int c = 0; c < nc; ++c) {
            const bool last = c == nc - 1;
            uint8_t* stage = stage0;
            if (store_choice) {
                if (lane == 0) bulk_wait_read0();  // the previous store has read chb
                __syncwarp();                      // ... before any lane writes it again
            }
            if (PM == 2 && c > 0 && status == 0) {
                // long periods: a new batch is decided while this chunk's load is in flight
                const int cs = c * kHWarpW, wc = last ? P.W_last : kHWarpW;
                if ((cs + wc - 1) / P.period >= jb + 32) {
                    const int jn = cs / P.period;
                    unsigned ns = 0, nq = 0;
                    kb = period_batch<CHASE_LONG_CF>(traces + i * P.ld + P.a0 + P.off0, jn, P.W, P.period, P.phase_start, T, A_even,
                                      wl, invK, Kc, e8, ebase, ZB, pt, pf, K0w, hcf, cnr, cnab, lane, ns, nq);
                    if (jn + lane > jb + 31) {  // count only periods the last batch did not decide
                        n_slow += ns;
                        n_seq += nq;
                    }
                    jb = jn;
                }
            }
            mbar_wait(mbar, par);
            if (c == 0) {  // ---- per-trace setup
                // the record: model (fit_kernel) and this trace's eta-0 scalars (record [10..15], kernels.h)
                const double* rec = reinterpret_cast<const double*>(stage + P.stage_bytes - kRecBytes);
                const int prof = (int)rec[13];
                prof_i = prof;
                pf = profs + prof;
                pt = reinterpret_cast<const PairTable*>(heads + prof);
                e8 = ent8_all + prof * kNB;
                ebase = pt->base;
                ZB = kLineBase | (uint32_t)line_off(prof, kZeroLine);
                J = rec[12];
                status = (int)rec[5];
                wl = rec[3];
                if (status == 0 && !(rec[15] > 0.0)) status = CHASE_ERR_MAXCI;
                const int m = (int)rec[8];
                mb = (J > 0.0 && m >= 1 && m <= P.W) ? m - 1 : P.W;
                Kc = rec[10];
                invK = rec[11];
                // first chunk in which S can reach J: from a lower bound on the windows needed
                // the completion window w* (from s0) has (w*+1)*max_k s_k >= J, so w* >= rec[14] - 1
                // (rec[14] = J/(1.000001 max_k s_k) absorbs the roundings): its chunk is at least c_may
                c_may = J > 0.0 ? (rec[14] >= (double)P.W ? nc - 1 : (int)(fmax(rec[14] - 1.0, 0.0) * (1.0 / kHWarpW))) : nc;
                if (status == 0) {
                    const double c0 = rec[0], wsn = rec[1], wcs = rec[2];
                    const int n_a = haext_len(T);
                    int ph = lane_mod_T;
                    double amax = 0.0, amin = DBL_MAX;
                    for (int j = lane; j < n_a; j += 32) {
                        // A(phi) = (c0 + w_sin*S[phi]) + w_cos*C[phi]  (canonical fold of Eq. 1)
                        const int ph1 = ph + 1 == T ? 0 : ph + 1;
                        A_even[j] = __dadd_rn(__dadd_rn(c0, __dmul_rn(wsn, phS[ph])), __dmul_rn(wcs, phC[ph]));
                        A_odd[j] = __dadd_rn(__dadd_rn(c0, __dmul_rn(wsn, phS[ph1])), __dmul_rn(wcs, phC[ph1]));
                        amax = fmax(amax, fabs(A_even[j]));
                        amin = fmin(amin, A_even[j]);
                        ph += 32;
                        while (ph >= T) ph -= T;
                    }
                    if constexpr (PER && (PM != 4 || CHASE_P2_CF)) {
                        if (P.k0len > 0) {
                            if constexpr (PM == 2)  // (long P: the warp-wide table)
                                cfh_setup_long(K0w, A_even, T, n_a, P.period, P.phase_start, wl, invK, Kc, amax, amin,
                                               lane);
                            else
                                cfh_setup(K0w, A_even, T, n_a, P.period, P.phase_start, wl, invK, Kc, amax, lane);
                            hcf = K0w[n_a].x;
                            cnr = K0w[n_a].y;
                            cnab = K0w[n_a + 1].x;
                            cfull = K0w[n_a + 1].y == 1.0;
                        }
                    }
                    if constexpr (PM == 0 && CHASE_H0_FAST) {
                        // the one-fma key's bound: 6u (|A| + |w_lag| c)/Kc <= 126000u y_min, i.e.
                        // |A| + |w_lag| c <= 21000 y_min Kc (envelope.cpp shrinks by 2^-36)
                        amax = warp_max_d(amax);
                        const double lam = __dmul_rd(__dmul_rd(21000.0, pt->y_min), Kc);
                        if (!pt->k0 && invK != 0.0 && amax < lam && fabs(wl) <= DBL_MAX) {
                            const double awl = fabs(wl);
                            const double cl = awl > 0.0 ? __ddiv_rd(__dsub_rd(lam, amax), awl) : (double)FLT_MAX;
                            const float clf = cl >= (double)FLT_MAX ? FLT_MAX : __double2float_rd(cl);
                            if (clf >= FLT_MIN) {
                                fast = true;
                                clim_bits = __float_as_uint(clf);
                                wlK = __dmul_rn(wl, invK);
                                for (int j = lane; j < n_a; j += 32) {  // B = fl(A * fl(1/Kc)), in place
                                    A_even[j] = __dmul_rn(A_even[j], invK);
                                    A_odd[j] = __dmul_rn(A_odd[j], invK);
                                }
                            }
                        }
                    }
                }
                __syncwarp();
            } else {
                phase_c += P.phase_step;
                if (phase_c >= T) phase_c -= T;
            }
            const int kc = last ? P.kc_last : kHChunk;
            const int j0 = kc * lane;
            const int nwin = max(0, min(kc, (last ? P.W_last : kHWarpW) - j0));
            const float* tv = reinterpret_cast<const float*>(stage) + P.off0 + j0;  // tv[jj] = c[s0 + c*kHWarpW + j0 + jj]
            CHASE_CHECK(j0 + nwin <= kHWarpW && P.off0 + j0 + nwin + 4 <= (P.stage_bytes - kRecBytes) / 4);
            int phi0 = phase_c + (last ? lph_last : lph_full);
            if (phi0 >= T) phi0 -= T;
            const double* Ap = (phi0 & 1) ? A_odd + (phi0 - 1) : A_even + phi0;

            // The next chunk's load is issued as soon as nothing reads the stage any more:
            // right after the hot loop and the two sums that may still read it (the
            // baseline's completion chunk), except in the chunk where the job completes.
            bool issued = false;
            if (status == 0) {
                Acc a{0.0, 0.0, 0.0, 0.0, FLT_MAX, 0u, 0, 0};
                const int ngr = (PER || invK == 0.0) ? 0 : nwin >> 2;
                if (kLaneLocal && !last) {  // lane-local periods (P | kHChunk): fused decide + replay
                    uint8_t* chl = chb + j0;
#define CHASE_LANE_P(PC) period_lane<PC>(tv, PC, Ap, wl, invK, Kc, e8, ebase, ZB, pt, pf, prof_i, K0w + phi0, hcf, cnr, cnab, \
                                         chl, a, n_slow, n_seq, cfull)
                    if constexpr (PM >= 4) CHASE_LANE_P(PM - 2);
                    else period_lane<0>(tv, P.period, Ap, wl, invK, Kc, e8, ebase, ZB, pt, pf, prof_i, K0w + phi0, hcf,
                                        cnr, cnab, chl, a, n_slow, n_seq);
#undef CHASE_LANE_P
                    __syncwarp();
                    k_carry = chb[kHWarpW - 1];
                } else if (PM == 2) {  // long periods: 32-period batches
                    const int cs = c * kHWarpW;
                    if (c == 0) {  // the trace's first batch needs its model (the record, in this stage)
                        jb = 0;
                        kb = period_batch<CHASE_LONG_CF>(traces + i * P.ld + P.a0 + P.off0, jb, P.W, P.period, P.phase_start, T,
                                          A_even, wl, invK, Kc, e8, ebase, ZB, pt, pf, K0w, hcf, cnr, cnab, lane, n_slow, n_seq);
                    }
                    period_replay_batch(tv, nwin, cs + j0, P.period, jb, kb, prof_i, chb + j0, a);
                    __syncwarp();
                } else if (PM == 26 && CHASE_DAY_BLOCKS && !last) {  // daily periods, full chunk: 12-window blocks
                    period_day(tv, c * kHWarpW + j0, P.W, phi0, T, A_even, wl, invK, Kc, e8, ebase, ZB, pt, pf, K0w, hcf,
                               cnr, cnab, prof_i, chb + j0, a, n_slow, n_seq);
                    __syncwarp();
                    k_carry = chb[kHWarpW - 1];
                } else if (PER && P.k0len > 0) {  // lane-direct periods with the closed form
                    const int wc = last ? P.W_last : kHWarpW;
                    period_direct<kDirectP>(reinterpret_cast<const float*>(stage) + P.off0, tv, nwin, c * kHWarpW + j0,
                                  c * kHWarpW, P.W, P.period, phi0, T, A_even, wl, invK, Kc, e8, ebase, ZB, pt, pf, K0w,
                                  hcf, cnr, cnab, k_carry, prof_i, chb + j0, a, n_slow, n_seq);
                    __syncwarp();
                    k_carry = chb[wc - 1];
                } else if (PER) {  // decisions for the chunk's periods first, then the replay
                    const int wc = last ? P.W_last : kHWarpW;
                    period_decisions(reinterpret_cast<const float*>(stage) + P.off0, c * kHWarpW, wc, P.W, P.period,
                                     P.phase_start, T, A_even, wl, invK, Kc, e8, ebase, ZB, pt, pf, K0w, hcf, cnr, cnab,
                                     k_carry, chb, lane, n_slow, n_seq);
                    __syncwarp();
                    k_carry = chb[wc - 1];
                    if (P.period >= 16 && (P.period & 3) == 0) {  // aligned runs of one choice: the run-form replay
                        const uint8_t* chl = chb + j0;
                        const int w0 = c * kHWarpW + j0;
                        int q = 0;
                        while (q < nwin) {
                            const int e = min(nwin, ((w0 + q) / P.period + 1) * P.period - w0);
                            const double2 ln = lds_line(kLineBase + (uint32_t)line_off(prof_i, (int)chl[q]));
                            replay_run(a, ln, e - q, run_csum(tv, q, e, a.vmin));
                            q = e;
                        }
                    } else {
                        replay_groups(tv, nwin, chb + j0, prof_i, a);
                    }
                }
                bool redone = false;
                if constexpr (PM == 0 && CHASE_H0_FAST) {
                    if (fast) {
                        // every value's bits b, offset by bits(FLT_MIN): max(b - 0x00800000) (unsigned) <=
                        // clim_bits - 0x00800000 iff all lie in [FLT_MIN, c_lim]; the lag of the lane's
                        // first window is in the bound too
                        uint32_t bmax = __float_as_uint(tv[-1]) - 0x00800000u;
                        hot_groups_fast(tv, ngr, Ap, wlK, e8, ebase, ZB, reinterpret_cast<uint32_t*>(chb + j0), bmax, a);
                        if (4 * ngr < nwin) {  // cold: the ragged last chunk
                            uint32_t mt;
                            acc_merge(a, hot_tail_fast(tv, 4 * ngr, nwin, Ap, wlK, e8, ebase, ZB, chb + j0, &mt));
                            bmax = max(bmax, mt);
                        }
                        // a value outside [FLT_MIN, c_lim] (zero, subnormal, negative, inf/NaN, too
                        // large): the chunk is redone with the exact key, which also validates (cold)
                        if (__any_sync(kFull, bmax > clim_bits - 0x00800000u)) {
                            const double* rec = reinterpret_cast<const double*>(stage + P.stage_bytes - kRecBytes);
                            const ExactModel M{rec[0], rec[1], rec[2], wl, Kc, invK, phS, phC};
                            a = lane_exact(tv, nwin, phi0, T, M, e8, ebase, ZB, pt, pf, chb + j0);
                            n_slow += (unsigned)a.bad_pad;
                            redone = true;
                        } else if (a.slow & 0x20202020u) {  // deferred windows: canonical on the exact forecast
                            const double* rec = reinterpret_cast<const double*>(stage + P.stage_bytes - kRecBytes);
                            const ExactModel M{rec[0], rec[1], rec[2], wl, Kc, invK, phS, phC};
                            const SlowFix fx = fix_slow_exact(tv, nwin, phi0, T, M, pt, pf, chb + j0);
                            a.S = __dadd_rn(a.S, fx.S);
                            a.E = __dadd_rn(a.E, fx.E);
                            a.C = __dadd_rn(a.C, fx.C);
                            n_slow += (unsigned)fx.n;
                        }
                        redone = true;  // (every case handled)
                    }
                }
                if constexpr (PM == 0 && CHASE_H0_FAST == 2) {
                    // one-fma key only: a trace it does not cover (eta = 1, Kc out of range, a table
                    // beyond the bound) takes the exact key chunk by chunk (cold)
                    if (!redone) {
                        const double* rec = reinterpret_cast<const double*>(stage + P.stage_bytes - kRecBytes);
                        const ExactModel M{rec[0], rec[1], rec[2], wl, Kc, invK, phS, phC};
                        a = lane_exact(tv, nwin, phi0, T, M, e8, ebase, ZB, pt, pf, chb + j0, invK == 0.0);
                        n_slow += (unsigned)a.bad_pad;
                        redone = true;
                    }
                }
                if (!PER && !redone) {
                    hot_groups(tv, ngr, Ap, wl, invK, e8, ebase, ZB, reinterpret_cast<uint32_t*>(chb + j0), a);
                    if (4 * ngr < nwin) {  // cold: a ragged last chunk, or Kc outside [2^-900, 2^900]
                        if (invK == 0.0) {
                            a = fused_generic<true, false, float, true>(tv, 0, nwin, Ap, wl, invK, pt, pf->line,
                                                                        chb + j0, nullptr, Kc, pf);
                            n_slow += (unsigned)a.bad_pad;
                        } else {
                            acc_merge(a, hot_tail(tv, 4 * ngr, nwin, Ap, wl, invK, e8, ebase, ZB, chb + j0));
                        }
                    }
                    if (a.slow & 0x20202020u) {  // deferred windows: the canonical K-way rule
                        const SlowFix fx = fix_slow<float>(tv, nwin, Ap, wl, Kc, pt, pf, chb + j0);
                        a.S = __dadd_rn(a.S, fx.S);
                        a.E = __dadd_rn(a.E, fx.E);
                        a.C = __dadd_rn(a.C, fx.C);
                        n_slow += (unsigned)fx.n;
                    }
                }
                // validation: negatives via vmin, NaN/inf via the sum of c
                const bool bad = __any_sync(kFull, !(a.vmin >= 0.0f) || !(a.Cs <= DBL_MAX) || a.bad);
                // baseline: sum of c over the windows before w*_b
                const int jb = c * kHWarpW + j0;
                const double Cbt = jb + nwin <= mb ? a.Cs : (jb < mb ? partial_cs(tv, mb - jb) : 0.0);
                // does the job complete in this chunk? (warp totals of the samples done)
                bool completes = false;
                if (!bad && !done && c >= c_may) completes = warp_sum(__dadd_rn(Sl, a.S)) >= J;
                if (!completes) {
                    __syncwarp();  // every lane is done with the stage
                    if (last) issue(i + GW, 0);
                    else issue(i, c + 1);
                    issued = true;
                }
                if (bad) status = CHASE_ERR_DATA;
                if (status == 0) {
                    Cbl = __dadd_rn(Cbl, Cbt);
                    if (completes) {
                        const double S_prev = warp_sum(Sl);
                        const double incl = warp_incl_scan(a.S, lane);
                        const double ex = __shfl_up_sync(kFull, incl, 1);
                        const double before = __dadd_rn(S_prev, lane == 0 ? 0.0 : ex);
                        const bool full = __dadd_rn(before, a.S) < J;
                        const unsigned who = __ballot_sync(kFull, !full && before < J && nwin > 0);
                        if (who != 0) {  // this chunk completes the job
                            __syncwarp();
                            const double Eb = warp_sum(full ? __dadd_rn(El, a.E) : El);
                            const double Cb = warp_sum(full ? __dadd_rn(Cl, a.C) : Cl);
                            const int src = __ffs(who) - 1;
                            const int nw_src = max(0, min(kc, (last ? P.W_last : kHWarpW) - kc * src));
                            const Completion cp = find_completion<float>(
                                tv + kc * (src - lane), chb + kc * src, nw_src,
                                __shfl_sync(kFull, before, src), J, pf->line, lane);
                            if (lane == 0) {
                                double* r = P.raw + i * kRawDoubles;
                                r[0] = __dadd_rn(Eb, cp.Ep);
                                r[1] = __dadd_rn(Cb, cp.Cp);
                                r[2] = J;
                                r[3] = cp.f;
                                r[4] = (double)((int64_t)P.L + c * kHWarpW + kc * src + cp.w);
                                r[5] = cp.Pk;
                                r[6] = cp.cw;
                                r[7] = 1.0;
                            }
                            done = true;
                        }
                        // else: no window reached J in the scan order (non-dyadic rounding): carry on
                    }
                    if (!done) {
                        Sl = __dadd_rn(Sl, a.S);
                        El = __dadd_rn(El, a.E);
                        Cl = __dadd_rn(Cl, a.C);
                    }
                    if (store_choice) {  // the chunk's choices: one TMA bulk store from the staging buffer
                        __syncwarp();
                        if (lane == 0) {
                            fence_proxy_async();
                            bulk_s2g(P.choice + i * P.ld_c + c * kHWarpW, chb,
                                     (uint32_t)(last ? (P.W_last + 15) & ~15 : kHWarpW));
                            bulk_commit();
                        }
                    }
                }
            } else if (status == CHASE_ERR_MAXCI || status == CHASE_ERR_FIT) {
                // S:29 precedence: a bad value anywhere makes the trace status 4
                if (__any_sync(kFull, chunk_has_bad(tv, nwin))) status = CHASE_ERR_DATA;
            }

            if (last) {  // ---- end of trace: one transposed reduction of the four running sums
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
                __syncwarp();  // every lane is done with the stage
                if (last) issue(i + GW, 0);
                else issue(i, c + 1);
            }
            par ^= 1u;
        }
    }
    if (store_choice && lane == 0) bulk_wait_read0();  // staging buffers stay valid until read
    n_slow = __reduce_add_sync(kFull, n_slow);
    if (lane == 0 && n_slow)
        atomicAdd(reinterpret_cast<unsigned long long*>(&P.diag->n_slow_windows), (unsigned long long)n_slow);
    if constexpr (PER) {
        n_seq = __reduce_add_sync(kFull, n_seq);
        if (lane == 0 && n_seq)
            atomicAdd(reinterpret_cast<unsigned long long*>(&P.diag->n_seq_periods), (unsigned long long)n_seq);
    }
}
