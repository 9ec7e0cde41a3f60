// device_common.cuh — PTX helpers, the Eq. 6 rule and lookup, warp collectives
// (included by kernels.cu inside its anonymous namespace).

constexpr int kWarps = kThreads / 32;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kRecBytes = kRecDoubles * 8;

thread_local uint64_t g_launches = 0;

// Bounds checks of our own (compute-sanitizer is closed on this pool): a
// build with -DCHASE_CHECKED=1 (tools/build_variant.sh checked ...) traps on
// any shared-memory, stage or output index outside its buffer; the default
// build compiles them away.
#ifndef CHASE_CHECKED
#define CHASE_CHECKED 0
#endif
#define CHASE_CHECK(cond)                     \
    do {                                      \
        if (CHASE_CHECKED && !(cond)) __trap(); \
    } while (0)

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
__device__ __forceinline__ void bulk_wait_read1() {
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void st_na_v4(uint4* p, uint4 v) {  // streaming store, no L1 allocation
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
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
// its fp64 encoding, then at most one integer threshold test on hi32(y).
// Returns kZeroLine when y lies where only the canonical rule is trusted.
// Negative y (an unclamped forecast) lands in bucket 0 and decides like x = 0.
__device__ __forceinline__ uint32_t plan_lookup(double y, const PairTable* pt) {
    const int h = __double2hiint(y);
    const int idx = max(min((h >> kSH) - pt->base, kNBUsed - 1), 0);
    const uint2 e = pt->ent[idx];
    const int T1 = (int)e.x;
    const bool p1 = h < T1;
    const bool p2 = h > T1 + (int)(e.y >> 16);
    return p1 ? (e.y & 0xffu) : (p2 ? ((e.y >> 8) & 0xffu) : (uint32_t)kZeroLine);
}

// 1/Kc for the lookup; 0 when Kc is outside [2^-900, 2^900] (or 0 with
// eta < 1): the trace then takes the canonical path for every window.
__device__ __forceinline__ double per_trace_invK(const PairTable* pt, double Kc) {
    if (pt->k0) return 1.0;
    return (Kc >= 0x1p-900 && Kc <= 0x1p900) ? __ddiv_rn(1.0, Kc) : 0.0;
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
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, o));
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

__device__ __forceinline__ const ProfileTable* blob_profiles(const uint8_t* blob) {
    const TablesHeader* H = reinterpret_cast<const TablesHeader*>(blob);
    return reinterpret_cast<const ProfileTable*>(blob + H->off_prof);
}

// Records which sweep kernel ran (chase_diag_t.kernel_path; block 0 only).
__device__ __forceinline__ void mark_path(chase_diag_t* d, unsigned bit) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(reinterpret_cast<unsigned long long*>(&d->kernel_path), bit);
}
