// envelope.cpp — see envelope.h.  Host-only, long double (x87, 64-bit mantissa).
#include "envelope.h"

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <climits>
#include <cstdint>
#include <cstring>

namespace chase {
namespace {

using ld = long double;

constexpr ld kDelta = 0x1p-47L;        // 64u: required relative gap to every other line
// s = 2^-36 (131072u, 1.5e-11 relative): absorbs a key's error relative to
// x/Kc.  A key y inside a shrunk interval is at least y s/(1+s) from the
// verified interval's ends.  The kernels' keys: y = fl(x * fl(1/Kc)) of the
// canonical forecast x (|error| <= 2u relative; the headline, plan_kernel, the
// general sweep), and the decision periods' closed-form horizon mean (error
// kept below 120000u of the mean per period).  The bands this
// leaves around each breakpoint are far inside the hi32 test's own
// granularity (2^-20).
constexpr ld kShrink = 0x1p-36L;
constexpr double kYMax = 0x1p900;      // beyond: canonical path (overflow safety)
constexpr double kYMinK0 = 0x1p-900;   // eta == 1: below -> canonical (x == 0, underflow)

struct Line {
    int k;
    ld a, T;
};

inline ld cval(const Line& L, ld y) { return (L.a * y + 1.0L) / L.T; }

// Relative gap of line `o` over line `j` at y (y = inf: the limit).  Every term
// is positive, so this is accurate to a few long-double ulps (~1e-19).
ld gap(const Line& o, const Line& j, ld y, bool k0) {
    if (k0) return (o.a * j.T) / (j.a * o.T) - 1.0L;       // costs a x / T
    if (std::isinf(y)) {
        if (j.a > 0) return (o.a * j.T) / (j.a * o.T) - 1.0L;
        if (o.a > 0) return INFINITY;
        return j.T / o.T - 1.0L;
    }
    return cval(o, y) / cval(j, y) - 1.0L;
}

bool verify(const std::vector<Line>& L, int j, ld y, bool k0) {
    for (size_t o = 0; o < L.size(); ++o)
        if ((int)o != j && !(gap(L[o], L[j], y, k0) >= kDelta)) return false;
    return true;
}

double round_up_d(ld v) {
    double d = (double)v;
    if ((ld)d < v) d = std::nextafter(d, INFINITY);
    return d;
}
double round_down_d(ld v) {
    double d = (double)v;
    if ((ld)d > v) d = std::nextafter(d, -INFINITY);
    return d;
}

// Fast interval of line j inside [P, Q] (Q may be inf); false if empty.
bool fast_subinterval(const std::vector<Line>& L, int j, ld P, ld Q, ld* lo_out, ld* hi_out) {
    ld lo = P, hi = Q;
    const Line& J = L[j];
    for (size_t o = 0; o < L.size(); ++o) {
        if ((int)o == j) continue;
        // c_o(y) >= (1+d) c_j(y)  <=>  y * (a_o T_j - (1+d) a_j T_o) >= (1+d) T_o - T_j
        ld A = L[o].a * J.T - (1.0L + kDelta) * J.a * L[o].T;
        ld B = (1.0L + kDelta) * L[o].T - J.T;
        if (A > 0) lo = std::max(lo, B / A);
        else if (A < 0) hi = std::min(hi, B / A);
        else if (B > 0) return false;
    }
    if (!(lo <= hi)) return false;
    // Robust endpoint verification (the gap is linear-fractional, hence
    // monotone, in y on the interval): nudge inward until it passes.
    ld step = 0x1p-40L;
    for (int it = 0; it < 80 && !verify(L, j, lo, false); ++it, step *= 2) {
        lo = lo == 0 ? 0x1p-1000L : lo * (1.0L + step);
        if (!(lo <= hi)) return false;
    }
    if (!verify(L, j, lo, false)) return false;
    step = 0x1p-40L;
    for (int it = 0; it < 80 && !verify(L, j, hi, false); ++it, step *= 2) {
        hi = std::isinf(hi) ? std::max(lo * 2, (ld)1e30L) : hi * (1.0L - step);
        if (!(lo <= hi)) return false;
    }
    if (!verify(L, j, hi, false)) return false;
    *lo_out = lo;
    *hi_out = hi;
    return true;
}

double bucket_start(int base_raw, int b) {   // b in [1, kNBUsed - 1]
    uint64_t hi = (uint64_t)(uint32_t)((base_raw + b - 1) << kSH);
    uint64_t bits = hi << 32;
    double v;
    std::memcpy(&v, &bits, 8);
    return v;
}

}  // namespace

std::vector<FastInterval> build_pair_table(int K, const double* avg_power, const double* thr,
                                           double eta, double pmax, PairTable* out) {
    std::memset(out, 0, sizeof(*out));
    for (int k = 0; k < K; ++k) out->a[k] = eta * avg_power[k];   // same rounding as Eq. 6
    out->kbase = (1.0 - eta) * pmax;
    const bool k0 = !(out->kbase > 0.0);
    out->k0 = k0 ? 1 : 0;

    // Distinct lines, lowest index first (identical rows give bitwise-equal
    // costs, so first-min keeps the lowest).
    std::vector<Line> L;
    for (int k = 0; k < K; ++k) {
        bool dup = false;
        for (const Line& l : L)
            if (l.a == (ld)out->a[k] && l.T == (ld)thr[k]) dup = true;
        if (!dup) L.push_back({k, (ld)out->a[k], (ld)thr[k]});
    }

    std::vector<FastInterval> iv;
    if (k0) {
        // costs a_k x / Thr_k: one winner for every x > 0 if its ratio is
        // separated; x == 0 (all costs 0 -> index 0) stays canonical.
        int j = 0;
        for (size_t o = 1; o < L.size(); ++o)
            if (L[o].a * L[j].T < L[j].a * L[o].T) j = (int)o;
        ld amin = L[0].a;
        for (const Line& l : L) amin = std::min(amin, l.a);
        if (verify(L, j, 1.0L, true) && amin >= 0x1p-100L) iv.push_back({kYMinK0, kYMax, L[j].k});
    } else {
        std::vector<ld> pts{0.0L};
        for (size_t i = 0; i < L.size(); ++i)
            for (size_t o = i + 1; o < L.size(); ++o) {
                ld den = L[i].a * L[o].T - L[o].a * L[i].T;
                if (den == 0) continue;
                ld y = (L[i].T - L[o].T) / den;
                if (y > 0 && std::isfinite(y)) pts.push_back(y);
            }
        std::sort(pts.begin(), pts.end());
        pts.erase(std::unique(pts.begin(), pts.end()), pts.end());
        struct Seg { ld P, Q; int j; };
        std::vector<Seg> segs;
        for (size_t i = 0; i < pts.size(); ++i) {
            ld P = pts[i], Q = i + 1 < pts.size() ? pts[i + 1] : (ld)INFINITY;
            ld mid = std::isinf(Q) ? (P == 0 ? 1.0L : P * 2 + 1) : (P + Q) / 2;
            int j = 0;
            for (size_t o = 1; o < L.size(); ++o)
                if (cval(L[o], mid) < cval(L[j], mid)) j = (int)o;
            if (!segs.empty() && segs.back().j == j) segs.back().Q = Q;
            else segs.push_back({P, Q, j});
        }
        for (const Seg& s : segs) {
            ld lo, hi;
            if (!fast_subinterval(L, s.j, s.P, s.Q, &lo, &hi)) continue;
            double lo_d = lo == 0 ? 0.0 : round_up_d(lo * (1.0L + kShrink));
            double hi_d = std::isinf(hi) ? (double)INFINITY : round_down_d(hi * (1.0L - kShrink));
            hi_d = std::min(hi_d, kYMax);
            if (lo_d <= hi_d) iv.push_back({lo_d, hi_d, L[s.j].k});
        }
    }
    std::sort(iv.begin(), iv.end(), [](const FastInterval& a, const FastInterval& b) { return a.lo < b.lo; });
    out->n_intervals = (int)iv.size();
    // y_min: every positive finite endpoint of a verified (unshrunk) interval is
    // >= the smallest shrunk endpoint times (1 - 2^-35) (lo = lo_d/(1 + s),
    // hi = hi_d/(1 - s))
    double ymin = INFINITY;
    for (const FastInterval& f : iv)
        for (double v : {f.lo, f.hi})
            if (v > 0 && std::isfinite(v) && v < kYMax) ymin = std::min(ymin, v);
    out->y_min = std::isfinite(ymin) ? round_down_d((ld)ymin * (1.0L - 0x1p-35L)) : (double)INFINITY;

    // Bucket range: the 12-octave window [2^E0, 2^(E0+12)) holding the most
    // interval endpoints (endpoints outside it fall in the clamped end buckets,
    // which still take one exact threshold test, else the canonical path).
    std::vector<int> ex;
    for (const FastInterval& f : iv) {
        for (double v : {f.lo, f.hi}) {
            if (v > 0 && std::isfinite(v)) {
                int e;
                std::frexp(v, &e);
                ex.push_back(e - 1);  // floor(log2(v))
            }
        }
    }
    int E0 = 0;
    if (!ex.empty()) {
        int best = -1;
        for (int cand : ex) {
            const int e0 = cand - 1;
            int n = 0;
            for (int e : ex) n += (e >= e0 && e < e0 + 12) ? 1 : 0;
            if (n > best || (n == best && e0 < E0)) { best = n; E0 = e0; }
        }
        E0 = std::max(-1000, std::min(1000, E0));
    }
    const int base_raw = (E0 + 1023) << 6;
    out->base = base_raw - 1;

    auto hi32 = [](double v) -> int32_t {
        uint64_t b;
        std::memcpy(&b, &v, 8);
        return (int32_t)(uint32_t)(b >> 32);
    };
    auto enc = [](int32_t T1, int below, int above, int32_t delta) -> uint2 {
        if (delta < 0 || delta > 0xFFFF) { above = kZeroLine; delta = 0; }
        return make_uint2((uint32_t)T1, (uint32_t)below | ((uint32_t)above << 8) | ((uint32_t)delta << 16));
    };
    const uint2 all_slow = enc(INT32_MIN, kZeroLine, kZeroLine, 0);
    int n_test = 0;
    for (int b = 0; b < kNB; ++b) {
        if (b >= kNBUsed) { out->ent[b] = all_slow; continue; }
        double vb = b == 0 ? 0.0 : bucket_start(base_raw, b);
        double ve = b == kNBUsed - 1 ? (double)INFINITY : bucket_start(base_raw, b + 1);
        const FastInterval* cover = nullptr;
        const FastInterval* below = nullptr;
        const FastInterval* above = nullptr;
        for (const FastInterval& f : iv) {
            if (f.lo <= vb && f.hi >= ve) cover = &f;
            else if (f.lo <= vb && vb <= f.hi && f.hi < ve) below = &f;
            else if (vb < f.lo && f.lo < ve && f.hi >= ve) above = &f;
        }
        uint2 e;
        if (cover) {
            e = enc(INT32_MAX, cover->k, cover->k, 0);
        } else if (!below && !above) {
            e = all_slow;
        } else if (below && above) {
            // h < hi32(t_lo) => y < t_lo;  h > hi32(t_hi) => y > t_hi
            const int32_t T1 = hi32(below->hi), T2 = hi32(above->lo);
            e = enc(T1, below->k, above->k, T2 - T1);
            ++n_test;
        } else if (below) {
            e = enc(hi32(below->hi), below->k, kZeroLine, 0);
            ++n_test;
        } else {
            e = enc(hi32(above->lo), kZeroLine, above->k, 0);
            ++n_test;
        }
        out->ent[b] = e;
    }
    out->n_test = n_test;
    return iv;
}

}  // namespace chase
