// div_probe.cu — checks, on random and adversarial operands, that the
// Markstein sequence q = RN(a*y), r = fma(-q, b, a), q' = fma(r, y, q) with
// y = RN(1/b) returns the correctly rounded a/b (__ddiv_rn) — the candidate
// replacement for the per-row divides of the fit.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/div_probe tools/div_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    return x;
}

__global__ void probe(uint64_t seed, int64_t n, int mode, unsigned long long* bad, double* ex) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t u1 = mix(seed ^ (2 * t)), u2 = mix(seed ^ (2 * t + 1));
        double a, b;
        if (mode == 0) {  // mantissas uniform, exponents in +-8
            a = __longlong_as_double((long long)((u1 & 0x000FFFFFFFFFFFFFull) | ((uint64_t)(1023 + (int)(u1 >> 60) - 8) << 52)));
            b = __longlong_as_double((long long)((u2 & 0x000FFFFFFFFFFFFFull) | ((uint64_t)(1023 + (int)(u2 >> 60) - 8) << 52)));
        } else if (mode == 1) {  // b with all-ones or near-all-ones mantissa
            a = __longlong_as_double((long long)((u1 & 0x000FFFFFFFFFFFFFull) | (1023ull << 52)));
            b = __longlong_as_double((long long)((0x000FFFFFFFFFFFFFull - (u2 & 0xFFF)) | (1023ull << 52)));
        } else if (mode == 2) {  // fit-like: centred differences over a positive sigma
            const double x = 300.0 + (double)(u1 >> 11) * (400.0 / 9007199254740992.0);
            const double mu = 480.0 + (double)(u2 & 0xFFFFF) * 1e-4;
            a = x - mu;
            b = 20.0 + (double)(u2 >> 20) * (180.0 / 17592186044416.0);
        } else {  // a with all-ones mantissas, random b
            a = __longlong_as_double((long long)((0x000FFFFFFFFFFFFFull - (u1 & 0xFF)) | (1023ull << 52)));
            b = __longlong_as_double((long long)((u2 & 0x000FFFFFFFFFFFFFull) | (1023ull << 52)));
        }
        const double y = __drcp_rn(b);
        const double q0 = __dmul_rn(a, y);
        const double r = __fma_rn(-q0, b, a);
        const double q = __fma_rn(r, y, q0);
        const double ref = __ddiv_rn(a, b);
        if (__double_as_longlong(q) != __double_as_longlong(ref)) {
            const unsigned long long k = atomicAdd(bad, 1ull);
            if (k < 4) { ex[3 * k] = a; ex[3 * k + 1] = b; ex[3 * k + 2] = q - ref; }
        }
    }
}

int main() {
    unsigned long long* bad;
    double* ex;
    cudaMallocManaged(&bad, 8);
    cudaMallocManaged(&ex, 12 * 8);
    const int64_t n = 4000000000ll;
    for (int mode = 0; mode < 4; ++mode) {
        *bad = 0;
        probe<<<148 * 16, 256>>>(0x1234567ull + mode, n, mode, bad, ex);
        cudaDeviceSynchronize();
        printf("{\"mode\": %d, \"pairs\": %lld, \"mismatches\": %llu", mode, (long long)n, *bad);
        for (unsigned long long k = 0; k < (*bad < 4 ? *bad : 4); ++k)
            printf(", \"ex%llu\": [%.17g, %.17g, %.3g]", k, ex[3 * k], ex[3 * k + 1], ex[3 * k + 2]);
        printf("}\n");
    }
    return 0;
}
