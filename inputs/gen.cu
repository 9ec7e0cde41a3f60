// gen.cu — host and device fillers for the synthetic trace generator
// (harness inputs only; see chase_gen.h).  Built into inputs/libchasegen.so.
#include <cuda_runtime.h>
#include <stdint.h>

#include "chase_gen.h"

extern "C" {

// Host filler: out[i][t] for traces [trace0, trace0+n) (fp32, row stride ld).
void chasegen_fill_host(float* out, int64_t n, int64_t N, int64_t ld, uint64_t seed,
                        int64_t trace0, int32_t mode, int32_t T, int32_t phase0,
                        const int32_t* sin_q, const int32_t* year_q) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        uint64_t tr = (uint64_t)(trace0 + i);
        chasegen_params_t p = chasegen_params(seed, tr, mode, T);
        float* row = out + i * ld;
        for (int64_t t = 0; t < N; ++t)
            row[t] = (float)chasegen_value_q(&p, seed, tr, t, T, phase0, sin_q, year_q) * 0.015625f;
        for (int64_t t = N; t < ld; ++t) row[t] = 0.0f;
    }
}

void chasegen_profile_ids_host(uint8_t* out, int64_t n, uint64_t seed, int64_t trace0, int32_t n_profiles) {
    for (int64_t i = 0; i < n; ++i)
        out[i] = (uint8_t)chasegen_profile_id(seed, (uint64_t)(trace0 + i), n_profiles);
}

}  // extern "C"

__global__ void chasegen_fill_kernel(float* out, int64_t n, int64_t N, int64_t ld, uint64_t seed,
                                     int64_t trace0, int32_t mode, int32_t T, int32_t phase0,
                                     const int32_t* sin_q, const int32_t* year_q) {
    int64_t i = blockIdx.y + (int64_t)blockIdx.z * gridDim.y;
    if (i >= n) return;
    uint64_t tr = (uint64_t)(trace0 + i);
    chasegen_params_t p = chasegen_params(seed, tr, mode, T);
    float* row = out + i * ld;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ld;
         t += (int64_t)gridDim.x * blockDim.x)
        row[t] = t < N ? (float)chasegen_value_q(&p, seed, tr, t, T, phase0, sin_q, year_q) * 0.015625f
                       : 0.0f;
}

__global__ void chasegen_profile_ids_kernel(uint8_t* out, int64_t n, uint64_t seed, int64_t trace0,
                                            int32_t n_profiles) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = (uint8_t)chasegen_profile_id(seed, (uint64_t)(trace0 + i), n_profiles);
}

extern "C" {

// Device filler; sin_q / year_q are DEVICE pointers.  Returns cudaError_t.
int chasegen_fill_device(float* out, int64_t n, int64_t N, int64_t ld, uint64_t seed,
                         int64_t trace0, int32_t mode, int32_t T, int32_t phase0,
                         const int32_t* sin_q, const int32_t* year_q, void* stream) {
    if (n <= 0) return 0;
    int64_t gy = n < 65535 ? n : 65535;
    int64_t gz = (n + gy - 1) / gy;
    dim3 grid((unsigned)((ld + 1023) / 1024 < 16 ? (ld + 1023) / 1024 : 16), (unsigned)gy, (unsigned)gz);
    chasegen_fill_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(out, n, N, ld, seed, trace0, mode, T,
                                                                   phase0, sin_q, year_q);
    return (int)cudaGetLastError();
}

int chasegen_profile_ids_device(uint8_t* out, int64_t n, uint64_t seed, int64_t trace0,
                                int32_t n_profiles, void* stream) {
    if (n <= 0) return 0;
    chasegen_profile_ids_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        out, n, seed, trace0, n_profiles);
    return (int)cudaGetLastError();
}

}  // extern "C"
