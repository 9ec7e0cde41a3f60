// fp64_probe.cu — measures the B200's FP64 vector issue rate (DFMA, DADD,
// DMUL) to give the rolling-refit kernel an ALU roofline, and
// the cost of the conversions / special functions next to a DADD (FRND, F2I,
// DSETP, F2F.F64.F32, MUFU.RCP) that shape the SVR and MAPE kernels.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/fp64_probe tools/fp64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void probe(double* out, int iters, double a, double b) {
    double x[8];
    float f[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        x[k] = threadIdx.x * 1e-3 + k;
        f[k] = 1.0f + k * 0.001f;
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (OP == 0) x[k] = __fma_rn(x[k], a, b);
            else if (OP == 1) x[k] = __dadd_rn(x[k], b);
            else if (OP == 2) x[k] = __dmul_rn(x[k], a);
            else if (OP == 3) x[k] = floor(__dadd_rn(x[k], b));                       // DADD + FRND
            else if (OP == 4) x[k] = __dadd_rn(x[k], (double)(__double2int_rn(x[k]) & 1));  // F2I + I2F + DADD
            else if (OP == 5) x[k] = __dadd_rn(x[k], x[k] > a ? b : a);               // DSETP + DADD
            else if (OP == 6) {                                                         // FMUL + F2F.F64.F32 + DADD
                f[k] = __fmul_rn(f[k], 1.0001f);
                x[k] = __dadd_rn(x[k], (double)f[k]);
            } else {                                                                    // MUFU.RCP + FADD
                float r;
                asm("rcp.approx.f32 %0, %1;" : "=f"(r) : "f"(f[k]));
                f[k] = __fadd_rn(r, 1.0f);
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k] + f[k];
    if (s == 12345.678) out[0] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* d;
    cudaMalloc(&d, 8);
    const int iters = 20000, threads = 256, blocks = sms * 8;
    const char* names[8] = {"dfma", "dadd", "dmul", "dadd+frnd", "f2i+i2f+dadd", "dsetp+dadd", "fmul+f2f.f64.f32+dadd",
                            "mufu.rcp+fadd"};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int op = 0; op < 8; ++op) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            if (op == 0) probe<0><<<blocks, threads>>>(d, iters, 0.999999, 1e-9);
            else if (op == 1) probe<1><<<blocks, threads>>>(d, iters, 0.999999, 1e-9);
            else if (op == 2) probe<2><<<blocks, threads>>>(d, iters, 0.999999, 1e-9);
            else if (op == 3) probe<3><<<blocks, threads>>>(d, iters, 0.999999, 1.5);
            else if (op == 4) probe<4><<<blocks, threads>>>(d, iters, 0.999999, 1e-9);
            else if (op == 5) probe<5><<<blocks, threads>>>(d, iters, 0.5, 1e-9);
            else if (op == 6) probe<6><<<blocks, threads>>>(d, iters, 0.5, 1e-9);
            else probe<7><<<blocks, threads>>>(d, iters, 0.5, 1e-9);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double ops = (double)blocks * threads * iters * 8;
            if (rep == 2)
                printf("{\"op\": \"%s\", \"thread_ops_per_s\": %.4e, \"per_sm_per_clk_at_1965\": %.2f, \"ms\": %.3f, \"sms\": %d}\n",
                       names[op], ops / (ms * 1e-3), ops / (ms * 1e-3) / sms / 1.965e9, ms, sms);
        }
    }
    return 0;
}
