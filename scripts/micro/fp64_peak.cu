// FP64 non-tensor pipe peak on this GPU: independent DFMA / DMUL / DADD chains, all SMs.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void __launch_bounds__(512) kern(double* out, int iters, double a, double b) {
    constexpr int C = 8;
    double x[C];
#pragma unroll
    for (int c = 0; c < C; ++c) x[c] = threadIdx.x * 1e-9 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (OP == 0) x[c] = fma(x[c], a, b);
            if (OP == 1) x[c] = __dmul_rn(x[c], a);
            if (OP == 2) x[c] = __dadd_rn(x[c], b);
        }
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) s += x[c];
    if (s == 1234.5) out[0] = s;
}

int main() {
    double* out;
    cudaMalloc(&out, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 1 << 16, threads = 512, blocks = sms * 4;
    const char* names[] = {"dfma", "dmul", "dadd"};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    printf("{");
    for (int op = 0; op < 3; ++op) {
        float best = 1e30f;
        for (int r = 0; r < 4; ++r) {
            cudaEventRecord(e0);
            if (op == 0) kern<0><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
            if (op == 1) kern<1><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
            if (op == 2) kern<2><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        const double ops = 8.0 * iters * threads * (double)blocks;
        const double per_clk_sm = ops / (best * 1e-3) / sms;
        printf("%s\"%s_gops\": %.1f, \"%s_per_sm_per_ns\": %.2f", op ? ", " : "", names[op], ops / best / 1e6,
               names[op], per_clk_sm / 1e9);
    }
    printf(", \"sms\": %d}\n", sms);
    return 0;
}
