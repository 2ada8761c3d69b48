// Pure DMUL, pure DADD and a 1:1 independent DMUL/DADD mix, 8 chains per thread,
// 16 warps/SM: does the mix exceed the single-op rate (separate issue paths)?
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(512) k(double* out, int iters, double a, double b) {
    double x[8], y[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) { x[c] = threadIdx.x * 1e-9 + c; y[c] = c * 0.5; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (MODE == 0) x[c] = __dmul_rn(x[c], a);
            if (MODE == 1) x[c] = __dadd_rn(x[c], b);
            if (MODE == 2) { x[c] = __dmul_rn(x[c], a); y[c] = __dadd_rn(y[c], b); }
        }
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += x[c] + y[c];
    if (s == 1234.5) out[0] = s;
}

template <int MODE>
void run(const char* name, double* out, int sms) {
    const int iters = 1 << 15;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        k<MODE><<<sms * 2, 512>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double ops = (MODE == 2 ? 16.0 : 8.0) * iters * 512.0 * sms * 2;
    printf("%s: %.1f fp64 ops/clk/SM at 1965 MHz\n", name, ops / (best * 1e-3) / sms / 1.965e9);
}

int main() {
    double* out;
    cudaMalloc(&out, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0>("dmul", out, sms);
    run<1>("dadd", out, sms);
    run<2>("dmul+dadd", out, sms);
    return 0;
}
