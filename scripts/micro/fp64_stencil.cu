// Throughput of the x-march's arithmetic pattern alone (no memory): C independent chains of
// acc += w * x (DMUL + DADD, no FMA) per thread, W warps per SM; reports % of the measured
// 64 fp64 lanes/clk/SM.  nvcc -O3 -fmad=false -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

template <int C, int NT>
__global__ void __launch_bounds__(NT, 1) k(double* out, int iters, const double* wv) {
    double w[19], x[C + 18], acc[C];
#pragma unroll
    for (int e = 0; e < 19; ++e) w[e] = wv[e];
#pragma unroll
    for (int q = 0; q < C + 18; ++q) x[q] = threadIdx.x * 1e-3 + q;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < C; ++c) acc[c] = 0.0;
#pragma unroll
        for (int e = 0; e < 19; ++e)
#pragma unroll
            for (int c = 0; c < C; ++c) acc[c] += w[e] * x[c + e];
#pragma unroll
        for (int q = 0; q < C + 18; ++q) x[q] = acc[q % C] * 1e-3 + x[q]; // keep values live
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) s += acc[c];
    if (s == 1.5) out[0] = s;
}

template <int C, int NT>
void run(double* out, double* w, int sms) {
    const int iters = 2000;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(a);
        k<C, NT><<<sms, NT>>>(out, iters, w);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    // fp64 ops per iteration per thread: 19*C*2 (stencil) + (C+18)*2 (update)
    const double ops = (19.0 * C * 2 + (C + 18) * 2) * iters * NT * (double)sms;
    printf("C=%d NT=%d: %.1f%% of 64/clk/SM at 1965 MHz\n", C, NT, 100.0 * ops / (best * 1e-3) / (sms * 64.0 * 1.965e9));
}

int main() {
    double *out, *w;
    cudaMalloc(&out, 8);
    cudaMalloc(&w, 19 * 8);
    double hw[19];
    for (int e = 0; e < 19; ++e) hw[e] = 0.01 * (e + 1);
    cudaMemcpy(w, hw, sizeof hw, cudaMemcpyHostToDevice);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<1, 256>(out, w, sms);
    run<2, 256>(out, w, sms);
    run<4, 256>(out, w, sms);
    run<4, 128>(out, w, sms);
    run<4, 512>(out, w, sms);
    run<8, 256>(out, w, sms);
    return 0;
}
