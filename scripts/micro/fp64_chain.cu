// DMUL+DADD accumulate chains (acc += w*x, no FMA): throughput vs independent chains per
// thread at a fixed 16 warps/SM; plus the dependent DADD latency (one warp, one chain).
// nvcc -O3 -fmad=false -gencode arch=compute_100a,code=sm_100a -o fp64_chain fp64_chain.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void __launch_bounds__(512) chains(double* out, int iters, const double* w) {
    double acc[C], x[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        acc[c] = 0.0;
        x[c] = 1.0 + threadIdx.x * 1e-9 + c;
    }
    const double w0 = w[0], w1 = w[1];
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < C; ++c) acc[c] = acc[c] + w0 * x[c];
#pragma unroll
        for (int c = 0; c < C; ++c) acc[c] = acc[c] + w1 * x[c];
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) s += acc[c];
    if (s == 1234.5) out[0] = s;
}

__global__ void latency(double* out, int iters, double b, long long* cyc) {
    double a = threadIdx.x;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) a = a + b;
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) *cyc = t1 - t0;
    if (a == 1234.5) out[0] = a;
}

template <int C>
void run(double* out, double* w, int sms) {
    const int iters = 1 << 14, blocks = sms;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        chains<C><<<blocks, 512>>>(out, iters, w);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double ops = 4.0 * C * iters * 512.0 * blocks; // DMUL + DADD, two per iteration
    printf("chains=%d: %.2f fp64 Gop/s = %.1f%% of 64/clk/SM at 1965 MHz\n", C, ops / best / 1e6,
           100.0 * ops / (best * 1e-3) / (sms * 64.0 * 1.965e9));
}

int main() {
    double *out, *w;
    long long* cyc;
    cudaMalloc(&out, 8);
    cudaMalloc(&w, 16);
    cudaMalloc(&cyc, 8);
    double hw[2] = {0.999, 1e-3};
    cudaMemcpy(w, hw, 16, cudaMemcpyHostToDevice);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    latency<<<1, 32>>>(out, 1024, 1e-9, cyc);
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("dependent DADD latency: %.2f cycles\n", c / (1024.0 * 16));
    run<1>(out, w, sms);
    run<2>(out, w, sms);
    run<3>(out, w, sms);
    run<4>(out, w, sms);
    run<6>(out, w, sms);
    return 0;
}
