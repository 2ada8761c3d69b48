// Brownian paths on the device (BrownianBatch, stochastics.hpp:32-43).
//
// Host mode uploads BrownianBatch::values as is (parity mode: the reference's own
// xoshiro256++ stream, stochastics.cpp:24-57, generated on the host).  Philox mode
// is the counter-based generator for large runs: the increment of Lebesgue step k of
// global path g is sqrt(dt_leb) * N(0,1), the normal drawn by Box-Muller (same uniform
// mapping as stochastics.cpp:49-56) from Philox4x32-10 with key = seed and counter
// = (k/2, g_lo, g_hi, 0); it is invariant to how paths are sharded across GPUs.
// Prefix values are summed sequentially per path, values[0] = 0, like
// simulate_brownian (stochastics.cpp:94-98).
#include <cmath>

#include "s2b_internal.cuh"

namespace s2b {

namespace {

__device__ __forceinline__ void philox_round(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3,
                                             uint32_t k0, uint32_t k1) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t hi0 = __umulhi(M0, c0), lo0 = M0 * c0;
    const uint32_t hi1 = __umulhi(M1, c2), lo1 = M1 * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0;
    c1 = n1;
    c2 = n2;
    c3 = n3;
}

__device__ __forceinline__ uint4 philox4x32_10(uint4 ctr, uint2 key) {
    uint32_t c0 = ctr.x, c1 = ctr.y, c2 = ctr.z, c3 = ctr.w, k0 = key.x, k1 = key.y;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        philox_round(c0, c1, c2, c3, k0, k1);
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return make_uint4(c0, c1, c2, c3);
}

// increments into values[m][k+1]; values[m][0] = 0
__global__ void philox_increments_kernel(double* values, size_t steps, size_t M, uint64_t seed,
                                         uint64_t path_offset, double scale) {
    const size_t pairs = (steps + 1) / 2;
    const size_t id = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (id >= pairs * M) return;
    const size_t m = id / pairs, q = id % pairs;
    const uint64_t g = path_offset + m;
    const uint4 r = philox4x32_10(make_uint4(static_cast<uint32_t>(q), static_cast<uint32_t>(g),
                                             static_cast<uint32_t>(g >> 32), 0u),
                                  make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32)));
    const uint64_t x0 = (static_cast<uint64_t>(r.x) << 32) | r.y;
    const uint64_t x1 = (static_cast<uint64_t>(r.z) << 32) | r.w;
    const double u1 = (static_cast<double>(x0 >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = static_cast<double>(x1 >> 11) * 0x1.0p-53;
    const double rad = sqrt(-2.0 * log(u1));
    double sn, cs;
    sincospi(2.0 * u2, &sn, &cs);
    double* v = values + m * (steps + 1);
    const size_t k = 2 * q;
    v[k + 1] = scale * (rad * cs);
    if (k + 1 < steps) v[k + 2] = scale * (rad * sn);
    if (q == 0) v[0] = 0.0;
}

__global__ void prefix_kernel(double* values, size_t steps, size_t M) {
    const size_t m = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (m >= M) return;
    double* v = values + m * (steps + 1);
    double acc = 0.0;
    for (size_t k = 0; k < steps; ++k) {
        acc = acc + v[k + 1];
        v[k + 1] = acc;
    }
}

__global__ void broadcast_kernel(const double* __restrict__ src, double* __restrict__ dst, size_t n) {
    double* d = dst + blockIdx.y * n;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        d[i] = src[i];
}

} // namespace

// dst[m][:] = host_src[:] for m < M (one H2D copy, then a device broadcast).
void broadcast_rows(s2b_context* ctx, double* dst, const double* host_src, size_t n, size_t M) {
    DevBuf<double> tmp(n);
    S2B_CUDA(cudaMemcpyAsync(tmp.p, host_src, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    for (size_t m0 = 0; m0 < M; m0 += 65535) {
        const size_t mc = std::min<size_t>(65535, M - m0);
        dim3 g(static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 64)), static_cast<unsigned>(mc));
        broadcast_kernel<<<g, 256, 0, ctx->stream>>>(tmp.p, dst + m0 * n, n);
        S2B_LAUNCHED(ctx);
    }
    S2B_CUDA(cudaStreamSynchronize(ctx->stream));
}

s2b_paths* make_paths_host(s2b_context* ctx, double dt_leb, size_t steps, size_t M, uint64_t seed,
                           const double* values) {
    if (M == 0) fail(S2B_ERR_CONFIG, "paths: need at least one trajectory");
    if (steps == 0 || !(dt_leb > 0.0)) fail(S2B_ERR_CONFIG, "paths: need steps > 0 and dt_leb > 0");
    auto* p = new s2b_paths();
    p->ctx = ctx;
    p->dt_leb = dt_leb;
    p->steps = steps;
    p->M = M;
    p->seed = seed;
    p->d_values.alloc(M * (steps + 1));
    S2B_CUDA(cudaMemcpyAsync(p->d_values.p, values, p->d_values.bytes(), cudaMemcpyHostToDevice, ctx->stream));
    S2B_CUDA(cudaStreamSynchronize(ctx->stream));
    return p;
}

s2b_paths* make_paths_philox(s2b_context* ctx, double dt_leb, size_t steps, size_t M, uint64_t seed,
                             uint64_t path_offset) {
    if (M == 0) fail(S2B_ERR_CONFIG, "paths: need at least one trajectory");
    if (steps == 0 || !(dt_leb > 0.0)) fail(S2B_ERR_CONFIG, "paths: need steps > 0 and dt_leb > 0");
    auto* p = new s2b_paths();
    p->ctx = ctx;
    p->dt_leb = dt_leb;
    p->steps = steps;
    p->M = M;
    p->seed = seed;
    p->d_values.alloc(M * (steps + 1));
    const size_t work = ((steps + 1) / 2) * M;
    philox_increments_kernel<<<static_cast<unsigned>((work + 255) / 256), 256, 0, ctx->stream>>>(
        p->d_values.p, steps, M, seed, path_offset, std::sqrt(dt_leb));
    S2B_LAUNCHED(ctx);
    prefix_kernel<<<static_cast<unsigned>((M + 127) / 128), 128, 0, ctx->stream>>>(p->d_values.p, steps, M);
    S2B_LAUNCHED(ctx);
    S2B_CUDA(cudaStreamSynchronize(ctx->stream));
    return p;
}

} // namespace s2b
