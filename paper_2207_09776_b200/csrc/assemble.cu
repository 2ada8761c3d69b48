// Device-side operator assembly: the CommutatorSet of the reference's
// host pipeline -- assemble_drift / assemble_diffusion (operators.cpp:134-189) and
// precompute_commutators (operators.cpp:191-208) over the CSR algebra of sparse.cpp:126-261 --
// computed on the GPU, bit for bit.
//
// Every matrix of the set is a 2-D stencil: row r = (i, j) couples to (i+dx, j+dv) with
// |dx|, |dv| <= 3.  Each matrix is held as a dense "box" [49][n] (offset-major, zero where the
// CSR has no entry), one thread per row:
//  * A and B: the terms of operators.cpp in their order (h, fx, fv, gxx, gxv, gvv; sig, sigx,
//    sigv), each term's value formed exactly as kron / scale_rows / sparse_scale form it
//    (av*bv with identity factors 1.0, zv[r]*v, then *0.5 for the second derivatives), summed
//    into the running entry from 0.0 -- sparse_add's merge, where a missing entry is + 0.0;
//  * products C = L R: C[r, r+o] = sum over the left offsets o1 in ascending column order
//    (== ascending (dv, dx)) of L[r, o1] * R[r+o1, o-o1], from 0.0 -- spmm's (a-entry,
//    b-entry) accumulation order, sparse.cpp:210-222; commutators as spmm(a,b) - spmm(b,a)
//    entry by entry.
// Absent CSR entries are exact zeros here.  That changes no bit: a running sum that starts at
// +0.0 can only become -0.0 if every addend is -0.0, so adding the +-0 products of absent
// entries never alters a value, and the reference's pruning of exact zeros is reproduced when
// the boxes are packed back into CSR (row by row, ascending column, zeros dropped).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <vector>

#include "s2b_internal.cuh"
#include "spde2d_b200.hpp"

namespace s2b {
namespace {

constexpr int kR = 3, kW = 7, kB = kW * kW;

__host__ __device__ constexpr int bit(int dx, int dv) { return (dv + kR) * kW + (dx + kR); }

struct AsmGrid {
    int nx, nv;
    double sx1, sv1; // d1 scales 1/(2 delta)
    double sx2, sv2; // d2 scales 1/(delta^2)
    int mask;        // non-zero fields: h fx fv gxx gxv gvv sig sigx sigv
};

// A and B of row r into the boxes (terms in operators.cpp order)
__global__ void assemble_ab_kernel(AsmGrid g, const double* __restrict__ f, double* __restrict__ A,
                                   double* __restrict__ B) {
    const size_t n = static_cast<size_t>(g.nx) * g.nv;
    const size_t r = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (r >= n) return;
    const int i = static_cast<int>(r % g.nx), j = static_cast<int>(r / g.nx);
    double b[kB], a[kB];
#pragma unroll
    for (int q = 0; q < kB; ++q) b[q] = a[q] = 0.0;
    const bool xl = i > 0, xr = i + 1 < g.nx, vl = j > 0, vr = j + 1 < g.nv;
    // tridiag weights (sparse.cpp:100-102): {lo*s, mid*s, hi*s}; kron factor 1.0 multiplies
    // (the middle weight of D1 is 0 * s: pruned, so D1 rows have two entries)
    const double d1x[3] = {-1.0 * g.sx1, 0.0, 1.0 * g.sx1};
    const double d1v[3] = {-1.0 * g.sv1, 0.0, 1.0 * g.sv1};
    const double d2x[3] = {1.0 * g.sx2, -2.0 * g.sx2, 1.0 * g.sx2};
    const double d2v[3] = {1.0 * g.sv2, -2.0 * g.sv2, 1.0 * g.sv2};
    auto add = [&](double* box, int dx, int dv, double v) {
        if (v != 0.0) box[bit(dx, dv)] = box[bit(dx, dv)] + v; // CsrBuilder drops exact zeros
    };
    auto fld = [&](int k) { return f[static_cast<size_t>(k) * n + r]; };
    // B = h + fx Dx + fv Dv + (gxx Dxx)/2 + gxv DvDx + (gvv Dvv)/2
    if (g.mask & 1) add(b, 0, 0, fld(0));
    if (g.mask & 2) {
        const double z = fld(1);
        if (z != 0.0) {
            if (xl) add(b, -1, 0, z * (1.0 * d1x[0]));
            if (xr) add(b, 1, 0, z * (1.0 * d1x[2]));
        }
    }
    if (g.mask & 4) {
        const double z = fld(2);
        if (z != 0.0) {
            if (vl) add(b, 0, -1, z * (d1v[0] * 1.0));
            if (vr) add(b, 0, 1, z * (d1v[2] * 1.0));
        }
    }
    if (g.mask & 8) {
        const double z = fld(3);
        if (z != 0.0) {
            if (xl) add(b, -1, 0, (z * (1.0 * d2x[0])) * 0.5);
            add(b, 0, 0, (z * (1.0 * d2x[1])) * 0.5);
            if (xr) add(b, 1, 0, (z * (1.0 * d2x[2])) * 0.5);
        }
    }
    if (g.mask & 16) {
        const double z = fld(4);
        if (z != 0.0) {
            if (vl && xl) add(b, -1, -1, z * (d1v[0] * d1x[0]));
            if (vl && xr) add(b, 1, -1, z * (d1v[0] * d1x[2]));
            if (vr && xl) add(b, -1, 1, z * (d1v[2] * d1x[0]));
            if (vr && xr) add(b, 1, 1, z * (d1v[2] * d1x[2]));
        }
    }
    if (g.mask & 32) {
        const double z = fld(5);
        if (z != 0.0) {
            if (vl) add(b, 0, -1, (z * (d2v[0] * 1.0)) * 0.5);
            add(b, 0, 0, (z * (d2v[1] * 1.0)) * 0.5);
            if (vr) add(b, 0, 1, (z * (d2v[2] * 1.0)) * 0.5);
        }
    }
    // A = sig + sigx Dx + sigv Dv
    if (g.mask & 64) add(a, 0, 0, fld(6));
    if (g.mask & 128) {
        const double z = fld(7);
        if (z != 0.0) {
            if (xl) add(a, -1, 0, z * (1.0 * d1x[0]));
            if (xr) add(a, 1, 0, z * (1.0 * d1x[2]));
        }
    }
    if (g.mask & 256) {
        const double z = fld(8);
        if (z != 0.0) {
            if (vl) add(a, 0, -1, z * (d1v[0] * 1.0));
            if (vr) add(a, 0, 1, z * (d1v[2] * 1.0));
        }
    }
#pragma unroll
    for (int q = 0; q < kB; ++q) {
        A[static_cast<size_t>(q) * n + r] = a[q];
        B[static_cast<size_t>(q) * n + r] = b[q];
    }
}

// (L R)[r, o] from 0.0 over the left offsets o1 in ascending order; radii rl, rr of L and R
__device__ __forceinline__ double box_spmm(const double* __restrict__ L, const double* __restrict__ R, size_t n,
                                           int nx, int nv, int i, int j, size_t r, int dx, int dv, int rl, int rr) {
    double acc = 0.0;
    for (int dv1 = -rl; dv1 <= rl; ++dv1) {
        const int dv2 = dv - dv1;
        if (dv2 < -rr || dv2 > rr || j + dv1 < 0 || j + dv1 >= nv) continue;
        for (int dx1 = -rl; dx1 <= rl; ++dx1) {
            const int dx2 = dx - dx1;
            if (dx2 < -rr || dx2 > rr || i + dx1 < 0 || i + dx1 >= nx) continue;
            const double lv = L[static_cast<size_t>(bit(dx1, dv1)) * n + r];
            if (lv == 0.0) continue; // absent entry of L: spmm never visits it
            const size_t k = r + static_cast<size_t>(static_cast<long long>(dv1) * nx + dx1);
            acc += lv * R[static_cast<size_t>(bit(dx2, dv2)) * n + k];
        }
    }
    return acc;
}

// C = L R (sub == false) or C = L R - R L (the commutator [L, R])
__global__ void box_product_kernel(const double* __restrict__ L, const double* __restrict__ R, double* __restrict__ C,
                                   int nx, int nv, int rl, int rr, int commutator) {
    const size_t n = static_cast<size_t>(nx) * nv;
    const size_t r = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (r >= n) return;
    const int i = static_cast<int>(r % nx), j = static_cast<int>(r / nx);
    const int ro = min(kR, rl + rr);
    for (int dv = -kR; dv <= kR; ++dv)
        for (int dx = -kR; dx <= kR; ++dx) {
            double v = 0.0;
            const bool in = dx >= -ro && dx <= ro && dv >= -ro && dv <= ro && i + dx >= 0 && i + dx < nx &&
                            j + dv >= 0 && j + dv < nv;
            if (in) {
                const double lr = box_spmm(L, R, n, nx, nv, i, j, r, dx, dv, rl, rr);
                v = lr;
                if (commutator) {
                    const double rlp = box_spmm(R, L, n, nx, nv, i, j, r, dx, dv, rr, rl);
                    v = lr - rlp; // sparse_sub merge: absent entries enter as 0.0
                }
            }
            C[static_cast<size_t>(bit(dx, dv)) * n + r] = v;
        }
}

__global__ void count_kernel(const double* __restrict__ box, size_t n, size_t* __restrict__ cnt) {
    const size_t r = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (r >= n) return;
    size_t c = 0;
    for (int q = 0; q < kB; ++q) c += box[static_cast<size_t>(q) * n + r] != 0.0;
    cnt[r] = c;
}

// row r's non-zeros in ascending column order (== ascending offset bit)
__global__ void pack_kernel(const double* __restrict__ box, size_t n, int nx, const size_t* __restrict__ rp,
                            int* __restrict__ ci, double* __restrict__ v) {
    const size_t r = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (r >= n) return;
    size_t o = rp[r];
    for (int q = 0; q < kB; ++q) {
        const double x = box[static_cast<size_t>(q) * n + r];
        if (x != 0.0) {
            const int dx = q % kW - kR, dv = q / kW - kR;
            ci[o] = static_cast<int>(static_cast<long long>(r) + static_cast<long long>(dv) * nx + dx);
            v[o] = x;
            ++o;
        }
    }
}

spde2d::SparseMatrix pack(s2b_context* ctx, const double* box, int nx, int nv) {
    const size_t n = static_cast<size_t>(nx) * nv;
    const unsigned g = static_cast<unsigned>((n + 255) / 256);
    DevBuf<size_t> cnt(n + 1), rp(n + 1);
    S2B_CUDA(cudaMemsetAsync(cnt.p + n, 0, sizeof(size_t), ctx->stream));
    count_kernel<<<g, 256, 0, ctx->stream>>>(box, n, cnt.p);
    S2B_LAUNCHED(ctx);
    size_t tmp_bytes = 0;
    S2B_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt.p, rp.p, n + 1, ctx->stream));
    DevBuf<unsigned char> tmp(std::max<size_t>(1, tmp_bytes));
    S2B_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, cnt.p, rp.p, n + 1, ctx->stream));
    std::vector<size_t> hrp(n + 1);
    S2B_CUDA(cudaMemcpyAsync(hrp.data(), rp.p, (n + 1) * sizeof(size_t), cudaMemcpyDeviceToHost, ctx->stream));
    S2B_CUDA(cudaStreamSynchronize(ctx->stream));
    const size_t nnz = hrp[n];
    DevBuf<int> ci(std::max<size_t>(1, nnz));
    DevBuf<double> v(std::max<size_t>(1, nnz));
    pack_kernel<<<g, 256, 0, ctx->stream>>>(box, n, nx, rp.p, ci.p, v.p);
    S2B_LAUNCHED(ctx);
    std::vector<int32_t> hci(nnz);
    std::vector<double> hv(nnz);
    if (nnz) {
        S2B_CUDA(cudaMemcpyAsync(hci.data(), ci.p, nnz * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        S2B_CUDA(cudaMemcpyAsync(hv.data(), v.p, nnz * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    }
    S2B_CUDA(cudaStreamSynchronize(ctx->stream));
    return spde2d::SparseMatrix(n, n, std::move(hrp), std::move(hci), std::move(hv));
}

} // namespace

// The CommutatorSet of `fields` on the device, packed back into the reference's CSR.
spde2d::CommutatorSet device_commutators(s2b_context* ctx, const spde2d::GridSpec& grid,
                                         const spde2d::CoefficientFields& f, int order) {
    if (order < 1 || order > 3) fail(S2B_ERR_CONFIG, "commutator order must be in {1, 2, 3}");
    const int nx = static_cast<int>(grid.x.n), nv = static_cast<int>(grid.v.n);
    const size_t n = static_cast<size_t>(nx) * nv;
    if (n == 0) fail(S2B_ERR_CONFIG, "device assembly: empty grid");
    const spde2d::Field* all[9] = {&f.h, &f.fx, &f.fv, &f.gxx, &f.gxv, &f.gvv, &f.sig, &f.sigx, &f.sigv};
    const bool zero[9] = {f.zero_h, f.zero_fx, f.zero_fv, f.zero_gxx, f.zero_gxv, f.zero_gvv,
                          f.zero_sig, f.zero_sigx, f.zero_sigv};
    AsmGrid g{nx, nv, 1.0 / (2.0 * grid.x.delta), 1.0 / (2.0 * grid.v.delta), 1.0 / (grid.x.delta * grid.x.delta),
              1.0 / (grid.v.delta * grid.v.delta), 0};
    DevBuf<double> F(9 * n);
    for (int k = 0; k < 9; ++k) {
        if (zero[k]) continue;
        if (all[k]->nx() != grid.x.n || all[k]->nv() != grid.v.n)
            fail(S2B_ERR_DIMENSION, "coefficient field shape does not match the grid");
        g.mask |= 1 << k;
        S2B_CUDA(cudaMemcpyAsync(F.p + k * n, all[k]->data().data(), n * sizeof(double), cudaMemcpyHostToDevice,
                                 ctx->stream));
    }
    const unsigned blocks = static_cast<unsigned>((n + 127) / 128);
    DevBuf<double> A(kB * n), B(kB * n);
    assemble_ab_kernel<<<blocks, 128, 0, ctx->stream>>>(g, F.p, A.p, B.p);
    S2B_LAUNCHED(ctx);
    spde2d::CommutatorSet s;
    s.order = order;
    s.A = pack(ctx, A.p, nx, nv);
    s.B = pack(ctx, B.p, nx, nv);
    if (order >= 2) {
        DevBuf<double> A2(kB * n), BA(kB * n);
        box_product_kernel<<<blocks, 128, 0, ctx->stream>>>(A.p, A.p, A2.p, nx, nv, 1, 1, 0);
        S2B_LAUNCHED(ctx);
        box_product_kernel<<<blocks, 128, 0, ctx->stream>>>(B.p, A.p, BA.p, nx, nv, 1, 1, 1); // [B,A]
        S2B_LAUNCHED(ctx);
        s.A2 = pack(ctx, A2.p, nx, nv);
        s.BA = pack(ctx, BA.p, nx, nv);
        if (order >= 3) {
            DevBuf<double> C(kB * n);
            box_product_kernel<<<blocks, 128, 0, ctx->stream>>>(BA.p, A.p, C.p, nx, nv, 2, 1, 1); // [[B,A],A]
            S2B_LAUNCHED(ctx);
            s.BAA = pack(ctx, C.p, nx, nv);
            box_product_kernel<<<blocks, 128, 0, ctx->stream>>>(BA.p, B.p, C.p, nx, nv, 2, 1, 1); // [[B,A],B]
            S2B_LAUNCHED(ctx);
            s.BAB = pack(ctx, C.p, nx, nv);
        }
    }
    return s;
}

} // namespace s2b
