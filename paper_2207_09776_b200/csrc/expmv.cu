// expmv_into on a general CSR matrix (src/sparse.cpp:427-503), one vector.
//
// Used by the C++ API's expmv()/magnus_step for arbitrary sparse matrices (the
// Magnus solver itself runs the stencil engine in magnus.cu).  The row sums run
// in ascending column order from 0.0, which equals the reference's DIA order
// (ascending diagonal) for every non-zero term; ||M||_1 sums each column in
// ascending row order via a CSC view built on the host (index shuffle only).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include "s2b_internal.cuh"

namespace s2b {

namespace {

__global__ void colsum_kernel(size_t n, const size_t* cp, const double* cv, unsigned long long* best) {
    const size_t c = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (c >= n) return;
    double s = 0.0;
    for (size_t q = cp[c]; q < cp[c + 1]; ++q) s += fabs(cv[q]);
    atomicMax(best, static_cast<unsigned long long>(__double_as_longlong(s)) & 0x7FFFFFFFFFFFFFFFULL);
}

// next = M term; t = next*inv; term = t; accum += t; running |t|, |accum| maxima.
__global__ void csr_term_kernel(size_t n, const size_t* rp, const int* ci, const double* v, const double* term_in,
                                double* term_out, double* accum, double inv, unsigned long long* nb) {
    const size_t r = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    unsigned long long tb = 0, sb = 0;
    if (r < n) {
        double s = 0.0;
        for (size_t q = rp[r]; q < rp[r + 1]; ++q) s += v[q] * term_in[ci[q]];
        const double t = s * inv;
        term_out[r] = t;
        const double a = accum[r] + t;
        accum[r] = a;
        tb = static_cast<unsigned long long>(__double_as_longlong(t)) & 0x7FFFFFFFFFFFFFFFULL;
        sb = static_cast<unsigned long long>(__double_as_longlong(a)) & 0x7FFFFFFFFFFFFFFFULL;
    }
    for (int o = 16; o > 0; o >>= 1) {
        tb = max(tb, __shfl_xor_sync(0xffffffffu, tb, o));
        sb = max(sb, __shfl_xor_sync(0xffffffffu, sb, o));
    }
    if ((threadIdx.x & 31) == 0) {
        if (tb) atomicMax(&nb[0], tb);
        if (sb) atomicMax(&nb[1], sb);
    }
}

} // namespace

void expmv_csr(s2b_context* ctx, const s2b_csr* m, const double* x, double tol, double theta, double* y,
               int report[4]) {
    if (!(tol > 0.0)) fail(S2B_ERR_CONFIG, "expmv: tol must be positive");
    if (!(theta > 0.0)) fail(S2B_ERR_CONFIG, "expmv: theta must be positive");
    const size_t n = m->rows, nnz = n ? m->row_ptr[n] : 0;
    report[0] = 0;
    report[2] = 0;
    report[3] = 0;
    std::copy(x, x + n, y);
    if (n == 0) {
        report[1] = 1;
        return;
    }
    // CSC view (row order preserved inside each column)
    std::vector<size_t> cp(n + 1, 0);
    for (size_t q = 0; q < nnz; ++q) {
        if (m->col_idx[q] < 0 || static_cast<size_t>(m->col_idx[q]) >= n) fail(S2B_ERR_DIMENSION, "expmv: column out of range");
        cp[m->col_idx[q] + 1]++;
    }
    std::partial_sum(cp.begin(), cp.end(), cp.begin());
    std::vector<double> cv(std::max<size_t>(1, nnz));
    std::vector<size_t> fill(cp.begin(), cp.end() - 1);
    for (size_t r = 0; r < n; ++r)
        for (size_t q = m->row_ptr[r]; q < m->row_ptr[r + 1]; ++q) cv[fill[m->col_idx[q]]++] = m->values[q];
    DevBuf<size_t> d_rp(n + 1), d_cp(n + 1);
    DevBuf<int> d_ci(std::max<size_t>(1, nnz));
    DevBuf<double> d_v(std::max<size_t>(1, nnz)), d_cv(cv.size()), term[2] = {DevBuf<double>(n), DevBuf<double>(n)},
        acc(n);
    DevBuf<unsigned long long> nb(3);
    cudaStream_t st = ctx->stream;
    S2B_CUDA(cudaMemcpyAsync(d_rp.p, m->row_ptr, (n + 1) * sizeof(size_t), cudaMemcpyHostToDevice, st));
    S2B_CUDA(cudaMemcpyAsync(d_cp.p, cp.data(), (n + 1) * sizeof(size_t), cudaMemcpyHostToDevice, st));
    if (nnz) {
        S2B_CUDA(cudaMemcpyAsync(d_ci.p, m->col_idx, nnz * sizeof(int), cudaMemcpyHostToDevice, st));
        S2B_CUDA(cudaMemcpyAsync(d_v.p, m->values, nnz * sizeof(double), cudaMemcpyHostToDevice, st));
        S2B_CUDA(cudaMemcpyAsync(d_cv.p, cv.data(), nnz * sizeof(double), cudaMemcpyHostToDevice, st));
    }
    S2B_CUDA(cudaMemsetAsync(nb.p, 0, nb.bytes(), st));
    const unsigned g = static_cast<unsigned>((n + 255) / 256);
    colsum_kernel<<<g, 256, 0, st>>>(n, d_cp.p, d_cv.p, &nb.p[2]);
    S2B_LAUNCHED(ctx);
    unsigned long long nbits = 0;
    S2B_CUDA(cudaMemcpyAsync(&nbits, &nb.p[2], sizeof(nbits), cudaMemcpyDeviceToHost, st));
    S2B_CUDA(cudaStreamSynchronize(st));
    double norm;
    std::memcpy(&norm, &nbits, sizeof(norm));
    const double q = std::ceil(norm / theta);
    const int segments = q > 1.0 ? (q < 2147483647.0 ? static_cast<int>(q) : 2147483647) : 1;
    report[1] = segments;
    if (norm == 0.0) return;
    S2B_CUDA(cudaMemcpyAsync(acc.p, x, n * sizeof(double), cudaMemcpyHostToDevice, st));
    const unsigned long long inf_bits = 0x7FF0000000000000ULL;
    for (int seg = 0; seg < segments; ++seg) {
        S2B_CUDA(cudaMemcpyAsync(term[0].p, acc.p, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
        double prev = INFINITY;
        bool converged = false;
        int cur = 0;
        for (int k = 1; k <= 55; ++k) {
            S2B_CUDA(cudaMemsetAsync(nb.p, 0, 2 * sizeof(unsigned long long), st));
            const double inv = 1.0 / (static_cast<double>(segments) * k);
            csr_term_kernel<<<g, 256, 0, st>>>(n, d_rp.p, d_ci.p, d_v.p, term[cur].p, term[cur ^ 1].p, acc.p, inv, nb.p);
            S2B_LAUNCHED(ctx);
            cur ^= 1;
            unsigned long long h[2];
            S2B_CUDA(cudaMemcpyAsync(h, nb.p, sizeof(h), cudaMemcpyDeviceToHost, st));
            S2B_CUDA(cudaStreamSynchronize(st));
            report[3] += 1;
            if (h[0] >= inf_bits || h[1] >= inf_bits) {
                report[0] = 1; // Overflow
                return;
            }
            report[2] = std::max(report[2], k);
            double tn, sn;
            std::memcpy(&tn, &h[0], sizeof(tn));
            std::memcpy(&sn, &h[1], sizeof(sn));
            const double gate = tol * sn;
            if (tn <= gate && prev <= gate) {
                converged = true;
                break;
            }
            prev = tn;
        }
        if (!converged) {
            report[0] = 2; // ToleranceNotReached
            return;
        }
    }
    S2B_CUDA(cudaMemcpyAsync(y, acc.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    S2B_CUDA(cudaStreamSynchronize(st));
    for (size_t i = 0; i < n; ++i)
        if (!std::isfinite(y[i])) {
            report[0] = 1;
            return;
        }
}

} // namespace s2b
