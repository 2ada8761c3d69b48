// expmv_into on a general CSR matrix (src/sparse.cpp:427-503): the kernel-level entry of the
// reference API (sparse.hpp:144-151) with a caller-owned workspace (ExpmvWorkspace,
// sparse.hpp:121-130).
//
// One cooperative launch runs the whole segmented Taylor series: the stopping rule needs the
// path-wide maxima of every term, so each term is one grid-stride pass over the rows followed
// by one grid-wide barrier; every thread then reads the same two maxima and takes the same
// branch (converge / next term / Overflow / ToleranceNotReached), so no host round trip sits
// inside the series.  The maxima are 64-bit atomics on the IEEE bit patterns of |t| and |s|
// (order independent; NaN ranks above +inf, so every non-finite value is caught), in three
// rotating slots: the slot of term c is zeroed after term c-2's barrier, when its previous
// readers are done.
//
// Arithmetic (bitwise the reference's):
//   * ||M||_1: every column summed in ascending row order from 0.0 (one_norm, sparse.cpp:263-271)
//     through a CSC permutation built with the pattern;
//   * row sums in ascending column order from 0.0, which equals the reference's DIA fold
//     (ascending diagonal offsets, sparse.cpp:412-423) for every non-zero product, and its CSR
//     spmv fallback exactly;
//   * t = next * (1 / (s*k)), accum += t, the two-term gate, the 55-term cap, residual =
//     last tnorm/snorm ratio (max over segments on success, the last one on
//     ToleranceNotReached, +inf on Overflow), segments = max(1, ceil(norm/theta)).
//
// The workspace caches the device copy of the pattern: a call with the same row_ptr/col_idx
// (compared exactly against a host copy) only uploads the values and x -- the MagnusLogBuilder
// case, where every window refills the values of one union pattern.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

#include "s2b_internal.cuh"

namespace cg = cooperative_groups;

struct s2b_expmv_workspace {
    s2b_context* ctx = nullptr;
    size_t n = 0, nnz = 0;
    std::vector<size_t> h_rp;  // cached pattern (host copy for the exact comparison)
    std::vector<int32_t> h_ci;
    s2b::DevBuf<size_t> rp, cp;
    s2b::DevBuf<int> ci;
    s2b::DevBuf<size_t> perm; // CSC position -> CSR index (ascending row inside each column)
    s2b::DevBuf<double> v, y, acc, term[2];
    s2b::DevBuf<unsigned long long> nb; // [4][2]: three rotating term slots + the norm
    s2b::DevBuf<double> rep;            // status, residual, segments, max_terms, terms, final buffer
    double* h_rep = nullptr;            // pinned
    int grid = 0;
    bool have_pattern = false;
};

namespace s2b {

namespace {

constexpr int kExpmvThreads = 256;
constexpr int kExpmvMaxTerms = 55;
constexpr unsigned long long kAbsMask = 0x7FFFFFFFFFFFFFFFULL;
constexpr unsigned long long kInfB = 0x7FF0000000000000ULL;

struct CoopArgs {
    size_t n;
    const size_t* rp;
    const int* ci;
    const double* v;
    const size_t* cp;
    const size_t* perm;
    double* y;   // x in, the result out (or acc, see rep[5])
    double* acc;
    double* t0;
    double* t1;
    unsigned long long* nb;
    double* rep;
    double tol, theta;
};

__device__ __forceinline__ void block_max2(unsigned long long& a, unsigned long long& b, unsigned long long* slot) {
    for (int o = 16; o > 0; o >>= 1) {
        a = max(a, __shfl_xor_sync(0xffffffffu, a, o));
        b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    if ((threadIdx.x & 31) == 0) {
        if (a) atomicMax(&slot[0], a);
        if (b) atomicMax(&slot[1], b);
    }
}

__global__ void __launch_bounds__(kExpmvThreads) expmv_coop_kernel(CoopArgs a) {
    cg::grid_group grid = cg::this_grid();
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    const size_t gid = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    const bool leader = gid == 0;
    // ---- ||M||_1: max column abs-sum, each column in ascending row order
    {
        unsigned long long nb = 0, unused = 0;
        for (size_t c = gid; c < a.n; c += stride) {
            double s = 0.0;
            for (size_t q = a.cp[c]; q < a.cp[c + 1]; ++q) s += fabs(a.v[a.perm[q]]);
            nb = max(nb, static_cast<unsigned long long>(__double_as_longlong(s)) & kAbsMask);
        }
        block_max2(nb, unused, &a.nb[6]);
    }
    grid.sync();
    const double norm = __longlong_as_double(static_cast<long long>(__ldcg(&a.nb[6])));
    const double q = ceil(norm / a.theta);
    const int segments = q > 1.0 ? (q < 2147483647.0 ? static_cast<int>(q) : 2147483647) : 1;
    double residual = 0.0;
    int status = 0, max_terms = 0;
    long long terms = 0;
    double* y = a.y;
    double* acc = a.acc;
    int final_buf = 0;
    if (norm != 0.0) { // norm == 0: y = x (sparse.cpp:449)
        int c = 0; // global term counter: slot c % 3
        for (int seg = 0; seg < segments && status == 0; ++seg) {
            double prev = __longlong_as_double(static_cast<long long>(kInfB));
            double last_ratio = prev;
            bool converged = false;
            int cur = 0;
            for (int k = 1; k <= kExpmvMaxTerms; ++k, ++c) {
                // term_k = M term_{k-1} / (s k); term_0 = accum_0 = y
                const double* tin = k == 1 ? y : (cur ? a.t1 : a.t0);
                double* tout = cur ? a.t0 : a.t1;
                const double* ain = k == 1 ? y : acc;
                const double inv = 1.0 / (static_cast<double>(segments) * k);
                unsigned long long tb = 0, sb = 0;
                for (size_t r = gid; r < a.n; r += stride) {
                    double s = 0.0;
                    for (size_t p = a.rp[r]; p < a.rp[r + 1]; ++p) s += a.v[p] * tin[a.ci[p]];
                    const double t = s * inv;
                    tout[r] = t;
                    const double sum = ain[r] + t;
                    acc[r] = sum;
                    tb = max(tb, static_cast<unsigned long long>(__double_as_longlong(t)) & kAbsMask);
                    sb = max(sb, static_cast<unsigned long long>(__double_as_longlong(sum)) & kAbsMask);
                }
                unsigned long long* slot = a.nb + 2 * (c % 3);
                block_max2(tb, sb, slot);
                grid.sync();
                tb = __ldcg(&slot[0]);
                sb = __ldcg(&slot[1]);
                if (leader) { // the slot of term c + 2; its last readers finished before this barrier
                    unsigned long long* z = a.nb + 2 * ((c + 2) % 3);
                    z[0] = 0;
                    z[1] = 0;
                }
                cur ^= 1;
                ++terms;
                if (tb >= kInfB || sb >= kInfB) { // non-finite term or accum (sparse.cpp:473-477)
                    status = 1;
                    residual = __longlong_as_double(static_cast<long long>(kInfB));
                    break;
                }
                max_terms = max(max_terms, k);
                const double tn = __longlong_as_double(static_cast<long long>(tb));
                const double sn = __longlong_as_double(static_cast<long long>(sb));
                const double gate = a.tol * sn;
                last_ratio = sn > 0.0 ? tn / sn : 0.0;
                if (tn <= gate && prev <= gate) {
                    residual = fmax(residual, last_ratio);
                    converged = true;
                    ++c;
                    break;
                }
                prev = tn;
            }
            if (status != 0) break;
            if (!converged) { // sparse.cpp:486-491
                status = 2;
                residual = last_ratio;
                break;
            }
            double* tmp = y; // std::swap(y, ws.accum)
            y = acc;
            acc = tmp;
            final_buf ^= 1;
        }
    }
    if (leader) {
        a.rep[0] = status;
        a.rep[1] = residual;
        a.rep[2] = segments;
        a.rep[3] = max_terms;
        a.rep[4] = static_cast<double>(terms);
        a.rep[5] = final_buf;
    }
}

void upload_pattern(s2b_expmv_workspace* ws, const s2b_csr* m) {
    const size_t n = m->rows, nnz = n ? m->row_ptr[n] : 0;
    for (size_t q = 0; q < nnz; ++q)
        if (m->col_idx[q] < 0 || static_cast<size_t>(m->col_idx[q]) >= n)
            fail(S2B_ERR_DIMENSION, "expmv: column out of range");
    ws->h_rp.assign(m->row_ptr, m->row_ptr + n + 1);
    ws->h_ci.assign(m->col_idx, m->col_idx + nnz);
    // CSC permutation: rows visited in ascending order keep each column's entries row-ordered
    std::vector<size_t> cp(n + 1, 0), perm(std::max<size_t>(1, nnz));
    for (size_t q = 0; q < nnz; ++q) cp[m->col_idx[q] + 1]++;
    std::partial_sum(cp.begin(), cp.end(), cp.begin());
    std::vector<size_t> fill(cp.begin(), cp.end() - 1);
    for (size_t r = 0; r < n; ++r)
        for (size_t q = m->row_ptr[r]; q < m->row_ptr[r + 1]; ++q) perm[fill[m->col_idx[q]]++] = q;
    cudaStream_t st = ws->ctx->stream;
    if (ws->n != n) {
        ws->rp.alloc(n + 1);
        ws->cp.alloc(n + 1);
        ws->y.alloc(n);
        ws->acc.alloc(n);
        ws->term[0].alloc(n);
        ws->term[1].alloc(n);
    }
    if (ws->ci.n < std::max<size_t>(1, nnz)) {
        ws->ci.alloc(std::max<size_t>(1, nnz));
        ws->perm.alloc(std::max<size_t>(1, nnz));
        ws->v.alloc(std::max<size_t>(1, nnz));
    }
    S2B_CUDA(cudaMemcpyAsync(ws->rp.p, m->row_ptr, (n + 1) * sizeof(size_t), cudaMemcpyHostToDevice, st));
    S2B_CUDA(cudaMemcpyAsync(ws->cp.p, cp.data(), (n + 1) * sizeof(size_t), cudaMemcpyHostToDevice, st));
    if (nnz) {
        S2B_CUDA(cudaMemcpyAsync(ws->ci.p, m->col_idx, nnz * sizeof(int), cudaMemcpyHostToDevice, st));
        S2B_CUDA(cudaMemcpyAsync(ws->perm.p, perm.data(), nnz * sizeof(size_t), cudaMemcpyHostToDevice, st));
    }
    S2B_CUDA(cudaStreamSynchronize(st)); // the host staging vectors die here
    ws->n = n;
    ws->nnz = nnz;
    int per_sm = 0;
    S2B_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, expmv_coop_kernel, kExpmvThreads, 0));
    const size_t want = (n + kExpmvThreads - 1) / kExpmvThreads;
    ws->grid = static_cast<int>(std::max<size_t>(1, std::min<size_t>(want, static_cast<size_t>(std::max(1, per_sm)) * ws->ctx->num_sms)));
    ws->have_pattern = true;
}

bool same_pattern(const s2b_expmv_workspace* ws, const s2b_csr* m) {
    if (!ws->have_pattern || ws->n != m->rows) return false;
    const size_t nnz = m->rows ? m->row_ptr[m->rows] : 0;
    return nnz == ws->nnz && std::memcmp(ws->h_rp.data(), m->row_ptr, (m->rows + 1) * sizeof(size_t)) == 0 &&
           (nnz == 0 || std::memcmp(ws->h_ci.data(), m->col_idx, nnz * sizeof(int32_t)) == 0);
}

// x and y: host (device == false) or device pointers of n doubles.
void expmv_run(s2b_expmv_workspace* ws, const s2b_csr* m, const double* x, double tol, double theta, double* y,
               s2b_expmv_report* out, bool device) {
    if (!(tol > 0.0)) fail(S2B_ERR_CONFIG, "expmv: tol must be positive");
    if (!(theta > 0.0)) fail(S2B_ERR_CONFIG, "expmv: theta must be positive");
    const size_t n = m->rows;
    *out = s2b_expmv_report{};
    out->segments = 1;
    if (n == 0) return;
    if (!same_pattern(ws, m)) upload_pattern(ws, m);
    cudaStream_t st = ws->ctx->stream;
    const cudaMemcpyKind in = device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (ws->nnz) S2B_CUDA(cudaMemcpyAsync(ws->v.p, m->values, ws->nnz * sizeof(double), cudaMemcpyHostToDevice, st));
    S2B_CUDA(cudaMemcpyAsync(ws->y.p, x, n * sizeof(double), in, st));
    S2B_CUDA(cudaMemsetAsync(ws->nb.p, 0, ws->nb.bytes(), st));
    CoopArgs a{n, ws->rp.p, ws->ci.p, ws->v.p, ws->cp.p, ws->perm.p, ws->y.p, ws->acc.p, ws->term[0].p,
               ws->term[1].p, ws->nb.p, ws->rep.p, tol, theta};
    void* args[] = {&a};
    S2B_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(expmv_coop_kernel), dim3(ws->grid),
                                         dim3(kExpmvThreads), args, 0, st));
    S2B_LAUNCHED(ws->ctx);
    S2B_CUDA(cudaMemcpyAsync(ws->h_rep, ws->rep.p, 6 * sizeof(double), cudaMemcpyDeviceToHost, st));
    S2B_CUDA(cudaStreamSynchronize(st));
    const double* r = ws->h_rep;
    out->status = static_cast<int>(r[0]);
    out->residual = r[1];
    out->segments = static_cast<int>(r[2]);
    out->max_terms = static_cast<int>(r[3]);
    out->terms = static_cast<int64_t>(r[4]);
    const double* res = r[5] != 0.0 ? ws->acc.p : ws->y.p;
    S2B_CUDA(cudaMemcpyAsync(y, res, n * sizeof(double), device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    S2B_CUDA(cudaStreamSynchronize(st));
    if (out->status == 0 && !device) { // the final finite scan (sparse.cpp:495-501)
        for (size_t i = 0; i < n; ++i)
            if (!std::isfinite(y[i])) {
                out->status = 1;
                out->residual = HUGE_VAL;
                break;
            }
    }
}

} // namespace

s2b_expmv_workspace* expmv_workspace_create(s2b_context* ctx) {
    auto* ws = new s2b_expmv_workspace();
    try {
        ws->ctx = ctx;
        ws->nb.alloc(8);
        ws->rep.alloc(6);
        S2B_CUDA(cudaMallocHost(&ws->h_rep, 6 * sizeof(double)));
    } catch (...) {
        delete ws;
        throw;
    }
    return ws;
}

void expmv_workspace_destroy(s2b_expmv_workspace* ws) {
    if (!ws) return;
    if (ws->h_rep) cudaFreeHost(ws->h_rep);
    delete ws;
}

void expmv_into(s2b_expmv_workspace* ws, const s2b_csr* m, const double* x, double tol, double theta, double* y,
                s2b_expmv_report* rep, bool device) {
    expmv_run(ws, m, x, tol, theta, y, rep, device);
}

void expmv_csr(s2b_context* ctx, const s2b_csr* m, const double* x, double tol, double theta, double* y,
               int report[4]) {
    s2b_expmv_workspace* ws = expmv_workspace_create(ctx);
    s2b_expmv_report r{};
    try {
        expmv_run(ws, m, x, tol, theta, y, &r, false);
    } catch (...) {
        expmv_workspace_destroy(ws);
        throw;
    }
    expmv_workspace_destroy(ws);
    report[0] = r.status;
    report[1] = r.segments;
    report[2] = r.max_terms;
    report[3] = static_cast<int>(r.terms);
}

} // namespace s2b
