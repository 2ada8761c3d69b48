// Iterated stochastic Magnus on the GPU: the pass engine.
//
// Reference path replaced: solve_iterated_magnus (src/magnus.cpp:239-304) with
// MagnusLogBuilder::fill (:141-160), log_coefficients (:26-40),
// lebesgue_functionals (src/stochastics.cpp:121-141) and expmv_into
// (src/sparse.cpp:427-503).
//
// B200 design:
//  * The logarithm Y of every path-window is never materialised.  The six
//    CommutatorSet matrices are re-laid out once as 2-D stencil weights; when
//    they are x-invariant away from the two x-boundary columns on each side
//    (the Langevin families) they compress to W[pair][j][class] (a few 100 KB).
//  * All (path, window) functionals, the six scalar weights c_s and the
//    segment counts s = ceil(||Y||_1 / theta) are computed up front, in
//    parallel in time (functionals_kernel, norm_*_kernel).
//  * A "pass" applies ONE Taylor term to EVERY live path: each path runs its
//    own (window, segment, k) state machine, so paths never wait for each
//    other and the reference's per-path stopping rule (two consecutive term
//    inf-norms <= tol * ||accum||_inf, 55-term cap) is replicated exactly.
//    term_tma_kernel streams the path's term/accum rows through a TMA
//    (cp.async.bulk) shared-memory ring, keeps a (2Rv+1)-row register window
//    per thread and rebuilds Y for its row strip from the compressed weights;
//    per-path inf-norms are max-reduced with 64-bit atomics (order-independent,
//    hence deterministic).  control_kernel then advances every path's state
//    machine and compacts the live list.
//  * Bitwise parity: all arithmetic is separately rounded (-fmad=false) in the
//    reference's order: Y assembly in slot order from 0.0, the matvec summed
//    in ascending stencil offset (= the DIA diagonal order of sparse.cpp:412-423)
//    from 0.0, t = next * (1/(s*k)), accum += t.  Column sums for ||Y||_1 are
//    accumulated in ascending row order like one_norm (sparse.cpp:263-271).
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>

#include "magnus_common.cuh"

namespace s2b {

using namespace mg;

int mg::tma_popcount(int variant) { return __builtin_popcountll(kVariants[variant].mask); }

// term_tma_kernel's shared memory: the TMA rings and the coefficient table, plus YST doubles per
// strip row (term_kernel.cuh); the strip height is capped so that the total fits kTermSmem
size_t mg::tma_smem_fixed(int variant, size_t nx) {
    const size_t nye = static_cast<size_t>(kClasses) * tma_popcount(variant);
    const size_t H = kVariants[variant].rx <= 2 ? 2 : 4;
    return 128 + kStages * (nx + 2 * H) * 8 + kStages * nx * 8 + kPairSlots * nye * 8;
}
size_t mg::tma_strip_cap(int variant, size_t nx) {
    const size_t nye = static_cast<size_t>(kClasses) * tma_popcount(variant);
    const size_t yst = (nye + 1) & ~static_cast<size_t>(1);
    // resident CTAs per SM of the launch's block-size class (NtClass: 128 -> 4, 256 -> 2, 512 -> 1),
    // each with ~1 KB of static / reserved shared memory
    const size_t nt = (std::max<size_t>((nx + 1) / 2, nye) + 31) / 32 * 32;
    const size_t ctas = nt <= 128 ? 4 : (nt <= 256 ? 2 : 1);
    const size_t budget = std::min(kTermSmem, (228 * 1024) / ctas - 2048);
    const size_t fixed = tma_smem_fixed(variant, nx);
    return budget > fixed + 8 * yst * 8 ? (budget - fixed) / (yst * 8) : 8;
}

namespace {

// lebesgue_functionals (stochastics.cpp:121-141) + log_coefficients (magnus.cpp:26-40),
// one thread per (path, window): all windows of all paths at once.
__global__ void functionals_kernel(const double* __restrict__ values, size_t steps, size_t M,
                                   size_t dt_steps, size_t nwin, size_t w0, size_t nw, double dt,
                                   int order, double* __restrict__ ctab) {
    const size_t tid = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (tid >= M * nw) return;
    const size_t m = tid / nw, w = w0 + tid % nw;
    const size_t id = m * nwin + w;
    const double* p = values + m * (steps + 1);
    const size_t k0 = w * dt_steps, k1 = k0 + dt_steps;
    const double base = p[k0];
    double iw = 0.0, isw = 0.0, iw2 = 0.0;
    for (size_t j = 0; j < dt_steps; ++j) {
        const double wv = p[k0 + j] - base;
        const double s = static_cast<double>(j) * dt;
        iw += wv;
        isw += s * wv;
        iw2 += wv * wv;
    }
    const double h = static_cast<double>(k1 - k0) * dt;
    const double W = p[k1] - p[k0];
    const double IW = iw * dt, IsW = isw * dt, IW2 = iw2 * dt;
    double c[6] = {h, W, 0.0, 0.0, 0.0, 0.0};
    if (order >= 2) {
        c[2] = -0.5 * h;
        c[3] = IW - 0.5 * h * W;
    }
    if (order >= 3) {
        c[4] = 0.5 * IW2 - 0.5 * W * IW + h * W * W / 12.0;
        c[5] = IsW - 0.5 * h * IW - h * h * W / 12.0;
    }
    double* out = ctab + id * 6;
#pragma unroll
    for (int s = 0; s < 6; ++s) out[s] = c[s];
}

// Y value of one stencil bit at one row: MagnusLogBuilder::fill's fold (magnus.cpp:147-159),
// 0.0 start, slots in order, zero coefficients skipped.
__device__ __forceinline__ double y_entry(const OpView& op, const double* c, int bit, int i, int j) {
    double y = 0.0;
    const int q0 = op.pair_begin[bit], q1 = op.pair_begin[bit + 1];
    for (int q = q0; q < q1; ++q) {
        const double cs = c[op.pair_slot[q]];
        if (cs == 0.0) continue;
        const double wv = op.compressed
                              ? op.w[(static_cast<size_t>(q) * op.nv + j) * kClasses + xclass(i, op.nx)]
                              : op.w[static_cast<size_t>(q) * op.nx * op.nv + static_cast<size_t>(j) * op.nx + i];
        y += cs * wv;
    }
    return y;
}

// ||Y||_1 column sum of column (i, j): rows in ascending order (descending stencil bit),
// only rows inside the grid (one_norm, sparse.cpp:263-271).
__device__ double column_sum(const OpView& op, const double* c, const int* bits, int nbits, int i,
                             int j) {
    double s = 0.0;
    for (int e = nbits - 1; e >= 0; --e) {
        const int b = bits[e];
        const int dx = b % kBoxW - kBoxR, dv = b / kBoxW - kBoxR;
        const int ir = i - dx, jr = j - dv;
        if (ir < 0 || ir >= op.nx || jr < 0 || jr >= op.nv) continue;
        s += fabs(y_entry(op, c, b, ir, jr));
    }
    return s;
}

// Segment count per (path, window): s = max(1, ceil(norm/theta)), 0 marks norm == 0
// (expmv returns its input unchanged, sparse.cpp:449).  One block per (path, window).
// Compressed layout: only columns whose stencil rows touch a boundary class, plus one
// interior representative, are distinct.
__global__ void norm_kernel(OpView op, const int* __restrict__ bits, int nbits, int rx,
                            const double* __restrict__ ctab, size_t nwin, size_t w0, size_t nw,
                            double theta, int* __restrict__ stab, double* __restrict__ norms) {
    const size_t id = (blockIdx.x / nw) * nwin + w0 + blockIdx.x % nw;
    __shared__ double c[6];
    __shared__ unsigned long long red[32];
    if (threadIdx.x < 6) c[threadIdx.x] = ctab[id * 6 + threadIdx.x];
    __syncthreads();
    unsigned long long best = 0;
    const int lim = rx + 2; // i <= lim or i >= nx-1-lim are the distinct columns
    const int ncol_i = op.compressed ? min(op.nx, 2 * lim + 2) : op.nx;
    const int total = ncol_i * op.nv;
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
        const int ii = t % ncol_i, j = t / ncol_i;
        int i = ii;
        if (op.compressed && op.nx > 2 * lim + 2 && ii > lim) i = op.nx - (2 * lim + 2) + ii;
        const double s = column_sum(op, c, bits, nbits, i, j);
        best = umax64(best, abs_bits(s)); // colsums are >= 0; NaN ranks above +inf
    }
    best = warp_umax(best);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x < 32) {
        unsigned long long v = threadIdx.x < (blockDim.x + 31) / 32 ? red[threadIdx.x] : 0ULL;
        v = warp_umax(v);
        if (threadIdx.x == 0) {
            const double norm = __longlong_as_double(static_cast<long long>(v));
            int s = 0;
            if (norm != 0.0) {
                const double q = ceil(norm / theta);
                s = q > 1.0 ? (q < 2147483647.0 ? static_cast<int>(q) : INT_MAX) : 1;
            }
            stab[id] = s;
            if (norms) norms[id] = norm;
        }
    }
}

// ---- path state machine ---------------------------------------------------------
struct Ctl {
    int* win;       // current window
    int* seg;       // segment within the window
    int* k;         // next Taylor term (1-based)
    int* nseg;      // segments of the current window
    int* status;    // 0 live, 1 finished/paused-at-T, 2 blown
    int* par;       // which of the two buffers holds the current term/accum
    int* rec_next;  // next record index
    double* prev;   // previous term inf-norm
    long long* terms;
    long long* windows;
    long long* segments;
    unsigned long long* tn; // running max |t| (bits)
    unsigned long long* sn; // running max |accum| (bits)
    int* act_in;
    int* act_out;
    int* cnt; // cnt[0] live-in, cnt[1] live-out, cnt[2] records queued
    int4* recq; // (path, record, parity, -)
    uint8_t* rec_status; // [R][M]
    const int* stab;     // [M][nwin]
    const long long* rec_steps; // [R]
    int R;
    int nwin;
    int dt_steps;
    int win_stop; // pause when reaching this window
    int p_lo;     // paths below this index belong to another engine (hybrid runs)
    double tol;
    double cap;
    size_t M;
};

// Enter window `w` of path p whose state is in parity `par`: skip zero-norm windows,
// queue record snapshots at window ends, finish at win_stop.  Returns true if the path
// has a term to run.
__device__ bool enter_window(const Ctl& c, int p, int w, int par) {
    while (true) {
        if (w >= c.win_stop) {
            c.win[p] = w;
            c.status[p] = w >= c.nwin ? 1 : 0;
            return false;
        }
        const int s = c.stab[static_cast<size_t>(p) * c.nwin + w];
        if (s != 0) {
            c.win[p] = w;
            c.nseg[p] = s;
            c.seg[p] = 0;
            c.k[p] = 1;
            c.prev[p] = __longlong_as_double(static_cast<long long>(kInfBits));
            return true;
        }
        // norm == 0: exp(Y)u = u, the window completes immediately
        c.windows[p] += 1;
        const long long step = static_cast<long long>(w + 1) * c.dt_steps;
        int r = c.rec_next[p];
        while (r < c.R && c.rec_steps[r] == step) {
            c.rec_status[static_cast<size_t>(r) * c.M + p] = 0;
            if (r < c.R - 1) c.recq[atomicAdd(&c.cnt[2], 1)] = make_int4(p, r, par, 0);
            ++r;
        }
        c.rec_next[p] = r;
        ++w;
    }
}

__global__ void init_kernel(Ctl c, int first_window) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= static_cast<int>(c.M) || p < c.p_lo) return;
    if (c.status[p] == 2) return; // blown paths stay blown
    c.tn[p] = 0;
    c.sn[p] = 0;
    if (first_window == 0) { // the counters accumulate over the session (reset by session_reset)
        c.par[p] = 0;
        c.rec_next[p] = 0;
    }
    if (enter_window(c, p, first_window, c.par[p])) c.act_out[atomicAdd(&c.cnt[1], 1)] = p;
}

// After a pass: evaluate the stopping rule of expmv_into (sparse.cpp:463-492) and the
// window-level blow-up rule of solve_iterated_magnus (magnus.cpp:277-291) per live path.
// solve_iterated_magnus checks max|u| > cap after every window, including a zero-norm one
// (magnus.cpp:277-286).  Before the first real window u is phi; after one, max|u| <= cap
// was already checked.  So with max|phi| > cap a path whose first window has norm 0 is
// BlownUp at once (no record written), and every other path proceeds unchanged.
__global__ void phi_cap_kernel(const int* __restrict__ stab, int nwin, int* __restrict__ status, size_t M) {
    const size_t p = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (p < M && status[p] == 0 && stab[p * nwin] == 0) status[p] = 2;
}

__global__ void control_kernel(Ctl c) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= c.cnt[0]) return;
    const int p = c.act_in[a];
    const unsigned long long tb = c.tn[p], sb = c.sn[p];
    c.tn[p] = 0;
    c.sn[p] = 0;
    const int par = c.par[p] ^ 1; // the pass wrote the other buffer pair
    c.par[p] = par;
    c.terms[p] += 1;
    if (tb >= kInfBits || sb >= kInfBits) { // non-finite term or accum: Overflow
        c.status[p] = 2;
        return;
    }
    const double tn = __longlong_as_double(static_cast<long long>(tb));
    const double sn = __longlong_as_double(static_cast<long long>(sb));
    const double gate = c.tol * sn;
    const int k = c.k[p];
    if (tn <= gate && c.prev[p] <= gate) {
        const int seg = c.seg[p] + 1;
        c.segments[p] += 1;
        if (seg < c.nseg[p]) {
            c.seg[p] = seg;
            c.k[p] = 1;
            c.prev[p] = __longlong_as_double(static_cast<long long>(kInfBits));
        } else {
            // window done: u = accum, max|u| == sn (magnus.cpp:282-286)
            if (sn > c.cap) {
                c.status[p] = 2;
                return;
            }
            const int w = c.win[p];
            c.windows[p] += 1;
            const long long step = static_cast<long long>(w + 1) * c.dt_steps;
            int r = c.rec_next[p];
            while (r < c.R && c.rec_steps[r] == step) {
                c.rec_status[static_cast<size_t>(r) * c.M + p] = 0;
                if (r < c.R - 1) c.recq[atomicAdd(&c.cnt[2], 1)] = make_int4(p, r, par, 0);
                ++r;
            }
            c.rec_next[p] = r;
            if (!enter_window(c, p, w + 1, par)) return;
        }
    } else {
        if (k >= kMaxTerms) { // ToleranceNotReached
            c.status[p] = 2;
            return;
        }
        c.prev[p] = tn;
        c.k[p] = k + 1;
    }
    c.act_out[atomicAdd(&c.cnt[1], 1)] = p;
}

// The two-term engine's state machine (term2_kernel.cuh): one pass applied terms k and k+1.
// Term k is judged first with (tn, sn); only if the segment did not stop there is term k+1
// judged with (tn2, sn2) -- exactly the reference's sequence of single terms (sparse.cpp:463-492).
// par holds the accumulator buffer index (0..2) during the loop: s_k went to S[(par+2)%3],
// s_{k+1} to S[(par+1)%3]; tpar flips when the segment continues.
__device__ void finish_segment(const Ctl& c, int p, int par, double sn) {
    const int seg = c.seg[p] + 1;
    c.segments[p] += 1;
    if (seg < c.nseg[p]) {
        c.seg[p] = seg;
        c.k[p] = 1;
        c.prev[p] = __longlong_as_double(static_cast<long long>(kInfBits));
        c.act_out[atomicAdd(&c.cnt[1], 1)] = p;
        return;
    }
    if (sn > c.cap) { // window done: u = accum, max|u| == sn (magnus.cpp:282-286)
        c.status[p] = 2;
        return;
    }
    const int w = c.win[p];
    c.windows[p] += 1;
    const long long step = static_cast<long long>(w + 1) * c.dt_steps;
    int r = c.rec_next[p];
    while (r < c.R && c.rec_steps[r] == step) {
        c.rec_status[static_cast<size_t>(r) * c.M + p] = 0;
        if (r < c.R - 1) c.recq[atomicAdd(&c.cnt[2], 1)] = make_int4(p, r, par, 0);
        ++r;
    }
    c.rec_next[p] = r;
    if (enter_window(c, p, w + 1, par)) c.act_out[atomicAdd(&c.cnt[1], 1)] = p;
}

__global__ void control2_kernel(Ctl c, Term2Args x) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= c.cnt[0]) return;
    const int p = c.act_in[a];
    const unsigned long long tb1 = c.tn[p], sb1 = c.sn[p], tb2 = x.tn2[p], sb2 = x.sn2[p];
    c.tn[p] = 0;
    c.sn[p] = 0;
    x.tn2[p] = 0;
    x.sn2[p] = 0;
    const int sidx = c.par[p];
    const int s_next = sidx == 2 ? 0 : sidx + 1; // s_{k+1}
    const int s_k = sidx == 0 ? 2 : sidx - 1;    // s_k
    const int k = c.k[p];
    // term k
    c.terms[p] += 1;
    if (tb1 >= kInfBits || sb1 >= kInfBits) {
        c.status[p] = 2;
        return;
    }
    const double tn1 = __longlong_as_double(static_cast<long long>(tb1));
    const double sn1 = __longlong_as_double(static_cast<long long>(sb1));
    const double gate1 = c.tol * sn1;
    if (tn1 <= gate1 && c.prev[p] <= gate1) {
        c.par[p] = s_k;
        finish_segment(c, p, s_k, sn1);
        return;
    }
    if (k >= kMaxTerms) { // ToleranceNotReached
        c.status[p] = 2;
        return;
    }
    // term k + 1
    c.terms[p] += 1;
    if (tb2 >= kInfBits || sb2 >= kInfBits) {
        c.status[p] = 2;
        return;
    }
    const double tn2 = __longlong_as_double(static_cast<long long>(tb2));
    const double sn2 = __longlong_as_double(static_cast<long long>(sb2));
    const double gate2 = c.tol * sn2;
    c.par[p] = s_next;
    if (tn2 <= gate2 && tn1 <= gate2) {
        finish_segment(c, p, s_next, sn2);
        return;
    }
    if (k + 1 >= kMaxTerms) {
        c.status[p] = 2;
        return;
    }
    c.prev[p] = tn2;
    c.k[p] = k + 2;
    x.tpar[p] ^= 1;
    c.act_out[atomicAdd(&c.cnt[1], 1)] = p;
}

// After a two-term run: every accumulator back in S0 / S1 (the other engines and the session
// readers know two buffers), par in {0, 1}.
__global__ void normalize2_kernel(const int* __restrict__ par, const double* __restrict__ S2, double* __restrict__ S0,
                                  size_t n, size_t M, int p_lo) {
    for (size_t m = p_lo + blockIdx.y; m < M; m += gridDim.y) {
        if (par[m] != 2) continue;
        const double* src = S2 + m * n;
        double* dst = S0 + m * n;
        for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
             i += static_cast<size_t>(gridDim.x) * blockDim.x)
            dst[i] = src[i];
    }
}

__global__ void normalize2_flag_kernel(int* __restrict__ par, size_t M, int p_lo) {
    const size_t m = p_lo + blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (m < M && par[m] == 2) par[m] = 0;
}

// Copy queued record snapshots S[par][p] -> rec[r][p].
__global__ void record_kernel(const int* __restrict__ cnt, const int4* __restrict__ recq,
                              const double* __restrict__ S0, const double* __restrict__ S1,
                              double* const* __restrict__ rec, size_t n, const double* __restrict__ S2 = nullptr) {
    const int nq = cnt[2];
    for (int q = blockIdx.y; q < nq; q += gridDim.y) {
        const int4 e = recq[q];
        const double* src = (e.z == 2 ? S2 : e.z ? S1 : S0) + static_cast<size_t>(e.x) * n;
        double* dst = rec[e.y] + static_cast<size_t>(e.x) * n;
        for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
             i += static_cast<size_t>(gridDim.x) * blockDim.x)
            dst[i] = src[i];
    }
}

__global__ void swap_counts_kernel(int* cnt) {
    cnt[0] = cnt[1];
    cnt[1] = 0;
    cnt[2] = 0;
}

// ---- term kernels --------------------------------------------------------------

// Generic kernel: one thread per (path, point); any stencil, full or compressed weights.
__global__ void term_generic_kernel(TermArgs a, const int* __restrict__ bits, int nbits) {
    const int nx = a.op.nx, nv = a.op.nv;
    const size_t n = static_cast<size_t>(nx) * nv;
    const int blocks_per_path = static_cast<int>((n + blockDim.x - 1) / blockDim.x);
    const long long work = static_cast<long long>(a.cnt[0]) * blocks_per_path;
    __shared__ double c[6];
    __shared__ unsigned long long red[2][32];
    for (long long wi = blockIdx.x; wi < work; wi += gridDim.x) {
        const int p = a.act[wi / blocks_per_path];
        const size_t r = (wi % blocks_per_path) * static_cast<size_t>(blockDim.x) + threadIdx.x;
        __syncthreads();
        if (threadIdx.x < 6) c[threadIdx.x] = a.ctab[(static_cast<size_t>(p) * a.nwin + a.win[p]) * 6 + threadIdx.x];
        __syncthreads();
        const int kk = a.k[p];
        const int par = a.par[p];
        const double inv = 1.0 / (static_cast<double>(a.nseg[p]) * kk);
        const double* Sin = (par ? a.S1 : a.S0) + static_cast<size_t>(p) * n;
        const double* in = kk == 1 ? Sin : (par ? a.T1 : a.T0) + static_cast<size_t>(p) * n;
        double* Tout = (par ? a.T0 : a.T1) + static_cast<size_t>(p) * n;
        double* Sout = (par ? a.S0 : a.S1) + static_cast<size_t>(p) * n;
        unsigned long long tb = 0, sb = 0;
        if (r < n) {
            const int i = static_cast<int>(r % nx), j = static_cast<int>(r / nx);
            double y = 0.0;
            for (int e = 0; e < nbits; ++e) {
                const int b = bits[e];
                const int dx = b % kBoxW - kBoxR, dv = b / kBoxW - kBoxR;
                const int ii = i + dx, jj = j + dv;
                const double x = (ii >= 0 && ii < nx && jj >= 0 && jj < nv) ? in[static_cast<size_t>(jj) * nx + ii] : 0.0;
                y += y_entry(a.op, c, b, i, j) * x;
            }
            const double t = y * inv;
            const double s = Sin[r] + t;
            Tout[r] = t;
            Sout[r] = s;
            tb = abs_bits(t);
            sb = abs_bits(s);
        }
        tb = warp_umax(tb);
        sb = warp_umax(sb);
        if ((threadIdx.x & 31) == 0) {
            red[0][threadIdx.x >> 5] = tb;
            red[1][threadIdx.x >> 5] = sb;
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            const int nw = (blockDim.x + 31) / 32;
            unsigned long long t2 = threadIdx.x < nw ? red[0][threadIdx.x] : 0ULL;
            unsigned long long s2 = threadIdx.x < nw ? red[1][threadIdx.x] : 0ULL;
            t2 = warp_umax(t2);
            s2 = warp_umax(s2);
            if (threadIdx.x == 0) {
                if (t2) atomicMax(&a.tn[p], t2);
                if (s2) atomicMax(&a.sn[p], s2);
            }
        }
    }
}



// Generic term kernel, K live paths per work item: Y is folded per point from the (x- or
// v-dependent, uncompressible) weights, which are shared by every path -- each weight load
// now serves K paths, so the L2 traffic per path*point*term drops ~K-fold.  Same arithmetic
// per path as term_generic_kernel (fold in slot order from 0.0 skipping zero weights; sum
// in ascending stencil bit).
template <int K>
__global__ void __launch_bounds__(256) term_generic_k_kernel(TermArgs a, const int* __restrict__ bits, int nbits) {
    const int nx = a.op.nx, nv = a.op.nv;
    const size_t n = static_cast<size_t>(nx) * nv;
    const int blocks_per_path = static_cast<int>((n + blockDim.x - 1) / blockDim.x);
    const int live = a.cnt[0];
    const long long groups = (live + K - 1) / K;
    const long long work = groups * blocks_per_path;
    __shared__ double c[K][6];
    __shared__ unsigned long long red[K][2][32];
    for (long long wi = blockIdx.x; wi < work; wi += gridDim.x) {
        const long long g = wi / blocks_per_path;
        const size_t r = (wi % blocks_per_path) * static_cast<size_t>(blockDim.x) + threadIdx.x;
        int pk[K];
#pragma unroll
        for (int k = 0; k < K; ++k) pk[k] = g * K + k < live ? a.act[g * K + k] : -1;
        __syncthreads();
        if (threadIdx.x < K * 6) {
            const int k = threadIdx.x / 6, q = threadIdx.x % 6;
            c[k][q] = pk[k] >= 0 ? a.ctab[(static_cast<size_t>(pk[k]) * a.nwin + a.win[pk[k]]) * 6 + q] : 0.0;
        }
        __syncthreads();
        const double* in[K];
        const double* Sin[K];
        double* Tout[K];
        double* Sout[K];
        double inv[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int p = pk[k] >= 0 ? pk[k] : 0;
            const int kk = a.k[p], par = a.par[p];
            inv[k] = 1.0 / (static_cast<double>(a.nseg[p]) * kk);
            Sin[k] = (par ? a.S1 : a.S0) + static_cast<size_t>(p) * n;
            in[k] = kk == 1 ? Sin[k] : (par ? a.T1 : a.T0) + static_cast<size_t>(p) * n;
            Tout[k] = (par ? a.T0 : a.T1) + static_cast<size_t>(p) * n;
            Sout[k] = (par ? a.S0 : a.S1) + static_cast<size_t>(p) * n;
        }
        unsigned long long tb[K], sb[K];
#pragma unroll
        for (int k = 0; k < K; ++k) tb[k] = sb[k] = 0;
        if (r < n) {
            const int i = static_cast<int>(r % nx), j = static_cast<int>(r / nx);
            double acc[K];
#pragma unroll
            for (int k = 0; k < K; ++k) acc[k] = 0.0;
            for (int e = 0; e < nbits; ++e) {
                const int b = bits[e];
                const int dx = b % kBoxW - kBoxR, dv = b / kBoxW - kBoxR;
                const int ii = i + dx, jj = j + dv;
                const bool ok = ii >= 0 && ii < nx && jj >= 0 && jj < nv;
                const size_t nb = ok ? static_cast<size_t>(jj) * nx + ii : 0;
                double y[K];
#pragma unroll
                for (int k = 0; k < K; ++k) y[k] = 0.0;
                const int q0 = a.op.pair_begin[b], q1 = a.op.pair_begin[b + 1];
                for (int q = q0; q < q1; ++q) {
                    const int sl = a.op.pair_slot[q];
                    const double w = a.op.compressed
                                         ? a.op.w[(static_cast<size_t>(q) * nv + j) * kClasses + xclass(i, nx)]
                                         : a.op.w[static_cast<size_t>(q) * n + r];
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        const double cs = c[k][sl];
                        if (cs != 0.0) y[k] += cs * w;
                    }
                }
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const double x = ok && pk[k] >= 0 ? in[k][nb] : 0.0;
                    acc[k] += y[k] * x;
                }
            }
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (pk[k] < 0) continue;
                const double t = acc[k] * inv[k];
                const double sv = Sin[k][r] + t;
                Tout[k][r] = t;
                Sout[k][r] = sv;
                tb[k] = abs_bits(t);
                sb[k] = abs_bits(sv);
            }
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            tb[k] = warp_umax(tb[k]);
            sb[k] = warp_umax(sb[k]);
            if ((threadIdx.x & 31) == 0) {
                red[k][0][threadIdx.x >> 5] = tb[k];
                red[k][1][threadIdx.x >> 5] = sb[k];
            }
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            const int nw = (blockDim.x + 31) / 32;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                unsigned long long t2 = threadIdx.x < nw ? red[k][0][threadIdx.x] : 0ULL;
                unsigned long long s2 = threadIdx.x < nw ? red[k][1][threadIdx.x] : 0ULL;
                t2 = warp_umax(t2);
                s2 = warp_umax(s2);
                if (threadIdx.x == 0 && pk[k] >= 0) {
                    if (t2) atomicMax(&a.tn[pk[k]], t2);
                    if (s2) atomicMax(&a.sn[pk[k]], s2);
                }
            }
        }
    }
}

} // namespace

#ifndef S2B_GENK_K
#define S2B_GENK_K 4
#endif
bool generic_k_enabled() {
    const char* e = std::getenv("S2B_GENK");
    return !(e && e[0] == '0');
}

int grid_for(s2b_context* ctx, size_t work, int threads) {
    (void)threads;
    const size_t cap = static_cast<size_t>(ctx->num_sms) * 16;
    return static_cast<int>(std::max<size_t>(1, std::min(work, cap)));
}

// ---- operator preparation (host) ---------------------------------------------------
namespace {

struct SourceStencil {
    std::map<int, std::vector<double>> w; // bit -> full weight array (n)
};

} // namespace

s2b_operator* make_operator(s2b_context* ctx, const s2b_grid* grid, int order,
                            const s2b_csr sources[6]) {
    if (order < 1 || order > 3) fail(S2B_ERR_CONFIG, "operator: order must be in {1, 2, 3}");
    const size_t nx = grid->nx, nv = grid->nv, n = nx * nv;
    if (nx == 0 || nv == 0) fail(S2B_ERR_CONFIG, "operator: empty grid");
    static const int min_order[6] = {1, 1, 2, 2, 3, 3}; // slot_min_order, magnus.cpp:54
    std::vector<SourceStencil> st(6);
    int rx = 0, rv = 0;
    for (int s = 0; s < 6; ++s) {
        if (min_order[s] > order) continue;
        const s2b_csr& m = sources[s];
        if (m.rows == 0) fail(S2B_ERR_CONFIG, "operator: commutator set lacks a matrix required by the order");
        if (m.rows != n) fail(S2B_ERR_DIMENSION, "operator: matrix size does not match the grid");
        for (size_t r = 0; r < n; ++r) {
            const long long i = static_cast<long long>(r % nx), j = static_cast<long long>(r / nx);
            for (size_t q = m.row_ptr[r]; q < m.row_ptr[r + 1]; ++q) {
                const long long col = m.col_idx[q];
                if (col < 0 || static_cast<size_t>(col) >= n) fail(S2B_ERR_DIMENSION, "operator: column out of range");
                const long long dx = col % static_cast<long long>(nx) - i;
                const long long dv = col / static_cast<long long>(nx) - j;
                if (std::llabs(dx) > kBoxR || std::llabs(dv) > kBoxR)
                    fail(S2B_ERR_CONFIG, "operator: stencil radius exceeds 3 in x or v");
                rx = std::max<int>(rx, static_cast<int>(std::llabs(dx)));
                rv = std::max<int>(rv, static_cast<int>(std::llabs(dv)));
                const int b = box_bit(static_cast<int>(dx), static_cast<int>(dv));
                auto& arr = st[s].w[b];
                if (arr.empty()) arr.assign(n, 0.0);
                arr[r] = m.values[q];
            }
        }
    }
    auto* op = new s2b_operator();
    op->ctx = ctx;
    op->order = order;
    op->nx = nx;
    op->nv = nv;
    op->rx = rx;
    op->rv = rv;
    op->grid = *grid;
    op->dx_delta = (grid->bx - grid->ax) / static_cast<double>(nx + 1);
    op->dv_delta = (grid->bv - grid->av) / static_cast<double>(nv + 1);
    // pairs grouped by bit (ascending), slot order inside a bit
    op->pair_begin.assign(kBoxBits + 1, 0);
    std::vector<const std::vector<double>*> pw;
    for (int b = 0; b < kBoxBits; ++b) {
        op->pair_begin[b] = static_cast<int>(op->pair_slot.size());
        for (int s = 0; s < 6; ++s) {
            auto it = st[s].w.find(b);
            if (it == st[s].w.end()) continue;
            op->pair_slot.push_back(s);
            pw.push_back(&it->second);
            op->union_mask |= 1ULL << b;
        }
    }
    op->pair_begin[kBoxBits] = static_cast<int>(op->pair_slot.size());
    op->npairs = static_cast<int>(op->pair_slot.size());
    for (size_t q = 0; q < pw.size() && op->wfinite; ++q)
        for (double v : *pw[q])
            if (!std::isfinite(v)) {
                op->wfinite = false;
                break;
            }

    // x-invariance check: W(i, j) == W(class representative, j) bitwise for every pair
    bool comp = nx >= 5;
    auto rep = [&](size_t i) -> size_t { return (i >= 2 && i + 2 < nx) ? 2 : i; };
    for (size_t q = 0; comp && q < pw.size(); ++q) {
        const auto& w = *pw[q];
        for (size_t j = 0; comp && j < nv; ++j)
            for (size_t i = 0; i < nx; ++i)
                if (std::memcmp(&w[j * nx + i], &w[j * nx + rep(i)], sizeof(double)) != 0) {
                    comp = false;
                    break;
                }
    }
    op->compressed = comp ? 1 : 0;
    std::vector<double> hw;
    if (comp) {
        hw.assign(static_cast<size_t>(op->npairs) * nv * kClasses, 0.0);
        const size_t cls_i[kClasses] = {0, 1, 2, nx - 2, nx - 1};
        for (size_t q = 0; q < pw.size(); ++q)
            for (size_t j = 0; j < nv; ++j)
                for (int c = 0; c < kClasses; ++c)
                    hw[(q * nv + j) * kClasses + c] = (*pw[q])[j * nx + cls_i[c]];
    } else {
        hw.assign(static_cast<size_t>(op->npairs) * n, 0.0);
        for (size_t q = 0; q < pw.size(); ++q) std::copy(pw[q]->begin(), pw[q]->end(), hw.begin() + q * n);
        // point-major copy for the term_var kernels: one row's weights are one contiguous block
        const size_t npp = static_cast<size_t>(op->npairs | 1);
        std::vector<double> hp(npp * n, 0.0);
        for (size_t q = 0; q < pw.size(); ++q)
            for (size_t r = 0; r < n; ++r) hp[r * npp + q] = (*pw[q])[r];
        op->d_wpm.alloc(hp.size());
        S2B_CUDA(cudaMemcpy(op->d_wpm.p, hp.data(), hp.size() * sizeof(double), cudaMemcpyHostToDevice));
    }
    op->d_w.alloc(hw.size());
    op->d_pair_begin.alloc(op->pair_begin.size());
    op->d_pair_slot.alloc(std::max<size_t>(1, op->pair_slot.size()));
    S2B_CUDA(cudaMemcpy(op->d_w.p, hw.data(), hw.size() * sizeof(double), cudaMemcpyHostToDevice));
    S2B_CUDA(cudaMemcpy(op->d_pair_begin.p, op->pair_begin.data(), op->pair_begin.size() * sizeof(int),
                        cudaMemcpyHostToDevice));
    if (!op->pair_slot.empty())
        S2B_CUDA(cudaMemcpy(op->d_pair_slot.p, op->pair_slot.data(), op->pair_slot.size() * sizeof(int),
                            cudaMemcpyHostToDevice));

    // kernel variant: compressed weights, even nx (16-byte rows), nx <= 1024, mask fits
    op->variant = 0;
    int max_pairs = 0;
    for (int b = 0; b < kBoxBits; ++b) max_pairs = std::max(max_pairs, op->pair_begin[b + 1] - op->pair_begin[b]);
    if (comp && nx % 2 == 0 && nx >= 6 && nx <= 1024 && max_pairs <= kPairSlots) {
        for (int v = 1; v < static_cast<int>(sizeof(kVariants) / sizeof(kVariants[0])); ++v) {
            if ((op->union_mask & ~kVariants[v].mask) == 0) {
                op->variant = v;
                break;
            }
        }
    }
    if (op->variant) {
        // entry-major weights for the TMA kernel: q = cls * NBM + e over the variant's mask
        std::vector<int> e2bit;
        for (int b = 0; b < kBoxBits; ++b)
            if ((kVariants[op->variant].mask >> b) & 1) e2bit.push_back(b);
        const size_t nbm = e2bit.size(), nye = kClasses * nbm;
        std::vector<double> wt(nv * nye * kPairSlots, 0.0);
        std::vector<int> eslot(nye * kPairSlots, -1);
        for (int cls = 0; cls < kClasses; ++cls)
            for (size_t e = 0; e < nbm; ++e) {
                const size_t q = cls * nbm + e;
                const int b = e2bit[e];
                for (int pq = op->pair_begin[b], k = 0; pq < op->pair_begin[b + 1]; ++pq, ++k) {
                    eslot[q * kPairSlots + k] = op->pair_slot[pq];
                    for (size_t j = 0; j < nv; ++j)
                        wt[(j * nye + q) * kPairSlots + k] = hw[(static_cast<size_t>(pq) * nv + j) * kClasses + cls];
                }
            }
        // entries whose Y can differ between an x-boundary class and the interior, ignoring
        // offsets that leave the grid from that class (their neighbour is zero padding, so
        // the interior weight contributes the same +-0): the boundary warp loads only these
        // per lane and broadcasts the interior value for the rest
        const int cls_i[kClasses] = {0, 1, 2, static_cast<int>(nx) - 2, static_cast<int>(nx) - 1};
        op->bmask = 0;
        for (size_t e = 0; e < nbm; ++e) {
            const int dx = e2bit[e] % kBoxW - kBoxR;
            for (int cls : {0, 1, 3, 4}) {
                const int i = cls_i[cls];
                if (i + dx < 0 || i + dx >= static_cast<int>(nx)) continue; // leaves the grid
                for (int k = 0; k < kPairSlots && !((op->bmask >> e) & 1); ++k)
                    for (size_t j = 0; j < nv; ++j) {
                        const double wb = wt[(j * nye + cls * nbm + e) * kPairSlots + k];
                        const double wi = wt[(j * nye + 2 * nbm + e) * kPairSlots + k];
                        if (std::memcmp(&wb, &wi, sizeof(double)) != 0) {
                            op->bmask |= 1u << e;
                            break;
                        }
                    }
            }
        }
        // a specialised variant of the same mask whose compile-time boundary set covers bmask
        // (same entry order, so wt/eslot stay valid)
        for (int v = 1; v < kNumVariants; ++v)
            if (kVariants[v].mask == kVariants[op->variant].mask && (op->bmask & ~kVariants[v].bm) == 0 &&
                __builtin_popcount(kVariants[v].bm) < __builtin_popcount(kVariants[op->variant].bm))
                op->variant = v;
        op->d_wt.alloc(wt.size());
        op->d_eslot.alloc(eslot.size());
        S2B_CUDA(cudaMemcpy(op->d_wt.p, wt.data(), wt.size() * sizeof(double), cudaMemcpyHostToDevice));
        S2B_CUDA(cudaMemcpy(op->d_eslot.p, eslot.data(), eslot.size() * sizeof(int), cudaMemcpyHostToDevice));
    }
    return op;
}

void operator_info(const s2b_operator* op, int64_t info[6]) {
    info[0] = __builtin_popcountll(op->union_mask);
    info[1] = op->compressed;
    info[2] = op->rx;
    info[3] = op->rv;
    info[4] = op->npairs;
    info[5] = op->order;
}

// ---- session -------------------------------------------------------------------
struct MagnusSession {
    s2b_context* ctx = nullptr;
    const s2b_operator* op = nullptr;
    const s2b_paths* paths = nullptr;
    s2b_magnus_config cfg{};
    std::vector<double> record_times;
    WindowPlan plan;
    size_t M = 0, n = 0, nwin = 0;
    int R = 0;
    int cur_window = 0; // all live paths are paused at this window boundary
    std::vector<double> phi;

    DevBuf<double> T[2], S[2];
    std::vector<DevBuf<double>> rec; // R-1 record buffers
    DevBuf<double*> rec_ptrs;
    DevBuf<double> ctab;
    DevBuf<int> stab;
    DevBuf<int> iv;              // win seg k nseg status par rec_next  (7 x M)
    DevBuf<double> prev;
    DevBuf<long long> terms, windows, segments;
    DevBuf<double> sx; // accumulator scratch of the in-place cluster engine
    int sx_slots = 0;
    DevBuf<int> cl_work;            // path counter of the cluster kernel in hybrid runs
    DevBuf<double> mom_part, mom;   // moments: chunk partials, result
    bool nz = false;                // the datum holds no -0.0
    cudaStream_t stream2 = nullptr; // streaming passes beside the cluster kernel (hybrid)
    DevBuf<unsigned long long> tn, sn;
    DevBuf<int> act[2];
    DevBuf<int> cnt;
    DevBuf<int4> recq;
    DevBuf<uint8_t> rec_status;
    DevBuf<long long> rec_steps;
    DevBuf<int> bits;
    int nbits = 0;
    int* h_cnt = nullptr; // pinned
    int cur = 0;          // which act[] is the input list
    bool timing = false;
    bool use_cluster = false; // cluster-resident engine (cluster_magnus.cu) for this operator
    bool external_prepare = false; // ctab/stab written by the caller (adaptive driver)
    bool phi_over_cap = false;     // max|phi| > blowup_norm_cap (zero-norm first windows blow up)
    // two-term streaming engine (term2_kernel.cuh): third accumulator for paths >= s2_lo
    DevBuf<double> S2;
    size_t s2_lo = 0;
    DevBuf<int> tpar;
    DevBuf<unsigned long long> tn2, sn2;
    bool finished = false;         // finish() moved the buffers out: every later call is refused
    // streaming x-march engine (term_xs.cu): T/S are x-major while its pass loop runs
    bool use_xs = false;
    bool xs_slice = false; // the hybrid run's streaming slice on the x-march engine
    bool xs_major = false;
    DevBuf<double> yg;   // the window's folded Y rows per path
    DevBuf<int4> xs_meta; // per live path of a pass: (path, k, parity, segments)
    std::vector<cudaEvent_t> ev;
    s2b_magnus_stats stats{};

    Ctl ctl(int win_stop) {
        Ctl c{};
        c.win = iv.p;
        c.seg = iv.p + M;
        c.k = iv.p + 2 * M;
        c.nseg = iv.p + 3 * M;
        c.status = iv.p + 4 * M;
        c.par = iv.p + 5 * M;
        c.rec_next = iv.p + 6 * M;
        c.prev = prev.p;
        c.terms = terms.p;
        c.windows = windows.p;
        c.segments = segments.p;
        c.tn = tn.p;
        c.sn = sn.p;
        c.act_in = act[cur].p;
        c.act_out = act[cur ^ 1].p;
        c.cnt = cnt.p;
        c.recq = recq.p;
        c.rec_status = rec_status.p;
        c.stab = stab.p;
        c.rec_steps = rec_steps.p;
        c.R = R;
        c.nwin = static_cast<int>(nwin);
        c.dt_steps = static_cast<int>(plan.dt_steps);
        c.win_stop = win_stop;
        c.tol = cfg.expmv_tol;
        c.cap = cfg.blowup_norm_cap;
        c.M = M;
        return c;
    }
};

} // namespace s2b

namespace s2b {

void session_reset(MagnusSession* s);

namespace {

void run_records(MagnusSession& s, const double* S2base = nullptr) {
    if (s.R <= 1) return;
    if (s.xs_major) {
        xs_records(s.ctx, s.cnt.p, s.recq.p, s.S[0].p, s.S[1].p, S2base, s.rec_ptrs.p, static_cast<int>(s.op->nx),
                   static_cast<int>(s.op->nv), s.M);
        return;
    }
    dim3 grid(static_cast<unsigned>(std::min<size_t>((s.n + 255) / 256, 64)), 64);
    record_kernel<<<grid, 256, 0, s.ctx->stream>>>(s.cnt.p, s.recq.p, s.S[0].p, s.S[1].p, s.rec_ptrs.p, s.n, S2base);
    S2B_LAUNCHED(s.ctx);
}

void swap_lists(MagnusSession& s) {
    swap_counts_kernel<<<1, 1, 0, s.ctx->stream>>>(s.cnt.p);
    S2B_LAUNCHED(s.ctx);
    s.cur ^= 1;
}

TermArgs term_args(MagnusSession& s) {
    TermArgs a{};
    a.op = OpView{s.op->d_pair_begin.p, s.op->d_pair_slot.p, s.op->d_w.p, static_cast<int>(s.op->nx),
                  static_cast<int>(s.op->nv), s.op->compressed, s.op->d_wpm.p};
    a.ctab = s.ctab.p;
    a.nwin = static_cast<int>(s.nwin);
    a.act = s.act[s.cur].p;
    a.cnt = s.cnt.p;
    a.win = s.iv.p;
    a.k = s.iv.p + 2 * s.M;
    a.nseg = s.iv.p + 3 * s.M;
    a.par = s.iv.p + 5 * s.M;
    a.T0 = s.T[0].p;
    a.T1 = s.T[1].p;
    a.S0 = s.S[0].p;
    a.S1 = s.S[1].p;
    a.tn = s.tn.p;
    a.sn = s.sn.p;
    {
        const char* e = std::getenv("S2B_STRIP");
        a.strip_rows = e ? std::max(8, std::atoi(e)) : kStripRows;
        // few paths (adaptive rounds, hybrid slices, small sweeps): shorter strips keep every SM busy
        if (!e)
            while (a.strip_rows > 16 &&
                   s.M * ((s.op->nv + a.strip_rows - 1) / a.strip_rows) < 4 * static_cast<size_t>(s.ctx->num_sms))
                a.strip_rows /= 2;
        // term_tma_kernel keeps the strip's Y rows in shared memory: cap J by the budget, with
        // balanced strips
        if (s.op->variant != 0) {
            const size_t jmax = tma_strip_cap(s.op->variant, s.op->nx);
            if (static_cast<size_t>(a.strip_rows) > jmax) {
                const size_t nstr = (s.op->nv + jmax - 1) / jmax;
                a.strip_rows = static_cast<int>((s.op->nv + nstr - 1) / nstr);
            }
        }
    }
    a.nstrips = static_cast<int>((s.op->nv + a.strip_rows - 1) / a.strip_rows);
    {
        const char* e = std::getenv("S2B_TMA_SYNC");
        const int g = e ? std::atoi(e) : 2;
        a.sync_g = g == 1 || g == 4 ? g : 2;
    }
    a.wt = s.op->d_wt.p;
    a.eslot = s.op->d_eslot.p;
    const uint64_t mask = kVariants[s.op->variant].mask;
    int e = 0;
    for (int b = 0; b < kBoxBits; ++b)
        if ((mask >> b) & 1) a.e2bit[e++] = static_cast<int8_t>(b);
    return a;
}

void launch_term(MagnusSession& s) {
    TermArgs a = term_args(s);
    const int variant = s.op->variant;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (s.timing) {
        S2B_CUDA(cudaEventCreate(&e0));
        S2B_CUDA(cudaEventCreate(&e1));
        S2B_CUDA(cudaEventRecord(e0, s.ctx->stream));
    }
    if (s.xs_major) {
        launch_term_xs(s.ctx, s.op, a, s.iv.p + s.M, s.yg.p, s.xs_meta.p, s.M, s.nz);
    } else if (variant == 0) {
        const int bs = 256;
        const size_t blocks_per_path = (s.n + bs - 1) / bs;
        const int grid = grid_for(s.ctx, s.M * blocks_per_path, bs);
        constexpr int kGenK = S2B_GENK_K; // live paths per work item (shares every weight load)
        const int grid_k = grid_for(s.ctx, (s.M + kGenK - 1) / kGenK * blocks_per_path, bs);
        if (term_var_supported(s.op))
            launch_term_var(s.ctx, s.op, a, s.M);
        else if (generic_k_enabled())
        {
            term_generic_k_kernel<kGenK><<<grid_k, bs, 0, s.ctx->stream>>>(a, s.bits.p, s.nbits);
            s.ctx->k_stream = reinterpret_cast<const void*>(term_generic_k_kernel<kGenK>);
        } else {
            term_generic_kernel<<<grid, bs, 0, s.ctx->stream>>>(a, s.bits.p, s.nbits);
            s.ctx->k_stream = reinterpret_cast<const void*>(term_generic_kernel);
        }
    } else {
        const int nye = kClasses * tma_popcount(variant);
        const int nt = static_cast<int>((std::max<size_t>((s.op->nx + 1) / 2, nye) + 31) / 32 * 32);
        const int H = kVariants[variant].rx <= 2 ? 2 : 4;
        const size_t rw = 2 * static_cast<size_t>(nt) + 2 * H;
        const size_t smem = tma_smem_fixed(variant, s.op->nx) + static_cast<size_t>(a.strip_rows) * ((nye + 1) & ~1) * 8;
        (void)rw;
        const size_t work = s.M * static_cast<size_t>(a.nstrips);
        if (nt <= 128)
            launch_term_nt128(s.ctx, variant, a, nt, smem, work);
        else if (nt <= 256)
            launch_term_nt256(s.ctx, variant, a, nt, smem, work);
        else
            launch_term_nt512(s.ctx, variant, a, nt, smem, work);
    }
    S2B_LAUNCHED(s.ctx);
    s.stats.term_launches += 1;
    if (s.timing) {
        S2B_CUDA(cudaEventRecord(e1, s.ctx->stream));
        s.ev.push_back(e0);
        s.ev.push_back(e1);
    }
}

// The two-term engine applies to the compressed Langevin stencils (variants 7-9, even nx up to
// 1024).  It is opt-in (S2B_TERM2=1): bitwise equal to the one-term passes, but measured slower
// on B200 -- 0.30 vs 0.66 of HBM at 1024^2 (512 threads spill at 128 registers), 6.30e8 vs
// 6.69e8 windows/s at cfg4 and 1.38e9 vs 1.41e9 at cfg2 as the hybrid slice (one 241-register
// CTA per SM: the per-row barrier and the fold are exposed) -- see DESIGN.md.
bool term2_enabled(const MagnusSession& s) {
    const char* e = std::getenv("S2B_TERM2");
    if (!(e && e[0] == '1')) return false;
    const int v = s.op->variant;
    return v >= 7 && v <= 9 && s.op->nx % 2 == 0 && s.op->nx >= 6 && s.op->nx <= 1024;
}

Term2Args term2_args(MagnusSession& s) {
    // S2 holds paths [s2_lo, M) only: its base pointer is offset so that S2 + p*n addresses path p
    return Term2Args{s.S2.p - s.s2_lo * s.n, s.tpar.p, s.tn2.p, s.sn2.p};
}

void launch_term2(MagnusSession& s) {
    TermArgs a = term_args(s);
    const Term2Args b = term2_args(s);
    const int variant = s.op->variant;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (s.timing) {
        S2B_CUDA(cudaEventCreate(&e0));
        S2B_CUDA(cudaEventCreate(&e1));
        S2B_CUDA(cudaEventRecord(e0, s.ctx->stream));
    }
    const int nye = kClasses * tma_popcount(variant);
    const int yst = (nye + 1) & ~1;
    const int nt = static_cast<int>((std::max<size_t>((s.op->nx + 1) / 2, nye) + 31) / 32 * 32);
    const int H = kVariants[variant].rx <= 2 ? 2 : 4;
    const size_t rw = s.op->nx + 2 * H;
    if (s.xs_major) {
        launch_term_xs2(s.ctx, s.op, a, b, s.iv.p + s.M, s.yg.p, s.xs_meta.p, s.M, s.nz);
        S2B_LAUNCHED(s.ctx);
        s.stats.term_launches += 1;
        if (s.timing) {
            S2B_CUDA(cudaEventRecord(e1, s.ctx->stream));
            s.ev.push_back(e0);
            s.ev.push_back(e1);
        }
        return;
    }
    const size_t smem = 128 + (kStages * rw + kStages * s.op->nx + 2 * rw + 8 * static_cast<size_t>(yst) +
                               static_cast<size_t>(kPairSlots) * nye) * 8;
    const size_t work = s.M * static_cast<size_t>(a.nstrips);
    if (nt <= 128)
        launch_term2_nt128(s.ctx, variant, a, b, nt, smem, work);
    else if (nt <= 256)
        launch_term2_nt256(s.ctx, variant, a, b, nt, smem, work);
    else
        launch_term2_nt512(s.ctx, variant, a, b, nt, smem, work);
    S2B_LAUNCHED(s.ctx);
    s.stats.term_launches += 1;
    if (s.timing) {
        S2B_CUDA(cudaEventRecord(e1, s.ctx->stream));
        s.ev.push_back(e0);
        s.ev.push_back(e1);
    }
}

void collect_timing(MagnusSession& s) {
    for (size_t q = 0; q + 1 < s.ev.size(); q += 2) {
        float ms = 0.f;
        S2B_CUDA(cudaEventElapsedTime(&ms, s.ev[q], s.ev[q + 1]));
        s.stats.term_kernel_ms += ms;
        cudaEventDestroy(s.ev[q]);
        cudaEventDestroy(s.ev[q + 1]);
    }
    s.ev.clear();
}

} // namespace

MagnusSession* session_create(s2b_context* ctx, const s2b_operator* op, const s2b_magnus_config* cfg,
                              const double* phi, const s2b_paths* paths) {
    if (cfg->order < 1 || cfg->order > 3 || cfg->order > op->order)
        fail(S2B_ERR_CONFIG, "solve_iterated_magnus: unsupported order");
    if (cfg->order != op->order)
        fail(S2B_ERR_CONFIG, "solve_iterated_magnus: operator was prepared for a different order");
    if (!(cfg->expmv_tol > 0.0)) fail(S2B_ERR_CONFIG, "expmv: tol must be positive");
    if (!(cfg->expmv_theta > 0.0)) fail(S2B_ERR_CONFIG, "expmv: theta must be positive");
    const size_t n = op->nx * op->nv;
    for (size_t i = 0; i < n; ++i)
        if (!std::isfinite(phi[i])) fail(S2B_ERR_CONFIG, "solve_iterated_magnus: non-finite datum");
    auto* s = new MagnusSession();
    try {
        s->ctx = ctx;
        s->op = op;
        s->paths = paths;
        s->cfg = *cfg;
        s->record_times.assign(cfg->record_times, cfg->record_times + cfg->n_record);
        s->cfg.record_times = s->record_times.data();
        s->plan = plan_windows(cfg->dt, cfg->T, paths->dt_leb, paths->steps, cfg->record_times,
                               cfg->n_record, "solver");
        s->M = paths->M;
        s->n = n;
        s->nwin = s->plan.total_steps / s->plan.dt_steps;
        s->R = static_cast<int>(s->plan.record_steps.size());
        {
            // S2B_ENGINE=stream|cluster overrides the automatic choice (A/B measurements)
            const char* eng = std::getenv("S2B_ENGINE");
            const bool ok = op->variant != 0 &&
                            cluster_engine_supported(op->variant, static_cast<int>(op->nx), static_cast<int>(op->nv));
            s->use_cluster = ok && !(eng && std::strcmp(eng, "stream") == 0);
            s->use_xs = !s->use_cluster && term_xs_supported(op);
            s->xs_slice = s->use_cluster && term_xs_slice_supported(op);
            if (s->use_cluster && cluster_xmi_supported(op->variant, static_cast<int>(op->nx), static_cast<int>(op->nv)))
                s->sx.alloc(cluster_xmi_scratch(static_cast<int>(op->nx), static_cast<int>(op->nv), &s->sx_slots));
        }
        s->phi.assign(phi, phi + n);
        {
            double mx = 0.0;
            for (size_t i = 0; i < n; ++i) mx = std::max(mx, std::fabs(phi[i]));
            s->phi_over_cap = mx > cfg->blowup_norm_cap;
        }
        s->nz = true;
        for (size_t i = 0; i < n && s->nz; ++i) s->nz = !(phi[i] == 0.0 && std::signbit(phi[i]));
        const size_t M = s->M;
        for (int b = 0; b < 2; ++b) {
            s->T[b].alloc(M * n);
            s->S[b].alloc(M * n);
        }
        std::vector<double*> rp;
        for (int r = 0; r + 1 < s->R; ++r) {
            s->rec.emplace_back(M * n);
            rp.push_back(s->rec.back().p);
        }
        s->rec_ptrs.alloc(std::max<size_t>(1, rp.size()));
        if (!rp.empty())
            S2B_CUDA(cudaMemcpy(s->rec_ptrs.p, rp.data(), rp.size() * sizeof(double*), cudaMemcpyHostToDevice));
        s->ctab.alloc(M * s->nwin * 6);
        s->stab.alloc(M * s->nwin);
        s->iv.alloc(7 * M);
        s->prev.alloc(M);
        s->terms.alloc(M);
        s->windows.alloc(M);
        s->segments.alloc(M);
        s->tn.alloc(M);
        s->sn.alloc(M);
        s->act[0].alloc(M);
        s->act[1].alloc(M);
        s->cnt.alloc(4);
        s->recq.alloc(M * std::max(1, s->R));
        s->rec_status.alloc(static_cast<size_t>(s->R) * M);
        s->rec_steps.alloc(s->R);
        std::vector<long long> rs(s->plan.record_steps.begin(), s->plan.record_steps.end());
        S2B_CUDA(cudaMemcpy(s->rec_steps.p, rs.data(), rs.size() * sizeof(long long), cudaMemcpyHostToDevice));
        std::vector<int> bits;
        for (int b = 0; b < kBoxBits; ++b)
            if ((op->union_mask >> b) & 1) bits.push_back(b);
        s->nbits = static_cast<int>(bits.size());
        s->bits.alloc(std::max<size_t>(1, bits.size()));
        if (!bits.empty())
            S2B_CUDA(cudaMemcpy(s->bits.p, bits.data(), bits.size() * sizeof(int), cudaMemcpyHostToDevice));
        S2B_CUDA(cudaMallocHost(&s->h_cnt, 4 * sizeof(int)));

        session_reset(s);
    } catch (...) {
        delete s;
        throw;
    }
    return s;
}

void session_reset(MagnusSession* s) {
    if (s->finished) fail(S2B_ERR_CONFIG, "magnus session: reset after finish (the buffers belong to the ensemble)");
    const size_t M = s->M, n = s->n;
    broadcast_rows(s->ctx, s->S[0].p, s->phi.data(), n, M);
    S2B_CUDA(cudaMemsetAsync(s->iv.p, 0, s->iv.bytes(), s->ctx->stream));
    S2B_CUDA(cudaMemsetAsync(s->rec_status.p, 1, s->rec_status.bytes(), s->ctx->stream));
    S2B_CUDA(cudaMemsetAsync(s->cnt.p, 0, s->cnt.bytes(), s->ctx->stream));
    S2B_CUDA(cudaMemsetAsync(s->terms.p, 0, s->terms.bytes(), s->ctx->stream));
    S2B_CUDA(cudaMemsetAsync(s->windows.p, 0, s->windows.bytes(), s->ctx->stream));
    S2B_CUDA(cudaMemsetAsync(s->segments.p, 0, s->segments.bytes(), s->ctx->stream));
    s->cur = 0;
    s->cur_window = 0;
    s->stats = s2b_magnus_stats{};
    s->stats.gridpoints = static_cast<double>(n);
    S2B_CUDA(cudaStreamSynchronize(s->ctx->stream));
}

// Functionals, logarithm weights and segment counts of windows [w0, w1) of every path,
// all in parallel in time, from the device path values as they are now.
void prepare_windows(MagnusSession* s, size_t w0, size_t w1) {
    const size_t M = s->M, nw = w1 - w0;
    if (nw == 0) return;
    const s2b_operator* op = s->op;
    const size_t total = M * nw;
    functionals_kernel<<<static_cast<unsigned>((total + 127) / 128), 128, 0, s->ctx->stream>>>(
        s->paths->d_values.p, s->paths->steps, M, s->plan.dt_steps, s->nwin, w0, nw,
        s->paths->dt_leb, s->cfg.order, s->ctab.p);
    S2B_LAUNCHED(s->ctx);
    OpView ov{op->d_pair_begin.p, op->d_pair_slot.p, op->d_w.p, static_cast<int>(op->nx),
              static_cast<int>(op->nv), op->compressed};
    for (size_t m0 = 0; m0 < M; m0 += (1u << 30) / nw) {
        const size_t mc = std::min<size_t>(M - m0, (1u << 30) / nw);
        norm_kernel<<<static_cast<unsigned>(mc * nw), 256, 0, s->ctx->stream>>>(
            ov, s->bits.p, s->nbits, op->rx, s->ctab.p + m0 * s->nwin * 6, s->nwin, w0, nw,
            s->cfg.expmv_theta, s->stab.p + m0 * s->nwin, nullptr);
        S2B_LAUNCHED(s->ctx);
    }
    if (w0 == 0 && s->phi_over_cap) {
        phi_cap_kernel<<<static_cast<unsigned>((M + 255) / 256), 256, 0, s->ctx->stream>>>(
            s->stab.p, static_cast<int>(s->nwin), s->iv.p + 4 * M, M);
        S2B_LAUNCHED(s->ctx);
    }
}

// The streaming pass engine over paths [p_lo, M): one Taylor term of every live path per
// pass, per-path state machines in control_kernel (see the file header).
// x-major <-> row-major for the streaming x-march engine: every path's current accumulator
// S[par[p]][p] is transposed into T[par[p]][p] (the term buffers are dead at a window boundary),
// then the S and T buffers trade places.
void xs_relayout(MagnusSession* s, bool to_xmajor, int p_lo = 0) {
    const int nx = static_cast<int>(s->op->nx), nv = static_cast<int>(s->op->nv);
    if (p_lo > 0) { // a hybrid slice: the cluster kernel owns paths [0, p_lo) of the same buffers
        xs_transpose_paths_inplace(s->ctx, s->S[0].p, s->S[1].p, s->iv.p + 5 * s->M, p_lo, s->M, nx);
        s->xs_major = to_xmajor;
        return;
    }
    xs_transpose_paths(s->ctx, s->S[0].p, s->S[1].p, s->T[0].p, s->T[1].p, s->iv.p + 5 * s->M, s->M,
                       to_xmajor ? nv : nx, to_xmajor ? nx : nv);
    std::swap(s->S[0].p, s->T[0].p);
    std::swap(s->S[1].p, s->T[1].p);
    s->xs_major = to_xmajor;
}

void stream_loop(MagnusSession* s, int stop, int p_lo) {
    const bool xs = p_lo == 0 ? s->use_xs : s->xs_slice;
    if (xs) {
        if (!s->yg.p) s->yg.alloc(term_xs_y_doubles(s->op, s->M));
        if (!s->xs_meta.p) s->xs_meta.alloc(s->M);
        xs_relayout(s, true, p_lo);
    }
    {
        // (re)activate every live path at the current window boundary; window 0 also
        // initialises the per-path state (parity, records, counters)
        Ctl c = s->ctl(stop);
        c.p_lo = p_lo;
        S2B_CUDA(cudaMemsetAsync(s->cnt.p, 0, s->cnt.bytes(), s->ctx->stream));
        init_kernel<<<static_cast<unsigned>((s->M + 127) / 128), 128, 0, s->ctx->stream>>>(c, s->cur_window);
        S2B_LAUNCHED(s->ctx);
        run_records(*s);
        swap_lists(*s);
    }
    int chunk = 4;
    while (true) {
        S2B_CUDA(cudaMemcpyAsync(s->h_cnt, s->cnt.p, sizeof(int), cudaMemcpyDeviceToHost, s->ctx->stream));
        S2B_CUDA(cudaStreamSynchronize(s->ctx->stream));
        if (s->timing) collect_timing(*s);
        if (s->h_cnt[0] == 0) break;
        for (int q = 0; q < chunk; ++q) {
            launch_term(*s);
            Ctl c = s->ctl(stop);
            control_kernel<<<static_cast<unsigned>((s->M + 255) / 256), 256, 0, s->ctx->stream>>>(c);
            S2B_LAUNCHED(s->ctx);
            run_records(*s);
            swap_lists(*s);
            s->stats.passes += 1;
        }
        chunk = std::min(chunk * 2, 64);
    }
    if (xs) xs_relayout(s, false, p_lo);
}

// The two-term streaming engine over paths [p_lo, M): two Taylor terms of every live path per
// pass (term2_kernel.cuh) and control2_kernel; afterwards every accumulator is moved back to
// S0/S1 (normalize2_kernel), so the session looks exactly as after one-term passes.
void stream_loop2(MagnusSession* s, int stop, int p_lo) {
    const size_t M = s->M, n = s->n;
    const bool xs = s->use_xs && p_lo == 0 && term_xs2_enabled();
    if (!s->S2.p || s->s2_lo != static_cast<size_t>(p_lo)) {
        s->S2.release();
        s->S2.alloc((M - p_lo) * n);
        s->s2_lo = p_lo;
    }
    if (!s->tpar.p) {
        s->tpar.alloc(M);
        s->tn2.alloc(M);
        s->sn2.alloc(M);
    }
    S2B_CUDA(cudaMemsetAsync(s->tpar.p, 0, s->tpar.bytes(), s->ctx->stream));
    S2B_CUDA(cudaMemsetAsync(s->tn2.p, 0, s->tn2.bytes(), s->ctx->stream));
    S2B_CUDA(cudaMemsetAsync(s->sn2.p, 0, s->sn2.bytes(), s->ctx->stream));
    const double* S2base = s->S2.p - s->s2_lo * n;
    if (xs) {
        if (!s->yg.p) s->yg.alloc(term_xs_y_doubles(s->op, s->M));
        if (!s->xs_meta.p) s->xs_meta.alloc(s->M);
        xs_relayout(s, true);
    }
    {
        Ctl c = s->ctl(stop);
        c.p_lo = p_lo;
        S2B_CUDA(cudaMemsetAsync(s->cnt.p, 0, s->cnt.bytes(), s->ctx->stream));
        init_kernel<<<static_cast<unsigned>((M + 127) / 128), 128, 0, s->ctx->stream>>>(c, s->cur_window);
        S2B_LAUNCHED(s->ctx);
        run_records(*s, S2base);
        swap_lists(*s);
    }
    int chunk = 2;
    while (true) {
        S2B_CUDA(cudaMemcpyAsync(s->h_cnt, s->cnt.p, sizeof(int), cudaMemcpyDeviceToHost, s->ctx->stream));
        S2B_CUDA(cudaStreamSynchronize(s->ctx->stream));
        if (s->timing) collect_timing(*s);
        if (s->h_cnt[0] == 0) break;
        for (int q = 0; q < chunk; ++q) {
            launch_term2(*s);
            Ctl c = s->ctl(stop);
            control2_kernel<<<static_cast<unsigned>((M + 255) / 256), 256, 0, s->ctx->stream>>>(c, term2_args(*s));
            S2B_LAUNCHED(s->ctx);
            run_records(*s, S2base);
            swap_lists(*s);
            s->stats.passes += 1;
        }
        chunk = std::min(chunk * 2, 32);
    }
    dim3 g(static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 64)), static_cast<unsigned>(std::min<size_t>(M - p_lo, 65535)));
    if (M > static_cast<size_t>(p_lo)) {
        normalize2_kernel<<<g, 256, 0, s->ctx->stream>>>(s->iv.p + 5 * M, S2base, s->S[0].p, n, M, p_lo);
        S2B_LAUNCHED(s->ctx);
        normalize2_flag_kernel<<<static_cast<unsigned>((M - p_lo + 255) / 256), 256, 0, s->ctx->stream>>>(
            s->iv.p + 5 * M, M, p_lo);
        S2B_LAUNCHED(s->ctx);
    }
    if (xs) xs_relayout(s, false);
}

// Hybrid split: the clusters of the x-march engines pack 15 x 8 (256^2) or 7 x 16 (512^2) per
// B200, leaving 28 / 36 of the 148 SMs idle; the streaming engine runs a slice of the paths
// concurrently on those SMs.  Measured best slices: 0.11-0.14 at 256^2 (+12%), 0.2 at 512^2
// (+17%).  S2B_HYBRID overrides the slice (0 disables).
double hybrid_fraction(const MagnusSession* s) {
    const char* e = std::getenv("S2B_HYBRID");
    if (e) return std::atof(e);
    const int v = s->op->variant, nx = static_cast<int>(s->op->nx), nv = static_cast<int>(s->op->nv);
    // the x-march streaming slice (term_xs_kernel) is 1.2-1.45x term_tma_kernel per SM, so it takes a
    // larger share: cfg2 1.375e9 (tma, 0.12) -> 1.485e9 windows/s (xs, 0.16), cfg4 6.48e8 (tma,
    // 0.20) -> 7.04e8 (xs, 0.25), same run (scripts/xs_hybrid.sh)
    if (cluster_xm_supported(v, nx, nv))
        return nx == 256 ? (s->xs_slice ? 0.16 : 0.12) : (nx == 128 ? 0.06 : 0.0); // 120 / 132 / 148 SMs busy
    if (cluster_xmi_supported(v, nx, nv)) return s->xs_slice ? 0.25 : 0.20;
    return 0.0;
}

ClusterArgs cluster_args(MagnusSession* s, int stop) {
    ClusterArgs a{};
    a.wt = s->op->d_wt.p;
    a.eslot = s->op->d_eslot.p;
    a.nx = static_cast<int>(s->op->nx);
    a.nv = static_cast<int>(s->op->nv);
    a.ctab = s->ctab.p;
    a.stab = s->stab.p;
    a.nwin = static_cast<int>(s->nwin);
    a.win0 = s->cur_window;
    a.win1 = stop;
    a.dt_steps = static_cast<int>(s->plan.dt_steps);
    a.S0 = s->S[0].p;
    a.S1 = s->S[1].p;
    a.win = s->iv.p;
    a.status = s->iv.p + 4 * s->M;
    a.par = s->iv.p + 5 * s->M;
    a.rec_next = s->iv.p + 6 * s->M;
    a.terms = s->terms.p;
    a.windows = s->windows.p;
    a.segments = s->segments.p;
    a.rec = s->rec_ptrs.p;
    a.rec_status = s->rec_status.p;
    a.rec_steps = s->rec_steps.p;
    a.R = s->R;
    a.tol = s->cfg.expmv_tol;
    a.cap = s->cfg.blowup_norm_cap;
    a.M = static_cast<int>(s->M);
    a.work = s->cnt.p + 3;
    a.sx = s->sx.p;
    a.sx_slots = s->sx_slots;
    a.nz = s->nz ? 1 : 0;
    return a;
}

// Advance several sessions to their ends in batched persistent launches (a step-size sweep
// on shared paths: run_stepsize_sweep, experiment.cpp:486-551).  Sessions on the x-march
// engines share one launch per kMaxBatch; any other engine runs its sessions one by one.
void sessions_run_batched(MagnusSession* const* ss, int n) {
    int i = 0;
    while (i < n) {
        MagnusSession* s0 = ss[i];
        const int v = s0->op->variant, nx = static_cast<int>(s0->op->nx), nv = static_cast<int>(s0->op->nv);
        if (!s0->use_cluster || !cluster_batch_supported(v, nx, nv)) {
            session_advance(s0, s0->nwin);
            ++i;
            continue;
        }
        ClusterBatch cb{};
        cb.n = 0;
        cb.prefix[0] = 0;
        int j = i;
        for (; j < n && cb.n < kMaxBatch; ++j) {
            MagnusSession* s = ss[j];
            if (!s->use_cluster || s->op != s0->op || static_cast<size_t>(s->cur_window) >= s->nwin) break;
            if (!s->external_prepare) prepare_windows(s, s->cur_window, s->nwin);
            cb.a[cb.n] = cluster_args(s, static_cast<int>(s->nwin));
            cb.prefix[cb.n + 1] = cb.prefix[cb.n] + static_cast<int>(s->M);
            ++cb.n;
        }
        if (cb.n == 0) { // session already finished (or a different operator): plain path
            session_advance(s0, s0->nwin);
            ++i;
            continue;
        }
        cb.total = cb.prefix[cb.n];
        S2B_CUDA(cudaMemsetAsync(cb.a[0].work, 0, sizeof(int), s0->ctx->stream));
        launch_cluster_magnus(s0->ctx, v, cb);
        S2B_CUDA(cudaStreamSynchronize(s0->ctx->stream));
        for (int q = i; q < j; ++q) {
            ss[q]->stats.term_launches += 1;
            ss[q]->cur_window = static_cast<int>(ss[q]->nwin);
        }
        i = j;
    }
}

void session_advance(MagnusSession* s, size_t n_windows) {
    if (s->finished) fail(S2B_ERR_CONFIG, "magnus session: advance after finish");
    if (n_windows == 0 || static_cast<size_t>(s->cur_window) >= s->nwin) return;
    const int stop = static_cast<int>(std::min(s->nwin, s->cur_window + n_windows));
    if (!s->external_prepare) prepare_windows(s, s->cur_window, stop);
    const double hf = s->use_cluster ? hybrid_fraction(s) : 0.0;
    int Ms = (hf > 0.0 && hf < 1.0 && s->M >= 64 &&
              cluster_batch_supported(s->op->variant, static_cast<int>(s->op->nx), static_cast<int>(s->op->nv)))
                 ? static_cast<int>(static_cast<double>(s->M) * hf) : 0;
    // a slice of fewer than 64 paths is launch-bound (one pass per Taylor term, ~300 per window,
    // each a few microseconds of work): it would outlast the cluster kernel, so small runs stay
    // on the cluster engine alone (an explicit S2B_HYBRID keeps any slice, for A/B runs)
    if (Ms < 64 && !std::getenv("S2B_HYBRID")) Ms = 0;
    if (s->use_cluster && Ms > 0) {
        // hybrid: paths [0, M1) on the cluster engine (stream 1), [M1, M) on the streaming
        // engine concurrently (stream 2, on the SMs the clusters leave idle)
        const int M1 = static_cast<int>(s->M) - Ms;
        s->stats.hybrid_paths = Ms;
        if (!s->stream2) S2B_CUDA(cudaStreamCreateWithFlags(&s->stream2, cudaStreamNonBlocking));
        if (!s->cl_work.p) s->cl_work.alloc(1);
        cudaStream_t st1 = s->ctx->stream;
        ClusterBatch cb{};
        cb.a[0] = cluster_args(s, stop); // a.M stays the record-status stride; total bounds the run
        cb.a[0].work = s->cl_work.p;
        cb.n = 1;
        cb.prefix[0] = 0;
        cb.prefix[1] = cb.total = M1;
        S2B_CUDA(cudaMemsetAsync(s->cl_work.p, 0, sizeof(int), st1));
        cudaEvent_t prep, done, e0 = nullptr, e1 = nullptr;
        S2B_CUDA(cudaEventCreateWithFlags(&prep, cudaEventDisableTiming));
        S2B_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
        S2B_CUDA(cudaEventRecord(prep, st1));
        if (s->timing) {
            S2B_CUDA(cudaEventCreate(&e0));
            S2B_CUDA(cudaEventCreate(&e1));
            S2B_CUDA(cudaEventRecord(e0, st1));
        }
        launch_cluster_magnus(s->ctx, s->op->variant, cb);
        s->stats.term_launches += 1;
        // the streaming passes: the same session state, a context view on stream 2
        s2b_context c2 = *s->ctx;
        c2.stream = s->stream2;
        s2b_context* c1 = s->ctx;
        const bool tim = s->timing;
        S2B_CUDA(cudaStreamWaitEvent(s->stream2, prep, 0));
        s->ctx = &c2;
        s->timing = false;
        try {
            if (term2_enabled(*s))
                stream_loop2(s, stop, M1);
            else
                stream_loop(s, stop, M1);
        } catch (...) {
            s->ctx = c1;
            s->timing = tim;
            cudaStreamSynchronize(st1); // the cluster kernel still owns the session buffers
            cudaStreamSynchronize(s->stream2);
            cudaEventDestroy(prep);
            cudaEventDestroy(done);
            throw;
        }
        s->ctx = c1;
        s->timing = tim;
        c1->launches = c2.launches;
        c1->k_stream = c2.k_stream;
        S2B_CUDA(cudaEventRecord(done, s->stream2));
        S2B_CUDA(cudaStreamWaitEvent(st1, done, 0));
        if (s->timing) {
            S2B_CUDA(cudaEventRecord(e1, st1));
            s->ev.push_back(e0);
            s->ev.push_back(e1);
        }
        S2B_CUDA(cudaStreamSynchronize(st1));
        cudaEventDestroy(prep);
        cudaEventDestroy(done);
        if (s->timing) collect_timing(*s);
        s->cur_window = stop;
        return;
    }
    if (s->use_cluster) {
        // cluster-resident engine: every live path runs windows [cur, stop) on chip
        ClusterBatch cb{};
        cb.a[0] = cluster_args(s, stop);
        cb.n = 1;
        cb.prefix[0] = 0;
        cb.prefix[1] = cb.total = static_cast<int>(s->M);
        S2B_CUDA(cudaMemsetAsync(s->cnt.p + 3, 0, sizeof(int), s->ctx->stream));
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (s->timing) {
            S2B_CUDA(cudaEventCreate(&e0));
            S2B_CUDA(cudaEventCreate(&e1));
            S2B_CUDA(cudaEventRecord(e0, s->ctx->stream));
        }
        launch_cluster_magnus(s->ctx, s->op->variant, cb);
        s->stats.term_launches += 1;
        if (s->timing) {
            S2B_CUDA(cudaEventRecord(e1, s->ctx->stream));
            s->ev.push_back(e0);
            s->ev.push_back(e1);
        }
        S2B_CUDA(cudaStreamSynchronize(s->ctx->stream));
        if (s->timing) collect_timing(*s);
        s->cur_window = stop;
        return;
    }
    if (term2_enabled(*s) || (s->use_xs && term_xs2_enabled()))
        stream_loop2(s, stop, 0);
    else
        stream_loop(s, stop, 0);
    s->cur_window = stop;
}

void session_stats(const MagnusSession* s, s2b_magnus_stats* out) {
    if (s->finished) fail(S2B_ERR_CONFIG, "magnus session: stats after finish (read them from the ensemble)");
    *out = s->stats;
    std::vector<long long> t(s->M), w(s->M);
    S2B_CUDA(cudaMemcpy(t.data(), s->terms.p, s->M * sizeof(long long), cudaMemcpyDeviceToHost));
    S2B_CUDA(cudaMemcpy(w.data(), s->windows.p, s->M * sizeof(long long), cudaMemcpyDeviceToHost));
    std::vector<long long> g(s->M);
    S2B_CUDA(cudaMemcpy(g.data(), s->segments.p, s->M * sizeof(long long), cudaMemcpyDeviceToHost));
    out->path_terms = 0;
    out->path_windows = 0;
    out->path_segments = 0;
    {
        const int v = s->op->variant, nx = static_cast<int>(s->op->nx), nv = static_cast<int>(s->op->nv);
        out->engine = !s->use_cluster ? 0
                      : cluster_xm_supported(v, nx, nv) ? 2
                      : cluster_xmi_supported(v, nx, nv) ? 3 : 1;
    }
    for (size_t m = 0; m < s->M; ++m) {
        out->path_terms += t[m];
        out->path_windows += w[m];
        out->path_segments += g[m];
    }
}

void session_set_timing(MagnusSession* s, bool on) { s->timing = on; }

namespace {
__global__ void gather_kernel(const int* __restrict__ par, const double* __restrict__ S0,
                              const double* __restrict__ S1, double* __restrict__ dst, size_t n,
                              size_t M) {
    for (size_t m = blockIdx.y; m < M; m += gridDim.y) {
        const double* src = (par[m] ? S1 : S0) + m * n;
        double* d = dst + m * n;
        for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
             i += static_cast<size_t>(gridDim.x) * blockDim.x)
            d[i] = src[i];
    }
}
__global__ void live_status_kernel(const int* __restrict__ status, uint8_t* __restrict__ out, size_t M) {
    const size_t m = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (m < M) out[m] = status[m] == 2 ? 1 : 0;
}
} // namespace

s2b_ensemble* session_snapshot(MagnusSession* s) {
    if (s->finished) fail(S2B_ERR_CONFIG, "magnus session: snapshot after finish");
    auto* e = new s2b_ensemble();
    e->ctx = s->ctx;
    e->R = 1;
    e->M = s->M;
    e->nx = s->op->nx;
    e->nv = s->op->nv;
    e->seed = s->paths->seed;
    e->grid = s->op->grid;
    e->times.push_back(static_cast<double>(s->cur_window * s->plan.dt_steps) * s->paths->dt_leb);
    e->states.emplace_back(s->M * s->n);
    e->status.alloc(s->M);
    dim3 g(static_cast<unsigned>(std::min<size_t>((s->n + 255) / 256, 128)), static_cast<unsigned>(std::min<size_t>(s->M, 65535)));
    gather_kernel<<<g, 256, 0, s->ctx->stream>>>(s->iv.p + 5 * s->M, s->S[0].p, s->S[1].p, e->states[0].p, s->n, s->M);
    S2B_LAUNCHED(s->ctx);
    live_status_kernel<<<static_cast<unsigned>((s->M + 255) / 256), 256, 0, s->ctx->stream>>>(s->iv.p + 4 * s->M, e->status.p, s->M);
    S2B_LAUNCHED(s->ctx);
    e->terms.alloc(s->M);
    e->windows.alloc(s->M);
    S2B_CUDA(cudaMemcpyAsync(e->terms.p, s->terms.p, s->M * sizeof(long long), cudaMemcpyDeviceToDevice, s->ctx->stream));
    S2B_CUDA(cudaMemcpyAsync(e->windows.p, s->windows.p, s->M * sizeof(long long), cudaMemcpyDeviceToDevice, s->ctx->stream));
    S2B_CUDA(cudaStreamSynchronize(s->ctx->stream));
    return e;
}

s2b_ensemble* session_finish(MagnusSession* s) {
    if (s->finished) fail(S2B_ERR_CONFIG, "magnus session: finish called twice");
    if (static_cast<size_t>(s->cur_window) < s->nwin) session_advance(s, s->nwin - s->cur_window);
    auto* e = new s2b_ensemble();
    e->ctx = s->ctx;
    e->R = s->R;
    e->M = s->M;
    e->nx = s->op->nx;
    e->nv = s->op->nv;
    e->seed = s->paths->seed;
    e->grid = s->op->grid;
    for (size_t r = 0; r < static_cast<size_t>(s->R); ++r)
        e->times.push_back(static_cast<double>(s->plan.record_steps[r]) * s->paths->dt_leb);
    for (auto& b : s->rec) e->states.push_back(std::move(b));
    s->rec.clear();
    // final record: gather the current buffers into T[0]'s storage (no longer needed)
    DevBuf<double> fin = std::move(s->T[0]);
    dim3 g(static_cast<unsigned>(std::min<size_t>((s->n + 255) / 256, 128)), static_cast<unsigned>(std::min<size_t>(s->M, 65535)));
    gather_kernel<<<g, 256, 0, s->ctx->stream>>>(s->iv.p + 5 * s->M, s->S[0].p, s->S[1].p, fin.p, s->n, s->M);
    S2B_LAUNCHED(s->ctx);
    e->states.push_back(std::move(fin));
    e->status = std::move(s->rec_status);
    e->terms = std::move(s->terms);
    e->windows = std::move(s->windows);
    s->finished = true;
    S2B_CUDA(cudaStreamSynchronize(s->ctx->stream));
    return e;
}

namespace {
// sum_m u_m and sum_m u_m^2 over live (not blown) paths, ascending m, reading each path's
// current buffer; the statistic the multi-GPU path all-reduces.
// Two levels, deterministic: chunks of kMomChunk paths per block (ascending m inside a chunk),
// then the chunk partials summed in ascending chunk order.  One thread per point would walk
// all M paths serially (latency-bound, and page-hopping 512 KB per step).
constexpr int kMomChunk = 64;
__global__ void session_moments_kernel(const int* __restrict__ par, const int* __restrict__ status,
                                       const double* __restrict__ S0, const double* __restrict__ S1,
                                       size_t M, size_t n, double* __restrict__ part) {
    const size_t r = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (r >= n) return;
    const size_t m0 = static_cast<size_t>(blockIdx.y) * kMomChunk;
    const size_t m1 = m0 + kMomChunk < M ? m0 + kMomChunk : M;
    double s1 = 0.0, s2 = 0.0;
#pragma unroll 8
    for (size_t m = m0; m < m1; ++m) {
        const double u = (par[m] ? S1 : S0)[m * n + r];
        if (status[m] == 2) continue;
        s1 += u;
        s2 += u * u;
    }
    part[blockIdx.y * 2 * n + r] = s1;
    part[blockIdx.y * 2 * n + n + r] = s2;
}
__global__ void moments_finish_kernel(const double* __restrict__ part, size_t nch, size_t n, double* __restrict__ mom) {
    const size_t r = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (r >= 2 * n) return;
    double acc = 0.0;
    for (size_t c = 0; c < nch; ++c) acc += part[c * 2 * n + r];
    mom[r] = acc;
}
} // namespace

void session_moments(MagnusSession* s, double* host_out, double* live_out) {
    if (s->finished) fail(S2B_ERR_CONFIG, "magnus session: moments after finish");
    const size_t nch = (s->M + kMomChunk - 1) / kMomChunk;
    if (s->mom_part.n < nch * 2 * s->n) s->mom_part.alloc(nch * 2 * s->n);
    if (s->mom.n < 2 * s->n) s->mom.alloc(2 * s->n);
    dim3 g(static_cast<unsigned>((s->n + 255) / 256), static_cast<unsigned>(nch));
    session_moments_kernel<<<g, 256, 0, s->ctx->stream>>>(s->iv.p + 5 * s->M, s->iv.p + 4 * s->M, s->S[0].p,
                                                          s->S[1].p, s->M, s->n, s->mom_part.p);
    S2B_LAUNCHED(s->ctx);
    moments_finish_kernel<<<static_cast<unsigned>((2 * s->n + 255) / 256), 256, 0, s->ctx->stream>>>(
        s->mom_part.p, nch, s->n, s->mom.p);
    S2B_LAUNCHED(s->ctx);
    S2B_CUDA(cudaMemcpyAsync(host_out, s->mom.p, 2 * s->n * sizeof(double), cudaMemcpyDeviceToHost, s->ctx->stream));
    std::vector<int> st(s->M);
    S2B_CUDA(cudaMemcpyAsync(st.data(), s->iv.p + 4 * s->M, s->M * sizeof(int), cudaMemcpyDeviceToHost, s->ctx->stream));
    S2B_CUDA(cudaStreamSynchronize(s->ctx->stream));
    if (live_out) {
        size_t live = 0;
        for (int v : st) live += v != 2;
        *live_out = static_cast<double>(live);
    }
}

void session_destroy(MagnusSession* s) {
    if (!s) return;
    if (s->stream2) cudaStreamDestroy(s->stream2);
    for (auto ev : s->ev) cudaEventDestroy(ev);
    if (s->h_cnt) cudaFreeHost(s->h_cnt);
    delete s;
}

// ---- solve_adaptive_magnus (magnus.cpp:306-404) ------------------------------------
//
// Per path: attempt the window [k0, k0+len) at orders 3 and 2 from one functional build,
// accept the order-3 result when both expmv calls succeed and max|u3-u2| / max|u3| <= tau,
// otherwise shrink len by `shrink` (below one Lebesgue step: blown).  Accepted windows never
// cross a record time.  On the GPU every live path makes one attempt per round: the
// attempt's six weights go into a one-window session (any Magnus engine), which runs twice
// (Y3, then Y2 on the same input); a block per path reduces the gap and decides.  Paths
// that finished or blew up sit the round out (status 2 -> skipped by every engine).
namespace {

__device__ void window_weights(const double* p, long long k0, long long L, double dt, double c3[6], double c2[6]) {
    // lebesgue_functionals (stochastics.cpp:121-141) + log_coefficients (magnus.cpp:26-40)
    const double base = p[k0];
    double iw = 0.0, isw = 0.0, iw2 = 0.0;
    for (long long j = 0; j < L; ++j) {
        const double wv = p[k0 + j] - base;
        const double sj = static_cast<double>(j) * dt;
        iw += wv;
        isw += sj * wv;
        iw2 += wv * wv;
    }
    const double h = static_cast<double>(L) * dt;
    const double W = p[k0 + L] - p[k0];
    const double IW = iw * dt, IsW = isw * dt, IW2 = iw2 * dt;
    c3[0] = c2[0] = h;
    c3[1] = c2[1] = W;
    c3[2] = c2[2] = -0.5 * h;
    c3[3] = c2[3] = IW - 0.5 * h * W;
    c3[4] = 0.5 * IW2 - 0.5 * W * IW + h * W * W / 12.0;
    c3[5] = IsW - 0.5 * h * IW - h * h * W / 12.0;
    c2[4] = c2[5] = 0.0;
}

struct AdArgs {
    const double* values;
    size_t vstride;
    size_t M, n;
    double dt_leb;
    long long dt_steps, total;
    const long long* rec_steps;
    int R;
    long long* k0;
    long long* len;
    int* fresh;
    int* flags; // 0 live, 1 done, 2 blown
    int* rec;   // next record
    int* rec_lo;
    int* rec_hi;
    int* accept;
    double* ctab3;
    double* ctab2;
    int* live;
    double tau, shrink, cap;
};

__global__ void ad_prepare_kernel(AdArgs a) {
    const size_t m = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (m >= a.M) return;
    double* c3 = a.ctab3 + m * 6;
    double* c2 = a.ctab2 + m * 6;
    if (a.flags[m] != 0) {
        for (int q = 0; q < 6; ++q) c3[q] = c2[q] = 0.0;
        return;
    }
    if (a.fresh[m]) { // never step across the next record boundary
        const long long to_rec = a.rec_steps[a.rec[m]] - a.k0[m];
        a.len[m] = a.dt_steps < to_rec ? a.dt_steps : to_rec;
        a.fresh[m] = 0;
    }
    double w3[6], w2[6];
    window_weights(a.values + m * a.vstride, a.k0[m], a.len[m], a.dt_leb, w3, w2);
    for (int q = 0; q < 6; ++q) {
        c3[q] = w3[q];
        c2[q] = w2[q];
    }
    atomicAdd(a.live, 1);
}

// session control block for one attempt run: every live path at window 0 of parity 0
__global__ void ad_reset_kernel(int* iv, size_t M, const int* flags) {
    const size_t m = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (m >= M) return;
    for (int f = 0; f < 7; ++f) iv[f * M + m] = 0;
    iv[4 * M + m] = flags[m] != 0 ? 2 : 0;
}

__global__ void ad_save_status_kernel(const int* status, int* out, size_t M) {
    const size_t m = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (m < M) out[m] = status[m];
}

// gap = max|u3 - u2| / max|u3| (or the diff when max|u3| == 0) and the accept/shrink rule
__global__ void ad_gap_kernel(AdArgs a, const double* __restrict__ u3, const double* __restrict__ S0,
                              const double* __restrict__ S1, const int* __restrict__ par,
                              const int* __restrict__ st3, const int* __restrict__ st2) {
    __shared__ unsigned long long red[2][32];
    for (size_t m = blockIdx.x; m < a.M; m += gridDim.x) {
        if (a.flags[m] != 0) {
            if (threadIdx.x == 0) a.accept[m] = 0;
            continue;
        }
        bool ok = st3[m] != 2 && st2[m] != 2;
        unsigned long long db = 0, sb = 0;
        if (ok) { // both results finite (expmv Ok): the max is order independent on the bits
            const double* x3 = u3 + m * a.n;
            const double* x2 = (par[m] ? S1 : S0) + m * a.n;
            for (size_t i = threadIdx.x; i < a.n; i += blockDim.x) {
                db = umax64(db, abs_bits(x3[i] - x2[i]));
                sb = umax64(sb, abs_bits(x3[i]));
            }
        }
        db = warp_umax(db);
        sb = warp_umax(sb);
        if ((threadIdx.x & 31) == 0) {
            red[0][threadIdx.x >> 5] = db;
            red[1][threadIdx.x >> 5] = sb;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (unsigned q = 1; q < blockDim.x / 32; ++q) {
                db = umax64(db, red[0][q]);
                sb = umax64(sb, red[1][q]);
            }
            db = umax64(db, red[0][0]);
            sb = umax64(sb, red[1][0]);
            double gap = __longlong_as_double(static_cast<long long>(kInfBits));
            const double diff = __longlong_as_double(static_cast<long long>(db));
            const double scale = __longlong_as_double(static_cast<long long>(sb));
            if (ok) {
                gap = scale > 0.0 ? diff / scale : diff;
                ok = isfinite(gap);
            }
            if (ok && gap <= a.tau) {
                a.accept[m] = 1;
                a.k0[m] += a.len[m];
                a.fresh[m] = 1;
                int r = a.rec[m];
                a.rec_lo[m] = r;
                if (!isfinite(scale) || scale > a.cap) {
                    a.flags[m] = 2; // magnus.cpp:360-363
                } else {
                    while (r < a.R && a.rec_steps[r] == a.k0[m]) ++r;
                    if (a.k0[m] >= a.total) a.flags[m] = 1;
                }
                a.rec_hi[m] = r;
                a.rec[m] = r;
            } else {
                a.accept[m] = 0;
                const long long shrunk = static_cast<long long>(static_cast<double>(a.len[m]) * a.shrink);
                if (shrunk < 1) a.flags[m] = 2; // cannot refine below the Lebesgue grid
                else a.len[m] = shrunk;
            }
        }
        __syncthreads();
    }
}

// accepted paths: u <- u3, and the record snapshots taken at the new k0
__global__ void ad_commit_kernel(AdArgs a, const double* __restrict__ u3, double* __restrict__ U,
                                 double* const* __restrict__ recs, uint8_t* __restrict__ rec_status) {
    for (size_t m = blockIdx.y; m < a.M; m += gridDim.y) {
        if (!a.accept[m]) continue;
        const int lo = a.rec_lo[m], hi = a.rec_hi[m];
        const double* src = u3 + m * a.n;
        for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < a.n;
             i += static_cast<size_t>(gridDim.x) * blockDim.x) {
            const double v = src[i];
            U[m * a.n + i] = v;
            for (int r = lo; r < hi && r < a.R - 1; ++r) recs[r][m * a.n + i] = v;
        }
        if (blockIdx.x == 0 && threadIdx.x == 0)
            for (int r = lo; r < hi; ++r) rec_status[static_cast<size_t>(r) * a.M + m] = 0;
    }
}

} // namespace

s2b_ensemble* solve_adaptive(s2b_context* ctx, const s2b_operator* op, const s2b_magnus_config* cfg,
                             const s2b_adaptive_config* ad, const double* phi, const s2b_paths* paths,
                             s2b_magnus_stats* stats) {
    if (!ad || !ad->enabled) fail(S2B_ERR_CONFIG, "solve_adaptive_magnus: adaptive flag not set");
    if (!(ad->shrink > 0.0 && ad->shrink < 1.0))
        fail(S2B_ERR_CONFIG, "solve_adaptive_magnus: shrink factor must lie in (0, 1)");
    if (op->order < 3) fail(S2B_ERR_CONFIG, "solve_adaptive_magnus: needs order-3 commutators");
    const WindowPlan plan = plan_windows(cfg->dt, cfg->T, paths->dt_leb, paths->steps, cfg->record_times,
                                         cfg->n_record, "solver");
    const size_t M = paths->M, n = op->nx * op->nv;
    const int R = static_cast<int>(plan.record_steps.size());
    // the attempt runner: a one-window session (window = one Lebesgue step; the weights are
    // supplied per attempt), no norm cap inside (the cap applies to accepted windows only)
    s2b_magnus_config c1 = *cfg;
    c1.order = 3;
    c1.dt = paths->dt_leb;
    c1.T = paths->dt_leb;
    c1.blowup_norm_cap = HUGE_VAL;
    c1.record_times = nullptr;
    c1.n_record = 0;
    // s runs the order-3 attempts, s2 the order-2 ones: one batched launch carries both
    MagnusSession* s = session_create(ctx, op, &c1, phi, paths);
    MagnusSession* s2 = nullptr;
    auto* e = new s2b_ensemble();
    try {
        s2 = session_create(ctx, op, &c1, phi, paths);
        s->external_prepare = true;
        s2->external_prepare = true;
        e->ctx = ctx;
        e->R = R;
        e->M = M;
        e->nx = op->nx;
        e->nv = op->nv;
        e->seed = paths->seed;
        e->grid = op->grid;
        for (size_t r : plan.record_steps) e->times.push_back(static_cast<double>(r) * paths->dt_leb);
        e->status.alloc(static_cast<size_t>(R) * M);
        S2B_CUDA(cudaMemsetAsync(e->status.p, 1, e->status.bytes(), ctx->stream));
        for (int r = 0; r + 1 < R; ++r) e->states.emplace_back(M * n);
        DevBuf<double> U(M * n), A(M * n), ctab2(M * 6);
        broadcast_rows(ctx, U.p, phi, n, M);
        DevBuf<long long> k0(M), len(M), rsteps(R);
        DevBuf<int> fresh(M), flags(M), rec(M), rlo(M), rhi(M), acc(M), st3(M), live(1);
        std::vector<int> ones(M, 1);
        S2B_CUDA(cudaMemsetAsync(k0.p, 0, k0.bytes(), ctx->stream));
        S2B_CUDA(cudaMemcpyAsync(fresh.p, ones.data(), M * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
        S2B_CUDA(cudaMemsetAsync(flags.p, 0, flags.bytes(), ctx->stream));
        S2B_CUDA(cudaMemsetAsync(rec.p, 0, rec.bytes(), ctx->stream));
        std::vector<long long> rs(plan.record_steps.begin(), plan.record_steps.end());
        S2B_CUDA(cudaMemcpyAsync(rsteps.p, rs.data(), R * sizeof(long long), cudaMemcpyHostToDevice, ctx->stream));
        std::vector<double*> rp;
        for (auto& b : e->states) rp.push_back(b.p);
        DevBuf<double*> drp(std::max<size_t>(1, rp.size()));
        if (!rp.empty())
            S2B_CUDA(cudaMemcpyAsync(drp.p, rp.data(), rp.size() * sizeof(double*), cudaMemcpyHostToDevice, ctx->stream));
        AdArgs a{};
        a.values = paths->d_values.p;
        a.vstride = paths->steps + 1;
        a.M = M;
        a.n = n;
        a.dt_leb = paths->dt_leb;
        a.dt_steps = static_cast<long long>(plan.dt_steps);
        a.total = static_cast<long long>(plan.total_steps);
        a.rec_steps = rsteps.p;
        a.R = R;
        a.k0 = k0.p;
        a.len = len.p;
        a.fresh = fresh.p;
        a.flags = flags.p;
        a.rec = rec.p;
        a.rec_lo = rlo.p;
        a.rec_hi = rhi.p;
        a.accept = acc.p;
        a.ctab3 = s->ctab.p; // the session's window-0 weights
        a.ctab2 = ctab2.p;
        a.live = live.p;
        a.tau = ad->tolerance;
        a.shrink = ad->shrink;
        a.cap = cfg->blowup_norm_cap;
        const unsigned gm = static_cast<unsigned>((M + 255) / 256);
        OpView ov{op->d_pair_begin.p, op->d_pair_slot.p, op->d_w.p, static_cast<int>(op->nx),
                  static_cast<int>(op->nv), op->compressed};
        auto norms = [&](MagnusSession* q) {
            for (size_t m0 = 0; m0 < M; m0 += (1u << 30)) {
                const size_t mc = std::min<size_t>(M - m0, 1u << 30);
                norm_kernel<<<static_cast<unsigned>(mc), 256, 0, ctx->stream>>>(
                    ov, q->bits.p, q->nbits, op->rx, q->ctab.p + m0 * 6, 1, 0, 1, cfg->expmv_theta,
                    q->stab.p + m0, nullptr);
                S2B_LAUNCHED(ctx);
            }
        };
        auto load = [&](MagnusSession* q) {
            S2B_CUDA(cudaMemcpyAsync(q->S[0].p, U.p, U.bytes(), cudaMemcpyDeviceToDevice, ctx->stream));
            ad_reset_kernel<<<gm, 256, 0, ctx->stream>>>(q->iv.p, M, flags.p);
            S2B_LAUNCHED(ctx);
            S2B_CUDA(cudaMemsetAsync(q->cnt.p, 0, q->cnt.bytes(), ctx->stream));
            q->cur = 0;
            q->cur_window = 0;
        };
        const dim3 gg(static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 64)), static_cast<unsigned>(std::min<size_t>(M, 65535)));
        int h_live = 0;
        while (true) {
            S2B_CUDA(cudaMemsetAsync(live.p, 0, sizeof(int), ctx->stream));
            ad_prepare_kernel<<<gm, 256, 0, ctx->stream>>>(a);
            S2B_LAUNCHED(ctx);
            S2B_CUDA(cudaMemcpyAsync(&h_live, live.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
            S2B_CUDA(cudaStreamSynchronize(ctx->stream));
            if (h_live == 0) break;
            S2B_CUDA(cudaMemcpyAsync(s2->ctab.p, ctab2.p, M * 6 * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
            norms(s);  // order 3
            norms(s2); // order 2
            load(s);
            load(s2);
            MagnusSession* both[2] = {s, s2};
            sessions_run_batched(both, 2);
            ad_save_status_kernel<<<gm, 256, 0, ctx->stream>>>(s->iv.p + 4 * M, st3.p, M);
            S2B_LAUNCHED(ctx);
            gather_kernel<<<gg, 256, 0, ctx->stream>>>(s->iv.p + 5 * M, s->S[0].p, s->S[1].p, A.p, n, M);
            S2B_LAUNCHED(ctx);
            ad_gap_kernel<<<static_cast<unsigned>(std::min<size_t>(M, 65535)), 256, 0, ctx->stream>>>(
                a, A.p, s2->S[0].p, s2->S[1].p, s2->iv.p + 5 * M, st3.p, s2->iv.p + 4 * M);
            S2B_LAUNCHED(ctx);
            ad_commit_kernel<<<gg, 256, 0, ctx->stream>>>(a, A.p, U.p, drp.p, e->status.p);
            S2B_LAUNCHED(ctx);
        }
        if (stats) {
            session_stats(s, stats); // counters of the order-3 attempts plus the order-2 ones
            s2b_magnus_stats st2{};
            session_stats(s2, &st2);
            stats->path_terms += st2.path_terms;
            stats->path_segments += st2.path_segments;
            stats->term_launches += st2.term_launches;
        }
        e->states.push_back(std::move(U));
        S2B_CUDA(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
        delete e;
        session_destroy(s);
        session_destroy(s2);
        throw;
    }
    session_destroy(s);
    session_destroy(s2);
    return e;
}

} // namespace s2b
