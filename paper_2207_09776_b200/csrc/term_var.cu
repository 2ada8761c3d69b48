// Streaming Taylor-term kernel for x-dependent coefficients (uncompressed weights), e.g. the
// variable-coefficient Langevin family of cfg3: Y cannot be compressed to per-row registers,
// so each point's generator entries are folded from the source weights every term
// (MagnusLogBuilder::fill, magnus.cpp:141-160: slots ascending from 0.0, zero coefficients
// skipped) and applied in ascending stencil order (dia_mv, sparse.cpp:412-423) -- the same
// per-point arithmetic as term_generic_k_kernel, restructured so the fp64 pipe does the work:
//  * the union stencil and the number of source pairs of every stencil entry are compile-time
//    (exactly the operator's: MASK, PCNT), so every neighbour offset is an immediate into a
//    shared-memory row ring, and a point's weights are loaded up front, all in flight at once
//    (only the slot of each pair -- which path coefficient -- is read at run time);
//  * the fold has no zero-coefficient branch: with finite weights, adding c*w = +-0 to a
//    y that started at +0.0 changes no bit (a sum is -0 only if both addends are), which is
//    the reference's skip; the operator must have finite weights (checked at upload);
//  * a work item is (K live paths, strip of kRows output rows); the K paths share every weight
//    load (the weights are the same for all paths) and the CTA marches down the strip with
//    the term rows j-KRV .. j+KRV of all K paths in a ring (zero x-halo columns, zero rows
//    outside the grid), one __syncthreads per row;
//  * items are ordered path-group fastest, so the CTAs resident at one time work on the same
//    strip and its weights stay in L2 even when the whole weight set does not (1024^2).
#include <algorithm>
#include <cstdlib>
#include <initializer_list>

#include "magnus_common.cuh"

namespace s2b {
namespace mg {

namespace {

constexpr int kVarNT = 256;  // threads per CTA
constexpr int kVarRows = 32; // output rows per work item
constexpr int kRing = 8;     // ring rows per path (power of two, >= 2*KRV + 2)

// PCNT: 3 bits per stencil entry (mask rank) = its number of source pairs
template <uint64_t PCNT>
struct Pc {
    static constexpr int cnt(int e) { return static_cast<int>((PCNT >> (3 * e)) & 7); }
    static constexpr int off(int e) {
        int o = 0;
        for (int i = 0; i < e; ++i) o += cnt(i);
        return o;
    }
};

template <int K, uint64_t MASK, uint64_t PCNT, int KRX, int KRV, int XPT>
__global__ void __launch_bounds__(kVarNT, 1) term_var_kernel(TermArgs a, int strips) {
    static_assert(2 * KRV + 2 <= kRing, "ring too short");
    static_assert(K % 2 == 0, "pairs of paths share 16-byte coefficient loads");
    constexpr int NB = MaskInfo<MASK>::count();
    constexpr int NP = Pc<PCNT>::off(NB);
    const int nx = a.op.nx, nv = a.op.nv;
    const size_t n = static_cast<size_t>(nx) * nv;
    const int RWS = nx + 2 * KRX; // ring row stride (zero x-halo on both sides)
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;

    extern __shared__ __align__(16) double vsm[];
    double* ring = vsm;                                         // [K][kRing][RWS]
    double* cq = ring + static_cast<size_t>(K) * kRing * RWS;   // [NP][K] coefficient per pair
    __shared__ int bslot[NP];                                   // pair -> CommutatorSet slot
    __shared__ unsigned long long red[K][2][kVarNT / 32];

    for (int q = t; q < NP; q += kVarNT) bslot[q] = a.op.pair_slot[q];
    for (int q = t; q < K * kRing * RWS; q += kVarNT) ring[q] = 0.0; // x-halos stay zero
    __syncthreads();

    const int live = a.cnt[0];
    const int groups = (live + K - 1) / K;
    const long long items = static_cast<long long>(groups) * strips;
    for (long long it = blockIdx.x; it < items; it += gridDim.x) {
        const int strip = static_cast<int>(it / groups);
        const int g = static_cast<int>(it - static_cast<long long>(strip) * groups);
        const int j0 = strip * kVarRows, j1 = min(nv, j0 + kVarRows);
        int pk[K];
        const double* in[K];
        const double* Sin[K];
        double* Tout[K];
        double* Sout[K];
        double inv[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            pk[k] = g * K + k < live ? a.act[g * K + k] : -1;
            const int p = pk[k] >= 0 ? pk[k] : a.act[g * K];
            const int kk = a.k[p], par = a.par[p];
            inv[k] = 1.0 / (static_cast<double>(a.nseg[p]) * kk);
            Sin[k] = (par ? a.S1 : a.S0) + static_cast<size_t>(p) * n;
            in[k] = kk == 1 ? Sin[k] : (par ? a.T1 : a.T0) + static_cast<size_t>(p) * n;
            Tout[k] = (par ? a.T0 : a.T1) + static_cast<size_t>(p) * n;
            Sout[k] = (par ? a.S0 : a.S1) + static_cast<size_t>(p) * n;
        }
        __syncthreads(); // the previous item is done with cq and the ring
        for (int q = t; q < NP * K; q += kVarNT) {
            const int pq = q / K, k = q - pq * K;
            const int p = pk[k] >= 0 ? pk[k] : a.act[g * K];
            cq[q] = pk[k] >= 0 ? a.ctab[(static_cast<size_t>(p) * a.nwin + a.win[p]) * 6 + bslot[pq]] : 0.0;
        }
        // ring rows j0-KRV .. j0+KRV (zero outside the grid)
        for (int jr = j0 - KRV; jr <= j0 + KRV; ++jr) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                double* dst = ring + (static_cast<size_t>(k) * kRing + (jr & (kRing - 1))) * RWS + KRX;
#pragma unroll
                for (int u = 0; u < XPT; ++u) {
                    const int i = t + u * kVarNT;
                    if (i < nx)
                        dst[i] = (jr >= 0 && jr < nv && pk[k] >= 0) ? in[k][static_cast<size_t>(jr) * nx + i] : 0.0;
                }
            }
        }
        __syncthreads();

        unsigned long long tb[K], sb[K];
#pragma unroll
        for (int k = 0; k < K; ++k) tb[k] = sb[k] = 0;

        for (int j = j0; j < j1; ++j) {
            // prefetch: the ring's next row and this row's accumulator
            const int jn = j + KRV + 1;
            double nxt[K][XPT], sacc[K][XPT];
#pragma unroll
            for (int k = 0; k < K; ++k)
#pragma unroll
                for (int u = 0; u < XPT; ++u) {
                    const int i = t + u * kVarNT;
                    const bool ok = i < nx && pk[k] >= 0;
                    nxt[k][u] = (ok && jn < nv) ? in[k][static_cast<size_t>(jn) * nx + i] : 0.0;
                    sacc[k][u] = ok ? Sin[k][static_cast<size_t>(j) * nx + i] : 0.0;
                }
#pragma unroll
            for (int u = 0; u < XPT; ++u) {
                const int i = t + u * kVarNT;
                if (i >= nx) continue;
                const size_t r = static_cast<size_t>(j) * nx + i;
                double w[NP];
#pragma unroll
                for (int q = 0; q < NP; ++q) w[q] = __ldg(a.op.w + static_cast<size_t>(q) * n + r);
                double acc[K];
#pragma unroll
                for (int k = 0; k < K; ++k) acc[k] = 0.0;
#pragma unroll
                for (int dv = -KRV; dv <= KRV; ++dv) {
#pragma unroll
                    for (int dx = -KRX; dx <= KRX; ++dx) {
                        if (!MaskInfo<MASK>::has(dx, dv)) continue;
                        const int e = MaskInfo<MASK>::rank(box_bit(dx, dv));
                        const int q0 = Pc<PCNT>::off(e), nq = Pc<PCNT>::cnt(e);
                        double y[K];
#pragma unroll
                        for (int k = 0; k < K; ++k) y[k] = 0.0;
#pragma unroll
                        for (int c = 0; c < 7; ++c) {
                            if (c >= nq) break;
                            const int q = q0 + c;
#pragma unroll
                            for (int k = 0; k < K; k += 2) {
                                const double2 cs = *reinterpret_cast<const double2*>(cq + q * K + k);
                                y[k] += cs.x * w[q];
                                y[k + 1] += cs.y * w[q];
                            }
                        }
                        const int jr = (j + dv) & (kRing - 1);
#pragma unroll
                        for (int k = 0; k < K; ++k) {
                            const double x = ring[(static_cast<size_t>(k) * kRing + jr) * RWS + KRX + i + dx];
                            acc[k] += y[k] * x;
                        }
                    }
                }
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    if (pk[k] < 0) continue;
                    const double tv = acc[k] * inv[k];
                    const double sv = sacc[k][u] + tv;
                    Tout[k][r] = tv;
                    Sout[k][r] = sv;
                    tb[k] = umax64(tb[k], abs_bits(tv));
                    sb[k] = umax64(sb[k], abs_bits(sv));
                }
            }
            // row jn goes to slot jn & 7, which held row jn - 8, long out of the window
#pragma unroll
            for (int k = 0; k < K; ++k) {
                double* dst = ring + (static_cast<size_t>(k) * kRing + (jn & (kRing - 1))) * RWS + KRX;
#pragma unroll
                for (int u = 0; u < XPT; ++u) {
                    const int i = t + u * kVarNT;
                    if (i < nx) dst[i] = nxt[k][u];
                }
            }
            __syncthreads();
        }
        // path-wide maxima: warp -> CTA -> one atomic per path
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const unsigned long long wt = warp_umax(tb[k]), ws = warp_umax(sb[k]);
            if (lane == 0) {
                red[k][0][warp] = wt;
                red[k][1][warp] = ws;
            }
        }
        __syncthreads();
        if (warp == 0) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                unsigned long long t2 = lane < kVarNT / 32 ? red[k][0][lane] : 0ULL;
                unsigned long long s2 = lane < kVarNT / 32 ? red[k][1][lane] : 0ULL;
                t2 = warp_umax(t2);
                s2 = warp_umax(s2);
                if (lane == 0 && pk[k] >= 0) {
                    if (t2) atomicMax(&a.tn[pk[k]], t2);
                    if (s2) atomicMax(&a.sn[pk[k]], s2);
                }
            }
        }
    }
}

constexpr uint64_t pcnt_of(std::initializer_list<int> c) {
    uint64_t v = 0;
    int e = 0;
    for (int x : c) v |= static_cast<uint64_t>(x) << (3 * e++);
    return v;
}
// Langevin unions (both families share the pair structure up to order 2; order 3 differs)
constexpr uint64_t kPc19var = pcnt_of({2, 1, 2, 1, 2, 4, 2, 1, 3, 3, 3, 1, 2, 4, 2, 1, 2, 1, 2});
constexpr uint64_t kPc19con = pcnt_of({2, 1, 2, 1, 1, 4, 1, 1, 2, 3, 2, 1, 1, 4, 1, 1, 2, 1, 2});
constexpr uint64_t kPc11 = pcnt_of({1, 1, 2, 1, 1, 3, 1, 1, 2, 1, 1});
constexpr uint64_t kPc5 = pcnt_of({2, 1, 1, 1, 2});

uint64_t pcnt_from(const s2b_operator* op) {
    uint64_t v = 0;
    int e = 0;
    for (int b = 0; b < kBoxBits; ++b)
        if ((op->union_mask >> b) & 1) {
            const int c = op->pair_begin[b + 1] - op->pair_begin[b];
            if (c > 7 || e >= 21) return ~0ULL;
            v |= static_cast<uint64_t>(c) << (3 * e++);
        }
    return v;
}

template <int K, uint64_t MASK, uint64_t PCNT, int KRX, int KRV>
void launch_var_k(s2b_context* ctx, const TermArgs& a, size_t live_max) {
    constexpr int NP = Pc<PCNT>::off(MaskInfo<MASK>::count());
    const int nx = a.op.nx, nv = a.op.nv;
    const int strips = (nv + kVarRows - 1) / kVarRows;
    const size_t smem = (static_cast<size_t>(K) * kRing * (nx + 2 * KRX) + static_cast<size_t>(NP) * K) * 8;
    auto go = [&](auto kern) {
        S2B_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        int per_sm = 0;
        S2B_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kVarNT, smem));
        const size_t items = (live_max + K - 1) / K * static_cast<size_t>(strips);
        const size_t cap = static_cast<size_t>(std::max(1, per_sm)) * ctx->num_sms;
        const int grid = static_cast<int>(std::max<size_t>(1, std::min(items, cap)));
        kern<<<grid, kVarNT, smem, ctx->stream>>>(a, strips);
    };
    if (nx <= kVarNT)
        go(term_var_kernel<K, MASK, PCNT, KRX, KRV, 1>);
    else if (nx <= 2 * kVarNT)
        go(term_var_kernel<K, MASK, PCNT, KRX, KRV, 2>);
    else
        go(term_var_kernel<K, MASK, PCNT, KRX, KRV, 4>);
}

} // namespace

bool term_var_supported(const s2b_operator* op) {
    const char* e = std::getenv("S2B_TERMVAR");
    if (e && e[0] == '0') return false;
    if (op->compressed || !op->wfinite || op->nx < 1 || op->nx > 4 * static_cast<size_t>(kVarNT)) return false;
    const uint64_t pc = pcnt_from(op);
    return (op->union_mask == kMask19 && (pc == kPc19var || pc == kPc19con)) ||
           (op->union_mask == kMask11 && pc == kPc11) || (op->union_mask == kMask5 && pc == kPc5);
}

void launch_term_var(s2b_context* ctx, const s2b_operator* op, const TermArgs& a, size_t live_max) {
    const bool wide = op->nx > 2 * static_cast<size_t>(kVarNT);
    const uint64_t pc = pcnt_from(op);
    if (op->union_mask == kMask19 && pc == kPc19var) {
        if (wide) launch_var_k<2, kMask19, kPc19var, 2, 2>(ctx, a, live_max);
        else launch_var_k<4, kMask19, kPc19var, 2, 2>(ctx, a, live_max);
    } else if (op->union_mask == kMask19) {
        if (wide) launch_var_k<2, kMask19, kPc19con, 2, 2>(ctx, a, live_max);
        else launch_var_k<4, kMask19, kPc19con, 2, 2>(ctx, a, live_max);
    } else if (op->union_mask == kMask11) {
        if (wide) launch_var_k<2, kMask11, kPc11, 1, 2>(ctx, a, live_max);
        else launch_var_k<4, kMask11, kPc11, 1, 2>(ctx, a, live_max);
    } else {
        if (wide) launch_var_k<2, kMask5, kPc5, 1, 1>(ctx, a, live_max);
        else launch_var_k<4, kMask5, kPc5, 1, 1>(ctx, a, live_max);
    }
}

} // namespace mg
} // namespace s2b
