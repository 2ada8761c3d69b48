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
//  * the fold starts at its first product instead of 0.0 + it (one DADD fewer per stencil
//    entry and path: 19 of 118 fp64 ops at order 3): y can then differ from the reference's
//    only in the sign of a zero, and the apply's accumulator starts at +0.0, so it absorbs a
//    +-0 product without a bit changing (x + -0 == x for x != 0, +0 + -0 == +0);
//  * a work item is (K live paths, strip of kRows output rows); the K paths share every weight
//    load (the weights are the same for all paths) and the CTA marches down the strip with
//    the term rows j-KRV .. j+KRV of all K paths in a ring (zero x-halo columns, zero rows
//    outside the grid), one __syncthreads per row;
//  * items are ordered path-group fastest, so the CTAs resident at one time work on the same
//    strip and its weights stay in L2 even when the whole weight set does not (1024^2).
#include <algorithm>
#include <cstdlib>
#include <initializer_list>
#include <type_traits>
#include <utility>

#include "magnus_common.cuh"

namespace s2b {
namespace mg {

namespace {

constexpr int kVarNT = 256;  // threads per CTA
constexpr int kVarRows = 128; // output rows per work item (32: 2-4% slower)
constexpr int kRing = 8;     // ring rows per path (power of two, >= 2*KRV + 2)

template <int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
    [&]<int... I>(std::integer_sequence<int, I...>) {
        (f(std::integral_constant<int, I>{}), ...);
    }(std::make_integer_sequence<int, N>{});
}

// The operator's exact structure as a template parameter: the union stencil (mask), the number
// of source pairs of every stencil entry (3 bits per entry, mask rank order, 21 per word) and
// the CommutatorSet slot of every pair (3 bits per pair, 21 per word).
struct VarFam {
    uint64_t mask;
    uint64_t pc[2];
    uint64_t ps[4];
};
template <VarFam F>
struct Fam {
    static constexpr uint64_t MASK = F.mask;
    static constexpr int cnt(int e) { return static_cast<int>((F.pc[e / 21] >> (3 * (e % 21))) & 7); }
    static constexpr int off(int e) {
        int o = 0;
        for (int i = 0; i < e; ++i) o += cnt(i);
        return o;
    }
    static constexpr int slot(int q) { return static_cast<int>((F.ps[q / 21] >> (3 * (q % 21))) & 7); }
};

// structure encodings from lists (compile time) and from an operator (upload time)
constexpr VarFam fam_of_lists(uint64_t mask, std::initializer_list<int> counts, std::initializer_list<int> slots) {
    VarFam f{mask, {0, 0}, {0, 0, 0, 0}};
    int e = 0;
    for (int c : counts) {
        f.pc[e / 21] |= static_cast<uint64_t>(c) << (3 * (e % 21));
        ++e;
    }
    int q = 0;
    for (int sl : slots) {
        f.ps[q / 21] |= static_cast<uint64_t>(sl) << (3 * (q % 21));
        ++q;
    }
    return f;
}
// Langevin unions and the general kinetic SPDE of the paper
// (a/2 d_vv + v d_x + b d_v + c, sigma d_v + beta: fields gvv, fx, fv, h, sigv, sig; 23-point
// order-3 union, radius x 2 / v 3), pair structures as the host builder produces them
constexpr uint64_t kMask23 = mask_of({{0, -3}, {-1, -2}, {0, -2}, {1, -2}, {-2, -1}, {-1, -1}, {0, -1}, {1, -1},
                                      {2, -1}, {-2, 0}, {-1, 0}, {0, 0}, {1, 0}, {2, 0}, {-2, 1}, {-1, 1},
                                      {0, 1}, {1, 1}, {2, 1}, {-1, 2}, {0, 2}, {1, 2}, {0, 3}});
constexpr VarFam kFam19v = fam_of_lists(kMask19, {2, 1, 2, 1, 2, 4, 2, 1, 3, 3, 3, 1, 2, 4, 2, 1, 2, 1, 2},
    {4, 5, 2, 4, 5, 5, 3, 5, 0, 1, 4, 5, 3, 5, 5, 0, 4, 5, 0, 2, 3, 0, 4, 5, 5, 3, 5, 0, 1, 4, 5, 3, 5, 5, 4, 5, 2, 4, 5});
constexpr VarFam kFam19c = fam_of_lists(kMask19, {2, 1, 2, 1, 1, 4, 1, 1, 2, 3, 2, 1, 1, 4, 1, 1, 2, 1, 2},
    {4, 5, 2, 4, 5, 5, 3, 0, 1, 4, 5, 3, 5, 0, 4, 0, 2, 3, 0, 4, 5, 3, 0, 1, 4, 5, 3, 5, 4, 5, 2, 4, 5});
constexpr VarFam kFam11 = fam_of_lists(kMask11, {1, 1, 2, 1, 1, 3, 1, 1, 2, 1, 1},
    {2, 3, 0, 1, 3, 0, 0, 2, 3, 0, 3, 0, 1, 3, 2});
constexpr VarFam kFam5 = fam_of_lists(kMask5, {2, 1, 1, 1, 2}, {0, 1, 0, 0, 0, 0, 1});
constexpr VarFam kFamK11 = fam_of_lists(kMask11, {2, 1, 4, 1, 2, 4, 2, 1, 4, 1, 2},
    {2, 3, 3, 0, 1, 2, 3, 3, 0, 3, 0, 1, 2, 3, 0, 3, 3, 0, 1, 2, 3, 3, 2, 3});
constexpr VarFam kFamK23 = fam_of_lists(kMask23,
    {2, 2, 4, 2, 1, 3, 6, 3, 1, 1, 4, 6, 4, 1, 1, 3, 6, 3, 1, 2, 4, 2, 2},
    {4, 5, 4, 5, 2, 3, 4, 5, 4, 5, 5, 3, 4, 5, 0, 1, 2, 3, 4, 5, 3, 4, 5, 5, 5, 0, 3, 4, 5, 0, 1, 2,
     3, 4, 5, 0, 3, 4, 5, 5, 5, 3, 4, 5, 0, 1, 2, 3, 4, 5, 3, 4, 5, 5, 4, 5, 2, 3, 4, 5, 4, 5, 4, 5});
constexpr VarFam kFams[] = {kFam19v, kFam19c, kFam11, kFam5, kFamK11, kFamK23};


// TW: the weight rows stream through shared memory (TMA, double-buffered); otherwise (grids
// whose two weight rows do not fit next to the ring) each point loads its weights from L2.
// G path groups: the CTA has G x kVarNT threads; group g handles the KT = K / G paths
// [g*KT, (g+1)*KT) of the item at every point, so the K paths still share one copy of each
// weight row while a thread carries only KT paths' state (G = 2: 16 warps per SM).
template <int K, int FI, int KRX, int KRV, int XPT, bool TW, int G = 1>
__global__ void __launch_bounds__(kVarNT * G, 1) term_var_kernel(TermArgs a, int strips) {
    constexpr int NT = kVarNT * G;
    constexpr int KT = K / G;
    static_assert(K % G == 0, "paths per group");
    constexpr uint64_t MASK = kFams[FI].mask;
    using PF = Fam<kFams[FI]>;
    static_assert(2 * KRV + 2 <= kRing, "ring too short");
    constexpr int NB = MaskInfo<MASK>::count();
    constexpr int NP = PF::off(NB);
    const int nx = a.op.nx, nv = a.op.nv;
    const size_t n = static_cast<size_t>(nx) * nv;
    const int RWS = nx + 2 * KRX; // ring row stride (zero x-halo on both sides)
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int xt = t % kVarNT, grp = t / kVarNT; // x position, path group

    extern __shared__ __align__(128) double vsm[];
    double* wbuf = vsm;                                          // [2][nx][NPP] weights of rows j, j+1
    constexpr int NPP = NP | 1; // point-major weight stride (odd: conflict-free 8-byte lanes)
    const size_t WSTR = static_cast<size_t>(nx) * NPP; // one row's weights (nx even: 16-byte multiple)
    double* ring = wbuf + (TW ? 2 * WSTR : 0); // [K][kRing][RWS]
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ unsigned long long red[K][2][kVarNT / 32];

    for (int q = t; q < K * kRing * RWS; q += NT) ring[q] = 0.0; // x-halos stay zero
    if (TW && t == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t ph = 0; // parity of the next wait on each weight buffer (bit b)
    // Row jw's weights (NP rows of nx doubles) stream into buffer jw & 1.  Thread 0 arms the
    // buffer's barrier (expect_tx) while the buffer's previous phase is complete and before the
    // CTA barrier that precedes the copies; the NP bulk copies are then issued by threads spread
    // over every warp (one copy each), so no compute warp is delayed by the issue.
    auto arm = [&](int jw) { mbar_expect_tx(&bar[jw & 1], static_cast<uint32_t>(WSTR * 8)); };
    auto copies = [&](int jw) { // the row's weights are contiguous point-major: one bulk copy, last warp
        if (TW && t == NT - 32) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); // prior generic reads of the buffer
            tma_row(wbuf + (jw & 1) * WSTR, a.op.wpm + static_cast<size_t>(jw) * WSTR, static_cast<uint32_t>(WSTR * 8),
                    &bar[jw & 1]);
        }
    };

    const int live = a.cnt[0];
    const int groups = (live + K - 1) / K;
    const long long items = static_cast<long long>(groups) * strips;
    for (long long it = blockIdx.x; it < items; it += gridDim.x) {
        // TW (all weights L2-resident): strips fastest, so the CTAs resident at one time read
        // different weight rows (no L2-slice hot spot); otherwise path groups fastest, so they
        // share one strip's weights while the whole set does not fit L2
        const int strip = TW ? static_cast<int>(it % strips) : static_cast<int>(it / groups);
        const int g = TW ? static_cast<int>(it / strips) : static_cast<int>(it - static_cast<long long>(strip) * groups);
        const int vrows = (nv + strips - 1) / strips; // rows per item (host: kVarRows, S2B_VAR_ROWS)
        const int j0 = strip * vrows, j1 = min(nv, j0 + vrows);
        int pk[KT];
        const double* in[KT];
        const double* Sin[KT];
        double* Tout[KT];
        double* Sout[KT];
        double inv[KT];
        double c[KT][6];
#pragma unroll
        for (int k = 0; k < KT; ++k) {
            const int kg = grp * KT + k; // the path's index in the item
            pk[k] = g * K + kg < live ? a.act[g * K + kg] : -1;
            const int p = pk[k] >= 0 ? pk[k] : a.act[g * K];
            const int kk = a.k[p], par = a.par[p];
            inv[k] = 1.0 / (static_cast<double>(a.nseg[p]) * kk);
            Sin[k] = (par ? a.S1 : a.S0) + static_cast<size_t>(p) * n;
            in[k] = kk == 1 ? Sin[k] : (par ? a.T1 : a.T0) + static_cast<size_t>(p) * n;
            Tout[k] = (par ? a.T0 : a.T1) + static_cast<size_t>(p) * n;
            Sout[k] = (par ? a.S0 : a.S1) + static_cast<size_t>(p) * n;
            const double* cp = a.ctab + (static_cast<size_t>(p) * a.nwin + a.win[p]) * 6;
#pragma unroll
            for (int q = 0; q < 6; ++q) c[k][q] = pk[k] >= 0 ? cp[q] : 0.0;
        }
        __syncthreads(); // the previous item is done with the ring and both weight buffers
        if (TW && t == 0) {
            arm(j0);
            if (j0 + 1 < j1) arm(j0 + 1);
        }
        __syncthreads(); // armed before any copy lands
        if (TW) copies(j0);
        // ring rows j0-KRV .. j0+KRV (zero outside the grid)
        for (int jr = j0 - KRV; jr <= j0 + KRV; ++jr) {
#pragma unroll
            for (int k = 0; k < KT; ++k) {
                double* dst = ring + (static_cast<size_t>(grp * KT + k) * kRing + (jr & (kRing - 1))) * RWS + KRX;
#pragma unroll
                for (int u = 0; u < XPT; ++u) {
                    const int i = xt + u * kVarNT;
                    if (i < nx)
                        dst[i] = (jr >= 0 && jr < nv && pk[k] >= 0) ? in[k][static_cast<size_t>(jr) * nx + i] : 0.0;
                }
            }
        }
        __syncthreads();

        unsigned long long tb[KT], sb[KT];
#pragma unroll
        for (int k = 0; k < KT; ++k) tb[k] = sb[k] = 0;

        for (int j = j0; j < j1; ++j) {
            // the next row's weights (its buffer was last read in row j-1, before the barrier)
            if (TW && j + 1 < j1) copies(j + 1);
            // prefetch: the ring's next row and this row's accumulator
            const int jn = j + KRV + 1;
            double nxt[KT][XPT], sacc[KT][XPT];
#pragma unroll
            for (int k = 0; k < KT; ++k)
#pragma unroll
                for (int u = 0; u < XPT; ++u) {
                    const int i = xt + u * kVarNT;
                    const bool ok = i < nx && pk[k] >= 0;
                    nxt[k][u] = (ok && jn < nv) ? in[k][static_cast<size_t>(jn) * nx + i] : 0.0;
                    sacc[k][u] = ok ? Sin[k][static_cast<size_t>(j) * nx + i] : 0.0;
                }
            if (TW) {
                mbar_wait(&bar[j & 1], (ph >> (j & 1)) & 1u);
                ph ^= 1u << (j & 1);
            }
            const double* wr = wbuf + (j & 1) * WSTR;
#pragma unroll
            for (int u = 0; u < XPT; ++u) {
                const int i = xt + u * kVarNT;
                if (i >= nx) continue;
                const size_t r = static_cast<size_t>(j) * nx + i;
                double wg[TW ? 1 : NP]; // the point's weights, all loads in flight at once
                if constexpr (!TW) {
#pragma unroll
                    for (int q = 0; q < NP; ++q) wg[q] = __ldg(a.op.wpm + r * NPP + q);
                }
                double acc[KT];
#pragma unroll
                for (int k = 0; k < KT; ++k) acc[k] = 0.0;
                // stencil entries in ascending bit order (== ascending (dv, dx)), all compile-time
                static_for<NB>([&](auto E) {
                    constexpr int e = decltype(E)::value;
                    constexpr int b = MaskInfo<MASK>::bit_of(e);
                    constexpr int dx = b % kBoxW - kBoxR, dv = b / kBoxW - kBoxR;
                    constexpr int q0 = PF::off(e);
                    double y[KT];
#pragma unroll
                    for (int k = 0; k < KT; ++k) y[k] = 0.0;
                    static_for<PF::cnt(e)>([&](auto C) {
                        constexpr int q = q0 + decltype(C)::value;
                        constexpr int sl = PF::slot(q);
                        double w;
                        if constexpr (TW) w = wr[i * NPP + q];
                        else w = wg[q];
#pragma unroll
                        for (int k = 0; k < KT; ++k) y[k] = decltype(C)::value == 0 ? c[k][sl] * w : y[k] + c[k][sl] * w;
                    });
                    const int jr = (j + dv) & (kRing - 1);
#pragma unroll
                    for (int k = 0; k < KT; ++k) {
                        const double x = ring[(static_cast<size_t>(grp * KT + k) * kRing + jr) * RWS + KRX + i + dx];
                        acc[k] += y[k] * x;
                    }
                });
#pragma unroll
                for (int k = 0; k < KT; ++k) {
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
            for (int k = 0; k < KT; ++k) {
                double* dst = ring + (static_cast<size_t>(grp * KT + k) * kRing + (jn & (kRing - 1))) * RWS + KRX;
#pragma unroll
                for (int u = 0; u < XPT; ++u) {
                    const int i = xt + u * kVarNT;
                    if (i < nx) dst[i] = nxt[k][u];
                }
            }
            // buffer j & 1 is read in this row only: its next phase (row j + 2) may be armed
            if (TW && t == 0 && j + 2 < j1) arm(j + 2);
            __syncthreads();
        }
        // path-wide maxima: warp -> group -> one atomic per path (a group's warps are contiguous)
#pragma unroll
        for (int k = 0; k < KT; ++k) {
            const unsigned long long wt = warp_umax(tb[k]), ws = warp_umax(sb[k]);
            if (lane == 0) {
                red[grp * KT + k][0][warp % (kVarNT / 32)] = wt;
                red[grp * KT + k][1][warp % (kVarNT / 32)] = ws;
            }
        }
        __syncthreads();
        if (warp % (kVarNT / 32) == 0) { // the first warp of each group
#pragma unroll
            for (int k = 0; k < KT; ++k) {
                unsigned long long t2 = lane < kVarNT / 32 ? red[grp * KT + k][0][lane] : 0ULL;
                unsigned long long s2 = lane < kVarNT / 32 ? red[grp * KT + k][1][lane] : 0ULL;
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

// x-split variant of the TMA-weight kernel: a work item is (K paths, strip, x-part of NT
// columns), one point per thread, so a CTA's two weight rows and its ring are small enough for
// two CTAs per SM -- one CTA's per-row barrier and weight wait hide behind the other's math.
// The ring (RING = 2*KRV+2 rows, slot = row mod RING) holds the part's columns plus KRX halo
// columns on each side (the neighbour part's values, zero outside the grid).
// G path groups as in term_var_kernel: G x NT threads, group g carries KT = K / G paths.
template <int K, int FI, int KRX, int KRV, int NT, int G = 1>
__global__ void __launch_bounds__(NT * G, G > 1 ? 1 : (K == 2 ? 512 / NT : 256 / NT))
    term_varx_kernel(TermArgs a, int strips, int gfast) {
    constexpr int NTT = NT * G; // threads per CTA
    constexpr int KT = K / G;
    static_assert(K % G == 0, "paths per group");
    constexpr uint64_t MASK = kFams[FI].mask;
    using PF = Fam<kFams[FI]>;
    constexpr int RING = 2 * KRV + 2;
    constexpr int NB = MaskInfo<MASK>::count();
    constexpr int NP = PF::off(NB);
    constexpr int RWS = NT + 2 * KRX; // ring row stride
    const int nx = a.op.nx, nv = a.op.nv;
    const size_t n = static_cast<size_t>(nx) * nv;
    const int parts = (nx + NT - 1) / NT;
    const int tt = threadIdx.x, lane = tt & 31, warp = tt >> 5;
    const int t = tt % NT, grp = tt / NT; // column within the part, path group

    extern __shared__ __align__(128) double vsm[];
    constexpr int NPP = NP | 1;                       // point-major weight stride (odd: conflict-free)
    double* wbuf = vsm;                               // [2][NT][NPP] weights of rows j, j+1 (this part)
    double* ring = wbuf + 2 * static_cast<size_t>(NT) * NPP; // [K][RING][RWS]
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ unsigned long long red[K][2][NT / 32];

    for (int q = tt; q < K * RING * RWS; q += NTT) ring[q] = 0.0;
    if (tt == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t ph = 0;
    int xlo = 0, wpart = NT; // current part: first column, width in the grid
    // as term_var_kernel: thread 0 arms, the last warp issues one bulk copy of the part's
    // point-major weights per row (columns past the grid are never read)
    auto arm = [&](int jw) { mbar_expect_tx(&bar[jw & 1], static_cast<uint32_t>(wpart * NPP * 8)); };
    auto copies = [&](int jw) {
        if (tt == NTT - 32) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tma_row(wbuf + static_cast<size_t>(jw & 1) * NT * NPP,
                    a.op.wpm + (static_cast<size_t>(jw) * nx + xlo) * NPP, static_cast<uint32_t>(wpart * NPP * 8),
                    &bar[jw & 1]);
        }
    };
    auto slot = [](int jr) { return ((jr % RING) + RING) % RING; };

    const int live = a.cnt[0];
    const int groups = (live + K - 1) / K;
    const long long items = static_cast<long long>(groups) * strips * parts;
    for (long long it = blockIdx.x; it < items; it += gridDim.x) {
        // gfast (weights beyond L2): path groups fastest, so resident CTAs share a strip's weights
        const long long pg = static_cast<long long>(parts) * groups;
        const int part = gfast ? static_cast<int>((it / groups) % parts) : static_cast<int>(it % parts);
        const int strip = gfast ? static_cast<int>(it / pg) : static_cast<int>((it / parts) % strips);
        const int g = gfast ? static_cast<int>(it % groups) : static_cast<int>(it / (static_cast<long long>(parts) * strips));
        const int vrows = (nv + strips - 1) / strips; // rows per item (host: kVarRows, S2B_VAR_ROWS)
        const int j0 = strip * vrows, j1 = min(nv, j0 + vrows);
        xlo = part * NT;
        wpart = min(NT, nx - xlo);
        const int i = xlo + t;          // this thread's column
        const bool act = t < wpart;
        // halo column of this thread (t < 2*KRX): left xlo-KRX+t, right xlo+wpart+(t-KRX)
        const int hi_col = t < KRX ? xlo - KRX + t : xlo + wpart + (t - KRX);
        const int hi_loc = t < KRX ? t : KRX + wpart + (t - KRX);
        const bool has_h = t < 2 * KRX;
        const bool h_in = has_h && hi_col >= 0 && hi_col < nx;
        int pk[KT];
        const double* in[KT];
        const double* Sin[KT];
        double* Tout[KT];
        double* Sout[KT];
        double inv[KT];
        double c[KT][6];
#pragma unroll
        for (int k = 0; k < KT; ++k) {
            const int kg = grp * KT + k;
            pk[k] = g * K + kg < live ? a.act[g * K + kg] : -1;
            const int p = pk[k] >= 0 ? pk[k] : a.act[g * K];
            const int kk = a.k[p], par = a.par[p];
            inv[k] = 1.0 / (static_cast<double>(a.nseg[p]) * kk);
            Sin[k] = (par ? a.S1 : a.S0) + static_cast<size_t>(p) * n;
            in[k] = kk == 1 ? Sin[k] : (par ? a.T1 : a.T0) + static_cast<size_t>(p) * n;
            Tout[k] = (par ? a.T0 : a.T1) + static_cast<size_t>(p) * n;
            Sout[k] = (par ? a.S0 : a.S1) + static_cast<size_t>(p) * n;
            const double* cp = a.ctab + (static_cast<size_t>(p) * a.nwin + a.win[p]) * 6;
#pragma unroll
            for (int q = 0; q < 6; ++q) c[k][q] = pk[k] >= 0 ? cp[q] : 0.0;
        }
        __syncthreads(); // the previous item is done with the ring and both weight buffers
        if (tt == 0) {
            arm(j0);
            if (j0 + 1 < j1) arm(j0 + 1);
        }
        __syncthreads(); // armed before any copy lands
        copies(j0);
        auto fill = [&](int k, int jr, double v_own, double v_h) {
            double* dst = ring + (static_cast<size_t>(grp * KT + k) * RING + slot(jr)) * RWS;
            if (act) dst[KRX + t] = v_own;
            if (has_h) dst[hi_loc] = v_h;
            if (!act && t < NT) dst[KRX + t] = 0.0; // columns past the grid's edge
        };
        auto ldv = [&](int k, int jr, int col, bool ok) -> double {
            return (ok && jr >= 0 && jr < nv && pk[k] >= 0) ? in[k][static_cast<size_t>(jr) * nx + col] : 0.0;
        };
        for (int jr = j0 - KRV; jr <= j0 + KRV; ++jr)
#pragma unroll
            for (int k = 0; k < KT; ++k) fill(k, jr, ldv(k, jr, i, act), ldv(k, jr, hi_col, h_in));
        __syncthreads();

        unsigned long long tb[KT], sb[KT];
#pragma unroll
        for (int k = 0; k < KT; ++k) tb[k] = sb[k] = 0;

        for (int j = j0; j < j1; ++j) {
            if (j + 1 < j1) copies(j + 1);
            const int jn = j + KRV + 1;
            double nxt[KT], nxh[KT], sacc[KT];
#pragma unroll
            for (int k = 0; k < KT; ++k) {
                nxt[k] = ldv(k, jn, i, act);
                nxh[k] = ldv(k, jn, hi_col, h_in);
                sacc[k] = (act && pk[k] >= 0) ? Sin[k][static_cast<size_t>(j) * nx + i] : 0.0;
            }
            int sl[2 * KRV + 1];
#pragma unroll
            for (int d = 0; d <= 2 * KRV; ++d) sl[d] = slot(j - KRV + d);
            mbar_wait(&bar[j & 1], (ph >> (j & 1)) & 1u);
            ph ^= 1u << (j & 1);
            const double* wr = wbuf + static_cast<size_t>(j & 1) * NT * NPP;
            if (act) {
                const size_t r = static_cast<size_t>(j) * nx + i;
                double acc[KT];
#pragma unroll
                for (int k = 0; k < KT; ++k) acc[k] = 0.0;
                static_for<NB>([&](auto E) {
                    constexpr int e = decltype(E)::value;
                    constexpr int b = MaskInfo<MASK>::bit_of(e);
                    constexpr int dx = b % kBoxW - kBoxR, dv = b / kBoxW - kBoxR;
                    constexpr int q0 = PF::off(e);
                    double y[KT];
#pragma unroll
                    for (int k = 0; k < KT; ++k) y[k] = 0.0;
                    static_for<PF::cnt(e)>([&](auto C) {
                        constexpr int q = q0 + decltype(C)::value;
                        constexpr int ps = PF::slot(q);
                        const double w = wr[t * NPP + q];
#pragma unroll
                        for (int k = 0; k < KT; ++k) y[k] = decltype(C)::value == 0 ? c[k][ps] * w : y[k] + c[k][ps] * w;
                    });
                    const int rs = sl[dv + KRV];
#pragma unroll
                    for (int k = 0; k < KT; ++k) {
                        const double x = ring[(static_cast<size_t>(grp * KT + k) * RING + rs) * RWS + KRX + t + dx];
                        acc[k] += y[k] * x;
                    }
                });
#pragma unroll
                for (int k = 0; k < KT; ++k) {
                    if (pk[k] < 0) continue;
                    const double tv = acc[k] * inv[k];
                    const double sv = sacc[k] + tv;
                    Tout[k][r] = tv;
                    Sout[k][r] = sv;
                    tb[k] = umax64(tb[k], abs_bits(tv));
                    sb[k] = umax64(sb[k], abs_bits(sv));
                }
            }
            // row jn replaces row jn - RING (= j - KRV - 1, out of this row's window): every
            // thread is past its reads of that slot only after the barrier of row j - 1
#pragma unroll
            for (int k = 0; k < KT; ++k) fill(k, jn, nxt[k], nxh[k]);
            if (tt == 0 && j + 2 < j1) arm(j + 2); // buffer j & 1's next phase (see term_var_kernel)
            __syncthreads();
        }
#pragma unroll
        for (int k = 0; k < KT; ++k) {
            const unsigned long long wt = warp_umax(tb[k]), ws = warp_umax(sb[k]);
            if (lane == 0) {
                red[grp * KT + k][0][warp % (NT / 32)] = wt;
                red[grp * KT + k][1][warp % (NT / 32)] = ws;
            }
        }
        __syncthreads();
        if (warp % (NT / 32) == 0) { // the first warp of each group
#pragma unroll
            for (int k = 0; k < KT; ++k) {
                unsigned long long t2 = lane < NT / 32 ? red[grp * KT + k][0][lane] : 0ULL;
                unsigned long long s2 = lane < NT / 32 ? red[grp * KT + k][1][lane] : 0ULL;
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

bool fam_from_op(const s2b_operator* op, VarFam* f) {
    *f = VarFam{op->union_mask, {0, 0}, {0, 0, 0, 0}};
    int e = 0;
    for (int b = 0; b < kBoxBits; ++b)
        if ((op->union_mask >> b) & 1) {
            const int c = op->pair_begin[b + 1] - op->pair_begin[b];
            if (c > 7 || e >= 42) return false;
            f->pc[e / 21] |= static_cast<uint64_t>(c) << (3 * (e % 21));
            ++e;
        }
    if (op->pair_slot.size() > 84) return false;
    for (size_t q = 0; q < op->pair_slot.size(); ++q)
        f->ps[q / 21] |= static_cast<uint64_t>(op->pair_slot[q]) << (3 * (q % 21));
    return true;
}
bool same(const VarFam& a, const VarFam& b) {
    return a.mask == b.mask && a.pc[0] == b.pc[0] && a.pc[1] == b.pc[1] && a.ps[0] == b.ps[0] &&
           a.ps[1] == b.ps[1] && a.ps[2] == b.ps[2] && a.ps[3] == b.ps[3];
}
int fam_of(const s2b_operator* op) {
    VarFam f;
    if (!fam_from_op(op, &f)) return -1;
    for (int i = 0; i < static_cast<int>(sizeof(kFams) / sizeof(kFams[0])); ++i)
        if (same(f, kFams[i])) return i;
    return -1;
}

// shared memory of one CTA: two weight rows + the K-path ring must fit 227 KB
size_t var_smem(int np, int k, int nx, int krx) {
    return (2 * static_cast<size_t>(np | 1) * nx + static_cast<size_t>(k) * kRing * (nx + 2 * krx)) * 8;
}

constexpr int kVarxNT = 128; // columns (threads) per CTA of the x-split kernel

template <int K, int FI, int KRX, int KRV>
void launch_var_k(s2b_context* ctx, const TermArgs& a, size_t live_max) {
    constexpr int NP = Fam<kFams[FI]>::off(MaskInfo<kFams[FI].mask>::count());
    const int nx = a.op.nx, nv = a.op.nv;
    const char* er = std::getenv("S2B_VAR_ROWS");
    // up to 256 columns one item covers the whole grid height (cfg3: 2.82e8 vs 2.74e8 windows/s
    // with 128-row strips; the ring prologue and the two-row weight prefetch are paid once)
    int vr = er ? std::max(4, std::atoi(er)) : (nx <= 256 ? 256 : kVarRows);
    if (!er) // few paths: shorter items keep every SM busy
        while (vr > 16 && (live_max + K - 1) / K * static_cast<size_t>((nv + vr - 1) / vr) *
                                  static_cast<size_t>((nx + 127) / 128) < 4 * static_cast<size_t>(ctx->num_sms))
            vr /= 2;
    const int strips = (nv + vr - 1) / vr;
    // wide grids: the x-split TMA kernel (measured 2.04e8 vs 1.71e8 windows/s at 1024^2); up to
    // 256 columns the full-row kernel is ahead (1.65e8 vs 1.56e8 at cfg3).  S2B_VARX=0/1 forces.
    const char* ev = std::getenv("S2B_VARX");
    // the full-row kernel needs two weight rows + the ring in one CTA's shared memory
    const bool row_fits = NP <= 40 && var_smem(NP, K, nx, KRX) <= 227 * 1024;
    const bool varx = (ev ? ev[0] != '0' : nx > kVarNT) || !row_fits;
    if (varx) {
        // x-split TMA kernel, 4 paths per item, several CTAs per SM (S2B_VARX_NT: columns per CTA)
        // G path groups per CTA: S2B_VARX_G=2 doubles the warps per SM; measured equal at cfg3k
        // and 14% slower at 1024^2 (cfg5 variable), so one group is the default
        const char* eg = std::getenv("S2B_VARX_G");
        const bool g2 = eg && eg[0] == '2';
        auto run = [&](auto ntag, auto ktag) {
            constexpr int NT = decltype(ntag)::value;
            constexpr int KX = decltype(ktag)::value; // paths per item
            auto launch = [&](auto kern, int nthreads) {
                const size_t smem = (2 * static_cast<size_t>(NP | 1) * NT + KX * static_cast<size_t>(2 * KRV + 2) * (NT + 2 * KRX)) * 8;
                S2B_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
                int per_sm = 0;
                S2B_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nthreads, smem));
                const size_t parts = (nx + NT - 1) / NT;
                const size_t items = (live_max + KX - 1) / KX * static_cast<size_t>(strips) * parts;
                const size_t cap = static_cast<size_t>(std::max(1, per_sm)) * ctx->num_sms;
                const int grid = grid_cap(static_cast<int>(std::max<size_t>(1, std::min(items, cap))));
                kern<<<grid, nthreads, smem, ctx->stream>>>(a, strips, nx > 256 ? 1 : 0);
                ctx->k_stream = reinterpret_cast<const void*>(kern);
            };
            if (g2 && KX % 2 == 0)
                launch(term_varx_kernel<KX, FI, KRX, KRV, NT, (KX % 2 == 0 ? 2 : 1)>, NT * (KX % 2 == 0 ? 2 : 1));
            else
                launch(term_varx_kernel<KX, FI, KRX, KRV, NT>, NT);
        };
        const char* en = std::getenv("S2B_VARX_NT");
        const char* ek = std::getenv("S2B_VARX_K");
        if constexpr (NP > 40) { // many source pairs: 64-column parts keep two CTAs per SM
            if (en && std::atoi(en) == 128)
                run(std::integral_constant<int, 128>{}, std::integral_constant<int, 4>{});
            else if (ek && std::atoi(ek) == 2)
                run(std::integral_constant<int, 64>{}, std::integral_constant<int, 2>{});
            else
                run(std::integral_constant<int, 64>{}, std::integral_constant<int, 4>{});
            return;
        }
        if (ek && std::atoi(ek) == 2)
            run(std::integral_constant<int, kVarxNT>{}, std::integral_constant<int, 2>{});
        else if (en && std::atoi(en) == 64)
            run(std::integral_constant<int, 64>{}, std::integral_constant<int, 4>{});
        else
            run(std::integral_constant<int, kVarxNT>{}, std::integral_constant<int, 4>{});
        return;
    }
    const bool tw = nx <= kVarNT;
    const size_t smem = ((tw ? 2 * static_cast<size_t>(NP | 1) * nx : 0) +
                         static_cast<size_t>(K) * kRing * (nx + 2 * KRX)) * 8;
    auto go = [&](auto kern, int nt) {
        S2B_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        int per_sm = 0;
        S2B_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nt, smem));
        const size_t items = (live_max + K - 1) / K * static_cast<size_t>(strips);
        const size_t cap = static_cast<size_t>(std::max(1, per_sm)) * ctx->num_sms;
        const int grid = grid_cap(static_cast<int>(std::max<size_t>(1, std::min(items, cap))));
        kern<<<grid, nt, smem, ctx->stream>>>(a, strips);
        ctx->k_stream = reinterpret_cast<const void*>(kern);
    };
    // full-row TMA kernel: one group of 256 threads; S2B_VAR_G=2 runs two path groups (16 warps
    // per SM, 128 registers) -- measured 7% slower at cfg3 order 3 (each weight load then serves
    // 2 paths instead of 4), so it stays opt-in
    const char* eg = std::getenv("S2B_VAR_G");
    const bool g2 = K % 2 == 0 && eg && eg[0] == '2';
    if constexpr (NP <= 40) {
        if (tw && g2)
            go(term_var_kernel<K, FI, KRX, KRV, 1, true, (K % 2 == 0 ? 2 : 1)>, kVarNT * (K % 2 == 0 ? 2 : 1));
        else if (tw)
            go(term_var_kernel<K, FI, KRX, KRV, 1, true>, kVarNT);
        else if (nx <= 2 * kVarNT)
            go(term_var_kernel<K, FI, KRX, KRV, 2, false>, kVarNT);
        else
            go(term_var_kernel<K, FI, KRX, KRV, 4, false>, kVarNT);
    }
}


} // namespace

bool term_var_supported(const s2b_operator* op) {
    const char* e = std::getenv("S2B_TERMVAR");
    if (e && e[0] == '0') return false;
    if (op->compressed || !op->wfinite || op->nx < 2 || op->nx % 2 != 0 || op->nx > 4 * static_cast<size_t>(kVarNT))
        return false;
    return fam_of(op) >= 0;
}

void launch_term_var(s2b_context* ctx, const s2b_operator* op, const TermArgs& a, size_t live_max) {
    const bool wide = op->nx > 2 * static_cast<size_t>(kVarNT); // 2 paths per item at 1024^2
    switch (fam_of(op)) {
    case 0:
        if (wide) launch_var_k<2, 0, 2, 2>(ctx, a, live_max);
        else launch_var_k<4, 0, 2, 2>(ctx, a, live_max);
        break;
    case 1:
        if (wide) launch_var_k<2, 1, 2, 2>(ctx, a, live_max);
        else launch_var_k<4, 1, 2, 2>(ctx, a, live_max);
        break;
    case 2:
        if (wide) launch_var_k<2, 2, 1, 2>(ctx, a, live_max);
        else launch_var_k<4, 2, 1, 2>(ctx, a, live_max);
        break;
    case 3:
        if (wide) launch_var_k<2, 3, 1, 1>(ctx, a, live_max);
        else launch_var_k<4, 3, 1, 1>(ctx, a, live_max);
        break;
    case 4: // general kinetic SPDE, order 2
        launch_var_k<4, 4, 1, 2>(ctx, a, live_max);
        break;
    default: // general kinetic SPDE, order 3 (23 points, 64 source pairs)
        launch_var_k<4, 5, 2, 3>(ctx, a, live_max);
        break;
    }
}

} // namespace mg
} // namespace s2b
