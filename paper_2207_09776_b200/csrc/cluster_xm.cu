// Cluster-resident Magnus engine, x-march layout (the default for the Langevin variants).
//
// Same cluster decomposition as cluster_magnus.cu (one 8-CTA cluster per path, CTA `rank`
// owns rows [rank*RPC, (rank+1)*RPC), all Taylor terms of a window on chip), but the work
// is laid out so that the generator Y costs nothing inside the term loop:
//  * lane = row.  Thread (r, seg) owns row r of the CTA and the x-segment
//    [seg*L, (seg+1)*L); it marches along x.  Y is x-invariant away from the two x-boundary
//    columns on each side (the compressed operator), so the thread's row of Y lives in
//    registers for the whole window (the y_j of MagnusLogBuilder::fill, magnus.cpp:141-160)
//    and the march only loads the term: one value per stencil row per point, from a
//    per-row register ring.
//  * T and S are stored x-major ([x][row]): a warp's 32 lanes read 32 consecutive rows of
//    one column (conflict-free), and every offset of the unrolled march is an immediate.
//  * The KRV halo rows of the neighbours are pushed by the producer with DSMEM stores as
//    each term is computed, so the one cluster barrier per term (needed anyway for the
//    path-wide norms of expmv_into's stopping rule, sparse.cpp:463-492) also publishes the
//    halos.
//  * Path-wide maxima: 32-bit REDUX on the (hi, lo) words of the non-negative doubles,
//    every warp re-derives the decision from the 8 CTA slots (no broadcast barrier).
// The arithmetic per point is unchanged: Y.t summed from 0.0 in ascending (dv, dx) order
// (== ascending DIA diagonal, sparse.cpp:412-423), t = acc * (1/(s*k)), S += t, no FMA.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "magnus_common.cuh"

namespace cg = cooperative_groups;

namespace s2b {
namespace mg {

namespace {

#ifndef S2B_XM_P
#define S2B_XM_P 4
#endif
constexpr int kXmP = S2B_XM_P; // points in flight per thread (ILP of the stencil sums)
#ifndef S2B_XM_NT
#define S2B_XM_NT 256
#endif
constexpr int kXmNT = S2B_XM_NT; // threads per CTA

template <uint64_t MASK>
struct RowExt {
    static constexpr int lo(int dv) {
        for (int dx = -kBoxR; dx <= kBoxR; ++dx)
            if (MaskInfo<MASK>::has(dx, dv)) return dx;
        return 1;
    }
    static constexpr int hi(int dv) {
        for (int dx = kBoxR; dx >= -kBoxR; --dx)
            if (MaskInfo<MASK>::has(dx, dv)) return dx;
        return 0;
    }
    static constexpr int span(int dv) { return hi(dv) - lo(dv) + 1; }
    static constexpr int off(int dv) {
        int o = 0;
        for (int d = -kBoxR; d < dv; ++d) o += span(d);
        return o;
    }
    static constexpr int total() { return off(kBoxR + 1); }
};

__host__ __device__ constexpr int popc32(uint32_t v) { return v == 0 ? 0 : static_cast<int>(v & 1u) + popc32(v >> 1); }
__host__ __device__ constexpr int bm_rank(uint32_t bm, int e) { return popc32(bm & ((1u << e) - 1u)); }

template <uint64_t MASK, int KRX, int KRV, uint32_t BM, int NX, int RPC>
struct XmLayout {
    static constexpr int TR = RPC + 2 * KRV; // rows incl. halo
    static constexpr int TX = NX + 2 * KRX;  // columns incl. zero x-halo
    static constexpr int TBUF = TX * TR;
    static constexpr int NBM = MaskInfo<MASK>::count();
    static constexpr int NYE = kClasses * NBM;
    static constexpr int NBB = popc32(BM);
    static constexpr int SCR = RPC * (NX + 1); // row-major padded scratch (in T[1])
    static constexpr size_t bytes() {
        return 8 * (2 * static_cast<size_t>(TBUF) + static_cast<size_t>(NX) * RPC + 4 * static_cast<size_t>(NBB) * RPC);
    }
    static_assert(SCR <= TBUF, "transpose scratch must fit one term buffer");
};

// max over a warp of non-negative doubles (or +NaN), as their bit patterns
__device__ __forceinline__ unsigned long long warp_max_bits(unsigned long long b) {
    const unsigned hi = static_cast<unsigned>(b >> 32), lo = static_cast<unsigned>(b);
    const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
    return (static_cast<unsigned long long>(mh) << 32) | ml;
}

// cluster barrier: release/acquire at cluster scope (covers the DSMEM halo stores)
__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// |v| by clearing the sign bit (an integer op: no fp64 instruction)
__device__ __forceinline__ double abs_of(double v) {
    return __hiloint2double(__double2hiint(v) & 0x7fffffff, __double2loint(v));
}

__device__ __forceinline__ unsigned long long dbits(double v) {
    return static_cast<unsigned long long>(__double_as_longlong(v));
}

template <int KRX, int KRV, uint64_t MASK, uint32_t BM, int NX, int RPC, int NT, int P, bool NZ, int CL>
__global__ void __launch_bounds__(NT, 1) cluster_xm_kernel(ClusterBatch B) {
    constexpr int kXmCl = CL; // CTAs per path
    using L = XmLayout<MASK, KRX, KRV, BM, NX, RPC>;
    using RE = RowExt<MASK>;
    constexpr int TR = L::TR, TX = L::TX, TBUF = L::TBUF;
    constexpr int NBM = L::NBM, NYE = L::NYE, NBB = L::NBB;
    constexpr int NSEG = NT / RPC;
    constexpr int LX = NX / NSEG; // points per thread along x
    constexpr int NW = NT / 32;
    constexpr int KP = kPairSlots;
    constexpr int NWIN = RE::total();
    constexpr int RW = 8;                 // ring slots per stencil row (>= span + P - 1)
    constexpr int XB = LX < 32 ? LX : 32; // columns per march block (multiple of RW and P)
    static_assert(RE::span(0) + P - 1 <= RW && RE::span(1) + P - 1 <= RW && RE::span(2) + P - 1 <= RW, "ring size");
    static_assert(LX % XB == 0 && XB % RW == 0 && XB % P == 0, "march blocks");
    static_assert(NT % RPC == 0 && NX % NSEG == 0 && LX >= 4, "x-march shape");
    static_assert(RPC >= 2 * KRV, "halo rows come from one neighbour");

    cg::cluster_group cluster = cg::this_cluster();
    const int rank = static_cast<int>(cluster.block_rank());
    const int t = threadIdx.x;
    const int lane = t & 31, warp = t >> 5;
    const int r = t % RPC;
    const int seg = t / RPC;
    const int x0 = seg * LX;
    const int row0 = rank * RPC;
    const int nx = NX;
    const int n = NX * B.a[0].nv;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* T = reinterpret_cast<double*>(smem_raw); // [2][TX][TR]
    double* S = T + 2 * TBUF;                        // [NX][RPC]
    double* bY = S + NX * RPC;                       // [4][NBB][RPC] boundary-class Y
    double* scr = T + TBUF;                          // scratch aliasing T[1]
    // window-fold scratch: T[1], or both term buffers for a one-CTA path (no neighbour can
    // push into T[0] then; re-zeroed after use)
    double* yscr = CL == 1 ? T : scr;
    static_assert(RPC * L::NYE <= (CL == 1 ? 2 : 1) * TBUF, "Y fold scratch must fit the term buffers");
    __shared__ unsigned long long slots[2][kXmCl * NW][2]; // warp maxima of every rank, per parity
    __shared__ double c[6];
    __shared__ int next_path;

    for (int q = t; q < 2 * TBUF; q += NT) T[q] = 0.0;

    const bool has_lo = rank > 0, has_hi = rank < kXmCl - 1;
    // DSMEM halo push: rows r < KRV go to the lower neighbour's rows RPC + r, rows
    // r >= RPC - KRV to the upper neighbour's rows r - RPC
    double* rem = nullptr;
    if (r < KRV && has_lo)
        rem = cluster.map_shared_rank(T, rank - 1) + (x0 + KRX) * TR + (RPC + r + KRV);
    else if (r >= RPC - KRV && has_hi)
        rem = cluster.map_shared_rank(T, rank + 1) + (x0 + KRX) * TR + (r - RPC + KRV);
    const bool do_rem = rem != nullptr;
    unsigned long long* slot_dst = cluster.map_shared_rank(&slots[0][0][0], lane < kXmCl ? lane : 0);
    static_assert(kXmCl * NW <= 64, "slot reduction covers two entries per lane");
    int* next0 = cluster.map_shared_rank(&next_path, 0);

    // own (row, x) element offsets
    const int tb = (x0 + KRX) * TR + (r + KRV); // in a T buffer
    const int sb = x0 * RPC + r;                // in S

    // global <-> x-major S through the padded row-major scratch (coalesced both ways)
    auto load_state = [&](const double* g) {
        for (int q = t; q < RPC * NX; q += NT) scr[(q / NX) * (NX + 1) + q % NX] = g[q];
        __syncthreads();
        for (int q = t; q < RPC * NX; q += NT) S[q] = scr[(q % RPC) * (NX + 1) + q / RPC];
        __syncthreads();
    };
    auto store_state = [&](double* g) {
        for (int q = t; q < RPC * NX; q += NT) scr[(q % RPC) * (NX + 1) + q / RPC] = S[q];
        __syncthreads();
        for (int q = t; q < RPC * NX; q += NT) g[q] = scr[(q / NX) * (NX + 1) + q % NX];
        __syncthreads();
    };
    // T[1] held scratch: restore its zero halo (x columns; outer rows of the edge CTAs)
    auto clear_t1 = [&]() {
        for (int q = t; q < TBUF; q += NT) scr[q] = 0.0;
        __syncthreads();
    };

    uint32_t gterm = 0;

    while (true) {
        if (rank == 0 && t == 0) next_path = atomicAdd(B.a[0].work, 1);
        cluster_barrier();
        const int vp = *next0;
        cluster_barrier();
        if (vp >= B.total) break;
        int sidx = 0; // the session this virtual path belongs to
        while (sidx + 1 < B.n && vp >= B.prefix[sidx + 1]) ++sidx;
        const ClusterArgs& a = B.a[sidx];
        const int p = vp - B.prefix[sidx];
        if (a.status[p] != 0) continue;

        const int par = a.par[p];
        double* gstate = (par ? a.S1 : a.S0) + static_cast<size_t>(p) * n + static_cast<size_t>(row0) * nx;
        load_state(gstate);
        clear_t1();

        int w = a.win0, rec = a.rec_next[p];
        long long terms = 0, windows = 0, segments = 0;
        bool blown = false;
        double sn_last = 0.0;

        auto do_records = [&](int wdone) {
            const long long step = static_cast<long long>(wdone + 1) * a.dt_steps;
            while (rec < a.R && a.rec_steps[rec] == step) {
                if (rec < a.R - 1) {
                    store_state(a.rec[rec] + static_cast<size_t>(p) * n + static_cast<size_t>(row0) * nx);
                    clear_t1();
                }
                if (rank == 0 && t == 0) a.rec_status[static_cast<size_t>(rec) * a.M + p] = 0;
                ++rec;
            }
        };

        while (w < a.win1 && !blown) {
            const int sw = a.stab[static_cast<size_t>(p) * a.nwin + w];
            if (sw == 0) { // norm == 0: exp(Y)u = u (sparse.cpp:449)
                ++windows;
                do_records(w);
                ++w;
                continue;
            }
            if (t < 6) c[t] = a.ctab[(static_cast<size_t>(p) * a.nwin + w) * 6 + t];
            __syncthreads();
            // fill's fold for this CTA's rows, slots ascending from 0.0, into scratch
            for (int q = t; q < RPC * NYE; q += NT) {
                const int rr = q / NYE, e = q - rr * NYE;
                const double* wr = a.wt + (static_cast<size_t>(row0 + rr) * NYE + e) * KP;
                double y = 0.0;
#pragma unroll
                for (int k = 0; k < KP; ++k) {
                    const int sl = __ldg(a.eslot + e * KP + k);
                    if (sl < 0) continue;
                    const double cs = c[sl];
                    if (cs != 0.0) y += cs * __ldg(wr + k);
                }
                yscr[q] = y;
            }
            __syncthreads();
            double y[NBM]; // interior (class 2) Y of row r
#pragma unroll
            for (int e = 0; e < NBM; ++e) y[e] = yscr[r * NYE + 2 * NBM + e];
            if constexpr (NBB > 0) {
                for (int q = t; q < 4 * NBB * RPC; q += NT) {
                    const int rr = q % RPC, eb = (q / RPC) % NBB, k4 = q / (RPC * NBB);
                    const int cls = k4 < 2 ? k4 : k4 + 1;
                    int e = 0;
                    for (int m = 0, seen = 0; m < 32; ++m)
                        if ((BM >> m) & 1) {
                            if (seen == eb) {
                                e = m;
                                break;
                            }
                            ++seen;
                        }
                    bY[q] = yscr[rr * NYE + cls * NBM + e];
                }
            }
            __syncthreads();
            if constexpr (CL == 1) {
                for (int q = t; q < TBUF; q += NT) T[q] = 0.0;
            }
            clear_t1();

            for (int sgi = 0; sgi < sw && !blown; ++sgi) {
                // segment start: term = accum = y (sparse.cpp:452-453); halos to neighbours
#pragma unroll
                for (int i = 0; i < LX; ++i) {
                    const double v = S[sb + i * RPC];
                    T[tb + i * TR] = v;
                    if (do_rem) rem[i * TR] = v;
                }
                int cur = 0;
                cluster_barrier();
                double prev = __longlong_as_double(static_cast<long long>(kInfBits));
                bool converged = false;
                for (int k = 1; k <= kMaxTerms; ++k) {
                    const double inv = 1.0 / (static_cast<double>(sw) * k);
                    const double* tin = T + cur * TBUF + tb;
                    double* tout = T + (cur ^ 1) * TBUF + tb;
                    double* rout = rem + (cur ^ 1) * TBUF;
                    double* sp = S + sb;
                    double tm = 0.0, sm = 0.0; // NaN-ignoring maxima of |t|, |accum|
                    unsigned ex = 0;           // max exponent field of accum: all-ones = non-finite
                    // per-row register rings of RW (power of two) slots over absolute columns c:
                    // slot (c - lo) & (RW-1) is periodic in c, so the march is a loop over
                    // blocks of XB columns (the last block, which may touch the zero x-halo of
                    // the last segment, is a separate instance)
                    double win[(2 * KRV + 1) * RW];
#pragma unroll
                    for (int dv = -KRV; dv <= KRV; ++dv) {
                        if (RE::span(dv) > 0) {
#pragma unroll
                            for (int cc = 0; cc < RW; ++cc) // constant trip count: always unrolled
                                if (cc < RE::span(dv) - 1) win[(dv + KRV) * RW + cc] = tin[(RE::lo(dv) + cc) * TR + dv];
                        }
                    }
                    auto block = [&](const int cbase, auto last_tag) {
                        constexpr bool LAST = decltype(last_tag)::value;
                        const double* tinb = tin + cbase * TR;
                        double* toutb = tout + cbase * TR;
                        double* routb = rout + cbase * TR;
                        double* spb = sp + cbase * RPC;
                        const bool first_blk = cbase == 0;
                        (void)first_blk;
#pragma unroll
                        for (int g = 0; g < XB; g += P) {
#pragma unroll
                            for (int dv = -KRV; dv <= KRV; ++dv)
                                if (RE::span(dv) > 0) {
#pragma unroll
                                    for (int q = 0; q < P; ++q) {
                                        const int col = g + q + RE::hi(dv);
                                        win[(dv + KRV) * RW + ((col - RE::lo(dv)) & (RW - 1))] = tinb[col * TR + dv];
                                    }
                                }
                            int bcls[P];
#pragma unroll
                            for (int q = 0; q < P; ++q) {
                                const int i = g + q;
                                bcls[q] = -1;
                                if constexpr (NBB > 0) {
                                    if (i < 2 && first_blk && seg == 0) bcls[q] = i;
                                    if (LAST && i >= XB - 2 && seg == NSEG - 1) bcls[q] = 2 + (i - (XB - 2));
                                }
                            }
                            double acc[P];
#pragma unroll
                            for (int q = 0; q < P; ++q) acc[q] = 0.0;
#pragma unroll
                            for (int dv = -KRV; dv <= KRV; ++dv) {
#pragma unroll
                                for (int dx = -KRX; dx <= KRX; ++dx) {
                                    if (MaskInfo<MASK>::has(dx, dv)) {
                                        const int e = MaskInfo<MASK>::rank(box_bit(dx, dv));
#pragma unroll
                                        for (int q = 0; q < P; ++q) {
                                            double wv = y[e];
                                            if constexpr (NBB > 0) {
                                                if ((BM >> e) & 1) {
                                                    if (bcls[q] >= 0)
                                                        wv = bY[(bcls[q] * NBB + bm_rank(BM, e)) * RPC + r];
                                                }
                                            }
                                            const int col = g + q + dx;
                                            const double pr = wv * win[(dv + KRV) * RW + ((col - RE::lo(dv)) & (RW - 1))];
                                            // NZ: start at the first product, not 0.0 + it (only the
                                            // sign of an all-zero sum differs; the accumulator and
                                            // hence every state bit cannot, see DESIGN "Parity")
                                            acc[q] = (NZ && e == 0) ? pr : acc[q] + pr;
                                        }
                                    }
                                }
                            }
#pragma unroll
                            for (int q = 0; q < P; ++q) {
                                const int i = g + q;
                                const double tv = acc[q] * inv;
                                const double sv = spb[i * RPC] + tv;
                                toutb[i * TR] = tv;
                                if (do_rem) routb[i * TR] = tv;
                                spb[i * RPC] = sv;
                                if (fabs(tv) > tm) tm = abs_of(tv);
                                if (fabs(sv) > sm) sm = abs_of(sv);
                                ex = max(ex, static_cast<unsigned>(__double2hiint(sv)) & 0x7ff00000u);
                            }
                        }
                    };
#pragma unroll 1
                    for (int cbase = 0; cbase < LX - XB; cbase += XB) block(cbase, std::false_type{});
                    block(LX - XB, std::true_type{});
                    if (ex == 0x7ff00000u) sm = __longlong_as_double(0x7FF8000000000000LL); // non-finite
                    // path-wide max|t|, max|accum| (NaN-ranked): every warp pushes its maxima into
                    // a slot of every rank (lane l -> rank l, DSMEM), so no CTA barrier sits in the
                    // term loop; after the cluster barrier each warp reduces all CL x NW slots
                    const unsigned long long wtb = warp_max_bits(dbits(tm));
                    const unsigned long long wsb = warp_max_bits(dbits(sm));
                    const int kp = gterm & 1;
                    if (lane < kXmCl) {
                        slot_dst[((kp * kXmCl + rank) * NW + warp) * 2 + 0] = wtb;
                        slot_dst[((kp * kXmCl + rank) * NW + warp) * 2 + 1] = wsb;
                    }
                    cluster_barrier();
                    unsigned long long tball = 0ull, sball = 0ull;
#pragma unroll
                    for (int q = lane; q < kXmCl * NW; q += 32) {
                        tball = umax64(tball, slots[kp][q][0]);
                        sball = umax64(sball, slots[kp][q][1]);
                    }
                    tball = warp_max_bits(tball);
                    sball = warp_max_bits(sball);
                    int dec = 0;
                    if (tball >= kInfBits || sball >= kInfBits) {
                        dec = 2; // Overflow
                    } else {
                        const double tn = __longlong_as_double(static_cast<long long>(tball));
                        const double sn = __longlong_as_double(static_cast<long long>(sball));
                        const double gate = a.tol * sn;
                        if (tn <= gate && prev <= gate) dec = 1;
                        prev = tn;
                        sn_last = sn;
                    }
                    ++gterm;
                    ++terms;
                    cur ^= 1;
                    if (dec == 2) {
                        blown = true;
                        break;
                    }
                    if (dec == 1) {
                        converged = true;
                        break;
                    }
                }
                if (!blown && !converged) blown = true; // ToleranceNotReached
                if (!blown) ++segments;
            }
            if (blown) break;
            // window-level cap (magnus.cpp:282-286)
            if (sn_last > a.cap) {
                blown = true;
                break;
            }
            ++windows;
            do_records(w);
            ++w;
        }
        if (!blown) store_state(gstate);
        if (rank == 0 && t == 0) {
            a.terms[p] += terms;
            a.windows[p] += windows;
            a.segments[p] += segments;
            a.rec_next[p] = rec;
            a.win[p] = w;
            a.status[p] = blown ? 2 : (w >= a.nwin ? 1 : 0);
        }
        // the next path reuses every buffer (and the neighbours push halos into ours)
        cluster_barrier();
    }
}

template <int V, int NX, int RPC, int NT, bool NZ, int CL>
void launch_xm(s2b_context* ctx, const ClusterBatch& a) {
    constexpr Variant v = kVariants[V];
    constexpr int kXmCl = CL;
    auto kern = cluster_xm_kernel<v.rx, v.rv, v.mask, v.bm, NX, RPC, NT, kXmP, NZ, CL>;
    const size_t smem = XmLayout<v.mask, v.rx, v.rv, v.bm, NX, RPC>::bytes();
    S2B_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    cudaLaunchConfig_t cfg{};
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kXmCl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(kXmCl);
    int clusters = 0;
    S2B_CUDA(cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg));
    clusters = grid_cap(std::max(1, std::min(clusters, a.total)));
    cfg.gridDim = dim3(kXmCl * clusters);
    S2B_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
    ctx->k_cluster = reinterpret_cast<const void*>(kern);
}

bool xm_enabled() {
    const char* e = std::getenv("S2B_XM");
    return !(e && e[0] == '0');
}

} // namespace

// grids: 256^2 as 8 CTAs x 32 rows (15 clusters fit), 128^2 as 4 x 32 (33 fit), 64^2 as one
// CTA of 64 rows per path (148 fit)
bool cluster_xm_supported(int variant, int nx, int nv) {
    if (!xm_enabled()) return false;
    if (variant < 7 || variant > 9) return false;
    return nx == nv && (nx == 256 || nx == 128 || nx == 64);
}

namespace {
template <int V, bool NZ>
void launch_xm_grid(s2b_context* ctx, const ClusterBatch& a) {
    switch (a.a[0].nx) {
    case 256: launch_xm<V, 256, 32, kXmNT, NZ, 8>(ctx, a); break;
    case 128: launch_xm<V, 128, 32, kXmNT, NZ, 4>(ctx, a); break;
    case 64: launch_xm<V, 64, 64, kXmNT, NZ, 1>(ctx, a); break;
    default: fail(S2B_ERR_RUNTIME, "x-march cluster engine: unsupported grid");
    }
}
} // namespace

void launch_cluster_xm(s2b_context* ctx, int variant, const ClusterBatch& a) {
    bool nz = true;
    for (int i = 0; i < a.n; ++i) nz = nz && a.a[i].nz;
    switch (variant * 2 + (nz ? 1 : 0)) {
    case 14: launch_xm_grid<7, false>(ctx, a); break;
    case 15: launch_xm_grid<7, true>(ctx, a); break;
    case 16: launch_xm_grid<8, false>(ctx, a); break;
    case 17: launch_xm_grid<8, true>(ctx, a); break;
    case 18: launch_xm_grid<9, false>(ctx, a); break;
    case 19: launch_xm_grid<9, true>(ctx, a); break;
    default: fail(S2B_ERR_RUNTIME, "x-march cluster engine: unsupported variant");
    }
    S2B_LAUNCHED(ctx);
}

} // namespace mg
} // namespace s2b
