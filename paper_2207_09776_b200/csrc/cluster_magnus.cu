// Cluster-resident Magnus engine: one thread-block cluster owns one path for a whole range
// of windows; the path never leaves shared memory between Taylor terms.
//
// For grids whose per-path working set (term x2 + accumulator + the window's Y rows) fits
// the shared memory of an 8-CTA cluster (nx <= 256, nv a multiple of 32), the streaming
// pass engine's HBM round trip per Taylor term is replaced by shared-memory traffic: CTA
// `rank` owns rows [rank*RPC, (rank+1)*RPC) of the path, reads the two halo rows of its
// neighbours through DSMEM, and the per-term path-wide inf-norms (the stopping rule of
// expmv_into, sparse.cpp:463-492) are exchanged through rank 0's shared memory with one
// cluster barrier per term.  Y (MagnusLogBuilder::fill, magnus.cpp:141-160) is folded once
// per window for the CTA's rows instead of once per term.  The arithmetic per point is the
// streaming kernel's (bitwise the reference's): only where the data lives changes.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "magnus_common.cuh"

namespace cg = cooperative_groups;

namespace s2b {
namespace mg {

namespace {

constexpr int kBandThreads = 128; // 2 x-points per thread -> nx <= 256

template <uint64_t MASK, int KRX>
struct ClLayout {
    static constexpr int H = KRX <= 2 ? 2 : 4;
    static constexpr int NBM = MaskInfo<MASK>::count();
    static constexpr int NYE = kClasses * NBM;
    static constexpr int YST = (NYE + 1) & ~1;
    // T[2][RPC][RW], S[RPC][nx], Ys[RPC][YST]
    static size_t smem_bytes(int nx, int rpc) {
        const size_t rw = static_cast<size_t>(nx) + 2 * H;
        return 8 * (2 * static_cast<size_t>(rpc) * rw + static_cast<size_t>(rpc) * nx +
                    static_cast<size_t>(rpc) * YST);
    }
};

// Running inf-norms over a thread's points: fp64 max (NaN-ignoring, like std::max) plus a
// flag for a NaN accumulator.  A non-finite t always reaches its accumulator (s = S + t), so
// "flag or an infinite max" <=> some t or s of the term is not finite (-> Overflow).
struct NormAcc {
    double tm = 0.0, sm = 0.0;
    bool nan = false;
    __device__ __forceinline__ void add(double tA, double tB, double sA, double sB) {
        tm = fmax(tm, fmax(fabs(tA), fabs(tB)));
        sm = fmax(sm, fmax(fabs(sA), fabs(sB)));
        nan = nan || (sA != sA) || (sB != sB);
    }
    __device__ __forceinline__ unsigned long long tbits() const {
        return static_cast<unsigned long long>(__double_as_longlong(tm));
    }
    __device__ __forceinline__ unsigned long long sbits() const {
        return nan ? 0x7FF8000000000000ULL : static_cast<unsigned long long>(__double_as_longlong(sm));
    }
};

// CL CTAs per cluster, BANDS 128-thread row bands per CTA, RPB rows per band.
template <int KRX, int KRV, uint64_t MASK, uint32_t BM, int RPB, int CL, int BANDS>
__global__ void __launch_bounds__(BANDS * kBandThreads, (BANDS <= 2 ? 2 : 1)) cluster_magnus_kernel(ClusterArgs a) {
    constexpr int kCl = CL;
    constexpr int kBands = BANDS;
    constexpr int kClThreads = BANDS * kBandThreads;
    using L = ClLayout<MASK, KRX>;
    constexpr int H = L::H;
    constexpr int AOFF = (H - KRX) & ~1;
    constexpr int LAST = 1 + KRX + H;
    constexpr int NP = (LAST - AOFF) / 2 + 1;
    constexpr int WROWS = 2 * KRV + 1;
    constexpr int NBM = L::NBM;
    constexpr int NYE = L::NYE;
    constexpr int YST = L::YST;
    constexpr int KP = kPairSlots;
    constexpr int RPC = RPB * kBands; // rows owned by this CTA
    constexpr int NSTEPS = RPB + 2 * KRV;

    cg::cluster_group cluster = cg::this_cluster();
    const int rank = static_cast<int>(cluster.block_rank());
    const int nx = a.nx;
    const int n = nx * a.nv;
    const int row0 = rank * RPC; // first global row of this CTA
    const int RW = nx + 2 * H;
    const int t = threadIdx.x;
    const int band = t / kBandThreads;
    const int lt = t % kBandThreads;
    const int nint = (nx - 4) / 2;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* T = reinterpret_cast<double*>(smem_raw); // [2][RPC][RW]
    double* S = T + 2 * RPC * RW;                    // [RPC][nx]
    double* Ys = S + RPC * nx;                       // [RPC][YST]
    __shared__ unsigned long long slots[2][kCl][2];  // per-term CTA maxima (read on rank 0)
    __shared__ unsigned long long red[2][kClThreads / 32];
    __shared__ double c[6];
    __shared__ int next_path;
    __shared__ int decision; // 0 continue, 1 converged, 2 non-finite

    for (int q = t; q < 2 * RPC * RW; q += kClThreads) T[q] = 0.0; // zero x-halos, kept

    // neighbours' term buffers (DSMEM); only the edge bands read them, on their halo steps
    const double* Tn_lo = cluster.map_shared_rank(T, rank > 0 ? rank - 1 : rank);
    const double* Tn_hi = cluster.map_shared_rank(T, rank < kCl - 1 ? rank + 1 : rank);
    unsigned long long* slots0 = cluster.map_shared_rank(&slots[0][0][0], 0);
    int* next0 = cluster.map_shared_rank(&next_path, 0);

    const bool active = lt < nint + 2;
    const int p0 = lt < nint ? 2 * lt + 2 : (lt == nint ? 0 : nx - 2);
    const int clsA = lt < nint ? 2 : (lt == nint ? 0 : 3);
    const int clsB = lt < nint ? 2 : (lt == nint ? 1 : 4);
    const bool wfast = BM == 0 || __all_sync(0xffffffffu, lt < nint || !active);
    const int rb0 = band * RPB;
    const bool has_lo = rank > 0, has_hi = rank < kCl - 1;

    uint32_t gterm = 0; // cluster-uniform term counter (slot parity)

    while (true) {
        if (rank == 0 && t == 0) next_path = atomicAdd(a.work, 1);
        cluster.sync();
        const int p = *next0;
        cluster.sync(); // everyone has read next_path before rank 0 may overwrite it
        if (p >= a.M) break;
        if (a.status[p] != 0) continue;

        const int par = a.par[p];
        double* gstate = (par ? a.S1 : a.S0) + static_cast<size_t>(p) * n + static_cast<size_t>(row0) * nx;
        for (int q = t; q < RPC * nx; q += kClThreads) S[q] = gstate[q];

        int w = a.win0, rec = a.rec_next[p];
        long long terms = 0, windows = 0, segments = 0;
        bool blown = false;
        double sn_last = 0.0;

        auto do_records = [&](int wdone) {
            const long long step = static_cast<long long>(wdone + 1) * a.dt_steps;
            while (rec < a.R && a.rec_steps[rec] == step) {
                if (rec < a.R - 1) {
                    double* dst = a.rec[rec] + static_cast<size_t>(p) * n + static_cast<size_t>(row0) * nx;
                    for (int q = t; q < RPC * nx; q += kClThreads) dst[q] = S[q];
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
            // Y rows of this CTA for window w: fill's fold, slots ascending from 0.0
            for (int q = t; q < RPC * NYE; q += kClThreads) {
                const int r = q / NYE, e = q - r * NYE;
                const double* wr = a.wt + (static_cast<size_t>(row0 + r) * NYE + e) * KP;
                double y = 0.0;
#pragma unroll
                for (int k = 0; k < KP; ++k) {
                    const int sl = __ldg(a.eslot + e * KP + k);
                    if (sl < 0) continue;
                    const double cs = c[sl];
                    if (cs != 0.0) y += cs * __ldg(wr + k);
                }
                Ys[r * YST + e] = y;
            }

            for (int seg = 0; seg < sw && !blown; ++seg) {
                // segment start: term = accum = y (sparse.cpp:452-453)
                for (int r = band; r < RPC; r += kBands)
                    for (int i = lt; i < nx; i += kBandThreads) T[r * RW + H + i] = S[r * nx + i];
                int cur = 0;
                cluster.sync();
                double prev = __longlong_as_double(static_cast<long long>(kInfBits));
                bool converged = false;
                for (int k = 1; k <= kMaxTerms; ++k) {
                    const double inv = 1.0 / (static_cast<double>(sw) * k);
                    const double* Tin = T + cur * RPC * RW;
                    double* Tout = T + (cur ^ 1) * RPC * RW;
                    NormAcc acc;
                    double win[WROWS][2 * NP];
#pragma unroll
                    for (int s = 0; s < NSTEPS; ++s) {
                        const int ph = s % WROWS;
                        const int r = rb0 - KRV + s; // CTA-local input row
                        const double* src;
                        bool zero = false;
                        if (s < KRV || s >= RPB + KRV) {
                            // halo step: only the edge bands leave the CTA
                            if (r < 0) {
                                zero = !has_lo;
                                src = Tn_lo + cur * RPC * RW + (RPC + r) * RW;
                            } else if (r >= RPC) {
                                zero = !has_hi;
                                src = Tn_hi + cur * RPC * RW + (r - RPC) * RW;
                            } else {
                                src = Tin + r * RW;
                            }
                        } else {
                            src = Tin + r * RW;
                        }
                        if (zero) {
#pragma unroll
                            for (int q = 0; q < 2 * NP; ++q) win[ph][q] = 0.0;
                        } else {
                            const double2* s2 = reinterpret_cast<const double2*>(src + p0 + AOFF);
#pragma unroll
                            for (int q = 0; q < NP; ++q) {
                                const double2 v2 = s2[q];
                                win[ph][2 * q] = v2.x;
                                win[ph][2 * q + 1] = v2.y;
                            }
                        }
                        if (s >= 2 * KRV && active) {
                            const int jo = r - KRV;
                            const double* yrow = Ys + jo * YST;
                            double accA = 0.0, accB = 0.0;
                            // ascending stencil offset == ascending DIA diagonal (sparse.cpp:412-423)
                            if (wfast) {
                                const double2* y2 = reinterpret_cast<const double2*>(yrow + 2 * NBM);
#pragma unroll
                                for (int dv = -KRV; dv <= KRV; ++dv) {
                                    const int rr = ((ph - KRV + dv) % WROWS + WROWS) % WROWS;
#pragma unroll
                                    for (int dx = -KRX; dx <= KRX; ++dx) {
                                        if (MaskInfo<MASK>::has(dx, dv)) {
                                            const int e = MaskInfo<MASK>::rank(box_bit(dx, dv));
                                            const int col = H + dx - AOFF;
                                            const double wv = (e & 1) ? y2[e >> 1].y : y2[e >> 1].x;
                                            accA += wv * win[rr][col];
                                            accB += wv * win[rr][col + 1];
                                        }
                                    }
                                }
                            } else {
                                const double* yA = yrow + clsA * NBM;
                                const double* yB = yrow + clsB * NBM;
                            const double2* yi2 = reinterpret_cast<const double2*>(yrow + 2 * NBM);
#pragma unroll
                                for (int dv = -KRV; dv <= KRV; ++dv) {
                                    const int rr = ((ph - KRV + dv) % WROWS + WROWS) % WROWS;
#pragma unroll
                                    for (int dx = -KRX; dx <= KRX; ++dx) {
                                        if (MaskInfo<MASK>::has(dx, dv)) {
                                            const int e = MaskInfo<MASK>::rank(box_bit(dx, dv));
                                            const int col = H + dx - AOFF;
                                            double wA, wB;
                                            if ((BM >> e) & 1) { // per-lane boundary value
                                                wA = yA[e];
                                                wB = yB[e];
                                            } else { // interior value, broadcast
                                                wA = wB = (e & 1) ? yi2[e >> 1].y : yi2[e >> 1].x;
                                            }
                                            accA += wA * win[rr][col];
                                            accB += wB * win[rr][col + 1];
                                        }
                                    }
                                }
                            }
                            double2* sp = reinterpret_cast<double2*>(S + jo * nx + p0);
                            const double2 sv = *sp;
                            const double tA = accA * inv, tB = accB * inv;
                            const double sA = sv.x + tA, sB = sv.y + tB;
                            *reinterpret_cast<double2*>(Tout + jo * RW + H + p0) = make_double2(tA, tB);
                            *sp = make_double2(sA, sB);
                            acc.add(tA, tB, sA, sB);
                        }
                    }
                    // path-wide max|t|, max|accum|: CTA reduction, then through rank 0
                    unsigned long long tb = warp_umax(acc.tbits());
                    unsigned long long sb = warp_umax(acc.sbits());
                    if ((t & 31) == 0) {
                        red[0][t >> 5] = tb;
                        red[1][t >> 5] = sb;
                    }
                    __syncthreads();
                    const int kp = gterm & 1;
                    if (t == 0) {
                        unsigned long long t2 = 0, s2 = 0;
                        for (int q = 0; q < kClThreads / 32; ++q) {
                            t2 = umax64(t2, red[0][q]);
                            s2 = umax64(s2, red[1][q]);
                        }
                        slots0[(kp * kCl + rank) * 2 + 0] = t2;
                        slots0[(kp * kCl + rank) * 2 + 1] = s2;
                    }
                    cluster.sync();
                    if (t == 0) {
                        unsigned long long tball = 0, sball = 0;
#pragma unroll
                        for (int q = 0; q < kCl; ++q) {
                            tball = umax64(tball, slots0[(kp * kCl + q) * 2 + 0]);
                            sball = umax64(sball, slots0[(kp * kCl + q) * 2 + 1]);
                        }
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
                        decision = dec;
                    }
                    __syncthreads();
                    const int dec = decision;
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
            // window-level cap (magnus.cpp:282-286): max|u| == sn of the last term (thread 0)
            if (t == 0) decision = sn_last > a.cap ? 2 : 0;
            __syncthreads();
            if (decision == 2) {
                blown = true;
                break;
            }
            ++windows;
            do_records(w);
            ++w;
        }
        if (!blown)
            for (int q = t; q < RPC * nx; q += kClThreads) gstate[q] = S[q];
        if (rank == 0 && t == 0) {
            a.terms[p] += terms;
            a.windows[p] += windows;
            a.segments[p] += segments;
            a.rec_next[p] = rec;
            a.win[p] = w;
            a.status[p] = blown ? 2 : (w >= a.nwin ? 1 : 0);
        }
        // the next path overwrites S/T/Ys: every CTA must be past its reads of this one
        cluster.sync();
    }
}

template <int V, int RPB, int CL, int BANDS>
void launch_vr(s2b_context* ctx, const ClusterArgs& a) {
    constexpr Variant v = kVariants[V];
    auto kern = cluster_magnus_kernel<v.rx, v.rv, v.mask, v.bm, RPB, CL, BANDS>;
    const size_t smem = ClLayout<v.mask, v.rx>::smem_bytes(a.nx, RPB * BANDS);
    S2B_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    if (CL > 8) S2B_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg{};
    cfg.blockDim = dim3(BANDS * kBandThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(CL);
    int clusters = 0;
    S2B_CUDA(cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg));
    clusters = grid_cap(std::max(1, std::min(clusters, a.M)));
    cfg.gridDim = dim3(CL * clusters);
    S2B_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
    ctx->k_cluster = reinterpret_cast<const void*>(kern);
}

// Cluster shapes: 8 CTAs x 4 bands (one CTA per SM) is the default; S2B_CLUSTER=16 selects
// 16 CTAs x 2 bands (two CTAs per SM, more SMs filled but a wider barrier per term) —
// measured slower on B200 at 256^2 (8.3e8 vs 8.9e8 path*pt*windows/s).
bool use_wide_cluster() {
    static const bool wide = [] {
        const char* e = std::getenv("S2B_CLUSTER");
        return e && e[0] == '1' && e[1] == '6';
    }();
    return wide;
}

template <int V>
void launch_v(s2b_context* ctx, const ClusterArgs& a) {
    // the 16-CTA shape is instantiated only for the Langevin variants (compile time)
    if constexpr (V >= 7)
    if (use_wide_cluster() && a.nv % (16 * 2) == 0) {
        switch (a.nv / (16 * 2)) {
        case 1: launch_vr<V, 1, 16, 2>(ctx, a); return;
        case 2: launch_vr<V, 2, 16, 2>(ctx, a); return;
        case 4: launch_vr<V, 4, 16, 2>(ctx, a); return;
        case 8: launch_vr<V, 8, 16, 2>(ctx, a); return;
        }
    }
    switch (a.nv / (8 * 4)) {
    case 1: launch_vr<V, 1, 8, 4>(ctx, a); return;
    case 2: launch_vr<V, 2, 8, 4>(ctx, a); return;
    case 4: launch_vr<V, 4, 8, 4>(ctx, a); return;
    case 8: launch_vr<V, 8, 8, 4>(ctx, a); return;
    }
    fail(S2B_ERR_RUNTIME, "cluster engine: unsupported nv");
}

} // namespace

bool cluster_engine_supported(int variant, int nx, int nv) {
    if (cluster_xm_supported(variant, nx, nv) || cluster_xmi_supported(variant, nx, nv)) return true;
    if (variant < 1 || (variant > 4 && variant < 7) || variant > 9) return false;
    if (nx % 2 || nx < 6 || nx > 2 * kBandThreads) return false;
    const int rpb = nv / 32; // 8 CTAs x 4 bands (or 16 x 2)
    if (nv % 32 || (rpb != 1 && rpb != 2 && rpb != 4 && rpb != 8)) return false;
    const int rpc = rpb * 4;
    size_t smem = 0;
    switch (variant) {
    case 1: smem = ClLayout<kMask5, 1>::smem_bytes(nx, rpc); break;
    case 2: smem = ClLayout<kMask11, 1>::smem_bytes(nx, rpc); break;
    case 3: smem = ClLayout<kMask19, 2>::smem_bytes(nx, rpc); break;
    case 4: smem = ClLayout<kBox22, 2>::smem_bytes(nx, rpc); break;
    case 7: smem = ClLayout<kMask5, 1>::smem_bytes(nx, rpc); break;
    case 8: smem = ClLayout<kMask11, 1>::smem_bytes(nx, rpc); break;
    case 9: smem = ClLayout<kMask19, 2>::smem_bytes(nx, rpc); break;
    }
    return smem + 1024 <= 227 * 1024;
}

bool cluster_batch_supported(int variant, int nx, int nv) {
    return cluster_xm_supported(variant, nx, nv) || cluster_xmi_supported(variant, nx, nv);
}

void launch_cluster_magnus(s2b_context* ctx, int variant, const ClusterBatch& b) {
    const ClusterArgs& a = b.a[0];
    if (cluster_xm_supported(variant, a.nx, a.nv)) {
        launch_cluster_xm(ctx, variant, b);
        return;
    }
    if (cluster_xmi_supported(variant, a.nx, a.nv)) {
        launch_cluster_xmi(ctx, variant, b);
        return;
    }
    if (b.n != 1) fail(S2B_ERR_RUNTIME, "cluster engine: batched launch needs the x-march engines");
    switch (variant) {
    case 1: launch_v<1>(ctx, a); break;
    case 2: launch_v<2>(ctx, a); break;
    case 3: launch_v<3>(ctx, a); break;
    case 4: launch_v<4>(ctx, a); break;
    case 7: launch_v<7>(ctx, a); break;
    case 8: launch_v<8>(ctx, a); break;
    case 9: launch_v<9>(ctx, a); break;
    default: fail(S2B_ERR_RUNTIME, "cluster engine: unsupported variant");
    }
    S2B_LAUNCHED(ctx);
}

} // namespace mg
} // namespace s2b
