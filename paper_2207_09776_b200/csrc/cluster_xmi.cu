// Cluster-resident Magnus, in-place x-march: for grids whose term + accumulator do not fit
// a cluster's shared memory (512 x 512: 4 MB per path vs 3.6 MB in a 16-CTA cluster).
//
// Same decomposition and arithmetic as cluster_xm.cu (lane = row, x-march with the row's Y
// in registers, P points in flight, DSMEM halo push, one cluster barrier per Taylor term,
// REDUX norms), with two changes that halve the shared-memory footprint:
//  * the term is updated IN PLACE in one shared buffer.  Within a warp a column is loaded
//    into the register rings before it is overwritten (program order); across warps the
//    KRX columns a warp reads from its neighbour segments are preloaded into registers
//    before a CTA barrier, after which every warp overwrites only its own segment.  The
//    KRV halo rows received from the neighbour CTAs are double-buffered by term parity
//    (two slot sets per side, interleaved so that every row read is base + immediate).
//  * the accumulator lives in global memory (L2-resident: 2 MB per path, one slot per
//    resident cluster), x-major per CTA so that a warp's 32 rows are one 256-byte line;
//    each thread reads/writes only its own points, prefetched one step ahead.
// Everything else (window fold of Y, stopping rule, blow-up exits, records) is cluster_xm's.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "magnus_common.cuh"

namespace cg = cooperative_groups;

namespace s2b {
namespace mg {

namespace {

constexpr int kXiCl = 16;
constexpr int kXiNT = 256;
constexpr int kXiP = 4;

template <uint64_t MASK>
struct RowExtI {
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
    // right-halo preload: columns LX .. LX + hi(dv) - 1 of every stencil row
    static constexpr int rh_off(int dv) {
        int o = 0;
        for (int d = -kBoxR; d < dv; ++d) o += span(d) > 0 && hi(d) > 0 ? hi(d) : 0;
        return o;
    }
    static constexpr int rh_total() { return rh_off(kBoxR + 1); }
};

__host__ __device__ constexpr int popc32i(uint32_t v) { return v == 0 ? 0 : static_cast<int>(v & 1u) + popc32i(v >> 1); }
__host__ __device__ constexpr int bm_rank_i(uint32_t bm, int e) { return popc32i(bm & ((1u << e) - 1u)); }

template <uint64_t MASK, int KRX, int KRV, uint32_t BM, int NX, int RPC>
struct XiLayout {
    static constexpr int TRI = RPC + 4 * KRV; // own rows + two halo slot sets per side
    static constexpr int TX = NX + 2 * KRX;
    static constexpr int TBUF = TX * TRI;
    static constexpr int NBM = MaskInfo<MASK>::count();
    static constexpr int NYE = kClasses * NBM;
    static constexpr int NBB = popc32i(BM);
    static constexpr size_t bytes() {
        return 8 * (static_cast<size_t>(TBUF) + static_cast<size_t>(RPC) * NYE + 4 * static_cast<size_t>(NBB) * RPC);
    }
};

__device__ __forceinline__ unsigned long long warp_max_bits_i(unsigned long long b) {
    const unsigned hi = static_cast<unsigned>(b >> 32), lo = static_cast<unsigned>(b);
    const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
    return (static_cast<unsigned long long>(mh) << 32) | ml;
}

__device__ __forceinline__ double abs_of_i(double v) {
    return __hiloint2double(__double2hiint(v) & 0x7fffffff, __double2loint(v));
}

__device__ __forceinline__ void cluster_barrier_i() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int KRX, int KRV, uint64_t MASK, uint32_t BM, int NX, int RPC, int NT, int P, int CL, bool NZ>
__global__ void __launch_bounds__(NT, 1) cluster_xmi_kernel(ClusterBatch B) {
    using L = XiLayout<MASK, KRX, KRV, BM, NX, RPC>;
    using RE = RowExtI<MASK>;
    constexpr int TRI = L::TRI, TBUF = L::TBUF;
    constexpr int NBM = L::NBM, NYE = L::NYE, NBB = L::NBB;
    constexpr int NSEG = NT / RPC;
    constexpr int LX = NX / NSEG;
    constexpr int NW = NT / 32;
    constexpr int KP = kPairSlots;
    constexpr int RW = 8;  // ring slots per stencil row (>= span + P - 1)
    constexpr int XB = 32; // columns per march block (multiple of RW and P)
    static_assert(RE::span(0) + P - 1 <= RW && RE::span(1) + P - 1 <= RW && RE::span(2) + P - 1 <= RW, "ring size");
    static_assert(LX % XB == 0 && XB % RW == 0 && XB % P == 0, "march blocks");
    constexpr int NRH = RE::rh_total();
    static_assert(NT % RPC == 0 && NX % NSEG == 0 && LX % P == 0 && LX >= 4, "x-march shape");
    static_assert(RPC >= 2 * KRV, "halo rows come from one neighbour");
#define XI_RSPAN(dv) (RE::span(dv) + P - 1)
#define XI_ROFF(dv) (RE::off(dv) + ((dv) + KRV) * (P - 1))

    cg::cluster_group cluster = cg::this_cluster();
    const int rank = static_cast<int>(cluster.block_rank());
    const int t = threadIdx.x;
    const int lane = t & 31, warp = t >> 5;
    const int r = t % RPC;
    const int seg = t / RPC;
    const int x0 = seg * LX;
    const int row0 = rank * RPC;
    const int n = NX * B.a[0].nv;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* T = reinterpret_cast<double*>(smem_raw); // [TX][TRI]
    double* Ys = T + TBUF;                           // [RPC][NYE] window fold scratch
    double* bY = Ys + RPC * NYE;                     // [4][NBB][RPC]
    __shared__ unsigned long long slots[2][CL][2];
    __shared__ unsigned long long red[NW][2];
    __shared__ double c[6];
    __shared__ int next_path;

    for (int q = t; q < TBUF; q += NT) T[q] = 0.0;

    // row index inside a column: own rows at 2KRV + row; halo slot set `par` shifted by KRV
    auto ridx = [&](int row, int par) {
        int i = 2 * KRV + row;
        if (par) i += row < 0 ? -KRV : (row >= RPC ? KRV : 0);
        return i;
    };
    const bool has_lo = rank > 0, has_hi = rank < CL - 1;
    const int cb = (x0 + KRX) * TRI; // column x0 of this segment
    double* rem0 = nullptr; // halo push target in the neighbour's slot set 0 / 1
    double* rem1 = nullptr;
    if (r < KRV && has_lo) {
        double* nb = cluster.map_shared_rank(T, rank - 1);
        rem0 = nb + cb + ridx(RPC + r, 0);
        rem1 = nb + cb + ridx(RPC + r, 1);
    } else if (r >= RPC - KRV && has_hi) {
        double* nb = cluster.map_shared_rank(T, rank + 1);
        rem0 = nb + cb + ridx(r - RPC, 0);
        rem1 = nb + cb + ridx(r - RPC, 1);
    }
    const bool do_rem = rem0 != nullptr;
    unsigned long long* slot_dst = cluster.map_shared_rank(&slots[0][0][0], lane < CL ? lane : 0);
    int* next0 = cluster.map_shared_rank(&next_path, 0);
    double* own = T + cb + 2 * KRV + r;
    const int slot_id = static_cast<int>(blockIdx.x) / CL;
    double* SX = B.a[0].sx + (static_cast<size_t>(slot_id) * CL + rank) * NX * RPC; // [NX][RPC]
    double* sxp = SX + static_cast<size_t>(x0) * RPC + r;

    uint32_t gterm = 0;
    int ip = 0; // halo slot set holding the current term's input rows

    while (true) {
        if (rank == 0 && t == 0) next_path = atomicAdd(B.a[0].work, 1);
        cluster_barrier_i();
        const int vp = *next0;
        cluster_barrier_i();
        if (vp >= B.total) break;
        int sidx = 0; // the session this virtual path belongs to
        while (sidx + 1 < B.n && vp >= B.prefix[sidx + 1]) ++sidx;
        const ClusterArgs& a = B.a[sidx];
        const int p = vp - B.prefix[sidx];
        if (a.status[p] != 0) continue;

        const int par = a.par[p];
        double* gstate = (par ? a.S1 : a.S0) + static_cast<size_t>(p) * n + static_cast<size_t>(row0) * NX;
        for (int q = t; q < RPC * NX; q += NT) SX[(q % NX) * RPC + q / NX] = gstate[q];
        __syncthreads();

        int w = a.win0, rec = a.rec_next[p];
        long long terms = 0, windows = 0, segments = 0;
        bool blown = false;
        double sn_last = 0.0;

        auto store_rows = [&](double* g) {
            __syncthreads();
            for (int q = t; q < RPC * NX; q += NT) g[q] = SX[(q % NX) * RPC + q / NX];
        };
        auto do_records = [&](int wdone) {
            const long long step = static_cast<long long>(wdone + 1) * a.dt_steps;
            while (rec < a.R && a.rec_steps[rec] == step) {
                if (rec < a.R - 1) store_rows(a.rec[rec] + static_cast<size_t>(p) * n + static_cast<size_t>(row0) * NX);
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
            __syncthreads();
            if (t < 6) c[t] = a.ctab[(static_cast<size_t>(p) * a.nwin + w) * 6 + t];
            __syncthreads();
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
                Ys[q] = y;
            }
            __syncthreads();
            double y[NBM];
#pragma unroll
            for (int e = 0; e < NBM; ++e) y[e] = Ys[r * NYE + 2 * NBM + e];
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
                    bY[q] = Ys[rr * NYE + cls * NBM + e];
                }
                __syncthreads();
            }

            for (int sgi = 0; sgi < sw && !blown; ++sgi) {
                // segment start: term = accum = y (sparse.cpp:452-453), halos into slot set ip
                double* rseg = ip ? rem1 : rem0;
#pragma unroll 8
                for (int i = 0; i < LX; ++i) {
                    const double v = __ldcg(sxp + i * RPC);
                    own[i * TRI] = v;
                    if (do_rem) rseg[i * TRI] = v;
                }
                cluster_barrier_i();
                double prev = __longlong_as_double(static_cast<long long>(kInfBits));
                bool converged = false;
                for (int k = 1; k <= kMaxTerms; ++k) {
                    const double inv = 1.0 / (static_cast<double>(sw) * k);
                    const int op = ip ^ 1;
                    // per stencil row: base of row r+dv (own rows or halo slot set ip)
                    const double* rp[2 * KRV + 1];
#pragma unroll
                    for (int dv = -KRV; dv <= KRV; ++dv) rp[dv + KRV] = T + cb + ridx(r + dv, ip);
                    double* rout = op ? rem1 : rem0;
                    double tm = 0.0, sm = 0.0;
                    unsigned ex = 0;
                    // per-row register rings of RW (power of two) slots over absolute columns:
                    // slot (c - lo) & (RW-1), periodic in c, so the march can be a rolled loop
                    // over blocks of XB columns (a fully unrolled 64-point march exceeds the
                    // unroller's budget and would put the rings in local memory)
                    double win[(2 * KRV + 1) * RW];
                    double rh[NRH > 0 ? NRH : 1];
                    // prime (columns lo .. hi-1, incl. the left neighbour segment's) and the
                    // right neighbour segment's columns: read before anyone overwrites them
#pragma unroll
                    for (int dv = -KRV; dv <= KRV; ++dv) {
                        if (RE::span(dv) > 0) {
#pragma unroll
                            for (int cc = 0; cc < RW; ++cc) // constant trip counts: always unrolled
                                if (cc < RE::span(dv) - 1)
                                    win[(dv + KRV) * RW + cc] = rp[dv + KRV][(RE::lo(dv) + cc) * TRI];
#pragma unroll
                            for (int q = 0; q < kBoxR; ++q)
                                if (q < RE::hi(dv)) rh[RE::rh_off(dv) + q] = rp[dv + KRV][(LX + q) * TRI];
                        }
                    }
                    double snx[P];
#pragma unroll
                    for (int q = 0; q < P; ++q) snx[q] = __ldcg(sxp + q * RPC);
                    __syncthreads();
                    // one block of XB columns starting at cbase (a multiple of RW); LAST: the
                    // segment's final block (right-halo columns come from rh)
                    auto block = [&](const int cbase, auto last_tag) __attribute__((always_inline)) {
                        constexpr bool LAST = decltype(last_tag)::value;
                        const double* rpb[2 * KRV + 1];
#pragma unroll
                        for (int d = 0; d < 2 * KRV + 1; ++d) rpb[d] = rp[d] + cbase * TRI;
                        double* ownb = own + cbase * TRI;
                        double* routb = rout + cbase * TRI;
                        double* sxb = sxp + cbase * RPC;
                        const bool first_blk = cbase == 0;
                        (void)first_blk;
#pragma unroll
                        for (int g = 0; g < XB; g += P) {
                            double scur[P];
#pragma unroll
                            for (int q = 0; q < P; ++q) scur[q] = snx[q];
                            if (!LAST || g + P < XB) {
#pragma unroll
                                for (int q = 0; q < P; ++q) snx[q] = __ldcg(sxb + (g + P + q) * RPC);
                            }
#pragma unroll
                            for (int dv = -KRV; dv <= KRV; ++dv)
                                if (RE::span(dv) > 0) {
#pragma unroll
                                    for (int q = 0; q < P; ++q) {
                                        const int col = g + q + RE::hi(dv); // relative to cbase
                                        const int sl = (dv + KRV) * RW + ((col - RE::lo(dv)) & (RW - 1));
                                        if (LAST && col >= XB)
                                            win[sl] = rh[RE::rh_off(dv) + (col - XB)];
                                        else
                                            win[sl] = rpb[dv + KRV][col * TRI];
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
                                                        wv = bY[(bcls[q] * NBB + bm_rank_i(BM, e)) * RPC + r];
                                                }
                                            }
                                            const int col = g + q + dx;
                                            const double pr = wv * win[(dv + KRV) * RW + ((col - RE::lo(dv)) & (RW - 1))];
                                            // NZ (datum without -0.0): start at the first product, as
                                            // cluster_xm (DESIGN "Parity")
                                            acc[q] = (NZ && e == 0) ? pr : acc[q] + pr;
                                        }
                                    }
                                }
                            }
#pragma unroll
                            for (int q = 0; q < P; ++q) {
                                const int i = g + q;
                                const double tv = acc[q] * inv;
                                const double sv = scur[q] + tv;
                                ownb[i * TRI] = tv;
                                if (do_rem) routb[i * TRI] = tv;
                                __stcg(sxb + i * RPC, sv);
                                if (fabs(tv) > tm) tm = abs_of_i(tv);
                                if (fabs(sv) > sm) sm = abs_of_i(sv);
                                ex = max(ex, static_cast<unsigned>(__double2hiint(sv)) & 0x7ff00000u);
                            }
                        }
                    };
#pragma unroll 1
                    for (int cbase = 0; cbase < LX - XB; cbase += XB) block(cbase, std::false_type{});
                    block(LX - XB, std::true_type{});
                    if (ex == 0x7ff00000u) sm = __longlong_as_double(0x7FF8000000000000LL);
                    const unsigned long long wtb = warp_max_bits_i(static_cast<unsigned long long>(__double_as_longlong(tm)));
                    const unsigned long long wsb = warp_max_bits_i(static_cast<unsigned long long>(__double_as_longlong(sm)));
                    if (lane == 0) {
                        red[warp][0] = wtb;
                        red[warp][1] = wsb;
                    }
                    __syncthreads();
                    const int kp = gterm & 1;
                    if (warp == 0) {
                        const unsigned long long ct = warp_max_bits_i(lane < NW ? red[lane][0] : 0ull);
                        const unsigned long long cs = warp_max_bits_i(lane < NW ? red[lane][1] : 0ull);
                        if (lane < CL) {
                            slot_dst[(kp * CL + rank) * 2 + 0] = ct;
                            slot_dst[(kp * CL + rank) * 2 + 1] = cs;
                        }
                    }
                    cluster_barrier_i();
                    const unsigned long long tball = warp_max_bits_i(lane < CL ? slots[kp][lane][0] : 0ull);
                    const unsigned long long sball = warp_max_bits_i(lane < CL ? slots[kp][lane][1] : 0ull);
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
                    ip = op;
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
            if (sn_last > a.cap) { // window-level cap (magnus.cpp:282-286)
                blown = true;
                break;
            }
            ++windows;
            do_records(w);
            ++w;
        }
        if (!blown) store_rows(gstate);
        if (rank == 0 && t == 0) {
            a.terms[p] += terms;
            a.windows[p] += windows;
            a.segments[p] += segments;
            a.rec_next[p] = rec;
            a.win[p] = w;
            a.status[p] = blown ? 2 : (w >= a.nwin ? 1 : 0);
        }
        __syncthreads();
        cluster_barrier_i();
    }
#undef XI_RSPAN
#undef XI_ROFF
}

template <int V, int NX, int RPC, bool NZ>
void launch_xmi(s2b_context* ctx, const ClusterBatch& a) {
    constexpr Variant v = kVariants[V];
    auto kern = cluster_xmi_kernel<v.rx, v.rv, v.mask, v.bm, NX, RPC, kXiNT, kXiP, kXiCl, NZ>;
    const size_t smem = XiLayout<v.mask, v.rx, v.rv, v.bm, NX, RPC>::bytes();
    S2B_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    S2B_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg{};
    cfg.blockDim = dim3(kXiNT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kXiCl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(kXiCl);
    int clusters = 0;
    S2B_CUDA(cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg));
    clusters = grid_cap(std::max(1, std::min({clusters, a.total, a.a[0].sx_slots})));
    cfg.gridDim = dim3(kXiCl * clusters);
    S2B_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
    ctx->k_cluster = reinterpret_cast<const void*>(kern);
}

bool xmi_enabled() {
    const char* e = std::getenv("S2B_XMI");
    return !(e && e[0] == '0');
}

} // namespace

bool cluster_xmi_supported(int variant, int nx, int nv) {
    if (!xmi_enabled()) return false;
    if (variant < 7 || variant > 9) return false;
    return nx == 512 && nv == 512;
}

size_t cluster_xmi_scratch(int nx, int nv, int* slots) {
    *slots = 148 / kXiCl + 1; // upper bound on resident clusters
    return static_cast<size_t>(*slots) * static_cast<size_t>(nx) * nv;
}

void launch_cluster_xmi(s2b_context* ctx, int variant, const ClusterBatch& a) {
    bool nz = true;
    for (int i = 0; i < a.n; ++i) nz = nz && a.a[i].nz;
    const char* e = std::getenv("S2B_XMI_NZ"); // 0: the literal 0.0 + first product (A/B)
    if (e && e[0] == '0') nz = false;
    switch (variant * 2 + (nz ? 1 : 0)) {
    case 14: launch_xmi<7, 512, 32, false>(ctx, a); break;
    case 15: launch_xmi<7, 512, 32, true>(ctx, a); break;
    case 16: launch_xmi<8, 512, 32, false>(ctx, a); break;
    case 17: launch_xmi<8, 512, 32, true>(ctx, a); break;
    case 18: launch_xmi<9, 512, 32, false>(ctx, a); break;
    case 19: launch_xmi<9, 512, 32, true>(ctx, a); break;
    default: fail(S2B_ERR_RUNTIME, "in-place cluster engine: unsupported variant");
    }
    S2B_LAUNCHED(ctx);
}

} // namespace mg
} // namespace s2b
