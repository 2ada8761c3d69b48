// Streaming x-march Taylor-term engine for the compressed Langevin stencils (variants 7-9) on
// grids whose paths do not fit a cluster (1024^2: cfg5).
//
// term_tma_kernel gives each thread two x-points of a row and marches down v: every row costs
// it the Y row (19 broadcast loads), a ring wait, a CTA barrier every two rows and the loop
// bookkeeping, all for 2 points -- 60% of its issued instructions are not DMUL/DADD
// (profiles/r02_term_tma_cfg5_ncu.json).  This engine turns the march by 90 degrees, as the
// cluster x-march kernel (cluster_xm.cu) does on chip:
//  * lane = row (v), the thread marches along x.  Y is x-invariant away from the two x-boundary
//    columns on each side, so the thread's row of Y sits in registers for the whole work item
//    (the y_j of MagnusLogBuilder::fill, magnus.cpp:141-160) and the inner loop only loads the
//    term -- one value per stencil row per point, from per-row register rings.
//  * while a session runs on this engine its term and accumulator vectors are kept x-major in
//    HBM ([path][x][v]); the session transposes them on entry and exit of the pass loop and
//    record snapshots are written row-major (xs_* helpers below).  A work item is
//    (live path, 32-row block); it walks the x range in tiles of kCW columns.  One TMA tensor
//    copy brings the tile's term with its halo (zero outside the grid: TMA out-of-bounds fill)
//    as [x][36 rows] -- lane r reads row r + dv of column c, 32 consecutive doubles, no bank
//    conflict -- and one more the accumulator tile; outputs go straight from registers to
//    HBM, 32 consecutive doubles per warp store.
//  * the Y rows of a path are folded once per window (xs_fold_kernel, at the window's first
//    pass) into [path][v][YW] and copied with the item's first tile.
// The arithmetic per point is the reference's and every other engine's: Y.t summed from 0.0 in
// ascending (dv, dx) order (== ascending DIA diagonal, sparse.cpp:412-423), t = acc * (1/(s*k)),
// S += t, no FMA; maxima as integer maxima of |.| bit patterns (NaN ranks above Inf) exactly as
// term_tma_kernel, judged by control_kernel (sparse.cpp:463-492).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "magnus_common.cuh"

namespace s2b {
namespace mg {

namespace {

constexpr int kXsNT = 256;   // 8 warps x 32 rows
constexpr int kXsRows = 32;  // rows per work item (lane = row)
constexpr int kCW = 128;     // tile columns (16 per warp)
constexpr int kXsStages = 3; // tile ring depth

__host__ __device__ constexpr int popc32x(uint32_t v) { return v == 0 ? 0 : static_cast<int>(v & 1u) + popc32x(v >> 1); }
__host__ __device__ constexpr int bm_rankx(uint32_t bm, int e) { return popc32x(bm & ((1u << e) - 1u)); }

template <uint64_t MASK>
struct XsRow { // extent of stencil row dv along x
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
};

template <int KRX, int KRV, uint64_t MASK, uint32_t BM>
struct XsLayout {
    static constexpr int NBM = MaskInfo<MASK>::count();
    static constexpr int NBB = popc32x(BM);
    static constexpr int YW0 = NBM + 4 * NBB;
    static constexpr int YW = YW0 | 1;                 // odd row stride: lane reads conflict-free
    static constexpr int HV = KRV < 2 ? 2 : KRV;       // halo rows of the tile (>= 2: the box
                                                       // starts on an even row, 32-byte columns)
    static constexpr int TR = kXsRows + 2 * HV;        // tile rows incl. halo
    static constexpr int TX = kCW + 2 * KRX;           // tile columns incl. halo
    static constexpr int TBYTES = TR * TX * 8;
    static constexpr int SBYTES = kCW * kXsRows * 8;
    static constexpr int YBYTES = kXsRows * YW * 8;
    static constexpr int TOFF = 0;
    static constexpr int SOFF = (TBYTES + 127) / 128 * 128;
    static constexpr int STAGE = SOFF + SBYTES;        // multiple of 128
    static constexpr int YOFF = kXsStages * STAGE;     // two Y buffers (item parity)
    static constexpr int YSTR = (YBYTES + 127) / 128 * 128;
    static constexpr int BAROFF = YOFF + 2 * YSTR;
    static constexpr size_t bytes() { return 128 + BAROFF + 64; } // + alignment slack, barriers
    static_assert(TR * 8 % 16 == 0, "TMA box inner extent must be a multiple of 16 bytes");
    static_assert(YBYTES % 16 == 0, "Y rows: one bulk copy");
};

__device__ __forceinline__ void tma_tile3(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}

// st.global under a predicate (keeps an epilogue branch-free: the compiler otherwise wraps a
// conditional store and its operands in a divergent branch)
__device__ __forceinline__ void st_if(double* ptr, double v, bool p) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.f64 [%0], %1;\n\t}" ::"l"(ptr), "d"(v),
                 "r"(static_cast<int>(p)));
}

} // namespace

// T0, T1, S0, S1 with the term box (rows + halo, columns + halo); S0, S1 with the accumulator box
struct XsMaps {
    CUtensorMap t[4];
    CUtensorMap s[2];
};

namespace {

// MagnusLogBuilder::fill (magnus.cpp:141-160) for the paths that enter a window this pass
// (k == 1, seg == 0): entries [0, NBM) interior Y, then the boundary classes 0, 1, nx-2, nx-1 of
// the BM entries.  The fold is the one of every other engine: slots ascending from 0.0, zero
// coefficients skipped.
template <uint64_t MASK, uint32_t BM>
__global__ void xs_fold_kernel(TermArgs a, const int* __restrict__ seg, double* __restrict__ Yg, int YW, int yrows,
                               int4* __restrict__ meta4, const int* __restrict__ tpar) {
    constexpr int NBM = MaskInfo<MASK>::count();
    constexpr int NBB = popc32x(BM);
    constexpr int NYE = kClasses * NBM;
    constexpr int KP = kPairSlots;
    constexpr int NE = NBM + 4 * NBB;
    const int nv = a.op.nv;
    const int live = a.cnt[0];
    for (int q = blockIdx.y; q < live; q += gridDim.y) {
        const int p = a.act[q];
        // every live path's (path, k, parity, segments) for the term kernel's producer
        if (blockIdx.x == 0 && threadIdx.x == 0)
            meta4[q] = make_int4(p, a.k[p], a.par[p] | (tpar ? tpar[p] << 2 : 0), a.nseg[p]);
        if (a.k[p] != 1 || seg[p] != 0) continue;
        const double* c = a.ctab + (static_cast<size_t>(p) * a.nwin + a.win[p]) * 6;
        for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < nv * NE; u += gridDim.x * blockDim.x) {
            const int row = u / NE, j = u - row * NE;
            int cls = 2, e = j;
            if constexpr (NBB > 0) if (j >= NBM) {
                const int k4 = (j - NBM) / NBB, b = (j - NBM) - k4 * NBB;
                cls = k4 < 2 ? k4 : k4 + 1;
                for (int m = 0, seen = 0; m < 32; ++m)
                    if ((BM >> m) & 1) {
                        if (seen == b) {
                            e = m;
                            break;
                        }
                        ++seen;
                    }
            }
            const int ee = cls * NBM + e;
            const double* wr = a.wt + (static_cast<size_t>(row) * NYE + ee) * KP;
            double y = 0.0;
#pragma unroll
            for (int k = 0; k < KP; ++k) {
                const int sl = __ldg(a.eslot + ee * KP + k);
                if (sl < 0) continue;
                const double cs = __ldg(c + sl);
                if (cs != 0.0) y += cs * __ldg(wr + k);
            }
            Yg[(static_cast<size_t>(p) * yrows + row + 2) * YW + j] = y;
        }
    }
}

template <int KRX, int KRV, uint64_t MASK, uint32_t BM, bool NZ, int NVC>
__global__ void __launch_bounds__(kXsNT, 1)
    term_xs_kernel(const __grid_constant__ XsMaps maps, TermArgs a, const double* __restrict__ Yg, int yrows,
                   const int4* __restrict__ meta4, int nrb, int nxt, int pf) {
    using L = XsLayout<KRX, KRV, MASK, BM>;
    using RE = XsRow<MASK>;
    constexpr int NBM = L::NBM, NBB = L::NBB, YW = L::YW, TR = L::TR;
    constexpr int NW = kXsNT / 32;
    constexpr int LX = kCW / NW; // points per thread per tile
    constexpr int P = 4;         // points in flight (independent DADD chains)
    constexpr int RW = 8;        // ring slots per stencil row (>= span + P - 1, power of two)
    static_assert(RE::span(0) + P - 1 <= RW && RE::span(1) + P - 1 <= RW && RE::span(2) + P - 1 <= RW, "ring size");
    static_assert(LX % P == 0, "march groups");

    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int nx = a.op.nx, nv = NVC > 0 ? NVC : a.op.nv; // compile-time column height: immediate store offsets
    const size_t n = static_cast<size_t>(nx) * nv;

    extern __shared__ unsigned char smem_raw[];
    const uint32_t base_u = (smem_u32(smem_raw) + 127u) & ~127u;
    unsigned char* base = smem_raw + (base_u - smem_u32(smem_raw));
    const uint32_t full_u = base_u + L::BAROFF;
    __shared__ unsigned long long red[2][2][NW];
    __shared__ int meta[kXsStages][3];  // the step's path, parity (written by the producer)
    __shared__ double minv[kXsStages];  // 1 / (segments * k) of that path

    if (t == 0) {
        for (int s = 0; s < kXsStages; ++s) mbar_init(reinterpret_cast<uint64_t*>(base + L::BAROFF) + s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const long long items = static_cast<long long>(a.cnt[0]) * nrb;
    const long long mine = items > blockIdx.x ? (items - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const long long nsteps = mine * nxt;

    // step g: item blockIdx.x + (g / nxt) * gridDim.x, tile g % nxt
    // The producer (thread 0) reads each item's (path, k, parity, segments) one item ahead, so the
    // issue of an item's first tile never waits on a global load (a late producer holds every
    // warp at the next CTA barrier)
    const long long nitems = mine;
    auto item_meta = [&](long long it) -> int4 {
        return it < nitems ? __ldg(meta4 + (blockIdx.x + it * gridDim.x) / nrb) : make_int4(0, 1, 0, 1);
    };
    int4 cur_m = make_int4(0, 1, 0, 1), next_m = make_int4(0, 1, 0, 1);
    if (t == 0) next_m = item_meta(0);
    auto issue = [&](long long g) {
        const long long it = g / nxt;
        const int tile = static_cast<int>(g - it * nxt);
        if (tile == 0) {
            if (pf) {
                cur_m = next_m;
                next_m = item_meta(it + 1);
            } else {
                cur_m = item_meta(it);
            }
        }
        const long long wi = blockIdx.x + it * gridDim.x;
        const int p = cur_m.x, kk = cur_m.y, par = cur_m.z;
        const int rb = static_cast<int>(wi % nrb);
        const int slot = static_cast<int>(g % kXsStages);
        // read by every thread at the step, after at least one CTA barrier (kXsStages >= 2)
        meta[slot][0] = p;
        meta[slot][1] = par;
        minv[slot] = 1.0 / (static_cast<double>(cur_m.w) * kk);
        const uint32_t bar = full_u + 8 * slot;
        const uint32_t st = base_u + slot * L::STAGE;
        uint32_t bytes = L::TBYTES + L::SBYTES;
        if (tile == 0) bytes += L::YBYTES;
        mbar_expect_tx_u(bar, bytes);
        // the first term of a segment reads the accumulator as its input (term = accum = y)
        tma_tile3(st + L::TOFF, &maps.t[kk == 1 ? 2 + par : par], rb * kXsRows - L::HV, tile * kCW - KRX, p, bar);
        tma_tile3(st + L::SOFF, &maps.s[par], rb * kXsRows, tile * kCW, p, bar);
        if (tile == 0)
            tma_row_u(base_u + L::YOFF + static_cast<uint32_t>(it & 1) * L::YSTR,
                      Yg + (static_cast<size_t>(p) * yrows + static_cast<size_t>(rb) * kXsRows + 2) * YW, L::YBYTES, bar);
    };
    if (t == 0)
        for (long long g = 0; g < kXsStages && g < nsteps; ++g) issue(g);
    __syncthreads(); // the prologue's step metadata

    double y[NBM];
    double inv = 0.0;
    unsigned long long tm = 0, sm = 0;
    int p = 0, v = 0;
    double* Tout = nullptr;
    double* Sout = nullptr;

    for (long long g = 0; g < nsteps; ++g) {
        const long long it = g / nxt;
        const int tile = static_cast<int>(g - it * nxt);
        const int slot = static_cast<int>(g % kXsStages);
        mbar_wait_u(full_u + 8 * slot, static_cast<uint32_t>((g / kXsStages) & 1));
        const double* ybuf = reinterpret_cast<const double*>(base + L::YOFF + (it & 1) * L::YSTR);
        if (tile == 0) {
            const long long wi = blockIdx.x + it * gridDim.x;
            p = meta[slot][0];
            const int rb = static_cast<int>(wi % nrb);
            v = rb * kXsRows + lane;
            const int par = meta[slot][1];
            inv = minv[slot];
            const size_t pbase = static_cast<size_t>(p) * n;
            Tout = (par ? a.T0 : a.T1) + pbase;
            Sout = (par ? a.S0 : a.S1) + pbase;
#pragma unroll
            for (int e = 0; e < NBM; ++e) y[e] = ybuf[lane * YW + e];
            tm = 0;
            sm = 0;
        }
        const double* tt = reinterpret_cast<const double*>(base + slot * L::STAGE + L::TOFF);
        const double* ts = reinterpret_cast<const double*>(base + slot * L::STAGE + L::SOFF);
        const int xw = tile * kCW + warp * LX; // global x of the thread's first point
        // own element (segment column 0, row lane) in the term tile
        const double* tin = tt + (warp * LX + KRX) * TR + (lane + L::HV);
        const double* sp = ts + warp * LX * kXsRows + lane;
        double* to = Tout + static_cast<size_t>(xw) * nv + v;
        double* so = Sout + static_cast<size_t>(xw) * nv + v;

        auto march = [&](auto edge_tag) {
            constexpr int EDGE = decltype(edge_tag)::value; // 0 interior, 1 left (x = 0, 1), 2 right
            double win[(2 * KRV + 1) * RW];
#pragma unroll
            for (int dv = -KRV; dv <= KRV; ++dv) {
                if (RE::span(dv) > 0) {
#pragma unroll
                    for (int cc = 0; cc < RW; ++cc)
                        if (cc < RE::span(dv) - 1) win[(dv + KRV) * RW + cc] = tin[(RE::lo(dv) + cc) * TR + dv];
                }
            }
#pragma unroll
            for (int gq = 0; gq < LX; gq += P) {
#pragma unroll
                for (int dv = -KRV; dv <= KRV; ++dv)
                    if (RE::span(dv) > 0) {
#pragma unroll
                        for (int q = 0; q < P; ++q) {
                            const int col = gq + q + RE::hi(dv);
                            win[(dv + KRV) * RW + ((col - RE::lo(dv)) & (RW - 1))] = tin[col * TR + dv];
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
                                const int i = gq + q;
                                double wv = y[e];
                                if constexpr (NBB > 0 && EDGE != 0) {
                                    if ((BM >> e) & 1) {
                                        // class index among {0, 1, nx-2, nx-1}
                                        const int k4 = EDGE == 1 ? (i < 2 ? i : -1) : (i >= LX - 2 ? 2 + (i - (LX - 2)) : -1);
                                        if (k4 >= 0) wv = ybuf[lane * YW + NBM + k4 * NBB + bm_rankx(BM, e)];
                                    }
                                }
                                const int col = i + dx;
                                const double pr = wv * win[(dv + KRV) * RW + ((col - RE::lo(dv)) & (RW - 1))];
                                // NZ: start at the first product, not 0.0 + it (only the sign of an
                                // all-zero sum differs; the accumulator and hence every state bit
                                // cannot, see DESIGN "Parity")
                                acc[q] = (NZ && e == 0) ? pr : acc[q] + pr;
                            }
                        }
                    }
                }
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    const int i = gq + q;
                    const double tv = acc[q] * inv;
                    const double sv = sp[i * kXsRows] + tv;
                    to[static_cast<size_t>(i) * nv] = tv;
                    so[static_cast<size_t>(i) * nv] = sv;
                    tm = umax64(tm, abs_bits(tv));
                    sm = umax64(sm, abs_bits(sv));
                }
            }
        };
        if (NBB > 0 && tile == 0 && warp == 0)
            march(std::integral_constant<int, 1>{});
        else if (NBB > 0 && tile == nxt - 1 && warp == NW - 1)
            march(std::integral_constant<int, 2>{});
        else
            march(std::integral_constant<int, 0>{});

        const bool last = tile == nxt - 1;
        if (last) {
            const unsigned long long wt = warp_umax(tm), ws = warp_umax(sm);
            if (lane == 0) {
                red[it & 1][0][warp] = wt;
                red[it & 1][1][warp] = ws;
            }
        }
        __syncthreads(); // the slot (and, after an item's last tile, its Y buffer) is consumed
        if (t == 0) {
            if (last) {
                unsigned long long t2 = 0, s2 = 0;
#pragma unroll
                for (int w = 0; w < NW; ++w) {
                    t2 = umax64(t2, red[it & 1][0][w]);
                    s2 = umax64(s2, red[it & 1][1][w]);
                }
                if (t2) atomicMax(&a.tn[p], t2);
                if (s2) atomicMax(&a.sn[p], s2);
            }
            if (g + kXsStages < nsteps) issue(g + kXsStages);
        }
    }
}

// ---- two Taylor terms per pass (temporal blocking) ------------------------------------------
//
// term_xs2_kernel applies the generator twice per pass: t_k is computed into shared memory and
// never leaves the SM, so a pass reads t_{k-1}, s_{k-1} and writes t_{k+1}, s_{k+1} and s_k (the
// stopping rule may end the segment at k) -- 40 B per two terms instead of 64 B.  It follows
// term2_kernel's buffer protocol, so stream_loop2 / control2_kernel / normalize2 drive it
// unchanged: T[tpar] -> T[tpar^1] (t_{k+1}); S[sidx] -> S[(sidx+1)%3] (s_{k+1}), S[(sidx+2)%3]
// (s_k); maxima of term k in tn/sn, of term k+1 in tn2/sn2.
// Work item (path, block of output rows starting at v0); two item shapes (Xs2Layout::H):
//  * H (default): 32-row blocks, lane r is row v0+r in both phases.  Phase 1: t_k on the 32
//    rows over tile columns [jW+2, jW+W+2), then t_k's 2 halo rows on each side (recomputed by
//    the neighbouring items) by a 2-point march per lane; all of it into the shared t_k buffer TK
//    whose first 4 columns [jW-2, jW+2) were computed by the previous tile (the x-march runs
//    ahead by 2 columns; tile 0 computes columns 0, 1 itself and zeroes -2, -1); every lane also
//    forms s_k = s_{k-1} + t_k and writes it.  Phase 2: t_{k+1} = (Y t_k) / (s (k+1)) over
//    [jW, jW+W) and s_{k+1} = (s_{k-1} + t_k) + t_{k+1} -- the same operations on the same
//    operands as two single passes.
//  * !H (S2B_XS2H=0): 28-row blocks, lane r is row v0-2+r; lanes 0, 1, 30, 31 compute the halo
//    rows of t_k in phase 1 and idle in phase 2.
// Rows and columns outside the grid are zero in TK.
constexpr int kX2Out = 28; // output rows per item
constexpr int kX2Stages = 2;

// H = false: 28 output rows per item, lanes 0, 1, 30, 31 compute t_k's halo rows (idle in
// phase 2).  H = true: 32 output rows per item (every lane owns its row in both phases); the 4
// halo rows of t_k are computed by a 2-point march per lane (lanes = 4 rows x 8 column pairs of
// the warp's 16 columns).  Row strides 42 / 38 (not 40 / 36) keep those lanes' shared-memory
// accesses at most 2-way conflicted.
template <int KRX, int KRV, uint64_t MASK, uint32_t BM, bool H>
struct Xs2Layout {
    static constexpr int NBM = MaskInfo<MASK>::count();
    static constexpr int NBB = popc32x(BM);
    static constexpr int YW = (NBM + 4 * NBB) | 1;
    static constexpr int OUT = H ? 32 : kX2Out;   // output rows per item
    static constexpr int RO = H ? 0 : -2;         // lane r is row v0 + RO + r
    static constexpr int TR = H ? 42 : 36;        // input rows from v0-4 (H uses 40)
    static constexpr int TX = kCW + 6;            // input columns jW-2 .. jW+W+4
    static constexpr int SR = OUT;                // s_{k-1} rows v0 .. v0+OUT
    static constexpr int SX = kCW + 2;            // s_{k-1} columns jW .. jW+W+2
    static constexpr int KX = kCW + 4;            // t_k columns jW-2 .. jW+W+2
    static constexpr int KR = H ? 38 : 32;        // t_k column stride (rows from v0-2; H uses 36)
    static constexpr int YR = H ? 36 : 32;        // Y rows per item, from v0-2
    static constexpr int TBYTES = TR * TX * 8;
    static constexpr int SBYTES = SR * SX * 8;
    static constexpr int YBYTES = YR * YW * 8;
    static constexpr int SOFF = (TBYTES + 127) / 128 * 128;
    static constexpr int STAGE = SOFF + (SBYTES + 127) / 128 * 128;
    static constexpr int KOFF = kX2Stages * STAGE;
    static constexpr int YOFF = KOFF + (KX * KR * 8 + 127) / 128 * 128;
    static constexpr int YSTR = (YBYTES + 127) / 128 * 128;
    static constexpr int BAROFF = YOFF + 2 * YSTR;
    static constexpr size_t bytes() { return 128 + BAROFF + 64; }
    static_assert(KRX <= 2 && KRV <= 2, "two-term tiles carry 2 halo rows / columns per term");
    static_assert(SR * 8 % 16 == 0 && TR * 8 % 16 == 0 && YBYTES % 16 == 0, "TMA extents");
};

// The x-march of one thread over NPTS points of its row: point i reads the tile at
// tin[(i + dx) * CS + dv].  Points [0, LB) take the x-boundary classes 0, 1; points RB0, RB0+1
// (RB0 >= 0) the classes nx-2, nx-1 (Y entries of BM from yb, the row's boundary block).
// epi(i, acc) receives the point's stencil sum (summed from 0.0 in ascending (dv, dx) order, or
// from the first product under NZ).
template <int KRX, int KRV, uint64_t MASK, uint32_t BM, bool NZ, int CS, int NPTS, int LB, int RB0, class Epi>
__device__ __forceinline__ void xs_march(const double* tin, const double* y, const double* yb, Epi&& epi) {
    using RE = XsRow<MASK>;
    constexpr int NBB = popc32x(BM);
    constexpr int P = 4, RW = 8;
    static_assert(RE::span(0) + P - 1 <= RW && RE::span(1) + P - 1 <= RW && RE::span(2) + P - 1 <= RW, "ring size");
    double win[(2 * KRV + 1) * RW];
#pragma unroll
    for (int dv = -KRV; dv <= KRV; ++dv) {
        if (RE::span(dv) > 0) {
#pragma unroll
            for (int cc = 0; cc < RW; ++cc)
                if (cc < RE::span(dv) - 1) win[(dv + KRV) * RW + cc] = tin[(RE::lo(dv) + cc) * CS + dv];
        }
    }
#pragma unroll
    for (int gq = 0; gq < NPTS; gq += P) {
#pragma unroll
        for (int dv = -KRV; dv <= KRV; ++dv)
            if (RE::span(dv) > 0) {
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    if (gq + q < NPTS) {
                        const int col = gq + q + RE::hi(dv);
                        win[(dv + KRV) * RW + ((col - RE::lo(dv)) & (RW - 1))] = tin[col * CS + dv];
                    }
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
                        const int i = gq + q;
                        if (i < NPTS) {
                            double wv = y[e];
                            if constexpr (NBB > 0) {
                                if ((BM >> e) & 1) {
                                    const int k4 = i < LB ? i : (RB0 >= 0 && i >= RB0 && i < RB0 + 2 ? 2 + (i - RB0) : -1);
                                    if (k4 >= 0) wv = yb[k4 * NBB + bm_rankx(BM, e)];
                                }
                            }
                            const int col = i + dx;
                            const double pr = wv * win[(dv + KRV) * RW + ((col - RE::lo(dv)) & (RW - 1))];
                            acc[q] = (NZ && e == 0) ? pr : acc[q] + pr;
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int q = 0; q < P; ++q)
            if (gq + q < NPTS) epi(gq + q, acc[q]);
    }
}

// T0, T1, S0, S1, S2 with the input box; S0, S1, S2 with the accumulator box
struct Xs2Maps {
    CUtensorMap t[5];
    CUtensorMap s[3];
};

template <int KRX, int KRV, uint64_t MASK, uint32_t BM, bool NZ, int NVC, bool H>
__global__ void __launch_bounds__(kXsNT, 1)
    term_xs2_kernel(const __grid_constant__ Xs2Maps maps, TermArgs a, Term2Args b, const double* __restrict__ Yg,
                    int yrows, const int4* __restrict__ meta4, int nrb, int nxt) {
    using L = Xs2Layout<KRX, KRV, MASK, BM, H>;
    constexpr int NBM = L::NBM, YW = L::YW, KR = L::KR, SR = L::SR, RO = L::RO;
    constexpr int NW = kXsNT / 32;
    constexpr int LX = kCW / NW;
    static_assert(LX == 16, "16 columns per warp");

    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int nx = a.op.nx, nv = NVC > 0 ? NVC : a.op.nv;
    const size_t n = static_cast<size_t>(nx) * nv;

    extern __shared__ unsigned char smem_raw[];
    const uint32_t base_u = (smem_u32(smem_raw) + 127u) & ~127u;
    unsigned char* base = smem_raw + (base_u - smem_u32(smem_raw));
    const uint32_t full_u = base_u + L::BAROFF;
    double* TK = reinterpret_cast<double*>(base + L::KOFF); // [KX][KR]
    __shared__ unsigned long long red[2][4][NW];
    __shared__ int meta[kX2Stages][3];  // path, accumulator index, term parity
    __shared__ double minv[kX2Stages][2];

    for (int q = t; q < L::KX * KR; q += kXsNT) TK[q] = 0.0;
    if (t == 0) {
        for (int s = 0; s < kX2Stages; ++s) mbar_init(reinterpret_cast<uint64_t*>(base + L::BAROFF) + s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const long long items = static_cast<long long>(a.cnt[0]) * nrb;
    const long long mine = items > blockIdx.x ? (items - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const long long nsteps = mine * nxt;
    auto item_meta = [&](long long it) -> int4 {
        return it < mine ? __ldg(meta4 + (blockIdx.x + it * gridDim.x) / nrb) : make_int4(0, 1, 0, 1);
    };
    int4 cur_m = make_int4(0, 1, 0, 1), next_m = make_int4(0, 1, 0, 1);
    if (t == 0) next_m = item_meta(0);
    auto issue = [&](long long g) {
        const long long it = g / nxt;
        const int tile = static_cast<int>(g - it * nxt);
        if (tile == 0) {
            cur_m = next_m;
            next_m = item_meta(it + 1);
        }
        const long long wi = blockIdx.x + it * gridDim.x;
        const int p = cur_m.x, kk = cur_m.y, sidx = cur_m.z & 3, tp = cur_m.z >> 2;
        const int v0 = static_cast<int>(wi % nrb) * L::OUT;
        const int slot = static_cast<int>(g % kX2Stages);
        meta[slot][0] = p;
        meta[slot][1] = sidx;
        meta[slot][2] = tp;
        minv[slot][0] = 1.0 / (static_cast<double>(cur_m.w) * kk);
        minv[slot][1] = 1.0 / (static_cast<double>(cur_m.w) * (kk + 1));
        const uint32_t bar = full_u + 8 * slot;
        const uint32_t st = base_u + slot * L::STAGE;
        uint32_t bytes = L::TBYTES + L::SBYTES;
        if (tile == 0) bytes += L::YBYTES;
        mbar_expect_tx_u(bar, bytes);
        // term k-1: the accumulator itself at a segment's first term (term = accum = y)
        tma_tile3(st, &maps.t[kk == 1 ? 2 + sidx : tp], v0 - 4, tile * kCW - 2, p, bar);
        tma_tile3(st + L::SOFF, &maps.s[sidx], v0, tile * kCW, p, bar);
        if (tile == 0) // Y rows v0-2 .. v0-2+YR (padded layout: row v at index v + 2)
            tma_row_u(base_u + L::YOFF + static_cast<uint32_t>(it & 1) * L::YSTR,
                      Yg + (static_cast<size_t>(p) * yrows + static_cast<size_t>(v0)) * YW, L::YBYTES, bar);
    };
    if (t == 0)
        for (long long g = 0; g < kX2Stages && g < nsteps; ++g) issue(g);
    __syncthreads();

    double y[NBM];
    double inv1 = 0.0, inv2 = 0.0;
    unsigned long long tm1 = 0, sm1 = 0, tm2 = 0, sm2 = 0;
    int p = 0, v0 = 0;
    bool rowok = false, own = false;
    double* Tn = nullptr; // t_{k+1}
    double* Sa = nullptr; // s_{k+1}
    double* Sb = nullptr; // s_k

    for (long long g = 0; g < nsteps; ++g) {
        const long long it = g / nxt;
        const int tile = static_cast<int>(g - it * nxt);
        const int slot = static_cast<int>(g % kX2Stages);
        mbar_wait_u(full_u + 8 * slot, static_cast<uint32_t>((g / kX2Stages) & 1));
        const double* ybuf = reinterpret_cast<const double*>(base + L::YOFF + (it & 1) * L::YSTR);
        if (tile == 0) {
            const long long wi = blockIdx.x + it * gridDim.x;
            p = meta[slot][0];
            const int sidx = meta[slot][1], tp = meta[slot][2];
            v0 = static_cast<int>(wi % nrb) * L::OUT;
            const int vr = v0 + RO + lane;
            rowok = vr >= 0 && vr < nv;
            own = (H || (lane >= 2 && lane < 2 + kX2Out)) && vr < nv;
            inv1 = minv[slot][0];
            inv2 = minv[slot][1];
            const size_t pbase = static_cast<size_t>(p) * n;
            double* const S2 = b.S2;
            Tn = (tp ? a.T0 : a.T1) + pbase;
            Sa = (sidx == 0 ? a.S1 : sidx == 1 ? S2 : a.S0) + pbase;
            Sb = (sidx == 0 ? S2 : sidx == 1 ? a.S0 : a.S1) + pbase;
#pragma unroll
            for (int e = 0; e < NBM; ++e) y[e] = ybuf[(lane + RO + 2) * YW + e];
            tm1 = sm1 = tm2 = sm2 = 0;
        }
        const double* yb = ybuf + (lane + RO + 2) * YW + NBM;
        const double* tt = reinterpret_cast<const double*>(base + slot * L::STAGE);
        const double* ts = reinterpret_cast<const double*>(base + slot * L::STAGE + L::SOFF);
        const int jW = tile * kCW;
        const int vr = v0 + RO + lane;
        const size_t vo = static_cast<size_t>(vr);
        const int kr = lane + RO + 2; // this lane's row in the t_k buffer
        const int sr = lane + RO;     // ... in the s_{k-1} tile

        // Every warp runs ONE unrolled march per phase over its 16 columns; the x-boundary
        // columns (other Y classes) and the two columns past the grid are masked out of that
        // march's epilogue and handled by 2-point marches of the edge warps (small code: the
        // instruction cache holds the kernel).  Epilogues are branch-free: rows a lane does not
        // own are computed and dropped by predicated stores and selects.
        const bool edge_l = tile == 0 && warp == 0, edge_r = tile == nxt - 1 && warp == NW - 1;
        // ---- phase 1: t_k (and s_k) over columns [jW+2, jW+W+2) (+ columns 0, 1 at tile 0)
        {
            const int xa = jW + 2 + warp * LX;
            const int hi1 = edge_r ? LX - 4 : LX; // columns nx-2.. of the last tile: below
            double* const sbw = Sb + static_cast<size_t>(xa) * nv + vo; // column xa of this lane
            auto epi1 = [&](int x, double acc, bool keep) {
                double tv = acc * inv1;
                tv = rowok ? tv : 0.0;
                TK[(x - jW + 2) * KR + kr] = tv;
                const double sv = ts[(x - jW) * SR + sr] + tv;
                const bool w = own && keep;
                st_if(sbw + (x - xa) * nv, sv, w);
                tm1 = umax64(tm1, w ? abs_bits(tv) : 0ull);
                sm1 = umax64(sm1, w ? abs_bits(sv) : 0ull);
            };
            const double* tin = tt + (xa - jW + 2) * L::TR + (lane + RO + 4);
            xs_march<KRX, KRV, MASK, BM, NZ, L::TR, LX, 0, -1>(tin, y, yb,
                                                               [&](int i, double acc) { epi1(xa + i, acc, i < hi1); });
            if (edge_l) // columns 0, 1: classes 0, 1
                xs_march<KRX, KRV, MASK, BM, NZ, L::TR, 2, 2, -1>(tt + 2 * L::TR + (lane + RO + 4), y, yb,
                                                                   [&](int i, double acc) { epi1(i, acc, true); });
            if (edge_r) { // columns nx-2, nx-1: classes 3, 4; nx, nx+1 are outside the grid (zero)
                xs_march<KRX, KRV, MASK, BM, NZ, L::TR, 2, 0, 0>(tin + (LX - 4) * L::TR, y, yb,
                                                                  [&](int i, double acc) { epi1(xa + LX - 4 + i, acc, true); });
                TK[(xa + LX - 2 - jW + 2) * KR + kr] = 0.0;
                TK[(xa + LX - 1 - jW + 2) * KR + kr] = 0.0;
            }
            if constexpr (H) {
                // t_k's halo rows v0-2, v0-1, v0+32, v0+33 over the warp's 16 columns: lane =
                // (row h, column pair c); Y of that row read from shared memory
                const int h = lane >> 3, c = lane & 7;
                const int hr = h < 2 ? h : 32 + h; // row in the t_k buffer (v0 - 2 + hr)
                const int vh = v0 - 2 + hr;
                const bool hok = vh >= 0 && vh < nv;
                const double* yh = ybuf + hr * YW;
                const int xh = xa + 2 * c;
                const double* tinh = tt + (xh - jW + 2) * L::TR + (hr + 2);
                auto epih = [&](int x, double acc, bool keep) {
                    const double tv = acc * inv1;
                    TK[(x - jW + 2) * KR + hr] = hok && keep ? tv : 0.0;
                };
                if (edge_r && c == 6) // columns nx-2, nx-1
                    xs_march<KRX, KRV, MASK, BM, NZ, L::TR, 2, 0, 0>(tinh, yh, yh + NBM,
                                                                      [&](int i, double acc) { epih(xh + i, acc, true); });
                else // (edge_r, c == 7: columns nx, nx+1 are outside the grid)
                    xs_march<KRX, KRV, MASK, BM, NZ, L::TR, 2, 0, -1>(
                        tinh, yh, yh + NBM, [&](int i, double acc) { epih(xh + i, acc, !(edge_r && c == 7)); });
                if (edge_l && c == 0) // columns 0, 1
                    xs_march<KRX, KRV, MASK, BM, NZ, L::TR, 2, 2, -1>(tt + 2 * L::TR + (hr + 2), yh, yh + NBM,
                                                                       [&](int i, double acc) { epih(i, acc, true); });
            }
        }
        __syncthreads(); // t_k of the tile (+ the carried columns) complete
        // the 4 t_k columns the next tile needs on its left: read now, placed after the barrier
        double carry = 0.0;
        if (t < 4 * KR) carry = TK[kCW * KR + t];

        // ---- phase 2: t_{k+1}, s_{k+1} over [jW, jW+W) on lanes 2..29
        {
            const int xa = jW + warp * LX;
            const int lo2 = edge_l ? 2 : 0, hi2 = edge_r ? LX - 2 : LX;
            const size_t cw = static_cast<size_t>(xa) * nv + vo; // column xa of this lane
            double* const tnw = Tn + cw;
            double* const saw = Sa + cw;
            auto epi2 = [&](int x, double acc, bool keep) {
                const double tk = TK[(x - jW + 2) * KR + kr];
                const double sk = ts[(x - jW) * SR + sr] + tk;
                const double tv = acc * inv2;
                const double sv = sk + tv;
                const bool w = own && keep;
                st_if(tnw + (x - xa) * nv, tv, w);
                st_if(saw + (x - xa) * nv, sv, w);
                tm2 = umax64(tm2, w ? abs_bits(tv) : 0ull);
                sm2 = umax64(sm2, w ? abs_bits(sv) : 0ull);
            };
            const double* tin = TK + (xa - jW + 2) * KR + kr;
            xs_march<KRX, KRV, MASK, BM, NZ, KR, LX, 0, -1>(
                tin, y, yb, [&](int i, double acc) { epi2(xa + i, acc, i >= lo2 && i < hi2); });
            if (edge_l)
                xs_march<KRX, KRV, MASK, BM, NZ, KR, 2, 2, -1>(tin, y, yb,
                                                                [&](int i, double acc) { epi2(xa + i, acc, true); });
            if (edge_r)
                xs_march<KRX, KRV, MASK, BM, NZ, KR, 2, 0, 0>(
                    tin + (LX - 2) * KR, y, yb, [&](int i, double acc) { epi2(xa + LX - 2 + i, acc, true); });
        }

        const bool last = tile == nxt - 1;
        if (last) {
            const unsigned long long w1 = warp_umax(tm1), w2 = warp_umax(sm1), w3 = warp_umax(tm2), w4 = warp_umax(sm2);
            if (lane == 0) {
                red[it & 1][0][warp] = w1;
                red[it & 1][1][warp] = w2;
                red[it & 1][2][warp] = w3;
                red[it & 1][3][warp] = w4;
            }
        }
        __syncthreads(); // the stage and TK are consumed
        if (t < 4 * KR) { // next tile of this item: carry; first tile of an item: columns -2, -1 are zero
            if (!last)
                TK[t] = carry;
            else if (t < 2 * KR)
                TK[t] = 0.0;
        }
        if (t == 0) {
            if (last) {
                unsigned long long r[4] = {0, 0, 0, 0};
#pragma unroll
                for (int w = 0; w < NW; ++w)
#pragma unroll
                    for (int q = 0; q < 4; ++q) r[q] = umax64(r[q], red[it & 1][q][w]);
                if (r[0]) atomicMax(&a.tn[p], r[0]);
                if (r[1]) atomicMax(&a.sn[p], r[1]);
                if (r[2]) atomicMax(&b.tn2[p], r[2]);
                if (r[3]) atomicMax(&b.sn2[p], r[3]);
            }
            if (g + kX2Stages < nsteps) issue(g + kX2Stages);
        }
    }
}

// per-path transpose: dst[p][c][r] = src[p][r][c] of an R x C matrix (R, C multiples of 32);
// path p's source is S[par[p]], its destination T[par[p]] (par == nullptr: buffer 0)
__global__ void xs_transpose_kernel(const double* __restrict__ s0, const double* __restrict__ s1,
                                    double* __restrict__ d0, double* __restrict__ d1, const int* __restrict__ par,
                                    int R, int C, size_t M) {
    __shared__ double tile[32][33];
    const size_t n = static_cast<size_t>(R) * C;
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (size_t p = blockIdx.z; p < M; p += gridDim.z) {
        const int b = par ? par[p] : 0;
        const double* src = (b ? s1 : s0) + p * n;
        double* dst = (b ? d1 : d0) + p * n;
        for (int k = threadIdx.y; k < 32; k += blockDim.y)
            tile[k][threadIdx.x] = src[static_cast<size_t>(r0 + k) * C + c0 + threadIdx.x];
        __syncthreads();
        for (int k = threadIdx.y; k < 32; k += blockDim.y)
            dst[static_cast<size_t>(c0 + k) * R + r0 + threadIdx.x] = tile[threadIdx.x][k];
        __syncthreads();
    }
}

// in-place transpose of paths [p_lo, M) of square d x d states S[par[p]][p] (its own inverse):
// block (bi, bj), bi <= bj, swaps the transposed 32 x 32 tiles (bi, bj) and (bj, bi)
__global__ void xs_transpose_inplace_kernel(double* __restrict__ s0, double* __restrict__ s1,
                                            const int* __restrict__ par, int d, size_t p_lo, size_t M) {
    __shared__ double ta[32][33], tb[32][33];
    const int T = d / 32;
    int bi = 0, rem = blockIdx.x; // pair index -> (bi, bj), bj >= bi
    while (rem >= T - bi) {
        rem -= T - bi;
        ++bi;
    }
    const int bj = bi + rem;
    const size_t n = static_cast<size_t>(d) * d;
    for (size_t p = p_lo + blockIdx.z; p < M; p += gridDim.z) {
        double* m = (par[p] ? s1 : s0) + p * n;
        for (int k = threadIdx.y; k < 32; k += blockDim.y) {
            ta[k][threadIdx.x] = m[static_cast<size_t>(bi * 32 + k) * d + bj * 32 + threadIdx.x];
            tb[k][threadIdx.x] = m[static_cast<size_t>(bj * 32 + k) * d + bi * 32 + threadIdx.x];
        }
        __syncthreads();
        for (int k = threadIdx.y; k < 32; k += blockDim.y) {
            m[static_cast<size_t>(bi * 32 + k) * d + bj * 32 + threadIdx.x] = tb[threadIdx.x][k];
            m[static_cast<size_t>(bj * 32 + k) * d + bi * 32 + threadIdx.x] = ta[threadIdx.x][k];
        }
        __syncthreads();
    }
}

// queued record snapshots S[par][p] (x-major) -> rec[r][p] (row-major), as record_kernel
__global__ void xs_record_kernel(const int* __restrict__ cnt, const int4* __restrict__ recq,
                                 const double* __restrict__ S0, const double* __restrict__ S1,
                                 const double* __restrict__ S2, double* const* __restrict__ rec, int nx, int nv) {
    __shared__ double tile[32][33];
    const size_t n = static_cast<size_t>(nx) * nv;
    const int nq = cnt[2];
    const int v0 = blockIdx.x * 32, x0 = blockIdx.y * 32; // source rows are x, columns v
    for (int q = blockIdx.z; q < nq; q += gridDim.z) {
        const int4 e = recq[q];
        const double* src = (e.z == 2 ? S2 : e.z ? S1 : S0) + static_cast<size_t>(e.x) * n;
        double* dst = rec[e.y] + static_cast<size_t>(e.x) * n;
        for (int k = threadIdx.y; k < 32; k += blockDim.y)
            tile[k][threadIdx.x] = src[static_cast<size_t>(x0 + k) * nv + v0 + threadIdx.x];
        __syncthreads();
        for (int k = threadIdx.y; k < 32; k += blockDim.y)
            dst[static_cast<size_t>(v0 + k) * nx + x0 + threadIdx.x] = tile[threadIdx.x][k];
        __syncthreads();
    }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        S2B_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
        if (!f || q != cudaDriverEntryPointSuccess) fail(S2B_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeFn>(f);
    }
    return fn;
}

// L2 sector promotion of the tile copies (S2B_XS_L2 = 0 / 64 / 128 / 256 bytes).  The term
// box starts 2 rows above its 32-row block, so every column copy touches a 16-byte piece of
// each neighbouring block: 64-byte promotion measured best at cfg5 (1.33e9 windows/s vs 1.25e9
// without promotion and 1.17e9 with 256-byte promotion, same run)
CUtensorMapL2promotion xs_l2_promotion() {
    const char* e = std::getenv("S2B_XS_L2");
    const int b = e ? std::atoi(e) : 64;
    return b == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
           : b == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
           : b == 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE;
}

// [M][nx][nv] doubles, box {rows, cols, 1}; out-of-bounds elements read as +0.0
void encode_xmaj(CUtensorMap* m, const double* base, size_t M, int nx, int nv, int rows, int cols) {
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(nv), static_cast<cuuint64_t>(nx), static_cast<cuuint64_t>(M)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(nv) * 8, static_cast<cuuint64_t>(nx) * nv * 8};
    const cuuint32_t box[3] = {static_cast<cuuint32_t>(rows), static_cast<cuuint32_t>(cols), 1};
    const cuuint32_t es[3] = {1, 1, 1};
    const CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box,
                                   es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   xs_l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(S2B_ERR_CUDA, "cuTensorMapEncodeTiled failed (x-major term maps)");
}

template <int V>
struct XsV {
    static constexpr Variant v = kVariants[V];
    using L = XsLayout<v.rx, v.rv, v.mask, v.bm>;
};

int xs_yw(int variant) {
    switch (variant) {
    case 7: return XsV<7>::L::YW;
    case 8: return XsV<8>::L::YW;
    case 9: return XsV<9>::L::YW;
    default: return 0;
    }
}

// Y rows per path in the padded layout (row v at index v + 2; both kernels' blocks fit, even)
int xs_yrows(int nv) {
    const int r32 = (nv + kXsRows - 1) / kXsRows * kXsRows, r28 = (nv + kX2Out - 1) / kX2Out * kX2Out;
    return (std::max(r32, r28) + 4 + 1) & ~1;
}

// the window's Y rows of every path that enters a window this pass, and the pass's item metadata
template <int V>
void launch_xs_fold(s2b_context* ctx, const TermArgs& a, const int* seg, double* Yg, int4* meta4, const int* tpar,
                    size_t M) {
    constexpr Variant v = kVariants[V];
    using L = typename XsV<V>::L;
    const int nv = a.op.nv;
    dim3 grid(static_cast<unsigned>(std::max(1, (nv * (L::NBM + 4 * L::NBB) + 255) / 256)),
              static_cast<unsigned>(std::min<size_t>(std::max<size_t>(M, 1), 512)));
    xs_fold_kernel<v.mask, v.bm><<<grid, 256, 0, ctx->stream>>>(a, seg, Yg, L::YW, xs_yrows(nv), meta4, tpar);
    S2B_LAUNCHED(ctx);
}

template <int V, bool NZ>
void launch_xs_v(s2b_context* ctx, const TermArgs& a, const int* seg, double* Yg, int4* meta4, size_t live_max) {
    constexpr Variant v = kVariants[V];
    using L = typename XsV<V>::L;
    const int nx = a.op.nx, nv = a.op.nv;
    const size_t M = live_max;
    launch_xs_fold<V>(ctx, a, seg, Yg, meta4, nullptr, M);
    XsMaps maps{};
    const double* tb[4] = {a.T0, a.T1, a.S0, a.S1};
    for (int i = 0; i < 4; ++i) encode_xmaj(&maps.t[i], tb[i], M, nx, nv, L::TR, L::TX);
    encode_xmaj(&maps.s[0], a.S0, M, nx, nv, kXsRows, kCW);
    encode_xmaj(&maps.s[1], a.S1, M, nx, nv, kXsRows, kCW);
    // compile-time column heights of the benchmark grids (immediate store offsets): 1024^2 and the
    // hybrid slices at 256^2 / 512^2
    const int nvc = nv == 1024 ? 3 : nv == 512 ? 2 : nv == 256 ? 1 : 0;
    auto kern = nvc == 3   ? term_xs_kernel<v.rx, v.rv, v.mask, v.bm, NZ, 1024>
                : nvc == 2 ? term_xs_kernel<v.rx, v.rv, v.mask, v.bm, NZ, 512>
                : nvc == 1 ? term_xs_kernel<v.rx, v.rv, v.mask, v.bm, NZ, 256>
                           : term_xs_kernel<v.rx, v.rv, v.mask, v.bm, NZ, 0>;
    const size_t smem = L::bytes();
    static int configured_device[4] = {-1, -1, -1, -1};
    if (configured_device[nvc] != ctx->device) {
        S2B_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        configured_device[nvc] = ctx->device;
    }
    const int nrb = nv / kXsRows, nxt = nx / kCW;
    const size_t work = M * static_cast<size_t>(nrb);
    const int grid = grid_cap(static_cast<int>(std::max<size_t>(1, std::min<size_t>(work, ctx->num_sms))));
    const char* pfe = std::getenv("S2B_XS_PF");
    const int pf = pfe ? std::atoi(pfe) : 1;
    kern<<<grid, kXsNT, smem, ctx->stream>>>(maps, a, Yg, xs_yrows(nv), meta4, nrb, nxt, pf);
    S2B_LAUNCHED(ctx);
    ctx->k_stream = reinterpret_cast<const void*>(kern);
}

template <int V, bool NZ, bool H>
void launch_xs2_v(s2b_context* ctx, const TermArgs& a, const Term2Args& b, const int* seg, double* Yg, int4* meta4,
                  size_t live_max) {
    constexpr Variant v = kVariants[V];
    using L = Xs2Layout<v.rx, v.rv, v.mask, v.bm, H>;
    static_assert(L::YW == XsV<V>::L::YW, "one Y layout for both kernels");
    static_assert(L::bytes() <= 227 * 1024, "shared memory");
    const int nx = a.op.nx, nv = a.op.nv;
    const size_t M = live_max;
    launch_xs_fold<V>(ctx, a, seg, Yg, meta4, b.tpar, M);
    Xs2Maps maps{};
    const double* tb[5] = {a.T0, a.T1, a.S0, a.S1, b.S2};
    for (int i = 0; i < 5; ++i) encode_xmaj(&maps.t[i], tb[i], M, nx, nv, L::TR, L::TX);
    for (int i = 0; i < 3; ++i) encode_xmaj(&maps.s[i], tb[2 + i], M, nx, nv, L::SR, L::SX);
    auto kern = nv == 1024 ? term_xs2_kernel<v.rx, v.rv, v.mask, v.bm, NZ, 1024, H>
                           : term_xs2_kernel<v.rx, v.rv, v.mask, v.bm, NZ, 0, H>;
    const size_t smem = L::bytes();
    static int configured_device[2] = {-1, -1};
    if (configured_device[nv == 1024] != ctx->device) {
        S2B_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        configured_device[nv == 1024] = ctx->device;
    }
    const int nrb = (nv + L::OUT - 1) / L::OUT, nxt = nx / kCW;
    const size_t work = M * static_cast<size_t>(nrb);
    const int grid = grid_cap(static_cast<int>(std::max<size_t>(1, std::min<size_t>(work, ctx->num_sms))));
    kern<<<grid, kXsNT, smem, ctx->stream>>>(maps, a, b, Yg, xs_yrows(nv), meta4, nrb, nxt);
    S2B_LAUNCHED(ctx);
    ctx->k_stream = reinterpret_cast<const void*>(kern);
}

} // namespace

// two Taylor terms per pass on the x-march engine (stream_loop2 with term_xs2_kernel), the
// default; S2B_XS2=0 keeps one term per pass.  cfg5: 1.44e9 vs 1.25e9 windows/s (same run),
// fp64 pipe 56% of active cycles, DRAM 40 B per two path*gridpoint*terms
bool term_xs2_enabled() {
    const char* e = std::getenv("S2B_XS2");
    return !(e && e[0] == '0');
}

void launch_term_xs2(s2b_context* ctx, const s2b_operator* op, const TermArgs& a, const Term2Args& b, const int* seg,
                     double* Yg, int4* meta4, size_t M, bool nz) {
    // 32-row items with the halo rows of t_k done by separate 2-point marches (default; cfg5
    // 1.538e9 vs 1.472e9 windows/s for 28-row items with halo lanes, same run); S2B_XS2H=0: 28-row
    const char* he = std::getenv("S2B_XS2H");
    const bool h = !(he && he[0] == '0');
    switch (op->variant * 2 + (nz ? 1 : 0)) {
    case 14: (h ? launch_xs2_v<7, false, true> : launch_xs2_v<7, false, false>)(ctx, a, b, seg, Yg, meta4, M); break;
    case 15: (h ? launch_xs2_v<7, true, true> : launch_xs2_v<7, true, false>)(ctx, a, b, seg, Yg, meta4, M); break;
    case 16: (h ? launch_xs2_v<8, false, true> : launch_xs2_v<8, false, false>)(ctx, a, b, seg, Yg, meta4, M); break;
    case 17: (h ? launch_xs2_v<8, true, true> : launch_xs2_v<8, true, false>)(ctx, a, b, seg, Yg, meta4, M); break;
    case 18: (h ? launch_xs2_v<9, false, true> : launch_xs2_v<9, false, false>)(ctx, a, b, seg, Yg, meta4, M); break;
    case 19: (h ? launch_xs2_v<9, true, true> : launch_xs2_v<9, true, false>)(ctx, a, b, seg, Yg, meta4, M); break;
    default: fail(S2B_ERR_RUNTIME, "x-major two-term engine: unsupported variant");
    }
}

bool term_xs_supported(const s2b_operator* op) {
    const char* e = std::getenv("S2B_XS");
    if (e && e[0] == '0') return false;
    const int v = op->variant;
    if (v < 7 || v > 9) return false;
    return op->nx >= 2 * static_cast<size_t>(kCW) && op->nx % kCW == 0 && op->nv % kXsRows == 0 && op->nv >= kXsRows;
}

size_t term_xs_y_doubles(const s2b_operator* op, size_t M) {
    return M * static_cast<size_t>(xs_yrows(static_cast<int>(op->nv))) * static_cast<size_t>(xs_yw(op->variant));
}

void launch_term_xs(s2b_context* ctx, const s2b_operator* op, const TermArgs& a, const int* seg, double* Yg,
                    int4* meta4, size_t M, bool nz) {
    switch (op->variant * 2 + (nz ? 1 : 0)) {
    case 14: launch_xs_v<7, false>(ctx, a, seg, Yg, meta4, M); break;
    case 15: launch_xs_v<7, true>(ctx, a, seg, Yg, meta4, M); break;
    case 16: launch_xs_v<8, false>(ctx, a, seg, Yg, meta4, M); break;
    case 17: launch_xs_v<8, true>(ctx, a, seg, Yg, meta4, M); break;
    case 18: launch_xs_v<9, false>(ctx, a, seg, Yg, meta4, M); break;
    case 19: launch_xs_v<9, true>(ctx, a, seg, Yg, meta4, M); break;
    default: fail(S2B_ERR_RUNTIME, "x-major streaming engine: unsupported variant");
    }
}

// S[par[p]][p] (R x C) -> T[par[p]][p] (C x R) for every path; the caller swaps S and T after
void xs_transpose_paths(s2b_context* ctx, const double* S0, const double* S1, double* T0, double* T1,
                        const int* par, size_t M, int R, int C) {
    if (M == 0) return;
    dim3 grid(static_cast<unsigned>(C / 32), static_cast<unsigned>(R / 32),
              static_cast<unsigned>(std::min<size_t>(M, 65535)));
    xs_transpose_kernel<<<grid, dim3(32, 8), 0, ctx->stream>>>(S0, S1, T0, T1, par, R, C, M);
    S2B_LAUNCHED(ctx);
}

void xs_transpose_paths_inplace(s2b_context* ctx, double* S0, double* S1, const int* par, size_t p_lo, size_t M,
                                int d) {
    if (M <= p_lo) return;
    const int T = d / 32;
    dim3 grid(static_cast<unsigned>(T * (T + 1) / 2), 1, static_cast<unsigned>(std::min<size_t>(M - p_lo, 65535)));
    xs_transpose_inplace_kernel<<<grid, dim3(32, 8), 0, ctx->stream>>>(S0, S1, par, d, p_lo, M);
    S2B_LAUNCHED(ctx);
}

// the x-march engine for the streaming slice of a hybrid run (paths the cluster engine leaves
// to the idle SMs): square grids only (the slice is relaid out in place); S2B_XS_SLICE=0 keeps
// term_tma_kernel there
bool term_xs_slice_supported(const s2b_operator* op) {
    const char* e = std::getenv("S2B_XS_SLICE");
    if (e && e[0] == '0') return false;
    return term_xs_supported(op) && op->nx == op->nv;
}

void xs_records(s2b_context* ctx, const int* cnt, const int4* recq, const double* S0, const double* S1,
                const double* S2, double* const* rec, int nx, int nv, size_t M) {
    dim3 grid(static_cast<unsigned>(nv / 32), static_cast<unsigned>(nx / 32),
              static_cast<unsigned>(std::min<size_t>(std::max<size_t>(M, 1), 64)));
    xs_record_kernel<<<grid, dim3(32, 8), 0, ctx->stream>>>(cnt, recq, S0, S1, S2, rec, nx, nv);
    S2B_LAUNCHED(ctx);
}

} // namespace mg
} // namespace s2b
