// Two Taylor terms per pass (temporal blocking) for the streaming Magnus engine.
//
// term_tma_kernel moves 32 B per path*gridpoint*term (reads t_{k-1}, s_{k-1}; writes t_k,
// s_k).  This kernel applies the generator twice per pass: t_k never leaves the SM, so one pass
// reads t_{k-1}, s_{k-1} and writes t_{k+1}, s_{k+1} -- plus s_k, because the stopping rule of
// expmv_into (sparse.cpp:479-481) may end the segment at term k, and the result is then s_k:
// 40 B per two terms, 20 B per term.  Both terms use the same Y (one window, one segment), so
// t_{k+1} = (Y t_k) * (1/(s(k+1))) and s_{k+1} = s_k + t_{k+1} are the same operations on the
// same operands as two single passes: the outputs are bitwise those of term_tma_kernel.
// control2_kernel (magnus.cu) evaluates the rule for term k, then for term k+1 only if the
// segment did not stop at k; a pass at k = 55 also computes a term 56 that the rule never uses.
//
// Row pipeline of one work item (path, output rows [j0, jend)), one step per input row:
//   step s: input row r = j0 - 2KRV + s arrives (TMA ring, with s-row r - KRV);
//           t_{k+1} row j2 = r - 2KRV - 1 from a register window of t_k rows (loaded from the
//           two-row shared t_k exchange after the previous step's barrier), written with
//           s_{k+1} = s_k + t_{k+1} (s_k from a register FIFO);
//           t_k row jk = r - KRV from the input window (rows outside the grid are zero), into
//           the shared exchange; for jk inside the strip also s_k = s_{k-1} + t_k, written out.
// t_k is computed for KRV halo rows on each side of the strip (recomputed by the neighbours),
// which costs 2*KRV/J of the t_k arithmetic.  Buffers: T[tpar] -> T[tpar^1] (t_{k+1});
// S[sidx] -> S[(sidx+1)%3] (s_{k+1}) and S[(sidx+2)%3] (s_k).
#pragma once

#include "term_kernel.cuh"

namespace s2b {
namespace mg {

template <int KRX, int KRV, uint64_t MASK, uint32_t BM, int NTMAX, int MINB>
__global__ void __launch_bounds__(NTMAX, MINB) term2_kernel(TermArgs a, Term2Args b) {
    constexpr int H = KRX <= 2 ? 2 : 4;
    constexpr int AOFF = (H - KRX) & ~1;
    constexpr int LAST = 1 + KRX + H;
    constexpr int NP = (LAST - AOFF) / 2 + 1;
    constexpr int WROWS = 2 * KRV + 1;
    constexpr int NBM = MaskInfo<MASK>::count();
    constexpr int NYE = kClasses * NBM;
    constexpr int YST = (NYE + 1) & ~1;
    constexpr int YR = 8; // Y row ring (a row's Y serves t_k now and t_{k+1} KRV+1 steps later)
    constexpr int KP = kPairSlots;
    static_assert(KRV + 2 <= YR, "Y ring too short");
    const int J = a.strip_rows;

    const int nx = a.op.nx, nv = a.op.nv;
    const int n = nx * nv;
    const int NT = blockDim.x;
    const int RW = nx + 2 * H;
    const int t = threadIdx.x;
    const int nint = (nx - 4) / 2;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    double* rows = reinterpret_cast<double*>(smem_raw + 128); // kStages x RW (input rows)
    double* srow = rows + kStages * RW;                       // kStages x nx (s_{k-1} rows)
    double* tk = srow + kStages * nx;                         // 2 x RW (t_k exchange, zero x-halo)
    double* Ys = tk + 2 * RW;                                 // YR x YST
    double* cq = Ys + YR * YST;                               // KP x NYE
    const uint32_t full_u = smem_u32(full), rows_u = smem_u32(rows), srow_u = smem_u32(srow);
    __shared__ double c[6];
    __shared__ unsigned long long red[4][32];

    for (int q = t; q < kStages * RW; q += NT) rows[q] = 0.0;
    for (int q = t; q < 2 * RW; q += NT) tk[q] = 0.0;
    if (t == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const bool active = t < nint + 2;
    const int p0 = t < nint ? 2 * t + 2 : (t == nint ? 0 : nx - 2);
    const int clsA = t < nint ? 2 : (t == nint ? 0 : 3);
    const int clsB = t < nint ? 2 : (t == nint ? 1 : 4);
    const bool wfast = BM == 0 || __all_sync(0xffffffffu, t < nint || !active);

    const bool owner = t < NYE;
    double own_w[KP];
    const double* wrow = a.wt + (owner ? t * KP : 0);
    auto load_w = [&](int j) {
        if (owner) {
            const double2* src = reinterpret_cast<const double2*>(wrow + static_cast<size_t>(j) * NYE * KP);
#pragma unroll
            for (int k = 0; k < KP / 2; ++k) {
                const double2 v = __ldg(src + k);
                own_w[2 * k] = v.x;
                own_w[2 * k + 1] = v.y;
            }
        }
    };
    auto fold_y = [&](int slot) { // MagnusLogBuilder::fill: slots ascending from 0.0, zeros skipped
        if (owner) {
            double y = 0.0;
#pragma unroll
            for (int k = 0; k < KP; ++k) {
                const double cs = cq[k * NYE + t];
                if (cs != 0.0) y += cs * own_w[k];
            }
            Ys[slot * YST + t] = y;
        }
    };
    // Y . window for this thread's two points (ascending stencil order == ascending DIA diagonal)
    auto apply = [&](const double* yrow, const double (&w)[WROWS][2 * NP], int ph_center, double& accA,
                     double& accB) {
        accA = 0.0;
        accB = 0.0;
        if (wfast) {
            const double2* y2 = reinterpret_cast<const double2*>(yrow + 2 * NBM);
#pragma unroll
            for (int dv = -KRV; dv <= KRV; ++dv) {
                const int rr = ((ph_center + dv) % WROWS + WROWS) % WROWS;
#pragma unroll
                for (int dx = -KRX; dx <= KRX; ++dx) {
                    if (MaskInfo<MASK>::has(dx, dv)) {
                        const int e = MaskInfo<MASK>::rank(box_bit(dx, dv));
                        const int col = H + dx - AOFF;
                        const double wv = (e & 1) ? y2[e >> 1].y : y2[e >> 1].x;
                        accA += wv * w[rr][col];
                        accB += wv * w[rr][col + 1];
                    }
                }
            }
        } else {
            const double* yA = yrow + clsA * NBM;
            const double* yB = yrow + clsB * NBM;
            const double2* yi2 = reinterpret_cast<const double2*>(yrow + 2 * NBM);
#pragma unroll
            for (int dv = -KRV; dv <= KRV; ++dv) {
                const int rr = ((ph_center + dv) % WROWS + WROWS) % WROWS;
#pragma unroll
                for (int dx = -KRX; dx <= KRX; ++dx) {
                    if (MaskInfo<MASK>::has(dx, dv)) {
                        const int e = MaskInfo<MASK>::rank(box_bit(dx, dv));
                        const int col = H + dx - AOFF;
                        double wA, wB;
                        if ((BM >> e) & 1) {
                            wA = yA[e];
                            wB = yB[e];
                        } else {
                            wA = wB = (e & 1) ? yi2[e >> 1].y : yi2[e >> 1].x;
                        }
                        accA += wA * w[rr][col];
                        accB += wB * w[rr][col + 1];
                    }
                }
            }
        }
    };

    uint32_t gstep = 0;
    const long long work = static_cast<long long>(a.cnt[0]) * a.nstrips;
    for (long long wi = blockIdx.x; wi < work; wi += gridDim.x) {
        const int p = a.act[wi / a.nstrips];
        const int strip = static_cast<int>(wi % a.nstrips);
        const int j0 = strip * J;
        const int jend = min(j0 + J, nv);
        const int kk = a.k[p];
        const int sidx = a.par[p], tp = b.tpar[p];
        const double inv1 = 1.0 / (static_cast<double>(a.nseg[p]) * kk);
        const double inv2 = 1.0 / (static_cast<double>(a.nseg[p]) * (kk + 1));
        const size_t pbase = static_cast<size_t>(p) * n;
        // S[sidx], S[(sidx+1)%3], S[(sidx+2)%3] by selects (no local-memory array)
        double* const S0 = a.S0;
        double* const S1 = a.S1;
        double* const S2 = b.S2;
        const double* Sin = (sidx == 0 ? S0 : sidx == 1 ? S1 : S2) + pbase;
        const double* in = kk == 1 ? Sin : (tp ? a.T1 : a.T0) + pbase;
        double* Tout = (tp ? a.T0 : a.T1) + pbase;
        double* Sa = (sidx == 0 ? S1 : sidx == 1 ? S2 : S0) + pbase; // s_{k+1}
        double* Sb = (sidx == 0 ? S2 : sidx == 1 ? S0 : S1) + pbase; // s_k
        const int jlo = max(0, j0 - KRV), jhi = min(nv, jend + KRV); // t_k rows computed
        const int nsteps = (jend - j0) + 4 * KRV + 1;

        auto issue = [&](int s) {
            const uint32_t slot = (gstep + s) & (kStages - 1);
            const int r = j0 - 2 * KRV + s;
            const int rs = r - KRV; // s_{k-1} row for t_k row rs
            uint32_t bytes = 0;
            const bool has_in = r >= 0 && r < nv && r < jend + 2 * KRV;
            const bool has_s = rs >= j0 && rs < jend;
            if (has_in) bytes += nx * 8;
            if (has_s) bytes += nx * 8;
            const uint32_t bar = full_u + 8 * slot;
            if (bytes) {
                mbar_expect_tx_u(bar, bytes);
                if (has_in) tma_row_u(rows_u + 8 * (slot * RW + H), in + r * nx, nx * 8, bar);
                if (has_s) tma_row_u(srow_u + 8 * (slot * nx), Sin + rs * nx, nx * 8, bar);
            } else {
                mbar_arrive_u(bar);
            }
        };

        __syncthreads(); // the previous item is done with the rings, the exchange and Y
        if (t == 0)
            for (int s = 0; s < kStages - 1 && s < nsteps; ++s) issue(s);
        if (t < 6) c[t] = a.ctab[(static_cast<size_t>(p) * a.nwin + a.win[p]) * 6 + t];
        __syncthreads();
        if (owner) {
#pragma unroll
            for (int k = 0; k < KP; ++k) {
                const int sl = __ldg(a.eslot + t * KP + k);
                cq[k * NYE + t] = sl >= 0 ? c[sl] : 0.0;
            }
        }
        // Y of the first t_k row, then the weights of the next
        load_w(jlo);
        __syncthreads();
        fold_y(jlo & (YR - 1));
        if (jlo + 1 < jhi) load_w(jlo + 1);
        for (int q = t; q < 2 * RW; q += NT) tk[q] = 0.0; // exchange rows start as zero rows
        __syncthreads();

        double w1[WROWS][2 * NP], w2[WROWS][2 * NP];
        double skf[WROWS][2]; // s_k FIFO (row jk kept for KRV+1 steps)
#pragma unroll
        for (int r = 0; r < WROWS; ++r) {
#pragma unroll
            for (int q = 0; q < 2 * NP; ++q) w1[r][q] = w2[r][q] = 0.0;
            skf[r][0] = skf[r][1] = 0.0;
        }
        unsigned long long tb1 = 0, sb1 = 0, tb2 = 0, sb2 = 0;

        for (int base = 0; base < nsteps; base += WROWS) {
#pragma unroll
            for (int ph = 0; ph < WROWS; ++ph) {
                const int s = base + ph;
                if (s < nsteps) {
                    if (t == 0 && s + kStages - 1 < nsteps) issue(s + kStages - 1);
                    const int r = j0 - 2 * KRV + s;
                    const int jk = r - KRV;          // t_k row of this step
                    const int jt = jk - 1;           // t_k row published by the previous step
                    const int j2 = r - 2 * KRV - 1;  // t_{k+1} row of this step
                    // 1. the t_k row of the previous step into the second window (slot of step s-1)
                    const int ph2 = (ph + WROWS - 1) % WROWS;
                    {
                        const bool in_rows = jt >= jlo && jt < jhi;
                        const double2* src = reinterpret_cast<const double2*>(tk + (jt & 1) * RW + p0 + AOFF);
#pragma unroll
                        for (int q = 0; q < NP; ++q) {
                            const double2 v2 = in_rows ? src[q] : make_double2(0.0, 0.0);
                            w2[ph2][2 * q] = v2.x;
                            w2[ph2][2 * q + 1] = v2.y;
                        }
                    }
                    // 2. t_{k+1} row j2 (window centre = step s-1-KRV) and s_{k+1}
                    if (j2 >= j0 && j2 < jend && active) {
                        const int pc2 = (ph + 2 * WROWS - 1 - KRV) % WROWS;
                        const int pf = (ph + 2 * WROWS - KRV - 1) % WROWS; // FIFO slot of row j2
                        double accA, accB;
                        apply(Ys + (j2 & (YR - 1)) * YST, w2, pc2, accA, accB);
                        const double tA = accA * inv2, tB = accB * inv2;
                        const double sA = skf[pf][0] + tA, sB = skf[pf][1] + tB;
                        const int off = j2 * nx + p0;
                        *reinterpret_cast<double2*>(Tout + off) = make_double2(tA, tB);
                        *reinterpret_cast<double2*>(Sa + off) = make_double2(sA, sB);
                        tb2 = umax64(tb2, umax64(abs_bits(tA), abs_bits(tB)));
                        sb2 = umax64(sb2, umax64(abs_bits(sA), abs_bits(sB)));
                    }
                    // 3. the next t_k row's Y (one step ahead) and the weights after it
                    if (jk + 1 > jlo && jk + 1 < jhi) {
                        fold_y((jk + 1) & (YR - 1));
                        if (jk + 2 < jhi) load_w(jk + 2);
                    }
                    // 4. input row r into the first window, t_k row jk
                    const uint32_t g = gstep + s;
                    const uint32_t slot = g & (kStages - 1);
                    mbar_wait_u(full_u + 8 * slot, (g / kStages) & 1);
                    if (r >= 0 && r < nv && r < jend + 2 * KRV) {
                        const double2* src = reinterpret_cast<const double2*>(rows + slot * RW + p0 + AOFF);
#pragma unroll
                        for (int q = 0; q < NP; ++q) {
                            const double2 v2 = src[q];
                            w1[ph][2 * q] = v2.x;
                            w1[ph][2 * q + 1] = v2.y;
                        }
                    } else {
#pragma unroll
                        for (int q = 0; q < 2 * NP; ++q) w1[ph][q] = 0.0;
                    }
                    if (jk >= jlo && jk < jhi && active) {
                        const int pc1 = (ph + WROWS - KRV) % WROWS;
                        double accA, accB;
                        apply(Ys + (jk & (YR - 1)) * YST, w1, pc1, accA, accB);
                        const double tA = accA * inv1, tB = accB * inv1;
                        *reinterpret_cast<double2*>(tk + (jk & 1) * RW + H + p0) = make_double2(tA, tB);
                        if (jk >= j0 && jk < jend) {
                            const double2 sv = *reinterpret_cast<const double2*>(srow + slot * nx + p0);
                            const double sA = sv.x + tA, sB = sv.y + tB;
                            skf[ph][0] = sA;
                            skf[ph][1] = sB;
                            *reinterpret_cast<double2*>(Sb + jk * nx + p0) = make_double2(sA, sB);
                            tb1 = umax64(tb1, umax64(abs_bits(tA), abs_bits(tB)));
                            sb1 = umax64(sb1, umax64(abs_bits(sA), abs_bits(sB)));
                        }
                    }
                    __syncthreads(); // ring slot, Y row and the t_k exchange row consumed / published
                }
            }
        }
        gstep += nsteps;

        tb1 = warp_umax(tb1);
        sb1 = warp_umax(sb1);
        tb2 = warp_umax(tb2);
        sb2 = warp_umax(sb2);
        if ((t & 31) == 0) {
            red[0][t >> 5] = tb1;
            red[1][t >> 5] = sb1;
            red[2][t >> 5] = tb2;
            red[3][t >> 5] = sb2;
        }
        __syncthreads();
        if (t < 32) {
            const int nw = (NT + 31) / 32;
            unsigned long long v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) v[q] = warp_umax(t < nw ? red[q][t] : 0ULL);
            if (t == 0) {
                if (v[0]) atomicMax(&a.tn[p], v[0]);
                if (v[1]) atomicMax(&a.sn[p], v[1]);
                if (v[2]) atomicMax(&b.tn2[p], v[2]);
                if (v[3]) atomicMax(&b.sn2[p], v[3]);
            }
        }
    }
}

// (max threads, min resident blocks): two windows + the s_k FIFO need ~190 registers
template <int NTMAX> struct Nt2Class;
template <> struct Nt2Class<128> { static constexpr int minb = 2; };
template <> struct Nt2Class<256> { static constexpr int minb = 1; };
template <> struct Nt2Class<512> { static constexpr int minb = 1; };

template <int V, int NTMAX>
void launch_term2_nt(s2b_context* ctx, const TermArgs& a, const Term2Args& b, int nt, size_t smem, size_t work) {
    constexpr Variant v = kVariants[V];
    auto kern = term2_kernel<v.rx, v.rv, v.mask, v.bm, NTMAX, Nt2Class<NTMAX>::minb>;
    static int configured_device = -1;
    if (configured_device != ctx->device) {
        S2B_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        configured_device = ctx->device;
    }
    int blocks_per_sm = 1;
    S2B_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, nt, smem));
    blocks_per_sm = std::max(1, blocks_per_sm);
    const size_t cap = static_cast<size_t>(ctx->num_sms) * blocks_per_sm;
    const int grid = grid_cap(static_cast<int>(std::max<size_t>(1, std::min(work, cap))));
    kern<<<grid, nt, smem, ctx->stream>>>(a, b);
    ctx->k_stream = reinterpret_cast<const void*>(kern);
}

} // namespace mg
} // namespace s2b
