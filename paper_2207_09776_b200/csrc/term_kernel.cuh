// The TMA-fed compressed-stencil Taylor-term kernel (see magnus.cu for the engine).
#pragma once

#include "magnus_common.cuh"

namespace s2b {
namespace mg {

// One work item = (live path, strip of J = a.strip_rows output rows).
//
// Thread -> points: thread t < (nx-4)/2 owns the interior x-points 2t+2, 2t+3; the next two
// threads own the x-boundary pairs {0, 1} and {nx-2, nx-1}, so every warp but the last reads
// ONE interior Y set for both of its points.  Rows stream through a kStages-deep TMA ring
// (stage s carries input row j0-KRV+s and accum row j0-2KRV+s); each thread keeps a
// (2KRV+1)-row register window of its x-neighbourhood.  The Y rows of the whole strip (5
// x-classes x the mask's stencil points each) are folded into shared memory once per item, by
// all threads, before the row loop: no warp does extra work inside the loop, so the per-row
// barrier only waits for the ring (the host sizes J so that the strip's Y fits).
template <int KRX, int KRV, uint64_t MASK, uint32_t BM, int NTMAX, int MINB>
__global__ void __launch_bounds__(NTMAX, MINB) term_tma_kernel(TermArgs a) {
    constexpr int H = KRX <= 2 ? 2 : 4;             // zero halo (doubles) on each side
    constexpr int AOFF = (H - KRX) & ~1;            // first loaded smem index relative to p0
    constexpr int LAST = 1 + KRX + H;               // last needed smem index relative to p0
    constexpr int NP = (LAST - AOFF) / 2 + 1;       // 16-byte pairs loaded per row
    constexpr int WROWS = 2 * KRV + 1;
    constexpr int NBM = MaskInfo<MASK>::count();
    constexpr int NYE = kClasses * NBM;             // Y entries of one row
    constexpr int YST = (NYE + 1) & ~1;             // Y row stride (16-byte aligned rows)
    const int J = a.strip_rows;
    constexpr int KP = kPairSlots;

    const int nx = a.op.nx, nv = a.op.nv;
    const int n = nx * nv;
    const int NT = blockDim.x;
    const int RW = nx + 2 * H; // smem row width (doubles)
    const int t = threadIdx.x;
    const int nint = (nx - 4) / 2; // threads owning interior pairs

    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    double* rows = reinterpret_cast<double*>(smem_raw + 128); // kStages x RW
    double* srow = rows + kStages * RW;                       // kStages x nx
    double* cq = srow + kStages * nx;                         // KP x NYE
    double* Ys = cq + KP * NYE;                               // J x YST: the strip's Y rows
    const uint32_t full_u = smem_u32(full), rows_u = smem_u32(rows), srow_u = smem_u32(srow);
    __shared__ double c[6];
    __shared__ unsigned long long red[2][32];

    for (int q = t; q < kStages * RW; q += NT) rows[q] = 0.0;
    if (t == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // this thread's two x-points p0, p0+1 and their classes
    const bool active = t < nint + 2;
    const int p0 = t < nint ? 2 * t + 2 : (t == nint ? 0 : nx - 2);
    const int clsA = t < nint ? 2 : (t == nint ? 0 : 3);
    const int clsB = t < nint ? 2 : (t == nint ? 1 : 4);
    const bool wfast = BM == 0 || __all_sync(0xffffffffu, t < nint || !active);

    // MagnusLogBuilder::fill fold (slots ascending from 0.0, zero coefficients skipped) of every
    // Y entry of rows [j0, jend), spread over all threads
    auto fold_strip = [&](int j0, int jend) {
        const int total = (jend - j0) * NYE;
        for (int u = t; u < total; u += NT) {
            const int jr = u / NYE, e = u - jr * NYE;
            const double2* src = reinterpret_cast<const double2*>(a.wt + (static_cast<size_t>(j0 + jr) * NYE + e) * KP);
            double w[KP];
#pragma unroll
            for (int k = 0; k < KP / 2; ++k) {
                const double2 v = __ldg(src + k);
                w[2 * k] = v.x;
                w[2 * k + 1] = v.y;
            }
            double y = 0.0;
#pragma unroll
            for (int k = 0; k < KP; ++k) {
                const double cs = cq[k * NYE + e];
                if (cs != 0.0) y += cs * w[k];
            }
            Ys[jr * YST + e] = y;
        }
    };

    uint32_t gstep = 0; // running stage counter across work items (mbarrier phases)
    const long long work = static_cast<long long>(a.cnt[0]) * a.nstrips;
    for (long long wi = blockIdx.x; wi < work; wi += gridDim.x) {
        const int p = a.act[wi / a.nstrips];
        const int strip = static_cast<int>(wi % a.nstrips);
        const int j0 = strip * J;
        const int jend = min(j0 + J, nv);
        const int kk = a.k[p];
        const int par = a.par[p];
        const double inv = 1.0 / (static_cast<double>(a.nseg[p]) * kk);
        const size_t pbase = static_cast<size_t>(p) * n;
        const double* Sin = (par ? a.S1 : a.S0) + pbase;
        const double* in = kk == 1 ? Sin : (par ? a.T1 : a.T0) + pbase;
        double* Tout = (par ? a.T0 : a.T1) + pbase;
        double* Sout = (par ? a.S0 : a.S1) + pbase;
        const int nsteps = (jend - j0) + 2 * KRV;

        auto issue = [&](int s) {
            const uint32_t slot = (gstep + s) & (kStages - 1);
            const int r = j0 - KRV + s;
            const int ro = r - KRV;
            uint32_t bytes = 0;
            const bool has_in = r >= 0 && r < nv;
            const bool has_s = s >= 2 * KRV && ro < jend;
            if (has_in) bytes += nx * 8;
            if (has_s) bytes += nx * 8;
            const uint32_t bar = full_u + 8 * slot;
            if (bytes) {
                mbar_expect_tx_u(bar, bytes);
                if (has_in) tma_row_u(rows_u + 8 * (slot * RW + H), in + r * nx, nx * 8, bar);
                if (has_s) tma_row_u(srow_u + 8 * (slot * nx), Sin + ro * nx, nx * 8, bar);
            } else {
                mbar_arrive_u(bar);
            }
        };

        // ring refill with one CTA barrier per G = sync_g steps: a step s = 0 mod G refills the G
        // slots that steps s-G .. s-1 read, all released by the barrier after step s-1, with rows
        // s+8-G .. s+7 (8-G .. 7 rows ahead).  G = 1 is the classic one-barrier-per-row ring.
        const int G = a.sync_g;
        const int ahead = kStages - G;
        __syncthreads(); // previous item fully consumed the ring and the Y rows
        if (t == 0) {
            for (int s = 0; s < ahead && s < nsteps; ++s) issue(s);
        }
        if (t < 6) c[t] = a.ctab[(static_cast<size_t>(p) * a.nwin + a.win[p]) * 6 + t];
        __syncthreads();
        for (int q = t; q < NYE * KP; q += NT) { // the coefficient of every (entry, pair slot)
            const int e = q / KP, k = q - e * KP;
            const int sl = __ldg(a.eslot + e * KP + k);
            cq[k * NYE + e] = sl >= 0 ? c[sl] : 0.0;
        }
        __syncthreads();
        fold_strip(j0, jend);
        __syncthreads();

        double win[WROWS][2 * NP];
#pragma unroll
        for (int r = 0; r < WROWS; ++r)
#pragma unroll
            for (int q = 0; q < 2 * NP; ++q) win[r][q] = 0.0;
        unsigned long long tb = 0, sb = 0;

        for (int base = 0; base < nsteps; base += WROWS) {
#pragma unroll
            for (int ph = 0; ph < WROWS; ++ph) {
                const int s = base + ph;
                if (s < nsteps) {
                    if (t == 0 && (s & (G - 1)) == 0) {
                        for (int q = ahead; q < kStages; ++q)
                            if (s + q < nsteps) issue(s + q);
                    }
                    const uint32_t g = gstep + s;
                    const uint32_t slot = g & (kStages - 1);
                    mbar_wait_u(full_u + 8 * slot, (g / kStages) & 1);
                    const int r = j0 - KRV + s;
                    if (r >= 0 && r < nv) {
                        const double2* src = reinterpret_cast<const double2*>(rows + slot * RW + p0 + AOFF);
#pragma unroll
                        for (int q = 0; q < NP; ++q) {
                            const double2 v2 = src[q];
                            win[ph][2 * q] = v2.x;
                            win[ph][2 * q + 1] = v2.y;
                        }
                    } else {
#pragma unroll
                        for (int q = 0; q < 2 * NP; ++q) win[ph][q] = 0.0;
                    }
                    const int jo = r - KRV; // output row of this step
                    if (s >= 2 * KRV && jo < jend && active) {
                        const double2 sv = *reinterpret_cast<const double2*>(srow + slot * nx + p0);
                        const double* yrow = Ys + (jo - j0) * YST;
                        double accA = 0.0, accB = 0.0;
                        // ascending stencil offset == ascending DIA diagonal (sparse.cpp:412-423)
                        if (wfast) {
                            // interior Y row: one 16-byte broadcast load per two entries
                            const double2* y2 = reinterpret_cast<const double2*>(yrow + 2 * NBM);
#pragma unroll
                            for (int dv = -KRV; dv <= KRV; ++dv) {
                                const int rr = ((ph - KRV + dv) % WROWS + WROWS) % WROWS;
#pragma unroll
                                for (int dx = -KRX; dx <= KRX; ++dx) {
                                    if (MaskInfo<MASK>::has(dx, dv)) {
                                        const int e = MaskInfo<MASK>::rank(box_bit(dx, dv));
                                        const int col = H + dx - AOFF;
                                        const double w = (e & 1) ? y2[e >> 1].y : y2[e >> 1].x;
                                        accA += w * win[rr][col];
                                        accB += w * win[rr][col + 1];
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
                        const int off = jo * nx + p0;
                        const double tA = accA * inv;
                        const double sA = sv.x + tA;
                        const double tB = accB * inv;
                        const double sB = sv.y + tB;
                        *reinterpret_cast<double2*>(Tout + off) = make_double2(tA, tB);
                        *reinterpret_cast<double2*>(Sout + off) = make_double2(sA, sB);
                        tb = umax64(tb, umax64(abs_bits(tA), abs_bits(tB)));
                        sb = umax64(sb, umax64(abs_bits(sA), abs_bits(sB)));
                    }
                    if ((s & (G - 1)) == G - 1) __syncthreads(); // ring slots consumed by every thread
                }
            }
        }
        gstep += nsteps;

        tb = warp_umax(tb);
        sb = warp_umax(sb);
        if ((t & 31) == 0) {
            red[0][t >> 5] = tb;
            red[1][t >> 5] = sb;
        }
        __syncthreads();
        if (t < 32) {
            const int nw = (NT + 31) / 32;
            unsigned long long t2 = t < nw ? red[0][t] : 0ULL;
            unsigned long long s2 = t < nw ? red[1][t] : 0ULL;
            t2 = warp_umax(t2);
            s2 = warp_umax(s2);
            if (t == 0) {
                if (t2) atomicMax(&a.tn[p], t2);
                if (s2) atomicMax(&a.sn[p], s2);
            }
        }
    }
}

// Block-size classes: (max threads, min resident blocks) -> register budget.
template <int NTMAX> struct NtClass;
template <> struct NtClass<128> { static constexpr int minb = 4; };
template <> struct NtClass<256> { static constexpr int minb = 2; };
template <> struct NtClass<512> { static constexpr int minb = 1; };

template <int V, int NTMAX>
void launch_term_nt(s2b_context* ctx, const TermArgs& a, int nt, size_t smem, size_t work) {
    constexpr Variant v = kVariants[V];
    auto kern = term_tma_kernel<v.rx, v.rv, v.mask, v.bm, NTMAX, NtClass<NTMAX>::minb>;
    static int configured_device = -1;
    if (configured_device != ctx->device) {
        S2B_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kTermSmem)));
        configured_device = ctx->device;
    }
    int blocks_per_sm = 1;
    S2B_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, nt, smem));
    blocks_per_sm = std::max(1, blocks_per_sm);
    const size_t cap = static_cast<size_t>(ctx->num_sms) * blocks_per_sm;
    const int grid = grid_cap(static_cast<int>(std::max<size_t>(1, std::min(work, cap))));
    kern<<<grid, nt, smem, ctx->stream>>>(a);
    ctx->k_stream = reinterpret_cast<const void*>(kern);
}

} // namespace mg
} // namespace s2b
