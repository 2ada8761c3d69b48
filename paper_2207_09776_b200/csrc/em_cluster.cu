// Cluster-resident Euler-Maruyama (solve_euler, src/euler.cpp:95-182) for x-invariant
// coefficient fields (the constant Langevin family) at 256 x 256.
//
// One 8-CTA cluster owns one path for ALL of its steps: the state never leaves shared
// memory between steps.  CTA `rank` owns 32 rows; lane = row, each thread marches along
// x over a 32-point segment with P points in flight, the row's coefficient values in
// registers (x-invariant fields), the three stencil rows in per-row register rings.  The
// state is double-buffered x-major ([x][row], conflict-free column reads, immediate
// offsets); the one halo row on each side is pushed to the neighbour CTA with a DSMEM
// store as it is computed, and one cluster barrier per step publishes it.
//
// Arithmetic: euler_step_into (euler.cpp:28-86) term by term, separately rounded
// (-fmad=false): central differences, drift folded over the non-zero fields in the order
// h, fx, fv, gxx, gxv, gvv with the 1/2 applied as (0.5*g) [per row here: the same
// product], noise over sig, sigx, sigv, then (u + drift*dt) + noise*dW.
// Blow-up: the reference stops a path at the first step whose max|u+| is infinite
// (std::max ignores NaN): each thread keeps the first step at which it produced an
// infinite value and folds it into a per-path atomicMin; the statuses are derived from it,
// so no per-step reduction is needed (values computed after a blow-up are discarded).
#include <cooperative_groups.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <type_traits>

#include "s2b_internal.cuh"

namespace cg = cooperative_groups;

namespace s2b {

namespace {

constexpr int kEmCl = 8;

struct EmXmArgs {
    const double* rowf; // [9][nv] row values of the x-invariant fields
    const double* colf; // [9][nx] column values of the v-invariant (x-dependent) fields, 1/2 applied to g
    const double* fgen; // [9][nx][nv] every field per point, x-major (a warp's rows coalesce), 1/2 applied to g
    double st[5];
    double dt;
    const double* values; // [M][vstride] Brownian prefix values
    size_t vstride;
    int step_leb;
    int nsteps;
    const double* phi;
    double* const* rec; // R record buffers [M][n]
    const int* rec_k;   // E-M step index after which record r is taken (ascending)
    int R;
    int* blow; // [M] first step with an infinite value (INT_MAX: none)
    int M;
    int nv;
    int* work;
};

// NZ: the datum holds no -0.0.  E-M then never produces one (in round-to-nearest a sum is -0
// only if both addends are -0, and the update ends in uc + ...), so starting a fold at its
// first term instead of at 0.0 + term changes no bit of any state -- only the sign of an
// all-zero drift / noise, which is then added to a state that is never -0.  Saves two fp64
// ops of ~18 per point.
constexpr int em_first(int mask, int group) { return (mask & group) & -(mask & group); }
#define EM_ADD(bit, acc, term) \
    ((NZ && (bit) == em_first(MASK, (bit) < 64 ? 63 : 448)) ? (term) : (acc) + (term))

__device__ __forceinline__ void cl_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int NX, int RPC, int NT, int P, int MASK, bool NZ>
__global__ void __launch_bounds__(NT, 1) em_cluster_kernel(EmXmArgs a) {
    constexpr bool GXV = (MASK & 16) != 0;
    constexpr int TR = RPC + 2; // rows incl. one halo row each side
    constexpr int TX = NX + 2;  // columns incl. one zero column each side
    constexpr int TBUF = TX * TR;
    constexpr int NSEG = NT / RPC;
    constexpr int LX = NX / NSEG;
    constexpr int WS = GXV ? 3 : 1; // ring span of rows j-1, j+1
    constexpr int R0 = 3 + P - 1;   // ring slots of row j
    constexpr int R1 = WS + P - 1;  // ring slots of rows j-1, j+1
    static_assert(NT % RPC == 0 && NX % NSEG == 0 && LX % P == 0, "x-march shape");

    cg::cluster_group cluster = cg::this_cluster();
    const int rank = static_cast<int>(cluster.block_rank());
    const int t = threadIdx.x;
    const int r = t % RPC;
    const int seg = t / RPC;
    const int x0 = seg * LX;
    const int row0 = rank * RPC;
    const int j = row0 + r;
    const int n = NX * a.nv;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* U = reinterpret_cast<double*>(smem_raw); // [2][TX][TR]
    __shared__ int next_path;

    const bool has_lo = rank > 0, has_hi = rank < kEmCl - 1;
    // halo push targets: row 0 -> lower neighbour's row RPC, row RPC-1 -> upper's row -1
    double* rem = nullptr;
    if (r == 0 && has_lo) rem = cluster.map_shared_rank(U, rank - 1) + (x0 + 1) * TR + (RPC + 1);
    else if (r == RPC - 1 && has_hi) rem = cluster.map_shared_rank(U, rank + 1) + (x0 + 1) * TR + 0;
    const bool do_rem = rem != nullptr;
    int* next0 = cluster.map_shared_rank(&next_path, 0);
    const int tb = (x0 + 1) * TR + (r + 1);

    // this row's coefficients (x-invariant); 0.5*g formed as the reference forms it per point
    const double fh = (MASK & 1) ? a.rowf[0 * a.nv + j] : 0.0;
    const double ffx = (MASK & 2) ? a.rowf[1 * a.nv + j] : 0.0;
    const double ffv = (MASK & 4) ? a.rowf[2 * a.nv + j] : 0.0;
    const double hgxx = (MASK & 8) ? 0.5 * a.rowf[3 * a.nv + j] : 0.0;
    const double fgxv = (MASK & 16) ? a.rowf[4 * a.nv + j] : 0.0;
    const double hgvv = (MASK & 32) ? 0.5 * a.rowf[5 * a.nv + j] : 0.0;
    const double fsig = (MASK & 64) ? a.rowf[6 * a.nv + j] : 0.0;
    const double fsx = (MASK & 128) ? a.rowf[7 * a.nv + j] : 0.0;
    const double fsv = (MASK & 256) ? a.rowf[8 * a.nv + j] : 0.0;
    const double st0 = a.st[0], st1 = a.st[1], st2 = a.st[2], st3 = a.st[3], st4 = a.st[4];
    const double dt = a.dt;

    while (true) {
        if (rank == 0 && t == 0) next_path = atomicAdd(a.work, 1);
        cl_barrier();
        const int p = *next0;
        cl_barrier(); // everyone has read next_path; the previous path's pushes are done
        if (p >= a.M) break;

        // phi into buffer 0: own rows and the two halo rows (zero outside the grid), and
        // zero x-halo columns in both buffers
        for (int q = t; q < TR * NX; q += NT) {
            const int rr = q / NX - 1, x = q % NX;
            const int jj = row0 + rr;
            U[(x + 1) * TR + rr + 1] = (jj >= 0 && jj < a.nv) ? a.phi[static_cast<size_t>(jj) * NX + x] : 0.0;
        }
        for (int q = t; q < 2 * 2 * TR; q += NT) {
            const int b = q / (2 * TR), side = (q / TR) & 1, rr = q % TR;
            U[b * TBUF + (side ? TX - 1 : 0) * TR + rr] = 0.0;
        }
        if (!has_lo || !has_hi) { // outer halo rows of buffer 1 stay zero
            for (int x = t; x < TX; x += NT) {
                if (!has_lo) U[TBUF + x * TR + 0] = 0.0;
                if (!has_hi) U[TBUF + x * TR + RPC + 1] = 0.0;
            }
        }
        __syncthreads();

        const double* pv = a.values + static_cast<size_t>(p) * a.vstride;
        double dWn = pv[a.step_leb] - pv[0];
        int first = INT_MAX;
        int rec = 0;
        int cur = 0;
        for (int k = 0; k < a.nsteps; ++k) {
            const double dW = dWn;
            if (k + 1 < a.nsteps) dWn = pv[static_cast<size_t>(k + 2) * a.step_leb] - pv[static_cast<size_t>(k + 1) * a.step_leb];
            const double* uin = U + cur * TBUF + tb;
            double* uout = U + (cur ^ 1) * TBUF + tb;
            double* rout = rem + (cur ^ 1) * TBUF;
            // rings over absolute columns c >= -1: row j slot (c+1) mod R0 (columns c-1..c+1
            // live per point), rows j-1, j+1 slot (c - LO1) mod R1
            constexpr int LO1 = GXV ? -1 : 0;
            double w0[R0], wm[R1], wp[R1];
            w0[0] = uin[-TR];
            w0[1] = uin[0];
            if constexpr (GXV) {
                wm[0] = uin[-TR - 1];
                wp[0] = uin[-TR + 1];
                wm[1] = uin[-1];
                wp[1] = uin[1];
            }
            bool inf_seen = false;
#pragma unroll
            for (int i0 = 0; i0 < LX; i0 += P) {
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    const int c = i0 + q;
                    w0[(c + 2) % R0] = uin[(c + 1) * TR];
                    const int ch = GXV ? c + 1 : c;
                    wm[(ch - LO1) % R1] = uin[ch * TR - 1];
                    wp[(ch - LO1) % R1] = uin[ch * TR + 1];
                }
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    const int c = i0 + q;
                    const double uc = w0[(c + 1) % R0];
                    const double uxm = w0[c % R0];
                    const double uxp = w0[(c + 2) % R0];
                    const double uvm = wm[(c - LO1) % R1];
                    const double uvp = wp[(c - LO1) % R1];
                    const double dxu = (uxp - uxm) * st0;
                    const double dvu = (uvp - uvm) * st2;
                    double drift = 0.0; // (NZ: the first present term starts the fold, see em_first)
                    if (MASK & 1) drift = EM_ADD(1, drift, fh * uc);
                    if (MASK & 2) drift = EM_ADD(2, drift, ffx * dxu);
                    if (MASK & 4) drift = EM_ADD(4, drift, ffv * dvu);
                    if (MASK & 8) {
                        const double dxxu = (uxp - 2.0 * uc + uxm) * st1;
                        drift = EM_ADD(8, drift, hgxx * dxxu);
                    }
                    if (MASK & 16) {
                        const double upp = wp[(c + 1 - LO1) % R1], upm = wp[(c - 1 - LO1) % R1];
                        const double ump = wm[(c + 1 - LO1) % R1], umm = wm[(c - 1 - LO1) % R1];
                        const double dxvu = (upp - upm - ump + umm) * st4;
                        drift = EM_ADD(16, drift, fgxv * dxvu);
                    }
                    if (MASK & 32) {
                        const double dvvu = (uvp - 2.0 * uc + uvm) * st3;
                        drift = EM_ADD(32, drift, hgvv * dvvu);
                    }
                    double noise = 0.0;
                    if (MASK & 64) noise = EM_ADD(64, noise, fsig * uc);
                    if (MASK & 128) noise = EM_ADD(128, noise, fsx * dxu);
                    if (MASK & 256) noise = EM_ADD(256, noise, fsv * dvu);
                    const double next = uc + drift * dt + noise * dW;
                    uout[c * TR] = next;
                    if (do_rem) rout[c * TR] = next;
                    inf_seen |= fabs(next) == __longlong_as_double(0x7FF0000000000000LL);
                }
            }
            if (inf_seen && first == INT_MAX) first = k;
            cl_barrier();
            cur ^= 1;
            while (rec < a.R && a.rec_k[rec] == k) {
                double* dst = a.rec[rec] + static_cast<size_t>(p) * n + static_cast<size_t>(row0) * NX;
                const double* src = U + cur * TBUF;
                for (int q = t; q < RPC * NX; q += NT) dst[q] = src[(q % NX + 1) * TR + q / NX + 1];
                ++rec;
            }
        }
        if (first != INT_MAX) atomicMin(a.blow + p, first);
    }
}

// In-place variant for grids whose double-buffered state exceeds a cluster (512^2: 4 MB per
// path vs 3.6 MB in a 16-CTA cluster): one state buffer updated in place.  Within a warp a
// column is read into the register rings before it is overwritten (program order); the
// columns a warp reads from its neighbour segments (x0-1, x0+LX) are preloaded before a CTA
// barrier; the halo rows from the neighbour CTAs are double-buffered by step parity (two
// slot sets per side: row -1 at index 1 / 0, row RPC at RPC+2 / RPC+3).
// XD: fields that depend on x only (v-invariant; e.g. a(x), sigma(x) of the variable Langevin
// family): lane = row, so a warp's 32 lanes read the same column value (one L1 broadcast).
template <int NX, int RPC, int NT, int P, int MASK, int CL, int NP, bool NZ, int XD = 0>
__global__ void __launch_bounds__(NT, 1) em_cluster_ip_kernel(EmXmArgs a) {
    static_assert((MASK & 16) == 0, "in-place E-M: no mixed derivative");
    constexpr int TRI = RPC + 4;
    constexpr int TX = NX + 2;
    constexpr int TBUF = TX * TRI;
    constexpr int NSEG = NT / RPC;
    constexpr int LX = NX / NSEG;
    constexpr int R0 = P + 2; // row j ring: columns c-1 .. c+P
    static_assert(NT % RPC == 0 && NX % NSEG == 0 && LX % P == 0, "x-march shape");

    cg::cluster_group cluster = cg::this_cluster();
    const int rank = static_cast<int>(cluster.block_rank());
    const int t = threadIdx.x;
    const int r = t % RPC;
    const int seg = t / RPC;
    const int x0 = seg * LX;
    const int row0 = rank * RPC;
    const int j = row0 + r;
    const int n = NX * a.nv;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* U = reinterpret_cast<double*>(smem_raw); // [NP][TX][TRI]: NP paths per cluster
    __shared__ int next_path;

    auto ridx = [&](int row, int par) {
        int i = 2 + row;
        if (par) i += row < 0 ? -1 : (row >= RPC ? 1 : 0);
        return i;
    };
    const bool has_lo = rank > 0, has_hi = rank < CL - 1;
    const int cb = (x0 + 1) * TRI;
    double* rem0 = nullptr;
    double* rem1 = nullptr;
    if (r == 0 && has_lo) {
        double* nb = cluster.map_shared_rank(U, rank - 1);
        rem0 = nb + cb + ridx(RPC, 0);
        rem1 = nb + cb + ridx(RPC, 1);
    } else if (r == RPC - 1 && has_hi) {
        double* nb = cluster.map_shared_rank(U, rank + 1);
        rem0 = nb + cb + ridx(-1, 0);
        rem1 = nb + cb + ridx(-1, 1);
    }
    const bool do_rem = rem0 != nullptr;
    int* next0 = cluster.map_shared_rank(&next_path, 0);

    constexpr bool RV = XD != -1; // row values used at all
    const double fh = (RV && (MASK & 1)) ? a.rowf[0 * a.nv + j] : 0.0;
    const double ffx = (RV && (MASK & 2)) ? a.rowf[1 * a.nv + j] : 0.0;
    const double ffv = (RV && (MASK & 4)) ? a.rowf[2 * a.nv + j] : 0.0;
    const double hgxx = (RV && (MASK & 8)) ? 0.5 * a.rowf[3 * a.nv + j] : 0.0;
    const double hgvv = (RV && (MASK & 32)) ? 0.5 * a.rowf[5 * a.nv + j] : 0.0;
    const double fsig = (RV && (MASK & 64)) ? a.rowf[6 * a.nv + j] : 0.0;
    const double fsx = (RV && (MASK & 128)) ? a.rowf[7 * a.nv + j] : 0.0;
    const double fsv = (RV && (MASK & 256)) ? a.rowf[8 * a.nv + j] : 0.0;
    const double st0 = a.st[0], st1 = a.st[1], st2 = a.st[2], st3 = a.st[3];
    const double dt = a.dt;

    for (int q = t; q < NP * TBUF; q += NT) U[q] = 0.0; // zero x-halo columns and outer halo rows
    int ip = 0;                                         // halo slot set of the current input

    while (true) {
        if (rank == 0 && t == 0) next_path = atomicAdd(a.work, NP);
        cl_barrier();
        const int pbase = *next0;
        cl_barrier();
        if (pbase >= a.M) break;
        const int np = a.M - pbase < NP ? a.M - pbase : NP; // paths this cluster carries now

        // phi: own rows and (where a neighbour exists) the halo rows of slot set ip
        for (int q = t; q < np * (RPC + 2) * NX; q += NT) {
            const int pi = q / ((RPC + 2) * NX), qq = q % ((RPC + 2) * NX);
            const int rr = qq / NX - 1, x = qq % NX;
            const int jj = row0 + rr;
            if (jj < 0 || jj >= a.nv) continue;
            U[pi * TBUF + (x + 1) * TRI + ridx(rr, ip)] = a.phi[static_cast<size_t>(jj) * NX + x];
        }
        __syncthreads();

        const double* pv[NP];
        double dWn[NP];
        int first[NP];
#pragma unroll
        for (int pi = 0; pi < NP; ++pi) {
            pv[pi] = a.values + static_cast<size_t>(pbase + (pi < np ? pi : 0)) * a.vstride;
            dWn[pi] = pv[pi][a.step_leb] - pv[pi][0];
            first[pi] = INT_MAX;
        }
        int rec = 0;
        for (int k = 0; k < a.nsteps; ++k) {
            double dW[NP];
#pragma unroll
            for (int pi = 0; pi < NP; ++pi) {
                dW[pi] = dWn[pi];
                if (k + 1 < a.nsteps)
                    dWn[pi] = pv[pi][static_cast<size_t>(k + 2) * a.step_leb] - pv[pi][static_cast<size_t>(k + 1) * a.step_leb];
            }
            // columns x0-1 and x0+LX of row j belong to the neighbour segments: read them first
            double lft[NP], cur0[NP], right[NP];
#pragma unroll
            for (int pi = 0; pi < NP; ++pi) {
                const double* r0 = U + pi * TBUF + cb + 2 + r;
                lft[pi] = r0[-TRI];
                cur0[pi] = r0[0];
                right[pi] = r0[LX * TRI];
            }
            __syncthreads();
            if constexpr (XD == -1) {
                // general fields (one value per point and field, x-major table): each point's
                // fields are loaded ONCE per step for all NP paths of the cluster -- the
                // per-path point loop below would re-read them from L2 for every path
                const size_t colbase = static_cast<size_t>(x0) * NX + j;
                double w0[NP][R0];
                bool infs[NP];
#pragma unroll
                for (int pi = 0; pi < NP; ++pi) {
                    w0[pi][0] = lft[pi];
                    w0[pi][1] = cur0[pi];
                    infs[pi] = false;
                }
#pragma unroll
                for (int i0 = 0; i0 < LX; i0 += P) {
                    double fl[9][P];
#pragma unroll
                    for (int f = 0; f < 9; ++f)
                        if ((MASK >> f) & 1)
#pragma unroll
                            for (int q = 0; q < P; ++q)
                                fl[f][q] = __ldg(a.fgen + static_cast<size_t>(f) * n + colbase + static_cast<size_t>(i0 + q) * NX);
#pragma unroll
                    for (int pi = 0; pi < NP; ++pi) {
                        if (pi >= np) break;
                        const double* rm = U + pi * TBUF + cb + ridx(r - 1, ip);
                        const double* r0 = U + pi * TBUF + cb + 2 + r;
                        const double* rp = U + pi * TBUF + cb + ridx(r + 1, ip);
                        double* own = U + pi * TBUF + cb + 2 + r;
                        double* rout = (ip ? rem0 : rem1) + pi * TBUF;
                        double wm[P], wp[P];
#pragma unroll
                        for (int q = 0; q < P; ++q) {
                            const int c = i0 + q;
                            w0[pi][(c + 2) % R0] = c + 1 < LX ? r0[(c + 1) * TRI] : right[pi];
                            wm[q] = rm[c * TRI];
                            wp[q] = rp[c * TRI];
                        }
#pragma unroll
                        for (int q = 0; q < P; ++q) {
                            const int c = i0 + q;
                            const double uc = w0[pi][(c + 1) % R0];
                            const double uxm = w0[pi][c % R0];
                            const double uxp = w0[pi][(c + 2) % R0];
                            const double uvm = wm[q];
                            const double uvp = wp[q];
                            const double dxu = (uxp - uxm) * st0;
                            const double dvu = (uvp - uvm) * st2;
                            double drift = 0.0; // euler_step_into's fold (euler.cpp:51-80), see em_first
                            if (MASK & 1) drift = EM_ADD(1, drift, fl[0][q] * uc);
                            if (MASK & 2) drift = EM_ADD(2, drift, fl[1][q] * dxu);
                            if (MASK & 4) drift = EM_ADD(4, drift, fl[2][q] * dvu);
                            if (MASK & 8) {
                                const double dxxu = (uxp - 2.0 * uc + uxm) * st1;
                                drift = EM_ADD(8, drift, fl[3][q] * dxxu);
                            }
                            if (MASK & 32) {
                                const double dvvu = (uvp - 2.0 * uc + uvm) * st3;
                                drift = EM_ADD(32, drift, fl[5][q] * dvvu);
                            }
                            double noise = 0.0;
                            if (MASK & 64) noise = EM_ADD(64, noise, fl[6][q] * uc);
                            if (MASK & 128) noise = EM_ADD(128, noise, fl[7][q] * dxu);
                            if (MASK & 256) noise = EM_ADD(256, noise, fl[8][q] * dvu);
                            const double next = uc + drift * dt + noise * dW[pi];
                            own[c * TRI] = next;
                            if (do_rem) rout[c * TRI] = next;
                            infs[pi] |= fabs(next) == __longlong_as_double(0x7FF0000000000000LL);
                        }
                    }
                }
#pragma unroll
                for (int pi = 0; pi < NP; ++pi)
                    if (pi < np && infs[pi] && first[pi] == INT_MAX) first[pi] = k;
            } else
#pragma unroll
            for (int pi = 0; pi < NP; ++pi) {
                if (pi >= np) break;
                const double* rm = U + pi * TBUF + cb + ridx(r - 1, ip); // row j-1
                const double* r0 = U + pi * TBUF + cb + 2 + r;           // row j
                const double* rp = U + pi * TBUF + cb + ridx(r + 1, ip); // row j+1
                double* own = U + pi * TBUF + cb + 2 + r;
                double* rout = (ip ? rem0 : rem1) + pi * TBUF;           // neighbour slot set ip^1
                double w0[R0], wm[P], wp[P];
                w0[0] = lft[pi];
                w0[1] = cur0[pi];
                bool inf_seen = false;
#pragma unroll
                for (int i0 = 0; i0 < LX; i0 += P) {
#pragma unroll
                    for (int q = 0; q < P; ++q) {
                        const int c = i0 + q;
                        w0[(c + 2) % R0] = c + 1 < LX ? r0[(c + 1) * TRI] : right[pi];
                        wm[q] = rm[c * TRI];
                        wp[q] = rp[c * TRI];
                    }
#pragma unroll
                    for (int q = 0; q < P; ++q) {
                        const int c = i0 + q;
                        const double uc = w0[(c + 1) % R0];
                        const double uxm = w0[c % R0];
                        const double uxp = w0[(c + 2) % R0];
                        const double uvm = wm[q];
                        const double uvp = wp[q];
                        const double dxu = (uxp - uxm) * st0;
                        const double dvu = (uvp - uvm) * st2;
                        double drift = 0.0; // (NZ: the first present term starts the fold, see em_first)
                        if (MASK & 1) drift = EM_ADD(1, drift, (XD == -1 ? __ldg(a.fgen + 0 * static_cast<size_t>(n) + static_cast<size_t>(x0 + c) * NX + j) : fh) * uc);
                        if (MASK & 2) {
                            const double fx = XD == -1 ? __ldg(a.fgen + 1 * static_cast<size_t>(n) + static_cast<size_t>(x0 + c) * NX + j)
                                            : (XD & 2) ? __ldg(a.colf + 1 * NX + x0 + c) : ffx;
                            drift = EM_ADD(2, drift, fx * dxu);
                        }
                        if (MASK & 4) drift = EM_ADD(4, drift, (XD == -1 ? __ldg(a.fgen + 2 * static_cast<size_t>(n) + static_cast<size_t>(x0 + c) * NX + j) : ffv) * dvu);
                        if (MASK & 8) {
                            const double dxxu = (uxp - 2.0 * uc + uxm) * st1;
                            drift = EM_ADD(8, drift, (XD == -1 ? __ldg(a.fgen + 3 * static_cast<size_t>(n) + static_cast<size_t>(x0 + c) * NX + j) : hgxx) * dxxu);
                        }
                        if (MASK & 32) {
                            const double dvvu = (uvp - 2.0 * uc + uvm) * st3;
                            const double g = XD == -1 ? __ldg(a.fgen + 5 * static_cast<size_t>(n) + static_cast<size_t>(x0 + c) * NX + j)
                                           : (XD & 32) ? __ldg(a.colf + 5 * NX + x0 + c) : hgvv;
                            drift = EM_ADD(32, drift, g * dvvu);
                        }
                        double noise = 0.0;
                        if (MASK & 64) noise = EM_ADD(64, noise, (XD == -1 ? __ldg(a.fgen + 6 * static_cast<size_t>(n) + static_cast<size_t>(x0 + c) * NX + j) : fsig) * uc);
                        if (MASK & 128) noise = EM_ADD(128, noise, (XD == -1 ? __ldg(a.fgen + 7 * static_cast<size_t>(n) + static_cast<size_t>(x0 + c) * NX + j) : fsx) * dxu);
                        if (MASK & 256) {
                            const double sv = XD == -1 ? __ldg(a.fgen + 8 * static_cast<size_t>(n) + static_cast<size_t>(x0 + c) * NX + j)
                                            : (XD & 256) ? __ldg(a.colf + 8 * NX + x0 + c) : fsv;
                            noise = EM_ADD(256, noise, sv * dvu);
                        }
                        const double next = uc + drift * dt + noise * dW[pi];
                        own[c * TRI] = next;
                        if (do_rem) rout[c * TRI] = next;
                        inf_seen |= fabs(next) == __longlong_as_double(0x7FF0000000000000LL);
                    }
                }
                if (inf_seen && first[pi] == INT_MAX) first[pi] = k;
            }
            cl_barrier();
            ip ^= 1;
            while (rec < a.R && a.rec_k[rec] == k) {
                for (int pi = 0; pi < np; ++pi) {
                    double* dst = a.rec[rec] + static_cast<size_t>(pbase + pi) * n + static_cast<size_t>(row0) * NX;
                    for (int q = t; q < RPC * NX; q += NT) dst[q] = U[pi * TBUF + (q % NX + 1) * TRI + 2 + q / NX];
                }
                ++rec;
            }
        }
#pragma unroll
        for (int pi = 0; pi < NP; ++pi)
            if (pi < np && first[pi] != INT_MAX) atomicMin(a.blow + pbase + pi, first[pi]);
        __syncthreads();
    }
}

template <int MASK, int NX, int CL, int NP, bool NZ, int XD = 0>
void launch_em_ip(s2b_context* ctx, const EmXmArgs& a) {
    constexpr int RPC = 32, NT = 256, P = 4;
    auto kern = em_cluster_ip_kernel<NX, RPC, NT, P, MASK, CL, NP, NZ, XD>;
    const size_t smem = 8 * static_cast<size_t>(NP) * (NX + 2) * (RPC + 4);
    S2B_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    S2B_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg{};
    cfg.blockDim = dim3(NT);
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
    ctx->k_em = reinterpret_cast<const void*>(kern);
}

template <int MASK, bool NZ>
void launch_em(s2b_context* ctx, const EmXmArgs& a) {
    constexpr int NX = 256, RPC = 32, NT = 256, P = 4;
    auto kern = em_cluster_kernel<NX, RPC, NT, P, MASK, NZ>;
    const size_t smem = 8 * 2 * static_cast<size_t>(NX + 2) * (RPC + 2);
    S2B_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    cudaLaunchConfig_t cfg{};
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kEmCl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(kEmCl);
    int clusters = 0;
    S2B_CUDA(cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg));
    clusters = grid_cap(std::max(1, std::min(clusters, a.M)));
    cfg.gridDim = dim3(kEmCl * clusters);
    S2B_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
    ctx->k_em = reinterpret_cast<const void*>(kern);
}

__global__ void em_cluster_status_kernel(const int* blow, const int* rec_k, int R, uint8_t* status, int M) {
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= M) return;
    for (int r = 0; r < R; ++r) status[static_cast<size_t>(r) * M + m] = blow[m] <= rec_k[r] ? 1 : 0;
}

} // namespace

// 256^2: S2B_EM_NP (3) paths per cluster in place (one barrier per step for all); S2B_EM2=0 selects
// the double-buffered one-path kernel
#ifndef S2B_EM_NP
#define S2B_EM_NP 3
#endif
bool em_multi_path() {
    const char* e = std::getenv("S2B_EM2");
    return !(e && e[0] == '0');
}

// the paper's general kinetic SPDE: h (c), fx (transport), fv (b), gvv (a), sig (beta), sigv (sigma)
constexpr int kKineticMask = 1 | 2 | 4 | 32 | 64 | 256;

bool em_cluster_supported(const s2b_fields* f) {
    const char* e = std::getenv("S2B_EMXM");
    if (e && e[0] == '0') return false;
    const bool grid_ok = f->nx == f->nv && (f->nx == 64 || f->nx == 128 || f->nx == 256 || f->nx == 512);
    if (!grid_ok) return false;
    if (f->mask == kKineticMask) return em_multi_path() || f->nx != 256; // general fields per point (in place)
    if (f->mask != (2 | 32 | 256)) return false;
    if (f->nx < 256) return f->xinv || (f->sep && f->xdep == (32 | 256)); // in-place kernels only
    if (f->xinv) return true;
    // separable fields (each x- or v-invariant): the in-place kernels take x-dependent gvv / sigv
    // (and fx) from a column table; the double-buffered one-path kernel only row values
    return f->sep && f->xdep == (32 | 256) && (f->nx == 512 || em_multi_path());
}

void em_cluster_solve(s2b_context* ctx, const s2b_fields* f, double dt, const double* d_phi,
                      const s2b_paths* paths, int step_leb, int nsteps, const std::vector<int>& rec_k,
                      double* const* d_rec, uint8_t* d_status, bool no_neg_zero) {
    const int M = static_cast<int>(paths->M);
    DevBuf<int> blow(M), work(1), drec_k(rec_k.size());
    DevBuf<double*> drec(rec_k.size());
    std::vector<int> init(M, INT_MAX);
    S2B_CUDA(cudaMemcpyAsync(blow.p, init.data(), M * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    S2B_CUDA(cudaMemsetAsync(work.p, 0, sizeof(int), ctx->stream));
    S2B_CUDA(cudaMemcpyAsync(drec_k.p, rec_k.data(), rec_k.size() * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    S2B_CUDA(cudaMemcpyAsync(drec.p, d_rec, rec_k.size() * sizeof(double*), cudaMemcpyHostToDevice, ctx->stream));
    EmXmArgs a{};
    a.rowf = f->d_rowf.p;
    a.colf = f->d_colf.p;
    a.fgen = f->d_fgen.p;
    std::copy(f->st, f->st + 5, a.st);
    a.dt = dt;
    a.values = paths->d_values.p;
    a.vstride = paths->steps + 1;
    a.step_leb = step_leb;
    a.nsteps = nsteps;
    a.phi = d_phi;
    a.rec = drec.p;
    a.rec_k = drec_k.p;
    a.R = static_cast<int>(rec_k.size());
    a.blow = blow.p;
    a.M = M;
    a.nv = static_cast<int>(f->nv);
    a.work = work.p;
    constexpr int LC = 2 | 32 | 256; // the Langevin fields
    const int xd = f->xinv ? 0 : f->xdep;
    // small grids: 2-CTA (64^2, 6 paths per cluster) / 4-CTA (128^2, 3 paths) in-place clusters
    auto small = [&](auto nz_tag, auto xd_tag) {
        constexpr bool NZ = decltype(nz_tag)::value;
        constexpr int XD = decltype(xd_tag)::value;
        if (f->nx == 64) launch_em_ip<LC, 64, 2, 6, NZ, XD>(ctx, a);
        else launch_em_ip<LC, 128, 4, 3, NZ, XD>(ctx, a);
    };
    using T_ = std::true_type;
    using F_ = std::false_type;
    using X0 = std::integral_constant<int, 0>;
    using XV_ = std::integral_constant<int, 32 | 256>;
    if (f->mask == kKineticMask) { // general fields: every value per point from the halved table
        constexpr int KM = kKineticMask;
        if (f->nx == 64) launch_em_ip<KM, 64, 2, 6, false, -1>(ctx, a);
        else if (f->nx == 128) launch_em_ip<KM, 128, 4, 3, false, -1>(ctx, a);
        else if (f->nx == 256) launch_em_ip<KM, 256, 8, S2B_EM_NP, false, -1>(ctx, a);
        else launch_em_ip<KM, 512, 16, 1, false, -1>(ctx, a);
    } else if (f->nx < 256) {
        if (xd == 0) no_neg_zero ? small(T_{}, X0{}) : small(F_{}, X0{});
        else no_neg_zero ? small(T_{}, XV_{}) : small(F_{}, XV_{});
    } else if (xd == (32 | 256)) { // the variable Langevin family: a(x), sigma(x)
        constexpr int XV = 32 | 256;
        if (no_neg_zero) {
            if (f->nx == 512) launch_em_ip<LC, 512, 16, 1, true, XV>(ctx, a);
            else launch_em_ip<LC, 256, 8, S2B_EM_NP, true, XV>(ctx, a);
        } else {
            if (f->nx == 512) launch_em_ip<LC, 512, 16, 1, false, XV>(ctx, a);
            else launch_em_ip<LC, 256, 8, S2B_EM_NP, false, XV>(ctx, a);
        }
    } else if (no_neg_zero) {
        if (f->nx == 512) launch_em_ip<LC, 512, 16, 1, true>(ctx, a);
        else if (em_multi_path()) launch_em_ip<LC, 256, 8, S2B_EM_NP, true>(ctx, a);
        else launch_em<LC, true>(ctx, a);
    } else {
        if (f->nx == 512) launch_em_ip<LC, 512, 16, 1, false>(ctx, a);
        else if (em_multi_path()) launch_em_ip<LC, 256, 8, S2B_EM_NP, false>(ctx, a);
        else launch_em<LC, false>(ctx, a);
    }
    S2B_LAUNCHED(ctx);
    em_cluster_status_kernel<<<(M + 255) / 256, 256, 0, ctx->stream>>>(blow.p, drec_k.p, a.R, d_status, M);
    S2B_LAUNCHED(ctx);
    S2B_CUDA(cudaStreamSynchronize(ctx->stream));
}

} // namespace s2b
