// Euler-Maruyama on the GPU (solve_euler, src/euler.cpp:95-182).
//
// One launch advances every live path by one explicit step of euler_step_into
// (src/euler.cpp:28-86).  The arithmetic is the reference's, term by term and
// separately rounded (-fmad=false): central differences, the drift fold over the
// non-zero fields in the order h, fx, fv, gxx, gxv, gvv with the 1/2 applied as
// (0.5*g), the noise fold sig, sigx, sigv, then (u + drift*dt) + noise*dW.
// Blow-up follows the reference exactly: a path is flagged when max|u+| is not
// finite, and std::max there ignores NaN, so only an infinite |u+| flags it.
// dW is the difference of prefix values (euler.cpp:156), so E-M and Magnus consume
// the same paths.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <type_traits>
#include <vector>

#include "magnus_common.cuh"  // mbarrier / TMA helpers
#include "s2b_internal.cuh"

namespace s2b {

namespace {

struct EmArgs {
    const double* f; // 9 * n (only mask fields valid)
    const double* rowf; // [9][nv] row values when every field is x-invariant
    int mask;
    int nx, nv;
    double st[5];
    double dt;
    const double* values;
    size_t vstride; // steps + 1
    size_t k0, k1;  // Lebesgue indices: dW = values[k1] - values[k0]
    size_t k2;      // two-step kernel: the second step's dW = values[k2] - values[k1]
    const double* in;
    double* out;
    int* blown;
    size_t M;
};

template <bool GXV>
__global__ void __launch_bounds__(256) em_step_kernel(EmArgs a) {
    const int nx = a.nx, nv = a.nv;
    const size_t n = static_cast<size_t>(nx) * nv;
  for (size_t m = blockIdx.y; m < a.M; m += gridDim.y) {
    if (a.blown[m]) continue; // the reference stops a blown path (euler.cpp:159-162)
    const double* u = a.in + static_cast<size_t>(m) * n;
    double* o = a.out + static_cast<size_t>(m) * n;
    const double* pv = a.values + static_cast<size_t>(m) * a.vstride;
    const double dW = pv[a.k1] - pv[a.k0];
    bool inf_seen = false;
    for (size_t r = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; r < n;
         r += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(r % nx), j = static_cast<int>(r / nx);
        const double uc = u[r];
        const double uxm = i > 0 ? u[r - 1] : 0.0;
        const double uxp = i + 1 < nx ? u[r + 1] : 0.0;
        const double uvm = j > 0 ? u[r - nx] : 0.0;
        const double uvp = j + 1 < nv ? u[r + nx] : 0.0;
        const double dxu = (uxp - uxm) * a.st[0];
        const double dvu = (uvp - uvm) * a.st[2];
        const double* f = a.f;
        double drift = 0.0;
        if (a.mask & 1) drift += f[r] * uc;
        if (a.mask & 2) drift += f[n + r] * dxu;
        if (a.mask & 4) drift += f[2 * n + r] * dvu;
        if (a.mask & 8) {
            const double dxxu = (uxp - 2.0 * uc + uxm) * a.st[1];
            drift += 0.5 * f[3 * n + r] * dxxu;
        }
        if (GXV) {
            const bool up = j + 1 < nv, dn = j > 0, rt = i + 1 < nx, lf = i > 0;
            const double upp = (up && rt) ? u[r + nx + 1] : 0.0;
            const double upm = (up && lf) ? u[r + nx - 1] : 0.0;
            const double ump = (dn && rt) ? u[r - nx + 1] : 0.0;
            const double umm = (dn && lf) ? u[r - nx - 1] : 0.0;
            const double dxvu = (upp - upm - ump + umm) * a.st[4];
            drift += f[4 * n + r] * dxvu;
        }
        if (a.mask & 32) {
            const double dvvu = (uvp - 2.0 * uc + uvm) * a.st[3];
            drift += 0.5 * f[5 * n + r] * dvvu;
        }
        double noise = 0.0;
        if (a.mask & 64) noise += f[6 * n + r] * uc;
        if (a.mask & 128) noise += f[7 * n + r] * dxu;
        if (a.mask & 256) noise += f[8 * n + r] * dvu;
        const double next = uc + drift * a.dt + noise * dW;
        o[r] = next;
        inf_seen |= fabs(next) == __longlong_as_double(0x7FF0000000000000LL);
    }
    if (inf_seen) a.blown[m] = 1;
  }
}

// The reference's per-point update (euler.cpp:51-80) on register operands: the same
// expressions, in the same order, as em_step_kernel (without g^xv, which needs diagonals).
__device__ __forceinline__ double em_point(int mask, const double* fv, const double* st, double dt,
                                           double dW, double uc, double uxm, double uxp, double uvm,
                                           double uvp) {
    const double dxu = (uxp - uxm) * st[0];
    const double dvu = (uvp - uvm) * st[2];
    double drift = 0.0;
    if (mask & 1) drift += fv[0] * uc;
    if (mask & 2) drift += fv[1] * dxu;
    if (mask & 4) drift += fv[2] * dvu;
    if (mask & 8) {
        const double dxxu = (uxp - 2.0 * uc + uxm) * st[1];
        drift += 0.5 * fv[3] * dxxu;
    }
    if (mask & 32) {
        const double dvvu = (uvp - 2.0 * uc + uvm) * st[3];
        drift += 0.5 * fv[5] * dvvu;
    }
    double noise = 0.0;
    if (mask & 64) noise += fv[6] * uc;
    if (mask & 128) noise += fv[7] * dxu;
    if (mask & 256) noise += fv[8] * dvu;
    return uc + drift * dt + noise * dW;
}

// Row-marching streaming step (any fields without g^xv, even nx <= 1024): a work item is
// (group of P paths, strip of R rows); thread t owns x-points 2t, 2t+1 of every row (16-byte
// loads and stores), marches down the strip with rows j-1, j, j+1 of each path in registers
// and row j+2 in flight, and takes its x-neighbours from the adjacent lanes (warp-edge lanes
// read the one value across the warp boundary from L1).  The P paths share every field load.
// Items are ordered strip-fastest so neighbouring CTAs share halo rows in L2.
template <int P, int D, int MASK, bool XINV>
__global__ void __launch_bounds__(512, P == 1 ? 2 : 1) em_rows_kernel(EmArgs a, int R, int strips, int items) {
    const int nx = a.nx, nv = a.nv;
    const size_t n = static_cast<size_t>(nx) * nv;
    const int t = threadIdx.x, lane = t & 31;
    const int x0 = 2 * t;
    const bool act = x0 < nx;
    const int mask = MASK >= 0 ? MASK : a.mask;
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const int g = item / strips;
        const int j0 = (item - g * strips) * R, j1 = min(nv, j0 + R);
        const double* u[P];
        double* o[P];
        double dW[P];
        bool live[P];
        bool any = false;
        #pragma unroll
        for (int p = 0; p < P; ++p) {
            const size_t m = static_cast<size_t>(g) * P + p;
            live[p] = m < a.M && !a.blown[m];
            any |= live[p];
            const size_t mm = live[p] ? m : 0;
            u[p] = a.in + mm * n;
            o[p] = a.out + mm * n;
            const double* pv = a.values + mm * a.vstride;
            dW[p] = live[p] ? pv[a.k1] - pv[a.k0] : 0.0;
        }
        if (!any) continue; // the reference stops a blown path (euler.cpp:159-162)
        auto ld = [&](int p, int j) -> double2 {
            if (!act || !live[p] || j < 0 || j >= nv) return make_double2(0.0, 0.0);
            return __ldg(reinterpret_cast<const double2*>(u[p] + static_cast<size_t>(j) * nx + x0));
        };
        // rows j-1, j, j+1 in registers, rows j+2 .. j+1+D in flight
        double2 rm[P], rc[P], rp[P], rq[D][P];
        #pragma unroll
        for (int p = 0; p < P; ++p) {
            rm[p] = ld(p, j0 - 1);
            rc[p] = ld(p, j0);
            rp[p] = ld(p, j0 + 1);
            #pragma unroll
            for (int q = 0; q < D - 1; ++q) rq[q][p] = ld(p, j0 + 2 + q);
        }
        bool inf_seen[P];
        #pragma unroll
        for (int p = 0; p < P; ++p) inf_seen[p] = false;
        for (int j = j0; j < j1; ++j) {
            #pragma unroll
            for (int p = 0; p < P; ++p) rq[D - 1][p] = ld(p, j + 1 + D);
            const size_t r = static_cast<size_t>(j) * nx + x0;
            double fa[9], fb[9];
            #pragma unroll
            for (int k = 0; k < 9; ++k) {
                fa[k] = fb[k] = 0.0;
                if (k != 4 && (mask >> k & 1)) {
                    if (XINV) {
                        fa[k] = fb[k] = __ldg(a.rowf + k * nv + j);
                    } else if (act) {
                        const double2 fk = __ldg(reinterpret_cast<const double2*>(a.f + k * n + r));
                        fa[k] = fk.x;
                        fb[k] = fk.y;
                    }
                }
            }
            #pragma unroll
            for (int p = 0; p < P; ++p) {
                double left = __shfl_up_sync(0xffffffffu, rc[p].y, 1);
                double right = __shfl_down_sync(0xffffffffu, rc[p].x, 1);
                if (lane == 0) left = (act && live[p] && x0 > 0) ? __ldg(u[p] + r - 1) : 0.0;
                if (x0 + 2 >= nx) right = 0.0;
                else if (lane == 31) right = live[p] ? __ldg(u[p] + r + 2) : 0.0;
                if (!act || !live[p]) continue;
                const double na = em_point(mask, fa, a.st, a.dt, dW[p], rc[p].x, left, rc[p].y,
                                           rm[p].x, rp[p].x);
                const double nb = em_point(mask, fb, a.st, a.dt, dW[p], rc[p].y, rc[p].x, right,
                                           rm[p].y, rp[p].y);
                *reinterpret_cast<double2*>(o[p] + r) = make_double2(na, nb);
                const double inf = __longlong_as_double(0x7FF0000000000000LL);
                inf_seen[p] |= (fabs(na) == inf) | (fabs(nb) == inf);
            }
            #pragma unroll
            for (int p = 0; p < P; ++p) {
                rm[p] = rc[p];
                rc[p] = rp[p];
                rp[p] = rq[0][p];
                #pragma unroll
                for (int q = 0; q < D - 1; ++q) rq[q][p] = rq[q + 1][p];
            }
        }
        #pragma unroll
        for (int p = 0; p < P; ++p)
            if (inf_seen[p]) a.blown[static_cast<size_t>(g) * P + p] = 1;
    }
}

// Temporally blocked streaming step: TWO explicit steps per pass, u0 -> u1 -> u2, with u1
// never leaving the SM.  A work item is (path, strip of kTbRows output rows); rows of u0 stream
// through a TMA ring (kTbStages deep, zero x-halo), each u1 row is computed into a 4-row
// shared ring as soon as its three u0 rows are in, each u2 row as soon as its three u1 rows
// are, one CTA barrier per row.  HBM traffic per path*point*2 steps: read u0 + write u2
// (+ the 4 halo rows per strip) instead of 2 x (read + write).  The per-point arithmetic is
// em_point (the reference's); rows outside the grid are zero at every step, as in
// euler_step_into.  A blow-up (infinite |u|) in either step flags the path; the host only
// pairs steps whose intermediate state is not a record, so statuses and records are those of
// two single steps.
constexpr int kTbStages = 8;
constexpr int kTbRows = 32;

template <int MASK, bool XINV>
__global__ void __launch_bounds__(512, 2) em_tb_kernel(EmArgs a, int strips, int items) {
    const int nx = a.nx, nv = a.nv;
    const size_t n = static_cast<size_t>(nx) * nv;
    const int t = threadIdx.x;
    const int x0 = 2 * t;
    const bool act = x0 < nx;
    const int mask = MASK >= 0 ? MASK : a.mask;
    const int RW = nx + 4; // row stride: 2 zero doubles on each side (16-byte aligned data)
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    double* u0 = reinterpret_cast<double*>(smem_raw + 128); // [kTbStages][RW]
    double* u1 = u0 + kTbStages * RW;                      // [4][RW]
    for (int q = t; q < (kTbStages + 4) * RW; q += blockDim.x) u0[q] = 0.0;
    if (t == 0) {
        for (int s = 0; s < kTbStages; ++s) mg::mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    constexpr int LA = kTbStages - 2; // rows issued ahead (slot of row r-2 is free after row r's barrier)
    const double inf = __longlong_as_double(0x7FF0000000000000LL);
    uint32_t g = 0; // running row counter (mbarrier phases)
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const int m = item / strips;
        if (a.blown[m]) continue; // the reference stops a blown path (euler.cpp:159-162)
        const int trows = (nv + strips - 1) / strips; // rows per item (host: kTbRows, S2B_TB_ROWS)
        const int j0 = (item - m * strips) * trows, j1 = min(nv, j0 + trows);
        const double* u = a.in + static_cast<size_t>(m) * n;
        double* o = a.out + static_cast<size_t>(m) * n;
        const double* pv = a.values + static_cast<size_t>(m) * a.vstride;
        const double dW1 = pv[a.k1] - pv[a.k0], dW2 = pv[a.k2] - pv[a.k1];
        const int NR = (j1 - j0) + 4; // u0 rows j0-2 .. j1+1
        auto issue = [&](int s) {
            const uint32_t gs = g + s, slot = gs % kTbStages;
            const int r = j0 - 2 + s;
            if (r >= 0 && r < nv) {
                mg::mbar_expect_tx(&full[slot], static_cast<uint32_t>(nx * 8));
                mg::tma_row(u0 + slot * RW + 2, u + static_cast<size_t>(r) * nx, static_cast<uint32_t>(nx * 8), &full[slot]);
            } else {
                mg::mbar_arrive(&full[slot]);
            }
        };
        if (t == 0)
            for (int s = 0; s < LA && s < NR; ++s) issue(s);
        bool inf_seen = false;
        for (int s = 0; s < NR; ++s) {
            const uint32_t gs = g + s;
            mg::mbar_wait(&full[gs % kTbStages], (gs / kTbStages) & 1);
            const int r = j0 - 2 + s;
            const int q = r - 1; // u1 row of this step
            if (s >= 2 && q >= 0 && q < nv && act) {
                const double* A = u0 + ((gs - 1) % kTbStages) * RW + 2;       // row q
                const double* B = u0 + ((gs - 2) % kTbStages) * RW + 2;       // row q-1
                const double* C = u0 + (gs % kTbStages) * RW + 2;             // row q+1
                const double2 c2 = *reinterpret_cast<const double2*>(A + x0);
                const double2 b2 = q - 1 >= 0 ? *reinterpret_cast<const double2*>(B + x0) : make_double2(0.0, 0.0);
                const double2 d2 = q + 1 < nv ? *reinterpret_cast<const double2*>(C + x0) : make_double2(0.0, 0.0);
                const double lft = A[x0 - 1], rgt = A[x0 + 2];
                double fa[9], fb[9];
#pragma unroll
                for (int k = 0; k < 9; ++k) {
                    fa[k] = fb[k] = 0.0;
                    if (k != 4 && (mask >> k & 1)) {
                        if (XINV) {
                            fa[k] = fb[k] = __ldg(a.rowf + k * nv + q);
                        } else {
                            const double2 fk = __ldg(reinterpret_cast<const double2*>(a.f + k * n + static_cast<size_t>(q) * nx + x0));
                            fa[k] = fk.x;
                            fb[k] = fk.y;
                        }
                    }
                }
                const double na = em_point(mask, fa, a.st, a.dt, dW1, c2.x, lft, c2.y, b2.x, d2.x);
                const double nb = em_point(mask, fb, a.st, a.dt, dW1, c2.y, c2.x, rgt, b2.y, d2.y);
                *reinterpret_cast<double2*>(u1 + (q & 3) * RW + 2 + x0) = make_double2(na, nb);
                inf_seen |= (fabs(na) == inf) | (fabs(nb) == inf);
            }
            __syncthreads(); // u1 row q visible; every thread is done with u0 row r-2
            if (t == 0 && s + LA < NR) issue(s + LA);
            const int p = r - 2; // u2 row of this step
            if (p >= j0 && p < j1 && act) {
                const double* A = u1 + (p & 3) * RW + 2;
                const double* B = u1 + ((p - 1) & 3) * RW + 2;
                const double* C = u1 + ((p + 1) & 3) * RW + 2;
                const double2 c2 = *reinterpret_cast<const double2*>(A + x0);
                const double2 b2 = p - 1 >= 0 ? *reinterpret_cast<const double2*>(B + x0) : make_double2(0.0, 0.0);
                const double2 d2 = p + 1 < nv ? *reinterpret_cast<const double2*>(C + x0) : make_double2(0.0, 0.0);
                const double lft = A[x0 - 1], rgt = A[x0 + 2];
                double fa[9], fb[9];
#pragma unroll
                for (int k = 0; k < 9; ++k) {
                    fa[k] = fb[k] = 0.0;
                    if (k != 4 && (mask >> k & 1)) {
                        if (XINV) {
                            fa[k] = fb[k] = __ldg(a.rowf + k * nv + p);
                        } else {
                            const double2 fk = __ldg(reinterpret_cast<const double2*>(a.f + k * n + static_cast<size_t>(p) * nx + x0));
                            fa[k] = fk.x;
                            fb[k] = fk.y;
                        }
                    }
                }
                const double na = em_point(mask, fa, a.st, a.dt, dW2, c2.x, lft, c2.y, b2.x, d2.x);
                const double nb = em_point(mask, fb, a.st, a.dt, dW2, c2.y, c2.x, rgt, b2.y, d2.y);
                *reinterpret_cast<double2*>(o + static_cast<size_t>(p) * nx + x0) = make_double2(na, nb);
                inf_seen |= (fabs(na) == inf) | (fabs(nb) == inf);
            }
        }
        g += NR;
        if (inf_seen) a.blown[m] = 1;
    }
}

__global__ void em_record_status_kernel(const int* blown, uint8_t* status, size_t M) {
    const size_t m = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (m < M) status[m] = blown[m] ? 1 : 0;
}

} // namespace

s2b_fields* make_fields(s2b_context* ctx, const s2b_grid* grid, const double* const* fields9) {
    const size_t nx = grid->nx, nv = grid->nv, n = nx * nv;
    if (n == 0) fail(S2B_ERR_CONFIG, "fields: empty grid");
    auto* f = new s2b_fields();
    f->ctx = ctx;
    f->nx = nx;
    f->nv = nv;
    f->grid = *grid;
    f->d_f.alloc(9 * n);
    S2B_CUDA(cudaMemset(f->d_f.p, 0, f->d_f.bytes()));
    for (int k = 0; k < 9; ++k) {
        if (!fields9 || !fields9[k]) continue;
        bool nz = false;
        for (size_t r = 0; r < n; ++r)
            if (fields9[k][r] != 0.0) {
                nz = true;
                break;
            }
        if (!nz) continue; // CoefficientFields::refresh_zero_flags
        f->mask |= 1 << k;
        S2B_CUDA(cudaMemcpy(f->d_f.p + k * n, fields9[k], n * sizeof(double), cudaMemcpyHostToDevice));
    }
    // x-invariant fields (the constant Langevin family): row values for the cluster kernel
    f->xinv = true;
    std::vector<double> rowf(9 * nv, 0.0);
    for (int k = 0; k < 9 && f->xinv; ++k) {
        if (!(f->mask >> k & 1)) continue;
        for (size_t j = 0; j < nv && f->xinv; ++j) {
            const double* row = fields9[k] + j * nx;
            rowf[k * nv + j] = row[0];
            for (size_t i = 1; i < nx; ++i)
                if (std::memcmp(&row[i], &row[0], sizeof(double)) != 0) {
                    f->xinv = false;
                    break;
                }
        }
    }
    if (f->xinv) {
        f->d_rowf.alloc(9 * nv);
        S2B_CUDA(cudaMemcpy(f->d_rowf.p, rowf.data(), rowf.size() * sizeof(double), cudaMemcpyHostToDevice));
    }
    // separable fields: x-dependent ones must be v-invariant; rows of the others feed d_rowf
    {
        f->sep = true;
        f->xdep = 0;
        std::vector<double> colf(9 * nx, 0.0), rowf2(9 * nv, 0.0);
        for (int k = 0; k < 9 && f->sep; ++k) {
            if (!(f->mask >> k & 1)) continue;
            const double* F = fields9[k];
            bool xi = true, vi = true;
            for (size_t j = 0; j < nv && xi; ++j)
                for (size_t i = 1; i < nx; ++i)
                    if (std::memcmp(&F[j * nx + i], &F[j * nx], sizeof(double)) != 0) {
                        xi = false;
                        break;
                    }
            for (size_t j = 1; j < nv && vi; ++j)
                if (std::memcmp(&F[j * nx], &F[0], nx * sizeof(double)) != 0) vi = false;
            if (!xi && !vi) f->sep = false;
            if (!xi) f->xdep |= 1 << k;
            for (size_t i = 0; i < nx; ++i) colf[k * nx + i] = (k == 3 || k == 5) ? 0.5 * F[i] : F[i];
            for (size_t j = 0; j < nv; ++j) rowf2[k * nv + j] = F[j * nx];
        }
        if (f->sep && !f->xinv) {
            f->d_colf.alloc(9 * nx);
            S2B_CUDA(cudaMemcpy(f->d_colf.p, colf.data(), colf.size() * sizeof(double), cudaMemcpyHostToDevice));
            f->d_rowf.alloc(9 * nv); // x-invariant fields' row values (x-dependent rows unused)
            S2B_CUDA(cudaMemcpy(f->d_rowf.p, rowf2.data(), rowf2.size() * sizeof(double), cudaMemcpyHostToDevice));
        }
    }
    // general fields for the cluster E-M kernels: every field per point, 0.5 * g pre-applied
    // (the reference's (0.5 * g) product, the same rounding)
    if (!f->xinv && !(f->mask & 16)) {
        std::vector<double> fg(9 * n, 0.0);
        for (int k = 0; k < 9; ++k) {
            if (!(f->mask >> k & 1)) continue;
            for (size_t j = 0; j < nv; ++j) // x-major: [k][i][j]
                for (size_t i = 0; i < nx; ++i) {
                    const double v = fields9[k][j * nx + i];
                    fg[k * n + i * nv + j] = (k == 3 || k == 5) ? 0.5 * v : v;
                }
        }
        f->d_fgen.alloc(9 * n);
        S2B_CUDA(cudaMemcpy(f->d_fgen.p, fg.data(), fg.size() * sizeof(double), cudaMemcpyHostToDevice));
    }
    // EulerStencils::from_grid (euler.cpp:18-26)
    const double dx = (grid->bx - grid->ax) / static_cast<double>(nx + 1);
    const double dv = (grid->bv - grid->av) / static_cast<double>(nv + 1);
    f->st[0] = 1.0 / (2.0 * dx);
    f->st[1] = 1.0 / (dx * dx);
    f->st[2] = 1.0 / (2.0 * dv);
    f->st[3] = 1.0 / (dv * dv);
    f->st[4] = 1.0 / (4.0 * dx * dv);
    return f;
}

s2b_ensemble* solve_euler(s2b_context* ctx, const s2b_fields* f, const s2b_euler_config* cfg,
                          const double* phi, const s2b_paths* paths) {
    const WindowPlan plan = plan_windows(cfg->dt, cfg->T, paths->dt_leb, paths->steps,
                                         cfg->record_times, cfg->n_record, "solve_euler");
    const size_t M = paths->M, n = f->nx * f->nv;
    auto* e = new s2b_ensemble();
    try {
        e->ctx = ctx;
        e->R = plan.record_steps.size();
        e->M = M;
        e->nx = f->nx;
        e->nv = f->nv;
        e->seed = paths->seed;
        e->grid = f->grid;
        for (size_t r : plan.record_steps) e->times.push_back(static_cast<double>(r) * paths->dt_leb);
        e->status.alloc(e->R * M);
        const size_t nsteps = plan.total_steps / plan.dt_steps;
        if (em_cluster_supported(f) && M > 0) {
            // cluster-resident: every step of every path on chip, records written directly
            std::vector<int> rec_k;
            std::vector<double*> rp;
            for (size_t r : plan.record_steps) {
                rec_k.push_back(static_cast<int>(r / plan.dt_steps) - 1);
                e->states.emplace_back(M * n);
                rp.push_back(e->states.back().p);
            }
            DevBuf<double> dphi(n);
            S2B_CUDA(cudaMemcpyAsync(dphi.p, phi, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
            bool nz = true; // no -0.0 in the datum (see em_cluster.cu)
            for (size_t i = 0; i < n && nz; ++i) nz = !(phi[i] == 0.0 && std::signbit(phi[i]));
            em_cluster_solve(ctx, f, cfg->dt, dphi.p, paths, static_cast<int>(plan.dt_steps),
                             static_cast<int>(nsteps), rec_k, rp.data(), e->status.p, nz);
            return e;
        }
        DevBuf<double> U[2] = {DevBuf<double>(M * n), DevBuf<double>(M * n)};
        DevBuf<int> blown(M);
        S2B_CUDA(cudaMemsetAsync(blown.p, 0, blown.bytes(), ctx->stream));
        broadcast_rows(ctx, U[0].p, phi, n, M);
        EmArgs a{};
        a.f = f->d_f.p;
        a.mask = f->mask;
        a.nx = static_cast<int>(f->nx);
        a.nv = static_cast<int>(f->nv);
        std::copy(f->st, f->st + 5, a.st);
        a.dt = cfg->dt;
        a.values = paths->d_values.p;
        a.vstride = paths->steps + 1;
        a.blown = blown.p;
        a.M = M;
        const unsigned gx = static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 64));
        // the row-marching kernel: even nx up to 1024 points, no g^xv (S2B_EMROWS=0: the old one)
#ifndef S2B_EM_D
#define S2B_EM_D 2
#endif
        // paths per item, rows per strip, rows in flight: one path per item and two CTAs per SM
        // (64 registers) measured 0.745 of HBM at 1024^2 vs 0.56 for 2 paths x 4 rows (ncu)
        constexpr int kP = 2, kR = 32, kD = S2B_EM_D;
        const char* er = std::getenv("S2B_EMROWS");
        const bool rows = !(f->mask & 16) && f->nx % 2 == 0 && f->nx <= 1024 && !(er && er[0] == '0');
        const int nt = static_cast<int>(((f->nx / 2 + 31) / 32) * 32);
        const int strips = static_cast<int>((f->nv + kR - 1) / kR);
        const char* ep0 = std::getenv("S2B_EM_P");
        const int pit0 = ep0 && std::atoi(ep0) == 2 ? kP : 1;
        const size_t items_sz = ((M + pit0 - 1) / pit0) * static_cast<size_t>(strips);
        if (items_sz > static_cast<size_t>(INT_MAX)) fail(S2B_ERR_CONFIG, "solve_euler: too many paths");
        const int items = static_cast<int>(items_sz);
        a.rowf = f->d_rowf.p;
        using RowsFn = void (*)(EmArgs, int, int, int);
        const char* ep = std::getenv("S2B_EM_P"); // paths per item (A/B runs): 1 (default) or 2
        const int psel = ep ? std::atoi(ep) : 1;
        auto pick = [&](auto dtag) -> RowsFn {
            constexpr int D = decltype(dtag)::value;
            if (psel == 1)
                return f->mask == (2 | 32 | 256) ? (f->xinv ? em_rows_kernel<1, D, 2 | 32 | 256, true>
                                                            : em_rows_kernel<1, D, 2 | 32 | 256, false>)
                                                 : em_rows_kernel<1, D, -1, false>;
            return f->mask == (2 | 32 | 256) ? (f->xinv ? em_rows_kernel<kP, D, 2 | 32 | 256, true>
                                                        : em_rows_kernel<kP, D, 2 | 32 | 256, false>)
                                             : em_rows_kernel<kP, D, -1, false>;
        };
        const char* ed = std::getenv("S2B_EM_D"); // rows in flight (A/B runs)
        const int dsel = ed ? std::atoi(ed) : kD;
        RowsFn rows_fn = dsel == 2 ? pick(std::integral_constant<int, 2>{})
                         : dsel == 6 ? pick(std::integral_constant<int, 6>{})
                                     : pick(std::integral_constant<int, kD>{});
        const int pitem = psel == 1 ? 1 : kP;
        int rows_grid = 0;
        if (rows) {
            int per_sm = 0;
            S2B_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rows_fn, nt, 0));
            rows_grid = grid_cap(std::max(1, std::min(items, std::max(1, per_sm) * ctx->num_sms)));
        }
        // two steps per pass where the intermediate state is not a record (S2B_EMTB=0: never)
        const char* etb = std::getenv("S2B_EMTB");
        const bool tb = rows && !(etb && etb[0] == '0');
        const char* etr = std::getenv("S2B_TB_ROWS");
        const int tbr = etr ? std::max(4, std::atoi(etr)) : kTbRows;
        const int tb_strips = static_cast<int>((f->nv + tbr - 1) / tbr);
        const size_t tb_items_sz = M * static_cast<size_t>(tb_strips);
        if (tb && tb_items_sz > static_cast<size_t>(INT_MAX)) fail(S2B_ERR_CONFIG, "solve_euler: too many paths");
        const int tb_items = static_cast<int>(tb_items_sz);
        using TbFn = void (*)(EmArgs, int, int);
        TbFn tb_fn = f->mask == (2 | 32 | 256) ? (f->xinv ? em_tb_kernel<2 | 32 | 256, true> : em_tb_kernel<2 | 32 | 256, false>)
                                                 : em_tb_kernel<-1, false>;
        const size_t tb_smem = 128 + static_cast<size_t>(kTbStages + 4) * (f->nx + 4) * 8;
        int tb_grid = 0;
        if (tb) {
            S2B_CUDA(cudaFuncSetAttribute(tb_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(tb_smem)));
            int per_sm = 0;
            S2B_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tb_fn, nt, tb_smem));
            tb_grid = grid_cap(std::max(1, std::min(tb_items, std::max(1, per_sm) * ctx->num_sms)));
        }
        auto is_record = [&](size_t done) {
            return std::binary_search(plan.record_steps.begin(), plan.record_steps.end(), done);
        };
        size_t rec = 0;
        int cur = 0;
        for (size_t k = 0; k < nsteps;) {
            const bool two = tb && k + 1 < nsteps && !is_record((k + 1) * plan.dt_steps);
            a.k0 = k * plan.dt_steps;
            a.k1 = (k + 1) * plan.dt_steps;
            a.k2 = (k + 2) * plan.dt_steps;
            a.in = U[cur].p;
            a.out = U[cur ^ 1].p;
            dim3 grid(gx, static_cast<unsigned>(std::min<size_t>(M, 65535)));
            if (two) {
                tb_fn<<<tb_grid, nt, tb_smem, ctx->stream>>>(a, tb_strips, tb_items);
                ctx->k_em = reinterpret_cast<const void*>(tb_fn);
            } else if (rows) {
                rows_fn<<<rows_grid, nt, 0, ctx->stream>>>(a, kR, strips, items);
                ctx->k_em = reinterpret_cast<const void*>(rows_fn);
            } else if (f->mask & 16) {
                em_step_kernel<true><<<grid, 256, 0, ctx->stream>>>(a);
                ctx->k_em = reinterpret_cast<const void*>(em_step_kernel<true>);
            } else {
                em_step_kernel<false><<<grid, 256, 0, ctx->stream>>>(a);
                ctx->k_em = reinterpret_cast<const void*>(em_step_kernel<false>);
            }
            S2B_LAUNCHED(ctx);
            cur ^= 1;
            k += two ? 2 : 1;
            const size_t done = k * plan.dt_steps;
            while (rec < plan.record_steps.size() && plan.record_steps[rec] == done) {
                if (rec + 1 == plan.record_steps.size()) {
                    e->states.push_back(std::move(U[cur])); // last record: the final state itself
                } else {
                    DevBuf<double> snap(M * n);
                    S2B_CUDA(cudaMemcpyAsync(snap.p, U[cur].p, snap.bytes(), cudaMemcpyDeviceToDevice, ctx->stream));
                    e->states.push_back(std::move(snap));
                }
                em_record_status_kernel<<<static_cast<unsigned>((M + 255) / 256), 256, 0, ctx->stream>>>(
                    blown.p, e->status.p + rec * M, M);
                S2B_LAUNCHED(ctx);
                ++rec;
            }
        }
        S2B_CUDA(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
        delete e;
        throw;
    }
    return e;
}

namespace {
// max|out| per field with std::max semantics (euler.cpp:82): NaN never replaces the running
// maximum; on bit patterns, a NaN's |bits| exceed +inf's and are skipped.
__global__ void em_maxabs_kernel(const double* __restrict__ out, size_t n, unsigned long long* __restrict__ best) {
    const size_t m = blockIdx.y;
    unsigned long long b = 0;
    for (size_t r = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; r < n;
         r += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const unsigned long long v = static_cast<unsigned long long>(__double_as_longlong(out[m * n + r])) & 0x7FFFFFFFFFFFFFFFULL;
        if (v <= 0x7FF0000000000000ULL) b = max(b, v);
    }
    for (int o = 16; o > 0; o >>= 1) b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
    if ((threadIdx.x & 31) == 0 && b) atomicMax(&best[m], b);
}
} // namespace

// euler_step_into (euler.cpp:28-86) for M device fields: em_step_kernel's per-point
// arithmetic (the solver's general kernel) with dW = values[1] - values[0] for a
// two-column prefix table {0, dW[m]} -- exactly dW[m] -- and the caller's stencil scales.
void euler_step_batch(const s2b_fields* f, const double* st, const double* d_u, double* d_out, size_t M,
                      const double* dW, double dt, double* maxabs) {
    if (M == 0) return;
    s2b_context* ctx = f->ctx;
    S2B_CUDA(cudaSetDevice(ctx->device));
    const size_t n = f->nx * f->nv;
    std::vector<double> vals(2 * M);
    for (size_t m = 0; m < M; ++m) {
        vals[2 * m] = 0.0;
        vals[2 * m + 1] = dW[m];
    }
    DevBuf<double> dv(2 * M);
    DevBuf<int> blown(M);
    DevBuf<unsigned long long> best(M);
    S2B_CUDA(cudaMemcpyAsync(dv.p, vals.data(), vals.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    S2B_CUDA(cudaMemsetAsync(blown.p, 0, blown.bytes(), ctx->stream));
    S2B_CUDA(cudaMemsetAsync(best.p, 0, best.bytes(), ctx->stream));
    EmArgs a{};
    a.f = f->d_f.p;
    a.mask = f->mask;
    a.nx = static_cast<int>(f->nx);
    a.nv = static_cast<int>(f->nv);
    std::copy(st ? st : f->st, (st ? st : f->st) + 5, a.st);
    a.dt = dt;
    a.values = dv.p;
    a.vstride = 2;
    a.k0 = 0;
    a.k1 = 1;
    a.in = d_u;
    a.out = d_out;
    a.blown = blown.p;
    a.M = M;
    dim3 grid(static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 64)), static_cast<unsigned>(std::min<size_t>(M, 65535)));
    if (f->mask & 16)
        em_step_kernel<true><<<grid, 256, 0, ctx->stream>>>(a);
    else
        em_step_kernel<false><<<grid, 256, 0, ctx->stream>>>(a);
    S2B_LAUNCHED(ctx);
    if (maxabs) {
        for (size_t m0 = 0; m0 < M; m0 += 65535) {
            const size_t mc = std::min<size_t>(M - m0, 65535);
            em_maxabs_kernel<<<dim3(static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 32)), static_cast<unsigned>(mc)), 256, 0,
                               ctx->stream>>>(d_out + m0 * n, n, best.p + m0);
            S2B_LAUNCHED(ctx);
        }
        std::vector<unsigned long long> hb(M);
        S2B_CUDA(cudaMemcpyAsync(hb.data(), best.p, M * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
        S2B_CUDA(cudaStreamSynchronize(ctx->stream));
        for (size_t m = 0; m < M; ++m) std::memcpy(&maxabs[m], &hb[m], sizeof(double));
    } else {
        S2B_CUDA(cudaStreamSynchronize(ctx->stream));
    }
}

} // namespace s2b
