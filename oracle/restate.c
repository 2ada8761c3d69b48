/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle.  Never linked into, called by or
 * shipped with the product path (paper_2207_09776_b200/).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may use it.
 *
 * A plain-C restatement of the reference's hot path (arXiv 2207.09776 spec,
 * C++ library under /root/reference/proj).  Every function cites the
 * reference file:line it restates.  Arithmetic is written operation by
 * operation in the reference's order and compiled with -ffp-contract=off,
 * so on the same inputs it reproduces the reference bit for bit (pinned by
 * tests/test_oracle.py against oracle/_ref and tests/golden/).
 *
 * Sparse inputs are CSR exactly as spde2d::SparseMatrix stores them
 * (size_t row_ptr, int32 col_idx, double values; sparse.hpp:36-73).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- stochastics.cpp:13-57  NormalStream (splitmix64 -> xoshiro256++, Box-Muller) ---- */
static uint64_t rs_splitmix64(uint64_t *state) {
    uint64_t z = (*state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static uint64_t rs_rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

typedef struct { uint64_t s[4]; double cached; int has_cached; } rs_stream;

static void rs_stream_init(rs_stream *st, uint64_t seed, uint64_t traj) {
    uint64_t mix = seed;
    (void)rs_splitmix64(&mix);                 /* stochastics.cpp:26 */
    mix ^= (traj + 1) * 0xD1B54A32D192ED03ULL; /* :27 */
    for (int i = 0; i < 4; ++i) st->s[i] = rs_splitmix64(&mix);
    st->has_cached = 0;
    st->cached = 0.0;
}
static uint64_t rs_next_u64(rs_stream *st) { /* :31-41 xoshiro256++ */
    uint64_t *s = st->s;
    const uint64_t result = rs_rotl(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rs_rotl(s[3], 45);
    return result;
}
static double rs_next_normal(rs_stream *st) { /* :43-57 */
    if (st->has_cached) { st->has_cached = 0; return st->cached; }
    const double u1 = ((double)(rs_next_u64(st) >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = (double)(rs_next_u64(st) >> 11) * 0x1.0p-53;
    const double r = sqrt(-2.0 * log(u1));
    const double angle = 2.0 * 3.141592653589793 * u2;
    st->cached = r * sin(angle);
    st->has_cached = 1;
    return r * cos(angle);
}

/* stochastics.cpp:76-101: prefix values[m][0..steps] and increments (serial per path). */
void rs_simulate_brownian(size_t steps, double dt_leb, size_t M, uint64_t seed,
                          double *values, double *increments) {
    const double scale = sqrt(dt_leb);
    for (size_t m = 0; m < M; ++m) {
        rs_stream st;
        rs_stream_init(&st, seed, m);
        double *val = values + m * (steps + 1);
        val[0] = 0.0;
        for (size_t k = 0; k < steps; ++k) {
            const double inc = scale * rs_next_normal(&st);
            if (increments) increments[m * steps + k] = inc;
            val[k + 1] = val[k] + inc;
        }
    }
}

/* ---- stochastics.cpp:121-141  lebesgue_functionals: out = {h, W, IW, IsW, IW2} ---- */
void rs_functionals(const double *p, size_t k0, size_t k1, double dt, double out[5]) {
    const double base = p[k0];
    double iw = 0.0, isw = 0.0, iw2 = 0.0;
    for (size_t j = 0; j < k1 - k0; ++j) {
        const double w = p[k0 + j] - base;
        const double s = (double)j * dt;
        iw += w;
        isw += s * w;
        iw2 += w * w;
    }
    out[0] = (double)(k1 - k0) * dt; /* PathSegment::length, stochastics.hpp:58 */
    out[1] = p[k1] - p[k0];          /* terminal, stochastics.hpp:60 */
    out[2] = iw * dt;
    out[3] = isw * dt;
    out[4] = iw2 * dt;
}

/* ---- magnus.cpp:26-40  log_coefficients, slots B, A, A2, [B,A], [[B,A],A], [[B,A],B] ---- */
void rs_log_coefficients(int order, const double f[5], double c[6]) {
    const double h = f[0], W = f[1], IW = f[2], IsW = f[3], IW2 = f[4];
    for (int i = 0; i < 6; ++i) c[i] = 0.0;
    c[0] = h;
    c[1] = W;
    if (order >= 2) {
        c[2] = -0.5 * h;
        c[3] = IW - 0.5 * h * W;
    }
    if (order >= 3) {
        c[4] = 0.5 * IW2 - 0.5 * W * IW + h * W * W / 12.0;
        c[5] = IsW - 0.5 * h * IW - h * h * W / 12.0;
    }
}

/* A CSR source of the logarithm. */
typedef struct {
    const size_t *rp;
    const int32_t *ci;
    const double *v;
} rs_csr;

static int rs_cmp_i32(const void *a, const void *b) {
    const int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}
static int rs_cmp_i64(const void *a, const void *b) {
    const int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

/* magnus.cpp:88-139 union pattern (sorted unique columns per row) over the
 * sources present at `build_order` (slot_min_order, :54).  Returns nnz;
 * when rp/ci are non-NULL fills them.  srcs[s].rp == NULL marks an absent slot. */
size_t rs_union_pattern(size_t n, int build_order, const rs_csr srcs[6], size_t *rp, int32_t *ci) {
    static const int min_order[6] = {1, 1, 2, 2, 3, 3};
    size_t cap = 0;
    for (int s = 0; s < 6; ++s)
        if (min_order[s] <= build_order && srcs[s].rp) cap += srcs[s].rp[n];
    int32_t *scratch = (int32_t *)malloc((cap > 0 ? cap : 1) * sizeof(int32_t));
    size_t total = 0;
    if (rp) rp[0] = 0;
    for (size_t r = 0; r < n; ++r) {
        size_t cnt = 0;
        for (int s = 0; s < 6; ++s) {
            if (min_order[s] > build_order || !srcs[s].rp) continue;
            for (size_t k = srcs[s].rp[r]; k < srcs[s].rp[r + 1]; ++k) scratch[cnt++] = srcs[s].ci[k];
        }
        qsort(scratch, cnt, sizeof(int32_t), rs_cmp_i32);
        size_t u = 0;
        for (size_t k = 0; k < cnt; ++k)
            if (u == 0 || scratch[k] != scratch[u - 1]) scratch[u++] = scratch[k];
        if (ci) memcpy(ci + total, scratch, u * sizeof(int32_t));
        total += u;
        if (rp) rp[r + 1] = total;
    }
    free(scratch);
    return total;
}

/* magnus.cpp:141-160 fill: values = 0, then += c_s * v over slots in order,
 * skipping slots above `order` and zero coefficients. */
void rs_union_fill(size_t n, int build_order, int order, const rs_csr srcs[6], const double c[6],
                   const size_t *rp, const int32_t *ci, double *values) {
    static const int min_order[6] = {1, 1, 2, 2, 3, 3};
    memset(values, 0, rp[n] * sizeof(double));
    for (int s = 0; s < 6; ++s) {
        if (min_order[s] > build_order || !srcs[s].rp) continue;
        if (min_order[s] > order) continue;
        const double coef = c[s];
        if (coef == 0.0) continue;
        for (size_t r = 0; r < n; ++r) {
            size_t u = rp[r];
            for (size_t k = srcs[s].rp[r]; k < srcs[s].rp[r + 1]; ++k) {
                while (ci[u] != srcs[s].ci[k]) ++u;
                values[u] += coef * srcs[s].v[k];
            }
        }
    }
}

/* sparse.cpp:263-271 one_norm: max column abs-sum, entries visited in CSR order. */
double rs_one_norm(size_t n, const size_t *rp, const int32_t *ci, const double *v) {
    double *colsum = (double *)calloc(n > 0 ? n : 1, sizeof(double));
    for (size_t k = 0; k < rp[n]; ++k) colsum[ci[k]] += fabs(v[k]);
    double best = 0.0;
    for (size_t c = 0; c < n; ++c) best = best < colsum[c] ? colsum[c] : best; /* std::max */
    free(colsum);
    return best;
}

/* sparse.cpp:375-423 diagonal-major layout + matvec (ascending offsets, from 0.0). */
typedef struct {
    size_t ndiag;
    int64_t *off;
    size_t *begin;
    double *val;
} rs_dia;

static int rs_dia_build(size_t n, const size_t *rp, const int32_t *ci, const double *v, rs_dia *d) {
    const size_t nnz = rp[n];
    int64_t *offs = (int64_t *)malloc((nnz > 0 ? nnz : 1) * sizeof(int64_t));
    for (size_t r = 0; r < n; ++r)
        for (size_t k = rp[r]; k < rp[r + 1]; ++k) offs[k] = (int64_t)ci[k] - (int64_t)r;
    qsort(offs, nnz, sizeof(int64_t), rs_cmp_i64);
    size_t u = 0;
    for (size_t k = 0; k < nnz; ++k)
        if (u == 0 || offs[k] != offs[u - 1]) offs[u++] = offs[k];
    if (u > 64) { free(offs); return 0; } /* kMaxDiaDiagonals, sparse.cpp:373 */
    d->ndiag = u;
    d->off = offs;
    d->begin = (size_t *)malloc((u + 1) * sizeof(size_t));
    size_t total = 0;
    for (size_t k = 0; k < u; ++k) {
        d->begin[k] = total;
        total += n - (size_t)llabs(offs[k]);
    }
    d->begin[u] = total;
    d->val = (double *)calloc(total > 0 ? total : 1, sizeof(double));
    for (size_t r = 0; r < n; ++r) {
        for (size_t k = rp[r]; k < rp[r + 1]; ++k) {
            const int64_t off = (int64_t)ci[k] - (int64_t)r;
            size_t lo = 0, hi = u; /* lower_bound */
            while (lo < hi) { size_t mid = (lo + hi) / 2; if (offs[mid] < off) lo = mid + 1; else hi = mid; }
            const size_t r0 = off < 0 ? (size_t)(-off) : 0;
            d->val[d->begin[lo] + (r - r0)] = v[k];
        }
    }
    return 1;
}
static void rs_dia_free(rs_dia *d) { free(d->off); free(d->begin); free(d->val); }

static void rs_dia_mv(const rs_dia *d, size_t n, const double *x, double *y) {
    for (size_t i = 0; i < n; ++i) y[i] = 0.0;
    for (size_t k = 0; k < d->ndiag; ++k) {
        const int64_t off = d->off[k];
        const size_t r0 = off < 0 ? (size_t)(-off) : 0;
        const size_t len = d->begin[k + 1] - d->begin[k];
        const double *vv = d->val + d->begin[k];
        const double *xs = x + (size_t)((int64_t)r0 + off);
        double *ys = y + r0;
        for (size_t i = 0; i < len; ++i) ys[i] += vv[i] * xs[i];
    }
}

static void rs_csr_mv(size_t n, const size_t *rp, const int32_t *ci, const double *v,
                      const double *x, double *y) { /* sparse.cpp:236-247 */
    for (size_t r = 0; r < n; ++r) {
        double s = 0.0;
        for (size_t k = rp[r]; k < rp[r + 1]; ++k) s += v[k] * x[ci[k]];
        y[r] = s;
    }
}

/* sparse.cpp:427-503 expmv_into.  report = {status (0 Ok,1 Overflow,2 TolNotReached),
 * segments, max_terms, total_terms}; terms_per_seg (nullable, capacity cap_seg) gets K per segment. */
int rs_expmv(size_t n, const size_t *rp, const int32_t *ci, const double *v, const double *x,
             double tol, double theta, double *y, int report[4], int *terms_per_seg, int cap_seg,
             double *norm_out) {
    const int kMaxTerms = 55;
    const double norm = rs_one_norm(n, rp, ci, v);
    const double q = ceil(norm / theta);
    const int segments = q > 1.0 ? (int)q : 1;
    if (norm_out) *norm_out = norm;
    rs_dia dia;
    const int use_dia = rs_dia_build(n, rp, ci, v, &dia);
    double *term = (double *)malloc(n * sizeof(double));
    double *next = (double *)malloc(n * sizeof(double));
    double *accum = (double *)malloc(n * sizeof(double));
    memcpy(y, x, n * sizeof(double));
    report[0] = 0; report[1] = segments; report[2] = 0; report[3] = 0;
    int rc = 0;
    if (norm == 0.0 || n == 0) goto done;
    for (int seg = 0; seg < segments; ++seg) {
        memcpy(term, y, n * sizeof(double));
        memcpy(accum, y, n * sizeof(double));
        double prev_tnorm = INFINITY;
        int converged = 0;
        for (int k = 1; k <= kMaxTerms; ++k) {
            if (use_dia) rs_dia_mv(&dia, n, term, next);
            else rs_csr_mv(n, rp, ci, v, term, next);
            const double inv = 1.0 / ((double)segments * k);
            double tnorm = 0.0, snorm = 0.0;
            for (size_t i = 0; i < n; ++i) {
                const double t = next[i] * inv;
                term[i] = t;
                const double s = accum[i] + t;
                accum[i] = s;
                const double at = fabs(t), as = fabs(s);
                tnorm = tnorm < at ? at : tnorm; /* std::max(tnorm, |t|) */
                snorm = snorm < as ? as : snorm;
            }
            report[3] += 1;
            if (!isfinite(tnorm) || !isfinite(snorm)) { report[0] = 1; rc = 1; goto done; }
            if (k > report[2]) report[2] = k;
            const double gate = tol * snorm;
            if (tnorm <= gate && prev_tnorm <= gate) {
                if (terms_per_seg && seg < cap_seg) terms_per_seg[seg] = k;
                converged = 1;
                break;
            }
            prev_tnorm = tnorm;
        }
        if (!converged) { report[0] = 2; rc = 2; goto done; }
        memcpy(y, accum, n * sizeof(double));
    }
    for (size_t i = 0; i < n; ++i)
        if (!isfinite(y[i])) { report[0] = 1; rc = 1; break; }
done:
    if (use_dia) rs_dia_free(&dia);
    free(term); free(next); free(accum);
    return rc;
}

/* magnus.cpp:239-304 solve_iterated_magnus for ONE path (serial).  record_steps
 * ascending with last == total_steps; states_out [R][n]; status_out [R] (0 Ok, 1 blown);
 * win_terms (nullable) [nwin] gets the Taylor-term count S*K of each window;
 * win_segments (nullable) [nwin] the segment count s. */
void rs_magnus_path(size_t n, int order, const rs_csr srcs[6], const double *phi,
                    const double *path, double dt_leb, size_t dt_steps, size_t total_steps,
                    const size_t *record_steps, size_t nrec, double tol, double theta, double cap,
                    double *states_out, uint8_t *status_out, int *win_terms, int *win_segments) {
    size_t *rp = (size_t *)malloc((n + 1) * sizeof(size_t));
    const size_t nnz = rs_union_pattern(n, order, srcs, rp, NULL);
    int32_t *ci = (int32_t *)malloc((nnz > 0 ? nnz : 1) * sizeof(int32_t));
    rs_union_pattern(n, order, srcs, rp, ci);
    double *vals = (double *)malloc((nnz > 0 ? nnz : 1) * sizeof(double));
    double *u = (double *)malloc(n * sizeof(double));
    double *unext = (double *)malloc(n * sizeof(double));
    memcpy(u, phi, n * sizeof(double));
    for (size_t r = 0; r < nrec; ++r) status_out[r] = 1;
    size_t rec = 0, w = 0;
    int blown = 0;
    for (size_t k0 = 0; k0 < total_steps && !blown; k0 += dt_steps, ++w) {
        const size_t k1 = k0 + dt_steps;
        double f[5], c[6];
        rs_functionals(path, k0, k1, dt_leb, f);
        rs_log_coefficients(order, f, c);
        rs_union_fill(n, order, order, srcs, c, rp, ci, vals);
        int rep[4];
        rs_expmv(n, rp, ci, vals, u, tol, theta, unext, rep, NULL, 0, NULL);
        if (win_terms) win_terms[w] = rep[3];
        if (win_segments) win_segments[w] = rep[1];
        if (rep[0] != 0) { blown = 1; break; }
        double *tmp = u; u = unext; unext = tmp;
        double norm = 0.0;
        for (size_t i = 0; i < n; ++i) { const double a = fabs(u[i]); norm = norm < a ? a : norm; }
        if (!isfinite(norm) || norm > cap) { blown = 1; break; }
        while (rec < nrec && record_steps[rec] == k1) {
            memcpy(states_out + rec * n, u, n * sizeof(double));
            status_out[rec] = 0;
            ++rec;
        }
    }
    if (blown)
        for (size_t r = rec; r < nrec; ++r) status_out[r] = 1;
    free(rp); free(ci); free(vals); free(u); free(unext);
}

/* euler.cpp:28-86 euler_step_into.  fields[9] = h fx fv gxx gxv gvv sig sigx sigv
 * (NULL == identically zero, the zero_* flags); st = inv2dx invdx2 inv2dv invdv2 inv4dxdv
 * (EulerStencils::from_grid, euler.cpp:18-26).  Returns max|out|. */
double rs_euler_step(size_t nx, size_t nv, const double *const *f, const double st[5],
                     const double *u, double *out, double dW, double dt) {
    double maxabs = 0.0;
    for (size_t j = 0; j < nv; ++j) {
        const double *c = u + j * nx;
        const double *cm = j > 0 ? c - nx : NULL;
        const double *cp = j + 1 < nv ? c + nx : NULL;
        double *o = out + j * nx;
        for (size_t i = 0; i < nx; ++i) {
            const size_t id = j * nx + i;
            const double uc = c[i];
            const double uxm = i > 0 ? c[i - 1] : 0.0;
            const double uxp = i + 1 < nx ? c[i + 1] : 0.0;
            const double uvm = cm ? cm[i] : 0.0;
            const double uvp = cp ? cp[i] : 0.0;
            const double dxu = (uxp - uxm) * st[0];
            const double dvu = (uvp - uvm) * st[2];
            double drift = 0.0;
            if (f[0]) drift += f[0][id] * uc;
            if (f[1]) drift += f[1][id] * dxu;
            if (f[2]) drift += f[2][id] * dvu;
            if (f[3]) {
                const double dxxu = (uxp - 2.0 * uc + uxm) * st[1];
                drift += 0.5 * f[3][id] * dxxu;
            }
            if (f[4]) {
                const double upp = (cp && i + 1 < nx) ? cp[i + 1] : 0.0;
                const double upm = (cp && i > 0) ? cp[i - 1] : 0.0;
                const double ump = (cm && i + 1 < nx) ? cm[i + 1] : 0.0;
                const double umm = (cm && i > 0) ? cm[i - 1] : 0.0;
                const double dxvu = (upp - upm - ump + umm) * st[4];
                drift += f[4][id] * dxvu;
            }
            if (f[5]) {
                const double dvvu = (uvp - 2.0 * uc + uvm) * st[3];
                drift += 0.5 * f[5][id] * dvvu;
            }
            double noise = 0.0;
            if (f[6]) noise += f[6][id] * uc;
            if (f[7]) noise += f[7][id] * dxu;
            if (f[8]) noise += f[8][id] * dvu;
            const double nxt = uc + drift * dt + noise * dW;
            o[i] = nxt;
            const double a = fabs(nxt);
            maxabs = maxabs < a ? a : maxabs;
        }
    }
    return maxabs;
}

/* euler.cpp:95-182 solve_euler for ONE path. */
void rs_euler_path(size_t nx, size_t nv, const double *const *f, const double st[5],
                   const double *phi, const double *path, size_t step_leb, size_t total_steps,
                   double dt, const size_t *record_steps, size_t nrec, double *states_out,
                   uint8_t *status_out) {
    const size_t n = nx * nv;
    double *cur = (double *)malloc(n * sizeof(double));
    double *nxt = (double *)malloc(n * sizeof(double));
    memcpy(cur, phi, n * sizeof(double));
    for (size_t r = 0; r < nrec; ++r) status_out[r] = 1;
    size_t rec = 0;
    int blown = 0;
    const size_t nsteps = total_steps / step_leb;
    for (size_t k = 0; k < nsteps; ++k) {
        const double dW = path[(k + 1) * step_leb] - path[k * step_leb];
        const double norm = rs_euler_step(nx, nv, f, st, cur, nxt, dW, dt);
        double *tmp = cur; cur = nxt; nxt = tmp;
        if (!isfinite(norm)) { blown = 1; break; }
        const size_t done = (k + 1) * step_leb;
        while (rec < nrec && record_steps[rec] == done) {
            memcpy(states_out + rec * n, cur, n * sizeof(double));
            status_out[rec] = 0;
            ++rec;
        }
    }
    if (blown)
        for (size_t r = rec; r < nrec; ++r) status_out[r] = 1;
    free(cur); free(nxt);
}

/* exact_langevin.cpp:47-75 closed-form field; xn/vn are the grid nodes a+(i+1)delta. */
void rs_exact_field(size_t nx, size_t nv, const double *xn, const double *vn, double t, double a,
                    double sigma, double W, double IW, double *out) {
    const double gap = a - sigma * sigma;
    const double c2 = 2.0 / gap;
    const double t2 = t * t;
    const double t3 = t2 * t;
    const double qa = 3.0 * c2 / t3 + 0.5;
    const double qb = c2 / t + 0.5;
    const double qc = 3.0 * c2 / t2;
    const double det = 4.0 * qa * qb - qc * qc;
    const double sqrt3 = 1.7320508075688772, pi = 3.141592653589793;
    const double pref = sqrt3 / (pi * t2 * gap) * 2.0 * pi / sqrt(det);
    for (size_t j = 0; j < nv; ++j) {
        const double beta = vn[j] + sigma * W;
        for (size_t i = 0; i < nx; ++i) {
            const double alpha = xn[i] + sigma * IW;
            const double qd = 3.0 * c2 * beta / t2 - 6.0 * c2 * alpha / t3;
            const double qe = c2 * beta / t - 3.0 * c2 * alpha / t2;
            const double qf = c2 * (beta * beta / t - 3.0 * alpha * beta / t2 + 3.0 * alpha * alpha / t3);
            out[j * nx + i] = pref * exp((qb * qd * qd + qa * qe * qe - qc * qd * qe) / det - qf);
        }
    }
}

/* analysis.cpp:9-31 central_region (0 ok, 1 ConfigError). */
int rs_central_region(size_t d, int kappa, size_t *lo, size_t *hi) {
    if (d < 2 || kappa < 0) return 1;
    if (kappa >= 63 || ((size_t)1 << kappa) > d) return 1;
    const double half = (double)d / 2.0;
    const double width = (double)d / pow(2.0, kappa + 1);
    const int64_t lo1 = (int64_t)floor(half - width);
    const int64_t hi1 = (int64_t)floor(half + width);
    *lo = (size_t)(lo1 - 1 > 0 ? lo1 - 1 : 0);
    *hi = (size_t)(hi1 - 1 < (int64_t)d - 1 ? hi1 - 1 : (int64_t)d - 1);
    return *hi < *lo ? 1 : 0;
}

/* analysis.cpp:93-130 mean_rel_error and :53-91 mean_abs_error / avg.  States [M][n]
 * column-major (nx rows); status 0 Ok.  me_out (nullable) w*w in Field order.
 * Returns 0, or 1 when the reference blew up / has zero norm (ConfigError). */
int rs_errors(size_t nx, size_t lo, size_t hi, const double *ref, const uint8_t *ref_status,
              const double *app, const uint8_t *app_status, size_t M, double *err,
              size_t *blowups, double *ame, size_t *excluded, double *me_out) {
    const size_t n = nx * nx, w = hi - lo + 1;
    double sum = 0.0;
    *blowups = 0;
    for (size_t m = 0; m < M; ++m) {
        if (ref_status && ref_status[m] != 0) return 1;
        if (app_status && app_status[m] != 0) { ++*blowups; continue; }
        const double *rs = ref + m * n, *as = app + m * n;
        double num = 0.0, den = 0.0;
        for (size_t j = lo; j <= hi; ++j)
            for (size_t i = lo; i <= hi; ++i) {
                const double r = rs[j * nx + i];
                const double d = r - as[j * nx + i];
                num += d * d;
                den += r * r;
            }
        if (den == 0.0) return 1;
        sum += sqrt(num) / sqrt(den);
    }
    *err = *blowups > 0 ? INFINITY : sum / (double)M;
    double *me = (double *)calloc(w * w, sizeof(double));
    size_t used = 0;
    *excluded = 0;
    for (size_t m = 0; m < M; ++m) {
        if (app_status && app_status[m] != 0) { ++*excluded; continue; }
        ++used;
        const double *rs = ref + m * n, *as = app + m * n;
        for (size_t j = 0; j < w; ++j)
            for (size_t i = 0; i < w; ++i) {
                const size_t idx = (lo + j) * nx + lo + i;
                me[j * w + i] += fabs(rs[idx] - as[idx]);
            }
    }
    if (used > 0) {
        const double inv = 1.0 / (double)used;
        for (size_t k = 0; k < w * w; ++k) me[k] *= inv;
    }
    double s = 0.0;
    for (size_t k = 0; k < w * w; ++k) s += me[k];
    *ame = s / (double)(w * w);
    if (me_out) memcpy(me_out, me, w * w * sizeof(double));
    free(me);
    return 0;
}
