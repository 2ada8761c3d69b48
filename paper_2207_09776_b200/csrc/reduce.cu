// Closed-form reference and error norms on the GPU.
//
// exact_reference (src/exact_langevin.cpp:77-95) evaluates exact_langevin_field
// (:47-75) per path with (W, IW) of the window [0, t] taken by the same
// left-Riemann rule the solvers use.  The scalar constants (qa, qb, qc, det,
// pref) are formed on the host exactly as the reference forms them; the per-point
// expression is evaluated in the same operation order.  Only exp() differs
// (CUDA's vs glibc's, <= 1 ulp), so reference fields agree to ~1e-16 relative.
//
// The norms (src/analysis.cpp:53-130) keep the reference's summation order so
// that, given identical ensembles, they are bitwise the reference's:
// per path the region is swept j-major then i (num, den sequential), the per-path
// ratios are summed in ascending m; the ME matrix sums |ref-app| over ascending m
// per entry, then scales by 1/used; AME sums the ME entries in storage order.
// s2b_exact_errors fuses the reference field into those loops, so no reference
// ensemble is ever materialised, and also emits the moment sums (sum u, sum u^2)
// that the multi-GPU path all-reduces.
#include <cmath>
#include <numbers>

#include "s2b_internal.cuh"

namespace s2b {

namespace {

struct ExactParams {
    double t, t2, t3, c2, qa, qb, qc, det, pref, sigma;
    double ax, dx, av, dv;
    int nx, nv;
};

ExactParams exact_params(const s2b_grid& g, double t, double a, double sigma) {
    const double gap = a - sigma * sigma;
    if (!(a > 0.0) || sigma < 0.0 || !(gap > 0.0))
        fail(S2B_ERR_CONFIG, "exact Langevin solution needs a > 0 and a - sigma^2 > 0");
    if (!(t > 0.0)) fail(S2B_ERR_CONFIG, "exact_langevin_field: t must be positive");
    ExactParams p{};
    p.c2 = 2.0 / gap;
    p.t = t;
    p.t2 = t * t;
    p.t3 = p.t2 * t;
    p.qa = 3.0 * p.c2 / p.t3 + 0.5;
    p.qb = p.c2 / t + 0.5;
    p.qc = 3.0 * p.c2 / p.t2;
    p.det = 4.0 * p.qa * p.qb - p.qc * p.qc;
    p.pref = std::numbers::sqrt3 / (std::numbers::pi * p.t2 * gap) * 2.0 * std::numbers::pi / std::sqrt(p.det);
    p.sigma = sigma;
    p.ax = g.ax;
    p.av = g.av;
    p.dx = (g.bx - g.ax) / static_cast<double>(g.nx + 1);
    p.dv = (g.bv - g.av) / static_cast<double>(g.nv + 1);
    p.nx = static_cast<int>(g.nx);
    p.nv = static_cast<int>(g.nv);
    return p;
}

__device__ __forceinline__ double exact_value(const ExactParams& p, double W, double IW, int i, int j) {
    const double beta = (p.av + static_cast<double>(j + 1) * p.dv) + p.sigma * W;
    const double alpha = (p.ax + static_cast<double>(i + 1) * p.dx) + p.sigma * IW;
    const double qd = 3.0 * p.c2 * beta / p.t2 - 6.0 * p.c2 * alpha / p.t3;
    const double qe = p.c2 * beta / p.t - 3.0 * p.c2 * alpha / p.t2;
    const double qf = p.c2 * (beta * beta / p.t - 3.0 * alpha * beta / p.t2 + 3.0 * alpha * alpha / p.t3);
    return p.pref * exp((p.qb * qd * qd + p.qa * qe * qe - p.qc * qd * qe) / p.det - qf);
}

// (W, IW) over [0, k1] per path: lebesgue_functionals (stochastics.cpp:121-141).
__global__ void path_w_iw_kernel(const double* values, size_t stride, size_t k1, double dt, size_t M,
                                 double2* out) {
    const size_t m = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (m >= M) return;
    const double* p = values + m * stride;
    const double base = p[0];
    double iw = 0.0;
    for (size_t j = 0; j < k1; ++j) iw += p[j] - base;
    out[m] = make_double2(p[k1] - p[0], iw * dt);
}

__global__ void exact_field_kernel(ExactParams p, const double2* wiw, double* out, size_t M) {
    const size_t n = static_cast<size_t>(p.nx) * p.nv;
    for (size_t m = blockIdx.y; m < M; m += gridDim.y) {
        const double2 f = wiw[m];
        for (size_t r = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; r < n;
             r += static_cast<size_t>(gridDim.x) * blockDim.x) {
            const int i = static_cast<int>(r % p.nx), j = static_cast<int>(r / p.nx);
            out[m * n + r] = exact_value(p, f.x, f.y, i, j);
        }
    }
}

// Per path: ||ref-app||_F / ||ref||_F on the region; NaN for blown app paths,
// -1 flags a zero reference norm.  ref == nullptr: exact field from wiw.
__global__ void rel_kernel(const double* ref, const double2* wiw, ExactParams p, const double* app,
                           const uint8_t* app_status, size_t M, size_t n, int nx, int lo, int hi,
                           double* rel) {
    const size_t m = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (m >= M) return;
    if (app_status[m]) {
        rel[m] = __longlong_as_double(0x7FF8000000000000LL);
        return;
    }
    const double* a = app + m * n;
    double num = 0.0, den = 0.0;
    for (int j = lo; j <= hi; ++j)
        for (int i = lo; i <= hi; ++i) {
            const size_t idx = static_cast<size_t>(j) * nx + i;
            const double r = ref ? ref[m * n + idx] : exact_value(p, wiw[m].x, wiw[m].y, i, j);
            const double d = r - a[idx];
            num += d * d;
            den += r * r;
        }
    rel[m] = den == 0.0 ? -1.0 : sqrt(num) / sqrt(den);
}

// ME entry (i, j) of the region: sum over ascending m of |ref - app| (non-blown), * 1/used.
__global__ void me_kernel(const double* ref, const double2* wiw, ExactParams p, const double* app,
                          const uint8_t* app_status, size_t M, size_t n, int nx, int lo, int w,
                          size_t used, double* me) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= w * w) return;
    const int i = q % w, j = q / w;
    const size_t idx = static_cast<size_t>(lo + j) * nx + lo + i;
    double s = 0.0;
    for (size_t m = 0; m < M; ++m) {
        if (app_status[m]) continue;
        const double r = ref ? ref[m * n + idx] : exact_value(p, wiw[m].x, wiw[m].y, lo + i, lo + j);
        s += fabs(r - app[m * n + idx]);
    }
    if (used > 0) s *= 1.0 / static_cast<double>(used);
    me[q] = s;
}

// Sequential finishing sums (single thread: ascending order).
__global__ void finish_kernel(const double* rel, size_t M, const double* me, int ww, double* out) {
    double sum = 0.0;
    size_t blow = 0, used = 0, zero = 0;
    for (size_t m = 0; m < M; ++m) {
        const double r = rel[m];
        if (r != r) {
            ++blow;
            continue;
        }
        if (r < 0.0) ++zero;
        ++used;
        sum += r;
    }
    double ame = 0.0;
    for (int q = 0; q < ww; ++q) ame += me[q];
    out[0] = sum;
    out[1] = static_cast<double>(blow);
    out[2] = static_cast<double>(used);
    out[3] = static_cast<double>(zero);
    out[4] = ww > 0 ? ame / static_cast<double>(ww) : 0.0;
}

__global__ void moments_kernel(const double* app, const uint8_t* st, size_t M, size_t n, double* mom) {
    const size_t r = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (r >= n) return;
    double s1 = 0.0, s2 = 0.0;
    for (size_t m = 0; m < M; ++m) {
        if (st[m]) continue;
        const double u = app[m * n + r];
        s1 += u;
        s2 += u * u;
    }
    mom[r] = s1;
    mom[n + r] = s2;
}

} // namespace

void region_of(size_t d, int kappa, size_t* lo, size_t* hi) {
    if (d < 2) fail(S2B_ERR_CONFIG, "central_region: need d >= 2");
    if (kappa < 0) fail(S2B_ERR_CONFIG, "central_region: kappa must be non-negative");
    if (kappa >= 63 || (size_t{1} << kappa) > d) fail(S2B_ERR_CONFIG, "central_region: empty region, kappa too large");
    const double half = static_cast<double>(d) / 2.0;
    const double width = static_cast<double>(d) / std::pow(2.0, kappa + 1);
    const auto lo1 = static_cast<long long>(std::floor(half - width));
    const auto hi1 = static_cast<long long>(std::floor(half + width));
    *lo = static_cast<size_t>(std::max<long long>(lo1 - 1, 0));
    *hi = static_cast<size_t>(std::min<long long>(hi1 - 1, static_cast<long long>(d) - 1));
    if (*hi < *lo) fail(S2B_ERR_CONFIG, "central_region: empty region");
}

namespace {

void run_norms(s2b_context* ctx, const double* ref, const uint8_t* ref_status, const double2* wiw,
               const ExactParams& p, const s2b_ensemble* app, size_t app_record, int kappa,
               s2b_error_stats* out, double* me_out, double* per_path_rel, double* moments) {
    const size_t M = app->M, nx = app->nx, n = app->nx * app->nv;
    size_t lo, hi;
    region_of(nx, kappa, &lo, &hi); // n_x of the reference grid (analysis.cpp:56,96)
    if (hi >= app->nx || hi >= app->nv) fail(S2B_ERR_DIMENSION, "error norms: region exceeds the grid");
    if (ref_status) {
        std::vector<uint8_t> rs(M);
        S2B_CUDA(cudaMemcpy(rs.data(), ref_status, M, cudaMemcpyDeviceToHost));
        for (uint8_t v : rs)
            if (v) fail(S2B_ERR_CONFIG, "mean_rel_error: reference trajectory blew up");
    }
    const double* a = app->states[app_record].p;
    const uint8_t* ast = app->status.p + app_record * M;
    const int w = static_cast<int>(hi - lo + 1);
    DevBuf<double> rel(M), me(static_cast<size_t>(w) * w), fin(5);
    rel_kernel<<<static_cast<unsigned>((M + 127) / 128), 128, 0, ctx->stream>>>(
        ref, wiw, p, a, ast, M, n, static_cast<int>(nx), static_cast<int>(lo), static_cast<int>(hi), rel.p);
    S2B_LAUNCHED(ctx);
    // used count for ME
    std::vector<uint8_t> hs(M);
    S2B_CUDA(cudaMemcpyAsync(hs.data(), ast, M, cudaMemcpyDeviceToHost, ctx->stream));
    S2B_CUDA(cudaStreamSynchronize(ctx->stream));
    size_t used = 0;
    for (uint8_t v : hs) used += v == 0;
    me_kernel<<<static_cast<unsigned>((w * w + 127) / 128), 128, 0, ctx->stream>>>(
        ref, wiw, p, a, ast, M, n, static_cast<int>(nx), static_cast<int>(lo), w, used, me.p);
    S2B_LAUNCHED(ctx);
    finish_kernel<<<1, 1, 0, ctx->stream>>>(rel.p, M, me.p, w * w, fin.p);
    S2B_LAUNCHED(ctx);
    if (moments) {
        DevBuf<double> mom(2 * n);
        moments_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, ctx->stream>>>(a, ast, M, n, mom.p);
        S2B_LAUNCHED(ctx);
        S2B_CUDA(cudaMemcpyAsync(moments, mom.p, mom.bytes(), cudaMemcpyDeviceToHost, ctx->stream));
        S2B_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    double h[5];
    S2B_CUDA(cudaMemcpyAsync(h, fin.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    if (me_out) S2B_CUDA(cudaMemcpyAsync(me_out, me.p, me.bytes(), cudaMemcpyDeviceToHost, ctx->stream));
    if (per_path_rel) S2B_CUDA(cudaMemcpyAsync(per_path_rel, rel.p, rel.bytes(), cudaMemcpyDeviceToHost, ctx->stream));
    S2B_CUDA(cudaStreamSynchronize(ctx->stream));
    if (h[3] > 0) fail(S2B_ERR_CONFIG, "mean_rel_error: reference Frobenius norm is zero");
    out->sum_rel = h[0];
    out->blowups = static_cast<size_t>(h[1]);
    out->used = static_cast<size_t>(h[2]);
    out->excluded = out->blowups;
    out->err = out->blowups > 0 ? INFINITY : h[0] / static_cast<double>(M);
    out->ame = h[4];
    out->region_lo = lo;
    out->region_hi = hi;
}

} // namespace

s2b_ensemble* exact_reference(s2b_context* ctx, const s2b_grid* grid, double t, double a, double sigma,
                              const s2b_paths* paths) {
    const ExactParams p = exact_params(*grid, t, a, sigma);
    const size_t k1 = index_of(t, paths->dt_leb, paths->steps);
    if (k1 == 0) fail(S2B_ERR_CONFIG, "window: need t0 < t1 on the grid");
    const size_t M = paths->M, n = grid->nx * grid->nv;
    auto* e = new s2b_ensemble();
    e->ctx = ctx;
    e->R = 1;
    e->M = M;
    e->nx = grid->nx;
    e->nv = grid->nv;
    e->seed = paths->seed;
    e->grid = *grid;
    e->times.push_back(t);
    e->states.emplace_back(M * n);
    e->status.alloc(M);
    S2B_CUDA(cudaMemsetAsync(e->status.p, 0, M, ctx->stream));
    DevBuf<double2> wiw(M);
    path_w_iw_kernel<<<static_cast<unsigned>((M + 127) / 128), 128, 0, ctx->stream>>>(
        paths->d_values.p, paths->steps + 1, k1, paths->dt_leb, M, wiw.p);
    S2B_LAUNCHED(ctx);
    dim3 g(static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 256)), static_cast<unsigned>(std::min<size_t>(M, 65535)));
    exact_field_kernel<<<g, 256, 0, ctx->stream>>>(p, wiw.p, e->states[0].p, M);
    S2B_LAUNCHED(ctx);
    S2B_CUDA(cudaStreamSynchronize(ctx->stream));
    return e;
}

void exact_field(s2b_context* ctx, const s2b_grid* grid, double t, double a, double sigma, double W, double IW,
                 double* host_out) {
    const ExactParams p = exact_params(*grid, t, a, sigma);
    const size_t n = grid->nx * grid->nv;
    DevBuf<double2> wiw(1);
    DevBuf<double> out(n);
    const double2 h = make_double2(W, IW);
    S2B_CUDA(cudaMemcpyAsync(wiw.p, &h, sizeof(h), cudaMemcpyHostToDevice, ctx->stream));
    exact_field_kernel<<<static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 1024)), 256, 0, ctx->stream>>>(
        p, wiw.p, out.p, 1);
    S2B_LAUNCHED(ctx);
    S2B_CUDA(cudaMemcpyAsync(host_out, out.p, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    S2B_CUDA(cudaStreamSynchronize(ctx->stream));
}

void errors(s2b_context* ctx, const s2b_ensemble* ref, size_t ref_record, const s2b_ensemble* app,
            size_t app_record, int kappa, s2b_error_stats* out, double* me_out) {
    if (ref->nx != app->nx || ref->nv != app->nv) fail(S2B_ERR_DIMENSION, "error norms: grids differ");
    if (ref->M != app->M) fail(S2B_ERR_DIMENSION, "error norms: trajectory counts differ");
    if (ref->seed != app->seed) fail(S2B_ERR_CONFIG, "error norms: ensembles were built from different seeds");
    if (ref_record >= ref->R || app_record >= app->R) fail(S2B_ERR_DIMENSION, "error norms: record out of range");
    ExactParams dummy{};
    run_norms(ctx, ref->states[ref_record].p, ref->status.p + ref_record * ref->M, nullptr, dummy, app,
              app_record, kappa, out, me_out, nullptr, nullptr);
}

void exact_errors(s2b_context* ctx, const s2b_ensemble* app, size_t app_record, double a, double sigma,
                  const s2b_paths* paths, int kappa, s2b_error_stats* out, double* me_out,
                  double* per_path_rel, double* moments) {
    const s2b_grid* grid = &app->grid;
    if (app_record >= app->R) fail(S2B_ERR_DIMENSION, "error norms: record out of range");
    if (paths->M != app->M) fail(S2B_ERR_DIMENSION, "error norms: trajectory counts differ");
    if (paths->seed != app->seed) fail(S2B_ERR_CONFIG, "error norms: ensembles were built from different seeds");
    if (grid->nx != app->nx || grid->nv != app->nv) fail(S2B_ERR_DIMENSION, "error norms: grids differ");
    const double t = app->times[app_record];
    const ExactParams p = exact_params(*grid, t, a, sigma);
    const size_t k1 = index_of(t, paths->dt_leb, paths->steps);
    DevBuf<double2> wiw(app->M);
    path_w_iw_kernel<<<static_cast<unsigned>((app->M + 127) / 128), 128, 0, ctx->stream>>>(
        paths->d_values.p, paths->steps + 1, k1, paths->dt_leb, app->M, wiw.p);
    S2B_LAUNCHED(ctx);
    run_norms(ctx, nullptr, nullptr, wiw.p, p, app, app_record, kappa, out, me_out, per_path_rel, moments);
}

// sum_m u_m and sum_m u_m^2 over the non-blown paths of one record (ascending m per point)
void ensemble_moments(const s2b_ensemble* e, size_t record, double* host_moments, size_t* live) {
    if (record >= e->R) fail(S2B_ERR_DIMENSION, "ensemble moments: record out of range");
    s2b_context* ctx = e->ctx;
    const size_t M = e->M, n = e->nx * e->nv;
    const uint8_t* st = e->status.p + record * M;
    DevBuf<double> mom(2 * n);
    moments_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, ctx->stream>>>(e->states[record].p, st, M, n, mom.p);
    S2B_LAUNCHED(ctx);
    S2B_CUDA(cudaMemcpyAsync(host_moments, mom.p, mom.bytes(), cudaMemcpyDeviceToHost, ctx->stream));
    std::vector<uint8_t> hs(M);
    S2B_CUDA(cudaMemcpyAsync(hs.data(), st, M, cudaMemcpyDeviceToHost, ctx->stream));
    S2B_CUDA(cudaStreamSynchronize(ctx->stream));
    if (live) {
        size_t k = 0;
        for (uint8_t v : hs) k += v == 0;
        *live = k;
    }
}

} // namespace s2b
