// GPU-backed half of the C++ drop-in: the reference's solver, exact-solution and norm
// entry points (magnus.hpp:93-97, euler.hpp:46-49, exact_langevin.hpp:44-46,
// analysis.hpp:35-50, sparse.hpp:153-155) with their exact signatures, implemented on the
// C ABI (spde2d_b200.h).  Host types in, host types out; the data crosses to the GPU once
// per call.  Errors come back as the reference's exception classes; numerical failure is
// the per-path BlownUp status.  There is no CPU fallback: without a usable B200 every call
// throws std::runtime_error.
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <string>

#include "spde2d_b200.h"
#include "spde2d_b200.hpp"

namespace spde2d {

namespace {

void check(int rc) {
    if (rc == S2B_OK) return;
    const std::string msg = s2b_last_error();
    if (rc == S2B_ERR_CONFIG) throw ConfigError(msg);
    if (rc == S2B_ERR_DIMENSION) throw DimensionError(msg);
    throw std::runtime_error(msg);
}

// One context per process (device from S2B_DEVICE, default 0), created on first use.
s2b_context* context() {
    static std::once_flag once;
    static s2b_context* ctx = nullptr;
    std::call_once(once, [] {
        const char* d = std::getenv("S2B_DEVICE");
        check(s2b_context_create(d ? std::atoi(d) : 0, &ctx));
    });
    return ctx;
}

s2b_grid c_grid(const GridSpec& g) { return s2b_grid{g.x.a, g.x.b, g.x.n, g.v.a, g.v.b, g.v.n}; }

s2b_csr c_csr(const SparseMatrix& m) {
    return s2b_csr{m.rows(), m.row_ptr().data(), m.col_idx().data(), m.values().data()};
}

template <class T>
std::unique_ptr<T, int (*)(T*)> own(T* p, int (*d)(T*)) {
    return std::unique_ptr<T, int (*)(T*)>(p, d);
}

std::vector<double> flat_values(const BrownianBatch& b) {
    std::vector<double> v(b.M * (b.steps + 1));
    for (std::size_t m = 0; m < b.M; ++m) {
        if (b.values[m].size() != b.steps + 1) throw DimensionError("BrownianBatch: ragged values");
        std::memcpy(v.data() + m * (b.steps + 1), b.values[m].data(), (b.steps + 1) * sizeof(double));
    }
    return v;
}

s2b_paths* upload_paths(const BrownianBatch& b) {
    const std::vector<double> v = flat_values(b);
    s2b_paths* p = nullptr;
    check(s2b_paths_create_host(context(), b.dt_leb, b.steps, b.M, b.seed, v.data(), &p));
    return p;
}

// Device ensemble -> host SolutionEnsembles (blown paths get an empty state).
std::vector<SolutionEnsemble> download(s2b_ensemble* e, const GridSpec& grid, std::uint64_t seed,
                                       double seconds_per_path) {
    int64_t info[5];
    check(s2b_ensemble_info(e, info, nullptr));
    std::vector<double> times(static_cast<std::size_t>(info[0]));
    check(s2b_ensemble_info(e, info, times.data()));
    const std::size_t R = info[0], M = info[1], n = info[2];
    std::vector<SolutionEnsemble> out(R);
    std::vector<double> states(M * n);
    std::vector<std::uint8_t> status(M);
    for (std::size_t r = 0; r < R; ++r) {
        check(s2b_ensemble_download(e, r, states.data(), status.data()));
        SolutionEnsemble& s = out[r];
        s.grid = grid;
        s.t = times[r];
        s.seed = seed;
        s.states.resize(M);
        s.status.resize(M);
        s.seconds.assign(M, seconds_per_path);
        for (std::size_t m = 0; m < M; ++m) {
            s.status[m] = status[m] ? TrajectoryStatus::BlownUp : TrajectoryStatus::Ok;
            if (!status[m]) s.states[m].assign(states.begin() + m * n, states.begin() + (m + 1) * n);
        }
    }
    return out;
}

s2b_ensemble* upload_ensemble(const SolutionEnsemble& e) {
    const std::size_t M = e.trajectories(), n = e.grid.dim();
    std::vector<double> states(M * n, 0.0);
    std::vector<std::uint8_t> status(M);
    for (std::size_t m = 0; m < M; ++m) {
        status[m] = e.status[m] == TrajectoryStatus::Ok ? 0 : 1;
        if (!status[m]) {
            if (e.states[m].size() != n) throw DimensionError("SolutionEnsemble: state length mismatch");
            std::memcpy(states.data() + m * n, e.states[m].data(), n * sizeof(double));
        }
    }
    const s2b_grid g = c_grid(e.grid);
    s2b_ensemble* out = nullptr;
    check(s2b_ensemble_create_host(context(), &g, e.t, e.seed, M, states.data(), status.data(), &out));
    return out;
}

double elapsed_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

} // namespace

std::vector<SolutionEnsemble> solve_iterated_magnus(const MagnusConfig& cfg, const CommutatorSet& comms,
                                                    std::span<const double> phi, const BrownianBatch& batch,
                                                    double T, const GridSpec& grid) {
    if (cfg.order < 1 || cfg.order > 3 || cfg.order > comms.order)
        throw ConfigError("solve_iterated_magnus: unsupported order");
    if (phi.size() != grid.dim() || comms.B.rows() != grid.dim())
        throw DimensionError("solve_iterated_magnus: dimension mismatch");
    const auto t0 = std::chrono::steady_clock::now();
    const s2b_grid g = c_grid(grid);
    const SparseMatrix empty;
    // the operator is laid out for exactly the requested order (MagnusLogBuilder(comms, cfg.order))
    const s2b_csr src[6] = {c_csr(comms.B), c_csr(comms.A),
                            cfg.order >= 2 ? c_csr(comms.A2) : c_csr(empty),
                            cfg.order >= 2 ? c_csr(comms.BA) : c_csr(empty),
                            cfg.order >= 3 ? c_csr(comms.BAA) : c_csr(empty),
                            cfg.order >= 3 ? c_csr(comms.BAB) : c_csr(empty)};
    s2b_operator* op = nullptr;
    check(s2b_operator_create(context(), &g, cfg.order, src, &op));
    auto op_guard = own(op, s2b_operator_destroy);
    auto paths = own(upload_paths(batch), s2b_paths_destroy);
    const s2b_magnus_config c{cfg.order,       cfg.dt,           T, cfg.expmv_tol, cfg.expmv_theta,
                              cfg.blowup_norm_cap, cfg.record_times.data(), cfg.record_times.size()};
    s2b_ensemble* e = nullptr;
    check(s2b_solve_magnus(context(), op, &c, phi.data(), paths.get(), &e, nullptr));
    auto e_guard = own(e, s2b_ensemble_destroy);
    // per-path wall time is not observable on the GPU: report the mean (CSV uses total/M)
    return download(e, grid, batch.seed, elapsed_since(t0) / static_cast<double>(batch.M));
}

std::vector<SolutionEnsemble> solve_adaptive_magnus(const MagnusConfig& cfg, const CommutatorSet& comms,
                                                    std::span<const double> phi, const BrownianBatch& batch,
                                                    double T, const GridSpec& grid) {
    if (!cfg.adaptive.enabled) throw ConfigError("solve_adaptive_magnus: adaptive flag not set");
    if (!(cfg.adaptive.shrink > 0.0 && cfg.adaptive.shrink < 1.0))
        throw ConfigError("solve_adaptive_magnus: shrink factor must lie in (0, 1)");
    if (comms.order < 3) throw ConfigError("solve_adaptive_magnus: needs order-3 commutators");
    if (phi.size() != grid.dim() || comms.B.rows() != grid.dim())
        throw DimensionError("solve_adaptive_magnus: dimension mismatch");
    const auto t0 = std::chrono::steady_clock::now();
    const s2b_grid g = c_grid(grid);
    // MagnusLogBuilder(comms, 3): the union pattern of all six sources
    const s2b_csr src[6] = {c_csr(comms.B), c_csr(comms.A), c_csr(comms.A2),
                            c_csr(comms.BA), c_csr(comms.BAA), c_csr(comms.BAB)};
    s2b_operator* op = nullptr;
    check(s2b_operator_create(context(), &g, 3, src, &op));
    auto op_guard = own(op, s2b_operator_destroy);
    auto paths = own(upload_paths(batch), s2b_paths_destroy);
    const s2b_magnus_config c{3, cfg.dt, T, cfg.expmv_tol, cfg.expmv_theta, cfg.blowup_norm_cap,
                              cfg.record_times.data(), cfg.record_times.size()};
    const s2b_adaptive_config ad{1, cfg.adaptive.tolerance, cfg.adaptive.shrink};
    s2b_ensemble* e = nullptr;
    check(s2b_solve_adaptive_magnus(context(), op, &c, &ad, phi.data(), paths.get(), &e, nullptr));
    auto e_guard = own(e, s2b_ensemble_destroy);
    return download(e, grid, batch.seed, elapsed_since(t0) / static_cast<double>(batch.M));
}

std::vector<SolutionEnsemble> solve_euler(const EulerConfig& cfg, const CoefficientFields& fields,
                                          const GridSpec& grid, const Field& phi, const BrownianBatch& batch,
                                          double T) {
    if (phi.nx() != grid.x.n || phi.nv() != grid.v.n) throw DimensionError("solve_euler: datum shape mismatch");
    const auto t0 = std::chrono::steady_clock::now();
    const s2b_grid g = c_grid(grid);
    const Field* all[9] = {&fields.h, &fields.fx, &fields.fv, &fields.gxx, &fields.gxv,
                           &fields.gvv, &fields.sig, &fields.sigx, &fields.sigv};
    const bool zero[9] = {fields.zero_h,   fields.zero_fx,  fields.zero_fv,  fields.zero_gxx, fields.zero_gxv,
                          fields.zero_gvv, fields.zero_sig, fields.zero_sigx, fields.zero_sigv};
    const double* f9[9];
    for (int k = 0; k < 9; ++k) {
        if (!zero[k] && (all[k]->nx() != grid.x.n || all[k]->nv() != grid.v.n))
            throw DimensionError("coefficient field shape does not match the grid");
        f9[k] = zero[k] ? nullptr : all[k]->data().data();
    }
    s2b_fields* f = nullptr;
    check(s2b_fields_create(context(), &g, f9, &f));
    auto f_guard = own(f, s2b_fields_destroy);
    auto paths = own(upload_paths(batch), s2b_paths_destroy);
    const s2b_euler_config c{cfg.dt, T, cfg.record_times.data(), cfg.record_times.size()};
    s2b_ensemble* e = nullptr;
    check(s2b_solve_euler(context(), f, &c, phi.data().data(), paths.get(), &e));
    auto e_guard = own(e, s2b_ensemble_destroy);
    return download(e, grid, batch.seed, elapsed_since(t0) / static_cast<double>(batch.M));
}

SolutionEnsemble exact_reference(const GridSpec& grid, double t, const LangevinParams& params,
                                 const BrownianBatch& batch) {
    const auto t0 = std::chrono::steady_clock::now();
    const s2b_grid g = c_grid(grid);
    auto paths = own(upload_paths(batch), s2b_paths_destroy);
    s2b_ensemble* e = nullptr;
    check(s2b_exact_reference(context(), &g, t, params.a, params.sigma, paths.get(), &e));
    auto e_guard = own(e, s2b_ensemble_destroy);
    auto out = download(e, grid, batch.seed, elapsed_since(t0) / static_cast<double>(batch.M));
    return std::move(out.front());
}

namespace {
s2b_error_stats norms(const SolutionEnsemble& ref, const SolutionEnsemble& app, const CentralRegion& region,
                      Field* me) {
    if (ref.grid.x.n != app.grid.x.n || ref.grid.v.n != app.grid.v.n)
        throw DimensionError("error norms: grids differ");
    if (ref.trajectories() != app.trajectories()) throw DimensionError("error norms: trajectory counts differ");
    if (ref.seed != app.seed) throw ConfigError("error norms: ensembles were built from different seeds");
    auto r = own(upload_ensemble(ref), s2b_ensemble_destroy);
    auto a = own(upload_ensemble(app), s2b_ensemble_destroy);
    s2b_error_stats st{};
    const std::size_t w = region.size();
    std::vector<double> buf(w * w);
    check(s2b_errors(context(), r.get(), 0, a.get(), 0, region.kappa, &st, buf.data()));
    if (st.region_lo != region.lo || st.region_hi != region.hi)
        throw ConfigError("error norms: region does not match central_region(d, kappa)");
    if (me) {
        *me = Field(w, w);
        std::memcpy(me->data().data(), buf.data(), buf.size() * sizeof(double));
    }
    return st;
}
} // namespace

MeanAbsError mean_abs_error(const SolutionEnsemble& ref, const SolutionEnsemble& app, const CentralRegion& region) {
    MeanAbsError out;
    const s2b_error_stats st = norms(ref, app, region, &out.me);
    out.excluded = st.excluded;
    return out;
}

RelError mean_rel_error(const SolutionEnsemble& ref, const SolutionEnsemble& app, const CentralRegion& region) {
    const s2b_error_stats st = norms(ref, app, region, nullptr);
    return RelError{st.err, st.blowups};
}

std::vector<double> magnus_step(const SparseMatrix& y, std::span<const double> u, double tol) {
    return expmv(y, u, tol);
}

Field exact_langevin_field(const GridSpec& grid, double t, const LangevinParams& params,
                           const PathFunctionalsForExact& path) {
    const s2b_grid g = c_grid(grid);
    Field f(grid.x.n, grid.v.n);
    check(s2b_exact_field(context(), &g, t, params.a, params.sigma, path.W, path.IW, f.data().data()));
    return f;
}

ExpmvReport expmv_into(const SparseView& m, std::span<const double> x, std::vector<double>& y, double tol,
                       double theta, ExpmvWorkspace& ws) {
    if (m.rows != m.cols) throw DimensionError("expmv: matrix must be square");
    if (x.size() != m.cols) throw DimensionError("expmv: vector length mismatch");
    if (m.row_ptr.size() != m.rows + 1 || m.col_idx.size() != m.values.size() ||
        (m.rows && m.row_ptr[m.rows] != m.values.size()))
        throw DimensionError("expmv: malformed CSR view");
    if (!ws.device) {
        s2b_expmv_workspace* w = nullptr;
        check(s2b_expmv_workspace_create(context(), &w));
        ws.device = std::shared_ptr<s2b_expmv_workspace>(w, [](s2b_expmv_workspace* q) { s2b_expmv_workspace_destroy(q); });
    }
    const s2b_csr c{m.rows, m.row_ptr.data(), m.col_idx.data(), m.values.data()};
    y.resize(x.size());
    s2b_expmv_report r{};
    check(s2b_expmv_into(ws.device.get(), &c, x.data(), tol, theta, y.data(), &r));
    ws.terms = r.terms;
    ExpmvReport out;
    out.status = r.status == 0 ? ExpmvStatus::Ok : (r.status == 1 ? ExpmvStatus::Overflow : ExpmvStatus::ToleranceNotReached);
    out.residual = r.residual;
    out.segments = r.segments;
    out.max_terms = r.max_terms;
    return out;
}

std::vector<double> expmv(const SparseMatrix& m, std::span<const double> v, double tol, double theta) {
    ExpmvWorkspace ws;
    std::vector<double> y;
    const ExpmvReport rep = expmv_into(m.view(), v, y, tol, theta, ws);
    if (rep.status == ExpmvStatus::Overflow)
        throw ExpmvError(rep.status, rep.residual, "expmv: overflow (non-finite intermediate)");
    if (rep.status == ExpmvStatus::ToleranceNotReached)
        throw ExpmvError(rep.status, rep.residual,
                         "expmv: tolerance not reached within term budget, residual " + std::to_string(rep.residual));
    return y;
}

namespace {
// Device copy of the CoefficientFields the last euler_step_into call on this thread used;
// reused while the fields' contents (and shape) are unchanged, compared exactly.
struct StepFields {
    std::vector<double> data; // the non-zero fields, in field order
    int mask = -1;
    std::size_t nx = 0, nv = 0;
    s2b_fields* dev = nullptr;
    ~StepFields() {
        if (dev) s2b_fields_destroy(dev);
    }
};

s2b_fields* step_fields(const CoefficientFields& f, std::size_t nx, std::size_t nv) {
    thread_local StepFields cache;
    const Field* all[9] = {&f.h, &f.fx, &f.fv, &f.gxx, &f.gxv, &f.gvv, &f.sig, &f.sigx, &f.sigv};
    const bool zero[9] = {f.zero_h,   f.zero_fx,  f.zero_fv,  f.zero_gxx, f.zero_gxv,
                          f.zero_gvv, f.zero_sig, f.zero_sigx, f.zero_sigv};
    const std::size_t n = nx * nv;
    int mask = 0;
    for (int k = 0; k < 9; ++k) {
        if (zero[k]) continue;
        if (all[k]->nx() != nx || all[k]->nv() != nv) throw DimensionError("euler_step: coefficient field shape mismatch");
        mask |= 1 << k;
    }
    bool same = cache.dev && cache.mask == mask && cache.nx == nx && cache.nv == nv;
    for (int k = 0, q = 0; k < 9 && same; ++k)
        if (mask >> k & 1) same = std::memcmp(cache.data.data() + n * q++, all[k]->data().data(), n * sizeof(double)) == 0;
    if (same) return cache.dev;
    if (cache.dev) {
        s2b_fields_destroy(cache.dev);
        cache.dev = nullptr;
    }
    cache.data.clear();
    const double* f9[9] = {};
    for (int k = 0; k < 9; ++k)
        if (mask >> k & 1) {
            f9[k] = all[k]->data().data();
            cache.data.insert(cache.data.end(), all[k]->data().begin(), all[k]->data().end());
        }
    // the grid only fixes the shape here: the step takes the caller's stencil scales
    const s2b_grid g{-1.0, 1.0, nx, -1.0, 1.0, nv};
    check(s2b_fields_create(context(), &g, f9, &cache.dev));
    cache.mask = mask;
    cache.nx = nx;
    cache.nv = nv;
    return cache.dev;
}
} // namespace

double euler_step_into(const CoefficientFields& fields, const Field& u, Field& out, double dW, double dt,
                       const EulerStencils& st) {
    const std::size_t nx = u.nx(), nv = u.nv();
    if (out.nx() != nx || out.nv() != nv) throw DimensionError("euler_step: output shape mismatch");
    if (nx * nv == 0) return 0.0;
    s2b_fields* f = step_fields(fields, nx, nv);
    const double s5[5] = {st.inv2dx, st.invdx2, st.inv2dv, st.invdv2, st.inv4dxdv};
    double mx = 0.0;
    check(s2b_euler_step(f, s5, u.data().data(), out.data().data(), dW, dt, &mx));
    return mx;
}

Field euler_step(const CoefficientFields& fields, const Field& u, double dW, double dt, const EulerStencils& st) {
    Field out(u.nx(), u.nv());
    euler_step_into(fields, u, out, dW, dt, st);
    return out;
}

} // namespace spde2d
