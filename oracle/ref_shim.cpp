// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A flat extern "C" shim over the UNMODIFIED reference library (spde2d, built
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It lets
// the Python parity tests, the golden-fixture generator and bench.py's
// cpu_baseline / --impl reference legs call the reference's own public API:
//   operators   proj/include/spde2d/operators.hpp:60-88
//   stochastics proj/include/spde2d/stochastics.hpp:45-73
//   magnus      proj/include/spde2d/magnus.hpp:49-108
//   euler       proj/include/spde2d/euler.hpp:18-49
//   exact       proj/include/spde2d/exact_langevin.hpp:33-46
//   analysis    proj/include/spde2d/analysis.hpp:28-50
//   expmv       proj/include/spde2d/sparse.hpp:143-155
// Every entry point returns 0 on success or an error code
// (1 ConfigError, 2 DimensionError, 3 ExpmvError, 4 other) with the message
// available from ref_last_error().
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "spde2d/analysis.hpp"
#include "spde2d/euler.hpp"
#include "spde2d/exact_langevin.hpp"
#include "spde2d/magnus.hpp"
#include "spde2d/operators.hpp"
#include "spde2d/sparse.hpp"
#include "spde2d/stochastics.hpp"

using namespace spde2d;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 1;
    } catch (const DimensionError& e) {
        g_err = e.what();
        return 2;
    } catch (const ExpmvError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

struct OpsHandle {
    GridSpec grid;
    CoefficientFields fields;
    CommutatorSet comms;
};

const SparseMatrix* slot_of(const OpsHandle& h, int slot) {
    switch (slot) {
    case 0: return &h.comms.B;
    case 1: return &h.comms.A;
    case 2: return &h.comms.A2;
    case 3: return &h.comms.BA;
    case 4: return &h.comms.BAA;
    case 5: return &h.comms.BAB;
    default: return nullptr;
    }
}

Field* field_of(CoefficientFields& f, int which) {
    Field* all[] = {&f.h, &f.fx, &f.fv, &f.gxx, &f.gxv, &f.gvv, &f.sig, &f.sigx, &f.sigv};
    return (which >= 0 && which < 9) ? all[which] : nullptr;
}

BrownianBatch batch_from(const double* values, std::size_t M, std::size_t steps,
                         double dt_leb, std::uint64_t seed) {
    BrownianBatch b;
    b.T = static_cast<double>(steps) * dt_leb;
    b.dt_leb = dt_leb;
    b.M = M;
    b.seed = seed;
    b.steps = steps;
    b.values.resize(M);
    b.increments.resize(M);
    for (std::size_t m = 0; m < M; ++m) {
        const double* p = values + m * (steps + 1);
        b.values[m].assign(p, p + steps + 1);
        b.increments[m].resize(steps);
        for (std::size_t k = 0; k < steps; ++k) b.increments[m][k] = p[k + 1] - p[k];
    }
    return b;
}

void export_ensembles(const std::vector<SolutionEnsemble>& out, std::size_t M, std::size_t n,
                      double* states, std::uint8_t* status, double* seconds) {
    for (std::size_t r = 0; r < out.size(); ++r) {
        for (std::size_t m = 0; m < M; ++m) {
            const bool ok = out[r].status[m] == TrajectoryStatus::Ok;
            if (status) status[r * M + m] = ok ? 0 : 1;
            if (states) {
                double* dst = states + (r * M + m) * n;
                if (ok) {
                    std::memcpy(dst, out[r].states[m].data(), n * sizeof(double));
                } else {
                    for (std::size_t i = 0; i < n; ++i) dst[i] = std::nan("");
                }
            }
        }
    }
    if (seconds && !out.empty()) {
        for (std::size_t m = 0; m < M; ++m) seconds[m] = out[0].seconds[m];
    }
}

SolutionEnsemble ensemble_from(const GridSpec& grid, double t, std::uint64_t seed,
                               const double* states, const std::uint8_t* status,
                               std::size_t M) {
    SolutionEnsemble e;
    e.grid = grid;
    e.t = t;
    e.seed = seed;
    const std::size_t n = grid.dim();
    e.states.resize(M);
    e.status.resize(M);
    e.seconds.assign(M, 0.0);
    for (std::size_t m = 0; m < M; ++m) {
        const bool ok = status == nullptr || status[m] == 0;
        e.status[m] = ok ? TrajectoryStatus::Ok : TrajectoryStatus::BlownUp;
        if (ok) e.states[m].assign(states + m * n, states + (m + 1) * n);
    }
    return e;
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_max_threads() {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

// family: 0 langevin-constant, 1 langevin-variable, 2 explicit fields
// (fields9[k] == nullptr means identically zero; order h fx fv gxx gxv gvv sig sigx sigv).
int ref_ops_create(int family, double a, double sigma, std::size_t nx, std::size_t nv,
                   double ax, double bx, double av, double bv, int order,
                   const double* const* fields9, void** out) {
    return guarded([&] {
        auto h = std::make_unique<OpsHandle>();
        h->grid = GridSpec{build_grid(ax, bx, nx), build_grid(av, bv, nv)};
        if (family == 0) {
            h->fields = sample_coefficients(CoefficientFamily::langevin_constant(a, sigma), h->grid);
        } else if (family == 1) {
            h->fields = sample_coefficients(CoefficientFamily::langevin_variable(a, sigma), h->grid);
        } else {
            h->fields = sample_coefficients(CoefficientFamily::custom({}), h->grid);
            for (int k = 0; k < 9; ++k) {
                if (fields9 && fields9[k]) {
                    Field* f = field_of(h->fields, k);
                    std::memcpy(f->data().data(), fields9[k], nx * nv * sizeof(double));
                }
            }
            h->fields.refresh_zero_flags();
        }
        const SparseMatrix A = assemble_diffusion(h->fields, h->grid);
        const SparseMatrix B = assemble_drift(h->fields, h->grid);
        h->comms = precompute_commutators(A, B, order);
        *out = h.release();
    });
}

void ref_ops_destroy(void* h) { delete static_cast<OpsHandle*>(h); }

int ref_ops_csr(void* hv, int slot, std::size_t* rows, std::size_t* nnz,
                const std::size_t** rp, const std::int32_t** ci, const double** v) {
    return guarded([&] {
        auto* h = static_cast<OpsHandle*>(hv);
        const SparseMatrix* m = slot_of(*h, slot);
        if (!m) throw ConfigError("bad slot");
        *rows = m->rows();
        *nnz = m->nnz();
        *rp = m->row_ptr().data();
        *ci = m->col_idx().data();
        *v = m->values().data();
    });
}

int ref_ops_field(void* hv, int which, const double** data, int* is_zero) {
    return guarded([&] {
        auto* h = static_cast<OpsHandle*>(hv);
        Field* f = field_of(h->fields, which);
        if (!f) throw ConfigError("bad field");
        *data = f->data().data();
        const bool flags[9] = {h->fields.zero_h,   h->fields.zero_fx,  h->fields.zero_fv,
                               h->fields.zero_gxx, h->fields.zero_gxv, h->fields.zero_gvv,
                               h->fields.zero_sig, h->fields.zero_sigx, h->fields.zero_sigv};
        *is_zero = flags[which] ? 1 : 0;
    });
}

int ref_ops_diagonals(void* hv, int slot, std::size_t* ndiag) {
    return guarded([&] {
        auto* h = static_cast<OpsHandle*>(hv);
        *ndiag = slot_of(*h, slot)->nonzero_diagonals();
    });
}

int ref_gaussian_datum(void* hv, double* out) {
    return guarded([&] {
        auto* h = static_cast<OpsHandle*>(hv);
        const Field f = gaussian_datum(h->grid);
        std::memcpy(out, f.data().data(), f.size() * sizeof(double));
    });
}

int ref_node(void* hv, int axis, std::size_t i, double* out) {
    return guarded([&] {
        auto* h = static_cast<OpsHandle*>(hv);
        *out = axis == 0 ? h->grid.x.node(i) : h->grid.v.node(i);
    });
}

int ref_simulate_brownian(double T, double dt_leb, std::size_t M, std::uint64_t seed,
                          std::size_t* steps_out, double* values_out, double* inc_out) {
    return guarded([&] {
        const BrownianBatch b = simulate_brownian(T, dt_leb, M, seed);
        *steps_out = b.steps;
        for (std::size_t m = 0; m < M; ++m) {
            if (values_out)
                std::memcpy(values_out + m * (b.steps + 1), b.values[m].data(),
                            (b.steps + 1) * sizeof(double));
            if (inc_out)
                std::memcpy(inc_out + m * b.steps, b.increments[m].data(),
                            b.steps * sizeof(double));
        }
    });
}

int ref_functionals(const double* path, std::size_t len, std::size_t k0, std::size_t k1,
                    double dt_leb, double out5[5]) {
    return guarded([&] {
        std::vector<double> p(path, path + len);
        const ItoFunctionals f = lebesgue_functionals(PathSegment{&p, k0, k1, dt_leb});
        out5[0] = f.h;
        out5[1] = f.W;
        out5[2] = f.IW;
        out5[3] = f.IsW;
        out5[4] = f.IW2;
    });
}

// Union pattern + values of the order-`order` logarithm (MagnusLogBuilder, magnus.hpp:61-86).
// Call once with values == nullptr to get nnz; buffers sized rows+1 / nnz.
int ref_magnus_fill(void* hv, int build_order, int order, const double f5[5], std::size_t* nnz,
                    std::size_t* rp, std::int32_t* ci, double* values) {
    return guarded([&] {
        auto* h = static_cast<OpsHandle*>(hv);
        const MagnusLogBuilder builder(h->comms, build_order);
        *nnz = builder.nnz();
        if (!values) return;
        ItoFunctionals f;
        f.h = f5[0];
        f.W = f5[1];
        f.IW = f5[2];
        f.IsW = f5[3];
        f.IW2 = f5[4];
        std::vector<double> vals;
        builder.fill(order, f, vals);
        const SparseView view = builder.view_with(vals);
        std::memcpy(values, vals.data(), vals.size() * sizeof(double));
        std::memcpy(rp, view.row_ptr.data(), view.row_ptr.size() * sizeof(std::size_t));
        std::memcpy(ci, view.col_idx.data(), view.col_idx.size() * sizeof(std::int32_t));
    });
}

int ref_one_norm(std::size_t n, const std::size_t* rp, const std::int32_t* ci, const double* v,
                 double* out) {
    return guarded([&] {
        const std::size_t nnz = rp[n];
        SparseView view{n, n, {rp, n + 1}, {ci, nnz}, {v, nnz}};
        *out = one_norm(view);
    });
}

// expmv_into (sparse.hpp:149-151). status: 0 Ok, 1 Overflow, 2 ToleranceNotReached.
int ref_expmv(std::size_t n, const std::size_t* rp, const std::int32_t* ci, const double* v,
              const double* x, double tol, double theta, double* y, int* status,
              double* residual, int* segments, int* max_terms) {
    return guarded([&] {
        const std::size_t nnz = rp[n];
        SparseView view{n, n, {rp, n + 1}, {ci, nnz}, {v, nnz}};
        ExpmvWorkspace ws;
        std::vector<double> out;
        const ExpmvReport rep = expmv_into(view, {x, n}, out, tol, theta, ws);
        std::memcpy(y, out.data(), n * sizeof(double));
        *status = static_cast<int>(rep.status);
        *residual = rep.residual;
        *segments = rep.segments;
        *max_terms = rep.max_terms;
    });
}

// solve_iterated_magnus / solve_adaptive_magnus (magnus.hpp:93-108).
// states_out [R][M][n] (blown rows NaN), status_out [R][M] (0 Ok, 1 BlownUp).
int ref_solve_magnus(void* hv, int order, double dt, double tol, double theta, double cap,
                     int threads, int adaptive, double adaptive_tol, double adaptive_shrink,
                     const double* record_times, std::size_t nrec, const double* phi,
                     const double* values, std::size_t M, std::size_t steps, double dt_leb,
                     std::uint64_t seed, double T, std::size_t* nrec_out, double* states_out,
                     std::uint8_t* status_out, double* seconds_out) {
    return guarded([&] {
        auto* h = static_cast<OpsHandle*>(hv);
        MagnusConfig cfg;
        cfg.order = order;
        cfg.dt = dt;
        cfg.expmv_tol = tol;
        cfg.expmv_theta = theta;
        cfg.blowup_norm_cap = cap;
        cfg.threads = threads;
        cfg.adaptive.enabled = adaptive != 0;
        cfg.adaptive.tolerance = adaptive_tol;
        cfg.adaptive.shrink = adaptive_shrink;
        cfg.record_times.assign(record_times, record_times + nrec);
        const BrownianBatch batch = batch_from(values, M, steps, dt_leb, seed);
        const std::size_t n = h->grid.dim();
        const auto out = adaptive ? solve_adaptive_magnus(cfg, h->comms, {phi, n}, batch, T, h->grid)
                                  : solve_iterated_magnus(cfg, h->comms, {phi, n}, batch, T, h->grid);
        *nrec_out = out.size();
        export_ensembles(out, M, n, states_out, status_out, seconds_out);
    });
}

int ref_solve_euler(void* hv, double dt, int threads, const double* record_times,
                    std::size_t nrec, const double* phi, const double* values, std::size_t M,
                    std::size_t steps, double dt_leb, std::uint64_t seed, double T,
                    std::size_t* nrec_out, double* states_out, std::uint8_t* status_out,
                    double* seconds_out) {
    return guarded([&] {
        auto* h = static_cast<OpsHandle*>(hv);
        EulerConfig cfg;
        cfg.dt = dt;
        cfg.threads = threads;
        cfg.record_times.assign(record_times, record_times + nrec);
        const BrownianBatch batch = batch_from(values, M, steps, dt_leb, seed);
        const std::size_t n = h->grid.dim();
        const Field phif = devectorize({phi, n}, h->grid.x.n, h->grid.v.n);
        const auto out = solve_euler(cfg, h->fields, h->grid, phif, batch, T);
        *nrec_out = out.size();
        export_ensembles(out, M, n, states_out, status_out, seconds_out);
    });
}

int ref_euler_step(void* hv, const double* u, double dW, double dt, double* out,
                   double* maxabs) {
    return guarded([&] {
        auto* h = static_cast<OpsHandle*>(hv);
        const std::size_t nx = h->grid.x.n, nv = h->grid.v.n;
        const Field uf = devectorize({u, nx * nv}, nx, nv);
        Field of(nx, nv);
        *maxabs = euler_step_into(h->fields, uf, of, dW, dt, EulerStencils::from_grid(h->grid));
        std::memcpy(out, of.data().data(), nx * nv * sizeof(double));
    });
}

// exact_reference (exact_langevin.hpp:44-46): states_out [M][n].
int ref_exact_reference(void* hv, double t, double a, double sigma, const double* values,
                        std::size_t M, std::size_t steps, double dt_leb, std::uint64_t seed,
                        double* states_out) {
    return guarded([&] {
        auto* h = static_cast<OpsHandle*>(hv);
        const BrownianBatch batch = batch_from(values, M, steps, dt_leb, seed);
        const SolutionEnsemble e = exact_reference(h->grid, t, LangevinParams{a, sigma}, batch);
        const std::size_t n = h->grid.dim();
        for (std::size_t m = 0; m < M; ++m)
            std::memcpy(states_out + m * n, e.states[m].data(), n * sizeof(double));
    });
}

int ref_exact_field(void* hv, double t, double a, double sigma, double W, double IW,
                    double* out) {
    return guarded([&] {
        auto* h = static_cast<OpsHandle*>(hv);
        const Field f = exact_langevin_field(h->grid, t, LangevinParams{a, sigma},
                                             PathFunctionalsForExact{W, IW});
        std::memcpy(out, f.data().data(), f.size() * sizeof(double));
    });
}

int ref_central_region(std::size_t d, int kappa, std::size_t* lo, std::size_t* hi) {
    return guarded([&] {
        const CentralRegion r = central_region(d, kappa);
        *lo = r.lo;
        *hi = r.hi;
    });
}

// mean_rel_error + mean_abs_error + avg_mean_abs_error (analysis.hpp:35-50) on
// ensembles given as [M][n] arrays with status bytes (0 Ok).  me_out is w*w (Field order).
int ref_errors(void* hv, int kappa, const double* ref_states, const std::uint8_t* ref_status,
               const double* app_states, const std::uint8_t* app_status, std::size_t M,
               std::uint64_t seed, double* err, std::size_t* blowups, double* ame,
               std::size_t* excluded, double* me_out) {
    return guarded([&] {
        auto* h = static_cast<OpsHandle*>(hv);
        const SolutionEnsemble r = ensemble_from(h->grid, 1.0, seed, ref_states, ref_status, M);
        const SolutionEnsemble a = ensemble_from(h->grid, 1.0, seed, app_states, app_status, M);
        const CentralRegion region = central_region(h->grid.x.n, kappa);
        const RelError rel = mean_rel_error(r, a, region);
        *err = rel.err;
        *blowups = rel.blowups;
        const MeanAbsError me = mean_abs_error(r, a, region);
        *ame = avg_mean_abs_error(me.me);
        *excluded = me.excluded;
        if (me_out) std::memcpy(me_out, me.me.data().data(), me.me.size() * sizeof(double));
    });
}

} // extern "C"
