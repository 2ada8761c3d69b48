// The C ABI (include/spde2d_b200.h): handle lifetime, argument validation,
// exception -> error-code translation, and the host-side plan_windows rules.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "s2b_internal.cuh"
#include "spde2d_b200.hpp"

namespace s2b {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& what) { g_last_error = what; }

int grid_cap(int grid) {
    const char* e = std::getenv("S2B_GRID_CAP");
    if (!e) return grid;
    const int cap = std::atoi(e);
    return cap > 0 && cap < grid ? cap : grid;
}

namespace {

template <class F>
int guard(F&& f) {
    try {
        f();
        return S2B_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const spde2d::ConfigError& e) {
        g_last_error = e.what();
        return S2B_ERR_CONFIG;
    } catch (const spde2d::DimensionError& e) {
        g_last_error = e.what();
        return S2B_ERR_DIMENSION;
    } catch (const std::bad_alloc&) {
        g_last_error = "out of host memory";
        return S2B_ERR_RUNTIME;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return S2B_ERR_RUNTIME;
    }
}

void need(const void* p, const char* what) {
    if (!p) fail(S2B_ERR_CONFIG, std::string("null argument: ") + what);
}

} // namespace

void after_launch(s2b_context* ctx, const char* file, int line) {
    ctx->launches += 1;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        fail(S2B_ERR_CUDA, std::string("kernel launch failed at ") + file + ":" + std::to_string(line) + ": " +
                               cudaGetErrorString(e));
}

// BrownianBatch::index_of (stochastics.cpp:103-111)
size_t index_of(double t, double dt_leb, size_t steps) {
    const auto k = static_cast<long long>(std::llround(t / dt_leb));
    if (k < 0 || static_cast<size_t>(k) > steps ||
        std::abs(t - static_cast<double>(k) * dt_leb) > 1e-12 * std::max(1.0, std::abs(t)))
        fail(S2B_ERR_CONFIG, "time " + std::to_string(t) + " is not on the Lebesgue grid");
    return static_cast<size_t>(k);
}

// plan_windows (magnus.cpp:174-200); solve_euler uses the same rules (euler.cpp:102-122)
WindowPlan plan_windows(double dt, double T, double dt_leb, size_t steps, const double* record_times,
                        size_t n_record, const char* who) {
    WindowPlan plan;
    plan.total_steps = index_of(T, dt_leb, steps);
    plan.dt_steps = index_of(dt, dt_leb, steps);
    if (plan.dt_steps == 0) fail(S2B_ERR_CONFIG, std::string(who) + ": dt must be at least dt_leb");
    if (plan.total_steps % plan.dt_steps != 0)
        fail(S2B_ERR_CONFIG, std::string(who) + ": T must be an integer multiple of dt");
    if (n_record == 0) {
        plan.record_steps.push_back(plan.total_steps);
    } else {
        for (size_t q = 0; q < n_record; ++q) {
            const size_t k = index_of(record_times[q], dt_leb, steps);
            if (k == 0 || k > plan.total_steps || k % plan.dt_steps != 0)
                fail(S2B_ERR_CONFIG, std::string(who) + ": record time " + std::to_string(record_times[q]) +
                                         " is not a positive multiple of dt within [0, T]");
            plan.record_steps.push_back(k);
        }
        std::sort(plan.record_steps.begin(), plan.record_steps.end());
        if (plan.record_steps.back() != plan.total_steps) plan.record_steps.push_back(plan.total_steps);
    }
    return plan;
}

namespace {

spde2d::GridSpec grid_spec(const s2b_grid* g) {
    return spde2d::GridSpec{spde2d::build_grid(g->ax, g->bx, g->nx), spde2d::build_grid(g->av, g->bv, g->nv)};
}

spde2d::CoefficientFields host_fields(const s2b_grid* grid, int family, double a, double sigma,
                                      const double* const* fields9) {
    const spde2d::GridSpec g = grid_spec(grid);
    if (family == 0) return spde2d::sample_coefficients(spde2d::CoefficientFamily::langevin_constant(a, sigma), g);
    if (family == 1) return spde2d::sample_coefficients(spde2d::CoefficientFamily::langevin_variable(a, sigma), g);
    if (family != 2) fail(S2B_ERR_CONFIG, "unknown coefficient family");
    spde2d::CoefficientFields f = spde2d::sample_coefficients(spde2d::CoefficientFamily::custom({}), g);
    spde2d::Field* all[9] = {&f.h, &f.fx, &f.fv, &f.gxx, &f.gxv, &f.gvv, &f.sig, &f.sigx, &f.sigv};
    for (int k = 0; k < 9; ++k)
        if (fields9 && fields9[k]) std::memcpy(all[k]->data().data(), fields9[k], g.dim() * sizeof(double));
    f.refresh_zero_flags();
    return f;
}

s2b_csr csr_of(const spde2d::SparseMatrix& m) {
    s2b_csr c{};
    c.rows = m.rows();
    c.row_ptr = m.row_ptr().data();
    c.col_idx = m.col_idx().data();
    c.values = m.values().data();
    return c;
}

} // namespace
} // namespace s2b

using namespace s2b;

static MagnusSession* S(s2b_magnus_session* s) { return reinterpret_cast<MagnusSession*>(s); }
static const MagnusSession* S(const s2b_magnus_session* s) { return reinterpret_cast<const MagnusSession*>(s); }

extern "C" {

const char* s2b_last_error(void) { return g_last_error.c_str(); }
const char* s2b_version(void) { return "spde2d_b200 0.1 (sm_100a)"; }

int s2b_context_create(int device, s2b_context** out) {
    return guard([&] {
        need(out, "out");
        int count = 0;
        S2B_CUDA(cudaGetDeviceCount(&count));
        if (device < 0 || device >= count) fail(S2B_ERR_CONFIG, "no such CUDA device");
        S2B_CUDA(cudaSetDevice(device));
        cudaDeviceProp prop{};
        S2B_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10) fail(S2B_ERR_CUDA, std::string("sm_100a build needs a Blackwell B200, found ") + prop.name);
        auto* c = new s2b_context();
        c->device = device;
        c->num_sms = prop.multiProcessorCount;
        S2B_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        *out = c;
    });
}

int s2b_context_destroy(s2b_context* ctx) {
    return guard([&] {
        if (!ctx) return;
        cudaStreamSynchronize(ctx->stream);
        cudaStreamDestroy(ctx->stream);
        delete ctx;
    });
}

int s2b_context_synchronize(s2b_context* ctx) {
    return guard([&] {
        need(ctx, "ctx");
        S2B_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

void* s2b_context_stream(s2b_context* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }
int64_t s2b_context_launches(s2b_context* ctx) { return ctx ? ctx->launches : 0; }

int s2b_operator_create(s2b_context* ctx, const s2b_grid* grid, int order, const s2b_csr sources[6],
                        s2b_operator** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(grid, "grid");
        need(sources, "sources");
        need(out, "out");
        S2B_CUDA(cudaSetDevice(ctx->device));
        *out = make_operator(ctx, grid, order, sources);
    });
}

int s2b_operator_build(s2b_context* ctx, const s2b_grid* grid, int family, double a, double sigma,
                       const double* const* fields9, int order, s2b_operator** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(grid, "grid");
        need(out, "out");
        S2B_CUDA(cudaSetDevice(ctx->device));
        const spde2d::GridSpec g = grid_spec(grid);
        const spde2d::CoefficientFields f = host_fields(grid, family, a, sigma, fields9);
        const spde2d::CommutatorSet cs = spde2d::precompute_commutators(
            spde2d::assemble_diffusion(f, g), spde2d::assemble_drift(f, g), order);
        const s2b_csr src[6] = {csr_of(cs.B), csr_of(cs.A), csr_of(cs.A2), csr_of(cs.BA), csr_of(cs.BAA), csr_of(cs.BAB)};
        *out = make_operator(ctx, grid, order, src);
    });
}

int s2b_operator_info(const s2b_operator* op, int64_t info[6]) {
    return guard([&] {
        need(op, "op");
        operator_info(op, info);
    });
}

int s2b_operator_destroy(s2b_operator* op) {
    return guard([&] { delete op; });
}

int s2b_fields_create(s2b_context* ctx, const s2b_grid* grid, const double* const* fields9, s2b_fields** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(grid, "grid");
        need(out, "out");
        S2B_CUDA(cudaSetDevice(ctx->device));
        *out = make_fields(ctx, grid, fields9);
    });
}

int s2b_fields_build(s2b_context* ctx, const s2b_grid* grid, int family, double a, double sigma, s2b_fields** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(grid, "grid");
        need(out, "out");
        S2B_CUDA(cudaSetDevice(ctx->device));
        const spde2d::CoefficientFields f = host_fields(grid, family, a, sigma, nullptr);
        const double* f9[9] = {f.zero_h ? nullptr : f.h.data().data(),       f.zero_fx ? nullptr : f.fx.data().data(),
                               f.zero_fv ? nullptr : f.fv.data().data(),     f.zero_gxx ? nullptr : f.gxx.data().data(),
                               f.zero_gxv ? nullptr : f.gxv.data().data(),   f.zero_gvv ? nullptr : f.gvv.data().data(),
                               f.zero_sig ? nullptr : f.sig.data().data(),   f.zero_sigx ? nullptr : f.sigx.data().data(),
                               f.zero_sigv ? nullptr : f.sigv.data().data()};
        *out = make_fields(ctx, grid, f9);
    });
}

int s2b_fields_destroy(s2b_fields* f) {
    return guard([&] { delete f; });
}

int s2b_gaussian_datum(const s2b_grid* grid, double* out) {
    return guard([&] {
        need(grid, "grid");
        need(out, "out");
        const spde2d::Field f = spde2d::gaussian_datum(grid_spec(grid));
        std::memcpy(out, f.data().data(), f.size() * sizeof(double));
    });
}

struct s2b_host_ops {
    spde2d::GridSpec grid;
    spde2d::CoefficientFields fields;
    spde2d::CommutatorSet comms;
};

int s2b_host_ops_build(const s2b_grid* grid, int family, double a, double sigma, const double* const* fields9,
                       int order, s2b_host_ops** out) {
    return guard([&] {
        need(grid, "grid");
        need(out, "out");
        auto* h = new s2b_host_ops();
        try {
            h->grid = grid_spec(grid);
            h->fields = host_fields(grid, family, a, sigma, fields9);
            h->comms = spde2d::precompute_commutators(spde2d::assemble_diffusion(h->fields, h->grid),
                                                      spde2d::assemble_drift(h->fields, h->grid), order);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int s2b_host_ops_assemble_device(s2b_context* ctx, const s2b_grid* grid, int family, double a, double sigma,
                                 const double* const* fields9, int order, s2b_host_ops** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(grid, "grid");
        need(out, "out");
        S2B_CUDA(cudaSetDevice(ctx->device));
        auto* h = new s2b_host_ops();
        try {
            h->grid = grid_spec(grid);
            h->fields = host_fields(grid, family, a, sigma, fields9);
            h->comms = device_commutators(ctx, h->grid, h->fields, order);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int s2b_operator_build_device(s2b_context* ctx, const s2b_grid* grid, int family, double a, double sigma,
                              const double* const* fields9, int order, s2b_operator** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(grid, "grid");
        need(out, "out");
        S2B_CUDA(cudaSetDevice(ctx->device));
        const spde2d::GridSpec g = grid_spec(grid);
        const spde2d::CoefficientFields f = host_fields(grid, family, a, sigma, fields9);
        const spde2d::CommutatorSet cs = device_commutators(ctx, g, f, order);
        const s2b_csr src[6] = {csr_of(cs.B), csr_of(cs.A), csr_of(cs.A2), csr_of(cs.BA), csr_of(cs.BAA), csr_of(cs.BAB)};
        *out = make_operator(ctx, grid, order, src);
    });
}

int s2b_host_ops_csr(const s2b_host_ops* h, int slot, s2b_csr* out) {
    return guard([&] {
        need(h, "host_ops");
        need(out, "out");
        const spde2d::SparseMatrix* all[6] = {&h->comms.B, &h->comms.A, &h->comms.A2,
                                              &h->comms.BA, &h->comms.BAA, &h->comms.BAB};
        if (slot < 0 || slot > 5) fail(S2B_ERR_CONFIG, "host_ops: slot out of range");
        *out = csr_of(*all[slot]);
    });
}

int s2b_host_ops_field(const s2b_host_ops* h, int which, const double** data, int* is_zero) {
    return guard([&] {
        need(h, "host_ops");
        const spde2d::CoefficientFields& f = h->fields;
        const spde2d::Field* all[9] = {&f.h, &f.fx, &f.fv, &f.gxx, &f.gxv, &f.gvv, &f.sig, &f.sigx, &f.sigv};
        const bool z[9] = {f.zero_h, f.zero_fx, f.zero_fv, f.zero_gxx, f.zero_gxv, f.zero_gvv,
                           f.zero_sig, f.zero_sigx, f.zero_sigv};
        if (which < 0 || which > 8) fail(S2B_ERR_CONFIG, "host_ops: field out of range");
        *data = all[which]->data().data();
        *is_zero = z[which] ? 1 : 0;
    });
}

int s2b_host_ops_destroy(s2b_host_ops* h) {
    return guard([&] { delete h; });
}

int s2b_host_simulate_brownian(double T, double dt_leb, size_t M, uint64_t seed, double* values_out) {
    return guard([&] {
        need(values_out, "values_out");
        const spde2d::BrownianBatch b = spde2d::simulate_brownian(T, dt_leb, M, seed);
        for (size_t m = 0; m < M; ++m)
            std::memcpy(values_out + m * (b.steps + 1), b.values[m].data(), (b.steps + 1) * sizeof(double));
    });
}

int s2b_paths_create_host(s2b_context* ctx, double dt_leb, size_t steps, size_t M, uint64_t seed,
                          const double* values, s2b_paths** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(values, "values");
        need(out, "out");
        S2B_CUDA(cudaSetDevice(ctx->device));
        *out = make_paths_host(ctx, dt_leb, steps, M, seed, values);
    });
}

int s2b_paths_create_philox(s2b_context* ctx, double dt_leb, size_t steps, size_t M, uint64_t seed,
                            uint64_t path_offset, s2b_paths** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(out, "out");
        S2B_CUDA(cudaSetDevice(ctx->device));
        *out = make_paths_philox(ctx, dt_leb, steps, M, seed, path_offset);
    });
}

int s2b_paths_download(const s2b_paths* p, double* values_out) {
    return guard([&] {
        need(p, "paths");
        need(values_out, "values_out");
        S2B_CUDA(cudaMemcpy(values_out, p->d_values.p, p->d_values.bytes(), cudaMemcpyDeviceToHost));
    });
}

int s2b_paths_upload(s2b_paths* p, size_t k0, size_t k1, const double* values) {
    return guard([&] {
        need(p, "paths");
        need(values, "values");
        if (k1 < k0 || k1 > p->steps) fail(S2B_ERR_DIMENSION, "paths_upload: column range out of bounds");
        const size_t pitch = (p->steps + 1) * sizeof(double);
        S2B_CUDA(cudaMemcpy2DAsync(p->d_values.p + k0, pitch, values + k0, pitch, (k1 - k0 + 1) * sizeof(double),
                                   p->M, cudaMemcpyHostToDevice, p->ctx->stream));
    });
}

int s2b_paths_destroy(s2b_paths* p) {
    return guard([&] { delete p; });
}

int s2b_solve_magnus(s2b_context* ctx, const s2b_operator* op, const s2b_magnus_config* cfg, const double* phi,
                     const s2b_paths* paths, s2b_ensemble** out, s2b_magnus_stats* stats) {
    return guard([&] {
        need(ctx, "ctx");
        need(op, "op");
        need(cfg, "cfg");
        need(phi, "phi");
        need(paths, "paths");
        need(out, "out");
        S2B_CUDA(cudaSetDevice(ctx->device));
        MagnusSession* s = session_create(ctx, op, cfg, phi, paths);
        try {
            session_advance(s, static_cast<size_t>(-1) / 2);
            if (stats) session_stats(s, stats);
            *out = session_finish(s);
        } catch (...) {
            session_destroy(s);
            throw;
        }
        session_destroy(s);
    });
}

int s2b_solve_magnus_sweep(s2b_context* ctx, const s2b_operator* op, const s2b_magnus_config* cfgs, size_t ncfg,
                           const double* phi, const s2b_paths* paths, s2b_ensemble** outs, s2b_magnus_stats* stats) {
    return guard([&] {
        need(ctx, "ctx");
        need(op, "op");
        need(cfgs, "cfgs");
        need(phi, "phi");
        need(paths, "paths");
        need(outs, "outs");
        S2B_CUDA(cudaSetDevice(ctx->device));
        std::vector<MagnusSession*> ss;
        try {
            for (size_t i = 0; i < ncfg; ++i) ss.push_back(session_create(ctx, op, &cfgs[i], phi, paths));
            sessions_run_batched(ss.data(), static_cast<int>(ss.size()));
            for (size_t i = 0; i < ncfg; ++i) {
                if (stats) session_stats(ss[i], &stats[i]);
                outs[i] = session_finish(ss[i]);
            }
        } catch (...) {
            for (auto* s : ss) session_destroy(s);
            throw;
        }
        for (auto* s : ss) session_destroy(s);
    });
}

int s2b_solve_adaptive_magnus(s2b_context* ctx, const s2b_operator* op, const s2b_magnus_config* cfg,
                              const s2b_adaptive_config* adaptive, const double* phi, const s2b_paths* paths,
                              s2b_ensemble** out, s2b_magnus_stats* stats) {
    return guard([&] {
        need(ctx, "ctx");
        need(op, "op");
        need(cfg, "cfg");
        need(phi, "phi");
        need(paths, "paths");
        need(out, "out");
        S2B_CUDA(cudaSetDevice(ctx->device));
        *out = solve_adaptive(ctx, op, cfg, adaptive, phi, paths, stats);
    });
}

int s2b_solve_euler(s2b_context* ctx, const s2b_fields* f, const s2b_euler_config* cfg, const double* phi,
                    const s2b_paths* paths, s2b_ensemble** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(f, "fields");
        need(cfg, "cfg");
        need(phi, "phi");
        need(paths, "paths");
        need(out, "out");
        S2B_CUDA(cudaSetDevice(ctx->device));
        *out = solve_euler(ctx, f, cfg, phi, paths);
    });
}

int s2b_magnus_session_create(s2b_context* ctx, const s2b_operator* op, const s2b_magnus_config* cfg,
                              const double* phi, const s2b_paths* paths, s2b_magnus_session** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(op, "op");
        need(cfg, "cfg");
        need(phi, "phi");
        need(paths, "paths");
        need(out, "out");
        S2B_CUDA(cudaSetDevice(ctx->device));
        *out = reinterpret_cast<s2b_magnus_session*>(session_create(ctx, op, cfg, phi, paths));
    });
}

int s2b_magnus_session_advance(s2b_magnus_session* s, size_t n_windows) {
    return guard([&] {
        need(s, "session");
        session_advance(S(s), n_windows);
    });
}

int s2b_magnus_session_reset(s2b_magnus_session* s) {
    return guard([&] {
        need(s, "session");
        session_reset(S(s));
    });
}

int s2b_magnus_session_stats(const s2b_magnus_session* s, s2b_magnus_stats* stats) {
    return guard([&] {
        need(s, "session");
        need(stats, "stats");
        session_stats(S(s), stats);
    });
}

int s2b_magnus_session_set_timing(s2b_magnus_session* s, int enable) {
    return guard([&] {
        need(s, "session");
        session_set_timing(S(s), enable != 0);
    });
}

int s2b_magnus_session_ensemble(s2b_magnus_session* s, s2b_ensemble** out) {
    return guard([&] {
        need(s, "session");
        need(out, "out");
        *out = session_snapshot(S(s));
    });
}

int s2b_magnus_session_finish(s2b_magnus_session* s, s2b_ensemble** out) {
    return guard([&] {
        need(s, "session");
        need(out, "out");
        *out = session_finish(S(s));
    });
}

int s2b_magnus_session_moments(s2b_magnus_session* s, double* moments, double* live_paths) {
    return guard([&] {
        need(s, "session");
        need(moments, "moments");
        session_moments(S(s), moments, live_paths);
    });
}

int s2b_magnus_session_destroy(s2b_magnus_session* s) {
    return guard([&] { session_destroy(S(s)); });
}

int s2b_ensemble_create_host(s2b_context* ctx, const s2b_grid* grid, double t, uint64_t seed, size_t M,
                             const double* states, const uint8_t* status, s2b_ensemble** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(grid, "grid");
        need(states, "states");
        need(out, "out");
        S2B_CUDA(cudaSetDevice(ctx->device));
        auto* e = new s2b_ensemble();
        try {
            const size_t n = grid->nx * grid->nv;
            e->ctx = ctx;
            e->R = 1;
            e->M = M;
            e->nx = grid->nx;
            e->nv = grid->nv;
            e->seed = seed;
            e->grid = *grid;
            e->times.push_back(t);
            e->states.emplace_back(M * n);
            e->status.alloc(M);
            S2B_CUDA(cudaMemcpy(e->states[0].p, states, M * n * sizeof(double), cudaMemcpyHostToDevice));
            if (status)
                S2B_CUDA(cudaMemcpy(e->status.p, status, M, cudaMemcpyHostToDevice));
            else
                S2B_CUDA(cudaMemset(e->status.p, 0, M));
        } catch (...) {
            delete e;
            throw;
        }
        *out = e;
    });
}

int s2b_ensemble_info(const s2b_ensemble* e, int64_t info[5], double* times) {
    return guard([&] {
        need(e, "ensemble");
        info[0] = static_cast<int64_t>(e->R);
        info[1] = static_cast<int64_t>(e->M);
        info[2] = static_cast<int64_t>(e->nx * e->nv);
        info[3] = static_cast<int64_t>(e->nx);
        info[4] = static_cast<int64_t>(e->nv);
        if (times) std::copy(e->times.begin(), e->times.end(), times);
    });
}

int s2b_ensemble_download(const s2b_ensemble* e, size_t record, double* states, uint8_t* status) {
    return guard([&] {
        need(e, "ensemble");
        if (record >= e->R) fail(S2B_ERR_DIMENSION, "ensemble: record out of range");
        S2B_CUDA(cudaSetDevice(e->ctx->device));
        std::vector<uint8_t> st(e->M);
        S2B_CUDA(cudaMemcpy(st.data(), e->status.p + record * e->M, e->M, cudaMemcpyDeviceToHost));
        if (status) std::copy(st.begin(), st.end(), status);
        if (states) {
            const size_t n = e->nx * e->nv;
            S2B_CUDA(cudaMemcpy(states, e->states[record].p, e->M * n * sizeof(double), cudaMemcpyDeviceToHost));
            for (size_t m = 0; m < e->M; ++m)
                if (st[m])
                    for (size_t i = 0; i < n; ++i) states[m * n + i] = std::nan("");
        }
    });
}

int s2b_ensemble_counters(const s2b_ensemble* e, int64_t* terms, int64_t* windows) {
    return guard([&] {
        need(e, "ensemble");
        if (terms) {
            if (!e->terms.p) fail(S2B_ERR_CONFIG, "ensemble has no Magnus counters");
            S2B_CUDA(cudaMemcpy(terms, e->terms.p, e->M * sizeof(int64_t), cudaMemcpyDeviceToHost));
        }
        if (windows) {
            if (!e->windows.p) fail(S2B_ERR_CONFIG, "ensemble has no Magnus counters");
            S2B_CUDA(cudaMemcpy(windows, e->windows.p, e->M * sizeof(int64_t), cudaMemcpyDeviceToHost));
        }
    });
}

int s2b_ensemble_moments(const s2b_ensemble* e, size_t record, double* moments, size_t* live) {
    return guard([&] {
        need(e, "ensemble");
        need(moments, "moments");
        S2B_CUDA(cudaSetDevice(e->ctx->device));
        ensemble_moments(e, record, moments, live);
    });
}

int s2b_ensemble_destroy(s2b_ensemble* e) {
    return guard([&] { delete e; });
}

int s2b_exact_reference(s2b_context* ctx, const s2b_grid* grid, double t, double a, double sigma,
                        const s2b_paths* paths, s2b_ensemble** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(grid, "grid");
        need(paths, "paths");
        need(out, "out");
        S2B_CUDA(cudaSetDevice(ctx->device));
        *out = exact_reference(ctx, grid, t, a, sigma, paths);
    });
}

int s2b_exact_field(s2b_context* ctx, const s2b_grid* grid, double t, double a, double sigma, double W, double IW,
                    double* out) {
    return guard([&] {
        need(ctx, "ctx");
        need(grid, "grid");
        need(out, "out");
        S2B_CUDA(cudaSetDevice(ctx->device));
        exact_field(ctx, grid, t, a, sigma, W, IW, out);
    });
}

int s2b_errors(s2b_context* ctx, const s2b_ensemble* ref, size_t ref_record, const s2b_ensemble* app,
               size_t app_record, int kappa, s2b_error_stats* out, double* me_out) {
    return guard([&] {
        need(ctx, "ctx");
        need(ref, "ref");
        need(app, "app");
        need(out, "out");
        S2B_CUDA(cudaSetDevice(ctx->device));
        errors(ctx, ref, ref_record, app, app_record, kappa, out, me_out);
    });
}

int s2b_exact_errors(s2b_context* ctx, const s2b_ensemble* app, size_t app_record, double a, double sigma,
                     const s2b_paths* paths, int kappa, s2b_error_stats* out, double* me_out,
                     double* per_path_rel, double* moments) {
    return guard([&] {
        need(ctx, "ctx");
        need(app, "app");
        need(paths, "paths");
        need(out, "out");
        S2B_CUDA(cudaSetDevice(ctx->device));
        exact_errors(ctx, app, app_record, a, sigma, paths, kappa, out, me_out, per_path_rel, moments);
    });
}

int s2b_expmv(s2b_context* ctx, const s2b_csr* m, const double* x, double tol, double theta, double* y,
              int report[4]) {
    return guard([&] {
        need(ctx, "ctx");
        need(m, "matrix");
        need(x, "x");
        need(y, "y");
        need(report, "report");
        S2B_CUDA(cudaSetDevice(ctx->device));
        expmv_csr(ctx, m, x, tol, theta, y, report);
    });
}

int s2b_context_kernel_names(s2b_context* ctx, char* cluster, char* stream, size_t len) {
    return guard([&] {
        need(ctx, "ctx");
        auto put = [&](const void* fn, char* out) {
            if (!out || len == 0) return;
            const char* name = "";
            if (fn) S2B_CUDA(cudaFuncGetName(&name, fn));
            std::strncpy(out, name, len - 1);
            out[len - 1] = 0;
        };
        put(ctx->k_cluster, cluster);
        put(ctx->k_stream, stream);
    });
}

int s2b_context_em_kernel_name(s2b_context* ctx, char* out, size_t len) {
    return guard([&] {
        need(ctx, "ctx");
        if (!out || len == 0) return;
        const char* name = "";
        if (ctx->k_em) S2B_CUDA(cudaFuncGetName(&name, ctx->k_em));
        std::strncpy(out, name, len - 1);
        out[len - 1] = 0;
    });
}

int s2b_expmv_workspace_create(s2b_context* ctx, s2b_expmv_workspace** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(out, "out");
        S2B_CUDA(cudaSetDevice(ctx->device));
        *out = expmv_workspace_create(ctx);
    });
}

int s2b_expmv_workspace_destroy(s2b_expmv_workspace* ws) {
    return guard([&] { expmv_workspace_destroy(ws); });
}

int s2b_expmv_into(s2b_expmv_workspace* ws, const s2b_csr* m, const double* x, double tol, double theta,
                   double* y, s2b_expmv_report* report) {
    return guard([&] {
        need(ws, "workspace");
        need(m, "matrix");
        need(report, "report");
        if (m->rows) {
            need(x, "x");
            need(y, "y");
        }
        expmv_into(ws, m, x, tol, theta, y, report, false);
    });
}

int s2b_expmv_into_device(s2b_expmv_workspace* ws, const s2b_csr* m, const double* d_x, double tol, double theta,
                          double* d_y, s2b_expmv_report* report) {
    return guard([&] {
        need(ws, "workspace");
        need(m, "matrix");
        need(report, "report");
        if (m->rows) {
            need(d_x, "x");
            need(d_y, "y");
        }
        expmv_into(ws, m, d_x, tol, theta, d_y, report, true);
    });
}

int s2b_euler_step(const s2b_fields* f, const double* stencils, const double* u, double* out, double dW, double dt,
                   double* maxabs) {
    return guard([&] {
        need(f, "fields");
        need(u, "u");
        need(out, "out");
        const size_t n = f->nx * f->nv;
        DevBuf<double> du(n), dout(n);
        S2B_CUDA(cudaMemcpyAsync(du.p, u, n * sizeof(double), cudaMemcpyHostToDevice, f->ctx->stream));
        double mx = 0.0;
        euler_step_batch(f, stencils, du.p, dout.p, 1, &dW, dt, &mx);
        S2B_CUDA(cudaMemcpyAsync(out, dout.p, n * sizeof(double), cudaMemcpyDeviceToHost, f->ctx->stream));
        S2B_CUDA(cudaStreamSynchronize(f->ctx->stream));
        if (maxabs) *maxabs = mx;
    });
}

int s2b_euler_step_device(const s2b_fields* f, const double* stencils, const double* d_u, double* d_out, size_t M,
                          const double* dW, double dt, double* maxabs) {
    return guard([&] {
        need(f, "fields");
        if (M) {
            need(d_u, "u");
            need(d_out, "out");
            need(dW, "dW");
        }
        euler_step_batch(f, stencils, d_u, d_out, M, dW, dt, maxabs);
    });
}

} // extern "C"
