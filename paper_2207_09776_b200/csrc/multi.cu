// Path-sharded multi-GPU solves from the product API.
//
// The reference's unit of parallelism is the independent path loop (OpenMP over m,
// magnus.cpp:258-263, euler.cpp:142-145); nothing is exchanged inside the hot path.  Here
// every device of the node gets a contiguous range of global path ids (shard()), its own
// context and its own host thread, and runs the whole solve on its slice: operator build,
// Philox paths keyed by the GLOBAL path id (path_offset = the range start, so the paths do
// not depend on the device count), the Magnus / E-M engines, and the per-path norms.  The
// only collective is at the end, over NVLink with NCCL (loaded at run time, so the library
// itself has no NCCL dependency):
//   * one ncclAllReduce(sum, f64) of {ME sums, used, blow-ups, sum u, sum u^2, counters};
//   * one ncclAllGather of the per-path relative errors (padded to the largest range), so
//     Err = (sum over m ascending) / M is bitwise the one-device value (analysis.cpp:99-127).
// A device listed twice cannot join an NCCL clique; such a set (e.g. {0, 0} on a one-GPU
// box) runs the same shards and combines them on the host instead -- the same arithmetic,
// used by the tests to exercise sharding without a second GPU.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "s2b_internal.cuh"

namespace s2b {

struct NcclApi {
    void* lib = nullptr;
    ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;

    void load() {
        if (lib) return;
        lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) fail(S2B_ERR_RUNTIME, std::string("multi-GPU: cannot load libnccl.so.2: ") + dlerror());
        auto sym = [&](const char* name) {
            void* p = dlsym(lib, name);
            if (!p) fail(S2B_ERR_RUNTIME, std::string("multi-GPU: NCCL symbol missing: ") + name);
            return p;
        };
        comm_init_all = reinterpret_cast<decltype(comm_init_all)>(sym("ncclCommInitAll"));
        all_reduce = reinterpret_cast<decltype(all_reduce)>(sym("ncclAllReduce"));
        all_gather = reinterpret_cast<decltype(all_gather)>(sym("ncclAllGather"));
        group_start = reinterpret_cast<decltype(group_start)>(sym("ncclGroupStart"));
        group_end = reinterpret_cast<decltype(group_end)>(sym("ncclGroupEnd"));
        comm_destroy = reinterpret_cast<decltype(comm_destroy)>(sym("ncclCommDestroy"));
        error_string = reinterpret_cast<decltype(error_string)>(sym("ncclGetErrorString"));
    }
    void check(ncclResult_t r, const char* what) const {
        if (r != ncclSuccess) fail(S2B_ERR_RUNTIME, std::string(what) + ": " + error_string(r));
    }
};

namespace {
// what one device hands to the combine step (host copies)
struct Part {
    size_t offset = 0, count = 0;
    std::vector<double> rel;  // per-path ||ref-app||/||ref|| (NaN for blown paths)
    std::vector<double> pack; // [me sums (w*w)] used blowups [sum u (n)] [sum u^2 (n)] terms windows
    double ms = 0.0;
    int rc = S2B_OK;
    std::string err;
};
} // namespace

} // namespace s2b

struct s2b_multi {
    std::vector<int> devices;
    std::vector<s2b_context*> ctx;
    bool nccl = false;
    s2b::NcclApi api;
    std::vector<ncclComm_t> comms;
};

namespace s2b {

namespace {

void shard_range(size_t M, int rank, int world, size_t* off, size_t* cnt) {
    const size_t base = M / static_cast<size_t>(world), extra = M % static_cast<size_t>(world);
    const size_t r = static_cast<size_t>(rank);
    *cnt = base + (r < extra ? 1 : 0);
    *off = r * base + std::min(r, extra);
}

void check_rc(int rc) {
    if (rc != S2B_OK) fail(rc, s2b_last_error());
}

template <class T>
struct Owned {
    T* p = nullptr;
    int (*d)(T*);
    explicit Owned(int (*del)(T*)) : d(del) {}
    ~Owned() {
        if (p) d(p);
    }
};

enum class Scheme { Magnus, Euler };

struct Job {
    Scheme scheme;
    const s2b_grid* grid;
    const s2b_operator_spec* op;
    const s2b_magnus_config* mcfg;
    const s2b_euler_config* ecfg;
    const double* phi;
    double dt_leb;
    size_t steps, M;
    uint64_t seed;
    int kappa;
    size_t w2, n;
};

// The whole solve of one device's path range, on that device's host thread.
void run_part(s2b_context* ctx, const Job& j, Part& part) {
    if (part.count == 0) return;
    Owned<s2b_paths> paths(s2b_paths_destroy);
    check_rc(s2b_paths_create_philox(ctx, j.dt_leb, j.steps, part.count, j.seed, part.offset, &paths.p));
    Owned<s2b_ensemble> ens(s2b_ensemble_destroy);
    cudaEvent_t e0, e1;
    S2B_CUDA(cudaEventCreate(&e0));
    S2B_CUDA(cudaEventCreate(&e1));
    s2b_magnus_stats st{};
    if (j.scheme == Scheme::Magnus) {
        Owned<s2b_operator> op(s2b_operator_destroy);
        check_rc(s2b_operator_build(ctx, j.grid, j.op->family, j.op->a, j.op->sigma, j.op->fields9, j.op->order, &op.p));
        S2B_CUDA(cudaEventRecord(e0, ctx->stream));
        check_rc(s2b_solve_magnus(ctx, op.p, j.mcfg, j.phi, paths.p, &ens.p, &st));
        S2B_CUDA(cudaEventRecord(e1, ctx->stream));
    } else {
        Owned<s2b_fields> f(s2b_fields_destroy);
        if (j.op->family == 2)
            check_rc(s2b_fields_create(ctx, j.grid, j.op->fields9, &f.p));
        else
            check_rc(s2b_fields_build(ctx, j.grid, j.op->family, j.op->a, j.op->sigma, &f.p));
        S2B_CUDA(cudaEventRecord(e0, ctx->stream));
        check_rc(s2b_solve_euler(ctx, f.p, j.ecfg, j.phi, paths.p, &ens.p));
        S2B_CUDA(cudaEventRecord(e1, ctx->stream));
    }
    S2B_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    S2B_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    part.ms = ms;
    int64_t info[5];
    check_rc(s2b_ensemble_info(ens.p, info, nullptr));
    const size_t last = static_cast<size_t>(info[0]) - 1;
    part.pack.assign(j.w2 + 2 + 2 * j.n + 2, 0.0);
    double* mom = part.pack.data() + j.w2 + 2;
    if (j.kappa >= 0) {
        s2b_error_stats es{};
        part.rel.assign(part.count, 0.0);
        std::vector<double> me(j.w2);
        check_rc(s2b_exact_errors(ctx, ens.p, last, j.op->a, j.op->sigma, paths.p, j.kappa, &es, me.data(),
                                  part.rel.data(), mom));
        if (es.used)
            for (size_t q = 0; q < j.w2; ++q) part.pack[q] = me[q] * static_cast<double>(es.used);
        part.pack[j.w2] = static_cast<double>(es.used);
        part.pack[j.w2 + 1] = static_cast<double>(es.blowups);
    } else {
        size_t live = 0;
        check_rc(s2b_ensemble_moments(ens.p, last, mom, &live));
        part.pack[j.w2] = static_cast<double>(live);
        part.pack[j.w2 + 1] = static_cast<double>(part.count - live);
    }
    part.pack[j.w2 + 2 + 2 * j.n] = static_cast<double>(st.path_terms);
    part.pack[j.w2 + 3 + 2 * j.n] = static_cast<double>(st.path_windows);
}

// NCCL combine: all-reduce the packs, all-gather the per-path errors (rank order = path order).
void nccl_combine(s2b_multi* mg, std::vector<Part>& parts, size_t cmax, std::vector<double>& pack,
                  std::vector<double>& rel_all, bool with_rel) {
    const int W = static_cast<int>(mg->ctx.size());
    const size_t P = parts[0].pack.size();
    std::vector<DevBuf<double>> dpack(W), dsend(W), drecv(W);
    for (int r = 0; r < W; ++r) {
        S2B_CUDA(cudaSetDevice(mg->devices[r]));
        dpack[r].alloc(P);
        std::vector<double> p = parts[r].pack.empty() ? std::vector<double>(P, 0.0) : parts[r].pack;
        S2B_CUDA(cudaMemcpy(dpack[r].p, p.data(), P * sizeof(double), cudaMemcpyHostToDevice));
        if (with_rel) {
            dsend[r].alloc(std::max<size_t>(1, cmax));
            drecv[r].alloc(std::max<size_t>(1, cmax * W));
            std::vector<double> s(std::max<size_t>(1, cmax), NAN);
            std::copy(parts[r].rel.begin(), parts[r].rel.end(), s.begin());
            S2B_CUDA(cudaMemcpy(dsend[r].p, s.data(), s.size() * sizeof(double), cudaMemcpyHostToDevice));
        }
    }
    mg->api.check(mg->api.group_start(), "ncclGroupStart");
    for (int r = 0; r < W; ++r) {
        S2B_CUDA(cudaSetDevice(mg->devices[r]));
        mg->api.check(mg->api.all_reduce(dpack[r].p, dpack[r].p, P, ncclFloat64, ncclSum, mg->comms[r], mg->ctx[r]->stream),
                      "ncclAllReduce");
        if (with_rel && cmax)
            mg->api.check(mg->api.all_gather(dsend[r].p, drecv[r].p, cmax, ncclFloat64, mg->comms[r], mg->ctx[r]->stream),
                          "ncclAllGather");
    }
    mg->api.check(mg->api.group_end(), "ncclGroupEnd");
    for (int r = 0; r < W; ++r) {
        S2B_CUDA(cudaSetDevice(mg->devices[r]));
        S2B_CUDA(cudaStreamSynchronize(mg->ctx[r]->stream));
    }
    S2B_CUDA(cudaSetDevice(mg->devices[0]));
    pack.resize(P);
    S2B_CUDA(cudaMemcpy(pack.data(), dpack[0].p, P * sizeof(double), cudaMemcpyDeviceToHost));
    if (with_rel) {
        std::vector<double> g(cmax * W);
        if (cmax) S2B_CUDA(cudaMemcpy(g.data(), drecv[0].p, g.size() * sizeof(double), cudaMemcpyDeviceToHost));
        rel_all.clear();
        for (int r = 0; r < W; ++r) rel_all.insert(rel_all.end(), g.begin() + r * cmax, g.begin() + r * cmax + parts[r].count);
    }
}

void solve_multi(s2b_multi* mg, const Job& j, s2b_multi_stats* out, double* me_out, double* moments_out,
                 double* rel_out) {
    const int W = static_cast<int>(mg->ctx.size());
    std::vector<Part> parts(W);
    size_t cmax = 0;
    for (int r = 0; r < W; ++r) {
        shard_range(j.M, r, W, &parts[r].offset, &parts[r].count);
        cmax = std::max(cmax, parts[r].count);
    }
    // one host thread per device (its context, its stream); distinct devices run concurrently
    std::vector<std::thread> th;
    for (int r = 0; r < W; ++r)
        th.emplace_back([&, r] {
            try {
                S2B_CUDA(cudaSetDevice(mg->devices[r]));
                run_part(mg->ctx[r], j, parts[r]);
            } catch (const Error& e) {
                parts[r].rc = e.code;
                parts[r].err = e.what();
            } catch (const std::exception& e) {
                parts[r].rc = S2B_ERR_RUNTIME;
                parts[r].err = e.what();
            }
        });
    for (auto& t : th) t.join();
    for (int r = 0; r < W; ++r)
        if (parts[r].rc != S2B_OK) fail(parts[r].rc, "device " + std::to_string(mg->devices[r]) + ": " + parts[r].err);
    const size_t P = j.w2 + 2 + 2 * j.n + 2;
    for (auto& p : parts)
        if (p.pack.empty()) p.pack.assign(P, 0.0);
    std::vector<double> pack, rel_all;
    const bool with_rel = j.kappa >= 0;
    if (mg->nccl) {
        nccl_combine(mg, parts, cmax, pack, rel_all, with_rel);
    } else { // host combine, rank order (a device listed more than once)
        pack.assign(P, 0.0);
        for (const auto& p : parts) {
            for (size_t q = 0; q < P; ++q) pack[q] += p.pack[q];
            rel_all.insert(rel_all.end(), p.rel.begin(), p.rel.end());
        }
    }
    *out = s2b_multi_stats{};
    out->M_total = j.M;
    out->devices = W;
    out->nccl = mg->nccl ? 1 : 0;
    for (const auto& p : parts) out->max_solve_ms = std::max(out->max_solve_ms, p.ms);
    const double used = pack[j.w2], blown = pack[j.w2 + 1];
    out->errors.used = static_cast<size_t>(used);
    out->errors.blowups = static_cast<size_t>(blown);
    out->errors.excluded = out->errors.blowups;
    out->path_terms = static_cast<int64_t>(pack[j.w2 + 2 + 2 * j.n]);
    out->path_windows = static_cast<int64_t>(pack[j.w2 + 3 + 2 * j.n]);
    if (moments_out) std::memcpy(moments_out, pack.data() + j.w2 + 2, 2 * j.n * sizeof(double));
    if (with_rel) {
        // Err: the per-path ratios in ascending global m (analysis.cpp:99-127), inf if any blew up
        double s = 0.0;
        for (double v : rel_all)
            if (!std::isnan(v)) s += v;
        out->errors.sum_rel = s;
        out->errors.err = out->errors.blowups > 0 ? INFINITY : s / static_cast<double>(j.M);
        double ame = 0.0;
        for (size_t q = 0; q < j.w2; ++q) {
            const double v = used > 0 ? pack[q] / used : pack[q];
            if (me_out) me_out[q] = v;
            ame += v;
        }
        out->errors.ame = j.w2 ? ame / static_cast<double>(j.w2) : 0.0;
        size_t lo, hi;
        region_of(j.grid->nx, j.kappa, &lo, &hi);
        out->errors.region_lo = lo;
        out->errors.region_hi = hi;
        if (rel_out) std::memcpy(rel_out, rel_all.data(), rel_all.size() * sizeof(double));
    }
}

int multi_entry(s2b_multi* mg, const Job& j, s2b_multi_stats* out, double* me_out, double* moments_out,
                double* rel_out) {
    try {
        solve_multi(mg, j, out, me_out, moments_out, rel_out);
        return S2B_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return S2B_ERR_RUNTIME;
    }
}

} // namespace
} // namespace s2b

using namespace s2b;

extern "C" {

int s2b_shard(size_t M_total, int rank, int world, size_t* offset, size_t* count) {
    if (world < 1 || rank < 0 || rank >= world || !offset || !count) return S2B_ERR_CONFIG;
    shard_range(M_total, rank, world, offset, count);
    return S2B_OK;
}

int s2b_multi_create(const int* devices, int ndev, s2b_multi** out) {
    if (!devices || ndev < 1 || !out) return S2B_ERR_CONFIG;
    auto* mg = new s2b_multi();
    mg->devices.assign(devices, devices + ndev);
    for (int r = 0; r < ndev; ++r) {
        s2b_context* c = nullptr;
        const int rc = s2b_context_create(devices[r], &c);
        if (rc != S2B_OK) {
            s2b_multi_destroy(mg);
            return rc;
        }
        mg->ctx.push_back(c);
    }
    std::vector<int> sorted(mg->devices);
    std::sort(sorted.begin(), sorted.end());
    mg->nccl = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
    if (mg->nccl) {
        try {
            mg->api.load();
            mg->comms.resize(ndev);
            mg->api.check(mg->api.comm_init_all(mg->comms.data(), ndev, mg->devices.data()), "ncclCommInitAll");
        } catch (const Error& e) {
            mg->comms.clear();
            s2b_multi_destroy(mg);
            set_last_error(e.what());
            return e.code;
        }
    }
    *out = mg;
    return S2B_OK;
}

int s2b_multi_destroy(s2b_multi* mg) {
    if (!mg) return S2B_OK;
    for (auto c : mg->comms)
        if (c && mg->api.comm_destroy) mg->api.comm_destroy(c);
    for (auto c : mg->ctx) s2b_context_destroy(c);
    delete mg;
    return S2B_OK;
}

int s2b_multi_info(const s2b_multi* mg, int info[2]) {
    if (!mg || !info) return S2B_ERR_CONFIG;
    info[0] = static_cast<int>(mg->devices.size());
    info[1] = mg->nccl ? 1 : 0;
    return S2B_OK;
}

} // extern "C"

extern "C" {

int s2b_multi_solve_magnus(s2b_multi* mg, const s2b_grid* grid, const s2b_operator_spec* op,
                           const s2b_magnus_config* cfg, const double* phi, double dt_leb, size_t steps,
                           size_t M_total, uint64_t seed, int kappa, s2b_multi_stats* out, double* me_out,
                           double* moments_out, double* per_path_rel_out) {
    if (!mg || !grid || !op || !cfg || !phi || !out) return S2B_ERR_CONFIG;
    size_t w2 = 0;
    if (kappa >= 0) {
        size_t lo = 0, hi = 0;
        try {
            region_of(grid->nx, kappa, &lo, &hi);
        } catch (const Error& e) {
            set_last_error(e.what());
            return e.code;
        }
        w2 = (hi - lo + 1) * (hi - lo + 1);
    }
    const Job j{Scheme::Magnus, grid, op, cfg, nullptr, phi, dt_leb, steps, M_total, seed, kappa, w2,
                grid->nx * grid->nv};
    return multi_entry(mg, j, out, me_out, moments_out, per_path_rel_out);
}

int s2b_multi_solve_euler(s2b_multi* mg, const s2b_grid* grid, const s2b_operator_spec* fields,
                          const s2b_euler_config* cfg, const double* phi, double dt_leb, size_t steps,
                          size_t M_total, uint64_t seed, int kappa, s2b_multi_stats* out, double* me_out,
                          double* moments_out, double* per_path_rel_out) {
    if (!mg || !grid || !fields || !cfg || !phi || !out) return S2B_ERR_CONFIG;
    size_t w2 = 0;
    if (kappa >= 0) {
        size_t lo = 0, hi = 0;
        try {
            region_of(grid->nx, kappa, &lo, &hi);
        } catch (const Error& e) {
            set_last_error(e.what());
            return e.code;
        }
        w2 = (hi - lo + 1) * (hi - lo + 1);
    }
    const Job j{Scheme::Euler, grid, fields, nullptr, cfg, phi, dt_leb, steps, M_total, seed, kappa, w2,
                grid->nx * grid->nv};
    return multi_entry(mg, j, out, me_out, moments_out, per_path_rel_out);
}

} // extern "C"
