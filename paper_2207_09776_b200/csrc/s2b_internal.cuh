// Internal types shared by the CUDA translation units of libspde2d_b200.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "spde2d_b200.h"

namespace s2b {

// Error carrying one of the S2B_ERR_* codes across the C++ side of the C ABI.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& w) : std::runtime_error(w), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& what) { throw Error(code, what); }

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(S2B_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define S2B_CUDA(x) ::s2b::cuda_check((x), #x)
#define S2B_LAUNCHED(ctx) ::s2b::after_launch((ctx), __FILE__, __LINE__)

// Owning device buffer.
template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            n = o.n;
            o.p = nullptr;
            o.n = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t count) {
        release();
        if (count) S2B_CUDA(cudaMalloc(&p, count * sizeof(T)));
        n = count;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    size_t bytes() const { return n * sizeof(T); }
};

} // namespace s2b

// ---- handle definitions (opaque in the C header) -------------------------------
struct s2b_context {
    int device = 0;
    int num_sms = 0;
    cudaStream_t stream = nullptr;
    int64_t launches = 0;
    // the dominant kernels the Magnus engines launched last (their mangled names are what
    // bench.py matches against the ncu captures in profiles/)
    const void* k_cluster = nullptr;
    const void* k_stream = nullptr;
    const void* k_em = nullptr; // the E-M step kernel launched last (s2b_context_em_kernel_name)
};

namespace s2b {
void after_launch(s2b_context* ctx, const char* file, int line);
// S2B_GRID_CAP=n caps every persistent kernel's grid at n CTAs / clusters (never changes a
// result: work is drawn from counters or grid-strided).  The determinism stress tests vary
// it to change the interleaving of the synchronisation-heavy kernels.
int grid_cap(int grid);
}

// Stencil box addressing: bit b = (dv + 3) * 7 + (dx + 3) for |dx|, |dv| <= 3.
constexpr int kBoxR = 3;
constexpr int kBoxW = 2 * kBoxR + 1;
constexpr int kBoxBits = kBoxW * kBoxW;
constexpr int kClasses = 5; // x-classes of the compressed layout: 0, 1, interior, nx-2, nx-1

struct s2b_operator {
    s2b_context* ctx = nullptr;
    int order = 1;
    size_t nx = 0, nv = 0;
    int rx = 0, rv = 0;      // stencil radius actually used by the union pattern
    int compressed = 0;      // weights depend on (class(i), j) only
    uint64_t union_mask = 0; // union stencil bits
    int variant = 0;         // kernel instantiation id (see magnus.cu)
    // source-offset pairs, grouped by stencil bit in slot order
    std::vector<int> pair_begin; // kBoxBits + 1
    std::vector<int> pair_slot;  // npairs
    int npairs = 0;
    bool wfinite = true;      // every source weight finite (term_var's branch-free fold)
    s2b::DevBuf<int> d_pair_begin, d_pair_slot;
    s2b::DevBuf<double> d_wt; // entry-major weights of the TMA kernel variant
    s2b::DevBuf<int> d_eslot;
    uint32_t bmask = 0;       // Y entries that differ on x-boundary classes (in-grid offsets)
    // compressed: W[pair][j][cls]; full: W[pair][row]
    s2b::DevBuf<double> d_w;
    s2b::DevBuf<double> d_wpm; // uncompressed: point-major copy [row][x][npairs | 1] (term_var kernels)
    double dx_delta = 0.0, dv_delta = 0.0;
    s2b_grid grid{};
};

struct s2b_fields {
    s2b_context* ctx = nullptr;
    size_t nx = 0, nv = 0;
    int mask = 0;            // bit k set: field k (h fx fv gxx gxv gvv sig sigx sigv) non-zero
    s2b::DevBuf<double> d_f; // 9 * n, zero fields left unset
    double st[5] = {0, 0, 0, 0, 0}; // inv2dx invdx2 inv2dv invdv2 inv4dxdv
    s2b_grid grid{};
    bool xinv = false;          // every non-zero field constant along x (bitwise)
    s2b::DevBuf<double> d_rowf; // [9][nv] row values when xinv
    // separable: every non-zero field is x-invariant or v-invariant (bitwise); xdep = the
    // fields that depend on x, given per column in d_colf [9][nx] (g^xx, g^vv pre-halved)
    bool sep = false;
    int xdep = 0;
    s2b::DevBuf<double> d_colf;
    s2b::DevBuf<double> d_fgen; // [9][nx][nv] every field x-major, g^xx / g^vv pre-halved (cluster E-M)
};

struct s2b_paths {
    s2b_context* ctx = nullptr;
    double dt_leb = 0.0;
    size_t steps = 0, M = 0;
    uint64_t seed = 0;
    s2b::DevBuf<double> d_values; // [M][steps+1]
};

struct s2b_ensemble {
    s2b_context* ctx = nullptr;
    size_t R = 0, M = 0, nx = 0, nv = 0;
    std::vector<double> times;
    std::vector<s2b::DevBuf<double>> states; // R x [M][n]
    s2b::DevBuf<uint8_t> status;             // [R][M], 0 Ok
    s2b::DevBuf<long long> terms, windows;   // Magnus counters (optional)
    uint64_t seed = 0;
    s2b_grid grid{};
};

namespace s2b {

// plan_windows semantics (magnus.cpp:174-200) on the host.
struct WindowPlan {
    size_t dt_steps = 0, total_steps = 0;
    std::vector<size_t> record_steps;
};
size_t index_of(double t, double dt_leb, size_t steps);
WindowPlan plan_windows(double dt, double T, double dt_leb, size_t steps,
                        const double* record_times, size_t n_record, const char* who);

// Launch helpers implemented in the .cu files.
int grid_for(s2b_context* ctx, size_t work, int threads);
void broadcast_rows(s2b_context* ctx, double* dst, const double* host_src, size_t n, size_t M);

// Entry points behind the C ABI (implemented per .cu file).
s2b_operator* make_operator(s2b_context* ctx, const s2b_grid* grid, int order, const s2b_csr sources[6]);
void operator_info(const s2b_operator* op, int64_t info[6]);
struct MagnusSession;
MagnusSession* session_create(s2b_context* ctx, const s2b_operator* op, const s2b_magnus_config* cfg,
                              const double* phi, const s2b_paths* paths);
void session_reset(MagnusSession* s);
void session_advance(MagnusSession* s, size_t n_windows);
void session_stats(const MagnusSession* s, s2b_magnus_stats* out);
void session_set_timing(MagnusSession* s, bool on);
s2b_ensemble* session_snapshot(MagnusSession* s);
s2b_ensemble* session_finish(MagnusSession* s);
void sessions_run_batched(MagnusSession* const* ss, int n);
s2b_ensemble* solve_adaptive(s2b_context* ctx, const s2b_operator* op, const s2b_magnus_config* cfg,
                             const s2b_adaptive_config* ad, const double* phi, const s2b_paths* paths,
                             s2b_magnus_stats* stats);
void session_destroy(MagnusSession* s);
void session_moments(MagnusSession* s, double* host_out, double* live_out);
s2b_paths* make_paths_host(s2b_context* ctx, double dt_leb, size_t steps, size_t M, uint64_t seed,
                           const double* values);
s2b_paths* make_paths_philox(s2b_context* ctx, double dt_leb, size_t steps, size_t M, uint64_t seed,
                             uint64_t path_offset);
s2b_fields* make_fields(s2b_context* ctx, const s2b_grid* grid, const double* const* fields9);
// cluster-resident E-M (em_cluster.cu)
bool em_cluster_supported(const s2b_fields* f);
void em_cluster_solve(s2b_context* ctx, const s2b_fields* f, double dt, const double* d_phi,
                      const s2b_paths* paths, int step_leb, int nsteps, const std::vector<int>& rec_k,
                      double* const* d_rec, uint8_t* d_status, bool no_neg_zero);
s2b_ensemble* solve_euler(s2b_context* ctx, const s2b_fields* f, const s2b_euler_config* cfg,
                          const double* phi, const s2b_paths* paths);
s2b_ensemble* exact_reference(s2b_context* ctx, const s2b_grid* grid, double t, double a, double sigma,
                              const s2b_paths* paths);
void exact_field(s2b_context* ctx, const s2b_grid* grid, double t, double a, double sigma, double W, double IW,
                 double* host_out);
void errors(s2b_context* ctx, const s2b_ensemble* ref, size_t ref_record, const s2b_ensemble* app,
            size_t app_record, int kappa, s2b_error_stats* out, double* me_out);
void exact_errors(s2b_context* ctx, const s2b_ensemble* app, size_t app_record, double a, double sigma,
                  const s2b_paths* paths, int kappa, s2b_error_stats* out, double* me_out,
                  double* per_path_rel, double* moments);
s2b_expmv_workspace* expmv_workspace_create(s2b_context* ctx);
void expmv_workspace_destroy(s2b_expmv_workspace* ws);
void expmv_into(s2b_expmv_workspace* ws, const s2b_csr* m, const double* x, double tol, double theta, double* y,
                s2b_expmv_report* rep, bool device);
void euler_step_batch(const s2b_fields* f, const double* st, const double* d_u, double* d_out, size_t M,
                      const double* dW, double dt, double* maxabs);
void region_of(size_t d, int kappa, size_t* lo, size_t* hi); // central_region (analysis.cpp:9-31)
} // namespace s2b
namespace spde2d {
struct GridSpec;
struct CoefficientFields;
struct CommutatorSet;
}
namespace s2b {
// device-side assembly of the CommutatorSet (assemble.cu), packed into the reference's CSR
spde2d::CommutatorSet device_commutators(s2b_context* ctx, const spde2d::GridSpec& grid,
                                         const spde2d::CoefficientFields& f, int order);
void set_last_error(const std::string& what); // the calling thread's s2b_last_error()
void ensemble_moments(const s2b_ensemble* e, size_t record, double* host_moments, size_t* live);
void expmv_csr(s2b_context* ctx, const s2b_csr* m, const double* x, double tol, double theta, double* y,
               int report[4]);

} // namespace s2b
