/*
 * spde2d_b200.h — C ABI of the B200 hot path (the drop-in boundary).
 *
 * Plain pointers and sizes, POD structs, int return codes; no C++ or torch
 * types cross this boundary.  Each entry point replaces one reference
 * routine (file:line under /root/reference/proj):
 *
 *   s2b_operator_create      <- CommutatorSet consumption by MagnusLogBuilder
 *                               (include/spde2d/magnus.hpp:61-86, src/magnus.cpp:88-139)
 *   s2b_fields_create        <- CoefficientFields consumption by euler_step_into
 *                               (include/spde2d/operators.hpp:15-25, src/euler.cpp:28-86)
 *   s2b_paths_create_host    <- BrownianBatch (include/spde2d/stochastics.hpp:32-43)
 *   s2b_paths_create_philox  <- simulate_brownian (src/stochastics.cpp:76-101), counter-based
 *   s2b_solve_magnus         <- solve_iterated_magnus (include/spde2d/magnus.hpp:93-97,
 *                               src/magnus.cpp:239-304) incl. expmv_into (sparse.cpp:427-503)
 *   s2b_solve_euler          <- solve_euler (include/spde2d/euler.hpp:46-49, src/euler.cpp:95-182)
 *   s2b_exact_reference      <- exact_reference (include/spde2d/exact_langevin.hpp:44-46)
 *   s2b_errors               <- mean_rel_error / mean_abs_error / avg_mean_abs_error
 *                               (include/spde2d/analysis.hpp:35-50, src/analysis.cpp:53-130)
 *   s2b_exact_errors         <- exact_reference + the three norms, fused (no reference
 *                               ensemble is materialised), plus moment sums for the
 *                               cross-GPU allreduce
 *   s2b_expmv                <- expmv_into on a general CSR matrix (sparse.hpp:149-151)
 *   s2b_expmv_into           <- expmv_into + ExpmvWorkspace + ExpmvReport (sparse.hpp:106-151)
 *   s2b_euler_step           <- euler_step_into / euler_step (euler.hpp:19-40, euler.cpp:18-86)
 *
 * Error codes mirror the reference's exception classes (errors.hpp:10-19):
 * S2B_ERR_CONFIG <-> ConfigError, S2B_ERR_DIMENSION <-> DimensionError,
 * S2B_ERR_RUNTIME <-> std::runtime_error; numerical failure inside the solvers
 * is never an error — it is the per-path BlownUp status, as in the reference.
 * All calls are stream-ordered on the context's stream and synchronous at
 * return unless stated otherwise.  One context per GPU.
 */
#ifndef SPDE2D_B200_H
#define SPDE2D_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define S2B_OK 0
#define S2B_ERR_CONFIG 1
#define S2B_ERR_DIMENSION 2
#define S2B_ERR_EXPMV 3
#define S2B_ERR_RUNTIME 4
#define S2B_ERR_CUDA 5

typedef struct s2b_context s2b_context;
typedef struct s2b_operator s2b_operator;
typedef struct s2b_fields s2b_fields;
typedef struct s2b_paths s2b_paths;
typedef struct s2b_ensemble s2b_ensemble;
typedef struct s2b_magnus_session s2b_magnus_session;

/* GridSpec (grid.hpp:28-40): interior nodes a + (i+1)(b-a)/(n+1). */
typedef struct {
    double ax, bx;
    size_t nx;
    double av, bv;
    size_t nv;
} s2b_grid;

/* One spde2d::SparseMatrix in its CSR storage (sparse.hpp:36-73).  rows == 0 marks
 * an absent matrix (e.g. A2/BA/BAA/BAB of a lower-order CommutatorSet). */
typedef struct {
    size_t rows;
    const size_t *row_ptr;  /* rows + 1 */
    const int32_t *col_idx; /* row_ptr[rows] */
    const double *values;   /* row_ptr[rows] */
} s2b_csr;

/* MagnusConfig (magnus.hpp:19-28) + the horizon T. */
typedef struct {
    int order;
    double dt;
    double T;
    double expmv_tol;
    double expmv_theta;
    double blowup_norm_cap;
    const double *record_times; /* may be NULL when n_record == 0 (terminal only) */
    size_t n_record;
} s2b_magnus_config;

/* AdaptiveConfig (magnus.hpp:14-17): step-size control of solve_adaptive_magnus. */
typedef struct {
    int enabled;      /* must be non-zero for s2b_solve_adaptive_magnus */
    double tolerance; /* accepted order-2 / order-3 relative gap */
    double shrink;    /* window shrink factor in (0, 1) */
} s2b_adaptive_config;

/* EulerConfig (euler.hpp:12-16) + the horizon T. */
typedef struct {
    double dt;
    double T;
    const double *record_times;
    size_t n_record;
} s2b_euler_config;

/* Result of the norms (RelError + MeanAbsError summary, analysis.hpp:28-50). */
typedef struct {
    double err;       /* mean relative Frobenius error; +inf if any app path blew up */
    size_t blowups;   /* app paths blown up (mean_rel_error) */
    double ame;       /* avg_mean_abs_error of the ME matrix */
    size_t excluded;  /* app paths excluded from ME */
    double sum_rel;   /* sum over non-blown paths of ||ref-app||_F/||ref||_F (ascending m) */
    size_t used;      /* non-blown app paths */
    size_t region_lo; /* central region [lo, hi] */
    size_t region_hi;
} s2b_error_stats;

/* Per-run counters of the Magnus pass engine. */
typedef struct {
    int64_t passes;        /* stencil passes launched (one Taylor term of every live path) */
    int64_t path_terms;    /* sum over paths of Taylor terms applied (= S*K summed) */
    int64_t path_windows;  /* windows completed */
    int64_t term_launches; /* launches of the dominant term kernel */
    double term_kernel_ms; /* summed CUDA-event time of those launches (if timing enabled) */
    double gridpoints;     /* nx*nv */
    int64_t path_segments; /* sum over paths of Taylor segments (one k=1 term each) */
    int32_t engine;        /* 0 streaming passes, 1 cluster row-band, 2 cluster x-march, 3 in-place x-march */
    int64_t hybrid_paths;  /* paths the last cluster launch left to the streaming engine (idle SMs) */
} s2b_magnus_stats;

const char *s2b_last_error(void);
const char *s2b_version(void);

/* ---- context ---------------------------------------------------------------- */
int s2b_context_create(int device, s2b_context **out);
int s2b_context_destroy(s2b_context *ctx);
int s2b_context_synchronize(s2b_context *ctx);
/* The cudaStream_t (as void*) all work of this context is ordered on. */
void *s2b_context_stream(s2b_context *ctx);
/* Number of kernels launched by this context so far. */
int64_t s2b_context_launches(s2b_context *ctx);
/* Mangled names (cudaFuncGetName) of the dominant Magnus kernels this context launched last:
 * the cluster-resident engine's and the streaming pass engine's ("" if none), each copied
 * into a caller buffer of `len` bytes.  bench.py matches them against the ncu captures. */
int s2b_context_kernel_names(s2b_context *ctx, char *cluster, char *stream, size_t len);
/* Mangled name of the Euler-Maruyama step kernel this context launched last (em_cluster_ip,
 * em_tb, em_rows or em_step; "" if none), for bench.py's E-M capture check. */
int s2b_context_em_kernel_name(s2b_context *ctx, char *out, size_t len);

/* ---- operators ----------------------------------------------------------------
 * sources: B, A, A2, BA, BAA, BAB (the CommutatorSet slot order of magnus.cpp:42-52).
 * The CSR values are re-laid out as 2-D stencil weights, bit for bit. */
int s2b_operator_create(s2b_context *ctx, const s2b_grid *grid, int order,
                        const s2b_csr sources[6], s2b_operator **out);
/* Host-kept builder (operators.cpp semantics, our C++): family 0 langevin-constant,
 * 1 langevin-variable, 2 explicit fields (fields9: h fx fv gxx gxv gvv sig sigx sigv,
 * NULL = identically zero).  Builds the CSR CommutatorSet on the host and uploads it. */
int s2b_operator_build(s2b_context *ctx, const s2b_grid *grid, int family, double a,
                       double sigma, const double *const *fields9, int order,
                       s2b_operator **out);
/* info: [0] union stencil points, [1] compressed (x-invariant) layout flag,
 *       [2] radius x, [3] radius v, [4] source-offset pairs, [5] order */
int s2b_operator_info(const s2b_operator *op, int64_t info[6]);
int s2b_operator_destroy(s2b_operator *op);

/* Euler coefficient fields; fields9 entries NULL = identically zero. */
int s2b_fields_create(s2b_context *ctx, const s2b_grid *grid, const double *const *fields9,
                      s2b_fields **out);
int s2b_fields_build(s2b_context *ctx, const s2b_grid *grid, int family, double a, double sigma,
                     s2b_fields **out);
int s2b_fields_destroy(s2b_fields *f);

/* Gaussian datum phi = exp(-(x^2+v^2)/2) at interior nodes, host-computed (n doubles). */
int s2b_gaussian_datum(const s2b_grid *grid, double *out);

/* ---- host-kept builder (no GPU needed) -----------------------------------------
 * The CSR CommutatorSet and CoefficientFields exactly as the reference builds them
 * (operators.cpp:134-208 arithmetic order), for callers that hand CSR to
 * s2b_operator_create or want to inspect it.  Pointers returned by the accessors stay
 * valid until s2b_host_ops_destroy. */
typedef struct s2b_host_ops s2b_host_ops;
int s2b_host_ops_build(const s2b_grid *grid, int family, double a, double sigma,
                       const double *const *fields9, int order, s2b_host_ops **out);
int s2b_host_ops_csr(const s2b_host_ops *h, int slot, s2b_csr *out);
int s2b_host_ops_field(const s2b_host_ops *h, int which, const double **data, int *is_zero);
int s2b_host_ops_destroy(s2b_host_ops *h);
/* Device-side assembly: the same CommutatorSet computed on the GPU --
 * assemble_drift / assemble_diffusion (operators.cpp:134-189) and precompute_commutators
 * (operators.cpp:191-208) as per-row stencil kernels in the CSR algebra's accumulation order
 * (sparse.cpp:126-261), packed back into CSR with exact zeros pruned: bitwise the host
 * builder's (and the reference's) CSR.  The fields are sampled on the host as above. */
int s2b_host_ops_assemble_device(s2b_context *ctx, const s2b_grid *grid, int family, double a,
                                 double sigma, const double *const *fields9, int order,
                                 s2b_host_ops **out);
/* s2b_operator_build with the CommutatorSet assembled on the device. */
int s2b_operator_build_device(s2b_context *ctx, const s2b_grid *grid, int family, double a,
                              double sigma, const double *const *fields9, int order,
                              s2b_operator **out);
/* simulate_brownian (stochastics.cpp:76-101) on the host: values [M][steps+1]. */
int s2b_host_simulate_brownian(double T, double dt_leb, size_t M, uint64_t seed,
                               double *values_out);

/* ---- Brownian paths ------------------------------------------------------------
 * Host mode: prefix values [M][steps+1] exactly as BrownianBatch::values (parity mode).
 * Philox mode: N(0, dt_leb) increments from Philox4x32-10 keyed by (seed, path_offset+m)
 * with the Lebesgue step as counter, prefix-summed sequentially per path on the GPU. */
int s2b_paths_create_host(s2b_context *ctx, double dt_leb, size_t steps, size_t M,
                          uint64_t seed, const double *values, s2b_paths **out);
int s2b_paths_create_philox(s2b_context *ctx, double dt_leb, size_t steps, size_t M,
                            uint64_t seed, uint64_t path_offset, s2b_paths **out);
int s2b_paths_download(const s2b_paths *p, double *values_out);
/* Overwrite columns [k0, k1] of every path's prefix values from a host array laid out
 * like BrownianBatch::values ([M][steps+1]); the columns copied are the inputs of the
 * windows covering [k0, k1] (pinned host memory makes this an async DMA). */
int s2b_paths_upload(s2b_paths *p, size_t k0, size_t k1, const double *values);
int s2b_paths_destroy(s2b_paths *p);

/* ---- solvers -----------------------------------------------------------------
 * Results stay on the device in an ensemble (one record per record time, last = T). */
int s2b_solve_magnus(s2b_context *ctx, const s2b_operator *op, const s2b_magnus_config *cfg,
                     const double *phi, const s2b_paths *paths, s2b_ensemble **out,
                     s2b_magnus_stats *stats);
int s2b_solve_euler(s2b_context *ctx, const s2b_fields *f, const s2b_euler_config *cfg,
                    const double *phi, const s2b_paths *paths, s2b_ensemble **out);
/* A step-size sweep on shared paths (run_stepsize_sweep, experiment.cpp:486-551): ncfg
 * configurations (typically the same order at several dt) solved in batched launches -- one
 * persistent launch carries the paths of up to 8 configurations on the x-march engines.
 * outs[i] / stats[i] (stats may be NULL) as s2b_solve_magnus would return for cfgs[i]. */
int s2b_solve_magnus_sweep(s2b_context *ctx, const s2b_operator *op, const s2b_magnus_config *cfgs,
                           size_t ncfg, const double *phi, const s2b_paths *paths, s2b_ensemble **outs,
                           s2b_magnus_stats *stats);
/* solve_adaptive_magnus (magnus.cpp:306-404): orders 2 and 3 per window from one weight
 * build, accept order 3 when the relative gap <= tolerance, else shrink and retry.
 * cfg->order is ignored (the operator must carry order-3 commutators). */
int s2b_solve_adaptive_magnus(s2b_context *ctx, const s2b_operator *op, const s2b_magnus_config *cfg,
                              const s2b_adaptive_config *adaptive, const double *phi,
                              const s2b_paths *paths, s2b_ensemble **out, s2b_magnus_stats *stats);

/* Resident Magnus session: state stays in HBM, windows are advanced on demand.
 * The session borrows `op` and `paths`: both must outlive it (destroy the session first).
 * After s2b_magnus_session_finish the session's buffers belong to the returned ensemble:
 * advance / reset / stats / ensemble / moments / a second finish return S2B_ERR_CONFIG;
 * only destroy is valid. */
int s2b_magnus_session_create(s2b_context *ctx, const s2b_operator *op,
                              const s2b_magnus_config *cfg, const double *phi,
                              const s2b_paths *paths, s2b_magnus_session **out);
/* Advance every live path by up to n_windows windows (stops at T). */
int s2b_magnus_session_advance(s2b_magnus_session *s, size_t n_windows);
/* Reset every path to phi at window 0 (reuses all buffers; refused after finish). */
int s2b_magnus_session_reset(s2b_magnus_session *s);
int s2b_magnus_session_stats(const s2b_magnus_session *s, s2b_magnus_stats *stats);
/* Enable CUDA-event timing of every term-kernel launch (accumulated in the stats). */
int s2b_magnus_session_set_timing(s2b_magnus_session *s, int enable);
/* Snapshot of the current state (all paths) as a single-record ensemble at the current time. */
int s2b_magnus_session_ensemble(s2b_magnus_session *s, s2b_ensemble **out);
/* Finish: the ensemble of record times (valid once every path reached T). */
int s2b_magnus_session_finish(s2b_magnus_session *s, s2b_ensemble **out);
/* sum_m u_m and sum_m u_m^2 (2n doubles, host) over live paths at the current time;
 * live_paths (NULL-able) receives the number of non-blown paths. */
int s2b_magnus_session_moments(s2b_magnus_session *s, double *moments, double *live_paths);
int s2b_magnus_session_destroy(s2b_magnus_session *s);

/* ---- ensembles -------------------------------------------------------------- */
/* Upload a host SolutionEnsemble (states [M][n], status [M] 0 Ok; blown rows ignored). */
int s2b_ensemble_create_host(s2b_context *ctx, const s2b_grid *grid, double t, uint64_t seed,
                             size_t M, const double *states, const uint8_t *status,
                             s2b_ensemble **out);
/* info: [0] records, [1] M, [2] n, [3] nx, [4] nv */
int s2b_ensemble_info(const s2b_ensemble *e, int64_t info[5], double *times);
int s2b_ensemble_download(const s2b_ensemble *e, size_t record, double *states, uint8_t *status);
/* Per-path Taylor-term and window counters of a Magnus ensemble (NULL-able outputs). */
int s2b_ensemble_counters(const s2b_ensemble *e, int64_t *terms, int64_t *windows);
int s2b_ensemble_destroy(s2b_ensemble *e);

/* ---- exact solution + norms -------------------------------------------------- */
int s2b_exact_reference(s2b_context *ctx, const s2b_grid *grid, double t, double a,
                        double sigma, const s2b_paths *paths, s2b_ensemble **out);
/* One closed-form field (exact_langevin_field, exact_langevin.hpp:36-41) into host out[n]. */
int s2b_exact_field(s2b_context *ctx, const s2b_grid *grid, double t, double a, double sigma,
                    double W, double IW, double *out);
int s2b_errors(s2b_context *ctx, const s2b_ensemble *ref, size_t ref_record,
               const s2b_ensemble *app, size_t app_record, int kappa, s2b_error_stats *out,
               double *me_out);
/* Fused: exact field at the record's time (a, sigma; path functionals over [0, t]) vs app.
 * per_path_rel (M, NULL-able): ||ref-app||_F/||ref||_F (NaN for blown paths).
 * moments (2n, NULL-able): sum_m u_m and sum_m u_m^2 over non-blown paths. */
int s2b_exact_errors(s2b_context *ctx, const s2b_ensemble *app, size_t app_record, double a,
                     double sigma, const s2b_paths *paths, int kappa, s2b_error_stats *out,
                     double *me_out, double *per_path_rel, double *moments);

/* ---- general expmv ------------------------------------------------------------ */
int s2b_expmv(s2b_context *ctx, const s2b_csr *m, const double *x, double tol, double theta,
              double *y, int report[4]);

/* ---- kernel level: expmv_into with a workspace (sparse.hpp:106-151) ------------
 * s2b_expmv_workspace <- ExpmvWorkspace (sparse.hpp:121-130): caller-owned scratch that
 * caches the device copy of the last pattern (row_ptr / col_idx compared exactly), so a
 * MagnusLogBuilder refill only moves the values.  One cooperative launch per call runs the
 * whole segmented Taylor series (no host round trip per term).
 * s2b_expmv_into <- expmv_into (sparse.hpp:149-151, sparse.cpp:427-503): y = exp(M) x
 * (host x and y, n = m->rows doubles), report as ExpmvReport: status 0 Ok / 1 Overflow /
 * 2 ToleranceNotReached, residual = the achieved last-term/result ratio (max over segments;
 * the last ratio on ToleranceNotReached; +inf on Overflow), segments, max_terms, plus the
 * total Taylor terms applied.  On Overflow / ToleranceNotReached y holds the result of the
 * completed segments, as the reference's y does.
 * s2b_expmv_into_device: the same with x and y in device memory (no copies of the vectors). */
typedef struct s2b_expmv_workspace s2b_expmv_workspace;
typedef struct {
    int status;
    double residual;
    int segments;
    int max_terms;
    int64_t terms;
} s2b_expmv_report;
int s2b_expmv_workspace_create(s2b_context *ctx, s2b_expmv_workspace **out);
int s2b_expmv_workspace_destroy(s2b_expmv_workspace *ws);
int s2b_expmv_into(s2b_expmv_workspace *ws, const s2b_csr *m, const double *x, double tol,
                   double theta, double *y, s2b_expmv_report *report);
int s2b_expmv_into_device(s2b_expmv_workspace *ws, const s2b_csr *m, const double *d_x, double tol,
                          double theta, double *d_y, s2b_expmv_report *report);

/* ---- kernel level: one Euler-Maruyama step (euler.hpp:19-40, euler.cpp:18-86) ------
 * stencils[5] = EulerStencils {inv2dx, invdx2, inv2dv, invdv2, inv4dxdv} as the caller
 * passes them (NULL: EulerStencils::from_grid of the fields' grid).
 * s2b_euler_step <- euler_step_into: out = one explicit step of u (host fields of nx*nv
 * doubles, column-major) with increment dW; *maxabs (NULL-able) = max|out| with the
 * reference's std::max semantics (NaN entries ignored).
 * s2b_euler_step_device: M fields at once in device memory ([M][n] in, [M][n] out), dW[M]
 * and maxabs[M] (NULL-able) on the host. */
int s2b_euler_step(const s2b_fields *f, const double *stencils, const double *u, double *out,
                   double dW, double dt, double *maxabs);
int s2b_euler_step_device(const s2b_fields *f, const double *stencils, const double *d_u,
                          double *d_out, size_t M, const double *dW, double dt, double *maxabs);

/* Moments of one record: sum_m u_m and sum_m u_m^2 over the non-blown paths (2n doubles,
 * host), ascending m per point; live (NULL-able) = the number of non-blown paths. */
int s2b_ensemble_moments(const s2b_ensemble *e, size_t record, double *moments, size_t *live);

/* ---- multi-GPU (one node): path sharding + one NCCL reduction -----------
 * The reference parallelises over paths only (OpenMP, magnus.cpp:258-263,
 * euler.cpp:142-145).  s2b_multi owns one context per listed device and, when the devices
 * are distinct, an NCCL clique over them (ncclCommInitAll; NCCL is loaded at run time).
 * A solve splits the global paths [0, M_total) into contiguous ranges (s2b_shard), runs
 * each range on its device from its own host thread -- operator build, Philox paths keyed
 * by the global path id (path_offset = range start, so results do not depend on the device
 * count), the solver, the per-path norms -- then combines once: ncclAllReduce of the ME sums,
 * counts, moments and counters, ncclAllGather of the per-path errors, so Err is summed in
 * ascending global path order (bitwise the one-device value).  A device listed twice
 * combines on the host instead (same arithmetic; used to test sharding on one GPU). */
typedef struct s2b_multi s2b_multi;
/* Operator / coefficient description built on every device (s2b_operator_build arguments;
 * family 2 = explicit fields9).  a and sigma are also the LangevinParams of the exact norms. */
typedef struct {
    int family;
    double a;
    double sigma;
    const double *const *fields9;
    int order;
} s2b_operator_spec;
typedef struct {
    s2b_error_stats errors; /* combined norms vs the closed form (kappa >= 0) */
    int64_t path_terms;     /* Magnus Taylor terms over all paths */
    int64_t path_windows;
    double max_solve_ms;    /* slowest device's solver time (CUDA events on its stream) */
    size_t M_total;
    int devices;
    int nccl;               /* 1: combined with NCCL, 0: host combine */
} s2b_multi_stats;
/* shard(): contiguous range of `rank` among `world`; the first M % world ranks get one more. */
int s2b_shard(size_t M_total, int rank, int world, size_t *offset, size_t *count);
int s2b_multi_create(const int *devices, int ndev, s2b_multi **out);
int s2b_multi_destroy(s2b_multi *m);
/* info: [0] devices, [1] NCCL clique (1) or host combine (0) */
int s2b_multi_info(const s2b_multi *m, int info[2]);
/* kappa >= 0: norms against exact_reference(a, sigma) over the central region I^kappa (the
 * Langevin families); kappa < 0: moments and counts only.  me_out (w*w), moments_out (2n),
 * per_path_rel_out (M_total, global path order) are NULL-able host buffers. */
int s2b_multi_solve_magnus(s2b_multi *m, const s2b_grid *grid, const s2b_operator_spec *op,
                           const s2b_magnus_config *cfg, const double *phi, double dt_leb,
                           size_t steps, size_t M_total, uint64_t seed, int kappa,
                           s2b_multi_stats *out, double *me_out, double *moments_out,
                           double *per_path_rel_out);
int s2b_multi_solve_euler(s2b_multi *m, const s2b_grid *grid, const s2b_operator_spec *fields,
                          const s2b_euler_config *cfg, const double *phi, double dt_leb,
                          size_t steps, size_t M_total, uint64_t seed, int kappa,
                          s2b_multi_stats *out, double *me_out, double *moments_out,
                          double *per_path_rel_out);

#ifdef __cplusplus
}
#endif
#endif
