/*
 * mlnmf_b200.h -- C-ABI of the B200-native multilevel NMF solver.
 *
 * Drop-in boundary for the reference library `mlnmf` (/root/reference/proj).
 * The reference has no FFI; its boundary is the public C++ headers
 * proj/include/mlnmf/{matrix,solvers,multilevel,transfer,cost_model}.hpp.
 * Every entry point below cites the reference declaration it replaces.
 * Plain pointers and sizes only: matrices are caller-owned, row-major
 * (element (i,j) at i*cols + j, proj/include/mlnmf/matrix.hpp:47-52);
 * M is m x n (one column per vectorized image, pixel (i,j) of an h x w image at
 * row j*h + i, transfer.hpp:15-20), V is m x r, W is r x n.
 *
 * Errors: every int-returning call returns a status; the message of the last
 * failure on the calling thread is mlnmf_last_error().  The codes mirror the
 * reference's exception classes and its CLI exit codes
 * (proj/tools/mlnmf_main.cpp:214-233):
 *   MLNMF_ERR_INVALID  std::invalid_argument   (exit 2)
 *   MLNMF_ERR_DATA     mlnmf::DataError        (exit 3)
 *   MLNMF_ERR_NNLS_CAP mlnmf::NnlsCapExceeded  (exit 4)
 *   MLNMF_ERR_RUNTIME  std::runtime_error, CUDA and NCCL failures (exit 1)
 *
 * Threading: a session is single-owner and not thread-safe (the reference is
 * one logical thread per run).  The one-shot reference-shaped
 * calls use a per-thread default session.
 */
#ifndef MLNMF_B200_H_
#define MLNMF_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MLNMF_B200_VERSION 1

enum {
  MLNMF_OK = 0,
  MLNMF_ERR_RUNTIME = 1,
  MLNMF_ERR_INVALID = 2,
  MLNMF_ERR_DATA = 3,
  MLNMF_ERR_NNLS_CAP = 4
};

/* SolverKind (proj/include/mlnmf/cost_model.hpp:9) */
enum { MLNMF_ANLS = 0, MLNMF_MU = 1, MLNMF_HALS = 2 };
/* CycleKind (proj/include/mlnmf/multilevel.hpp:11) */
enum { MLNMF_SINGLE_LEVEL = 0, MLNMF_NESTED_ITERATION = 1, MLNMF_V_CYCLE = 2, MLNMF_FULL_MULTIGRID = 3 };
/* Budget::Mode (proj/include/mlnmf/solvers.hpp:37-41) */
enum { MLNMF_WORK_UNITS = 0, MLNMF_WALL_CLOCK_SECONDS = 1 };
/* storage / host buffer element types */
enum { MLNMF_F32 = 0, MLNMF_F64 = 1 };
/* M-streaming product implementation */
enum { MLNMF_GEMM_AUTO = 0, MLNMF_GEMM_SIMT = 1, MLNMF_GEMM_TCGEN05 = 2 };
/* error-sample implementation */
enum { MLNMF_ERROR_AUTO = 0, MLNMF_ERROR_GRAM = 1, MLNMF_ERROR_DIRECT = 2 };

typedef struct mlnmf_session mlnmf_session;
typedef struct mlnmf_trace mlnmf_trace;

typedef struct {
  int device;      /* CUDA device ordinal */
  int dtype;       /* MLNMF_F32 / MLNMF_F64 storage of M, V, W on the device */
  int exact;       /* 1: the reference's operation order (fp64 runs bit-identical) */
  int gemm_path;   /* MLNMF_GEMM_* */
  int error_mode;  /* MLNMF_ERROR_* */
  int world;       /* ranks sharing the problem (columns of M sharded) */
  int rank;        /* this rank */
  const void* nccl_id; /* 128-byte ncclUniqueId when world > 1 */
} mlnmf_options;

/* Synthetic BASELINE.json data generator. */
typedef struct {
  size_t h, w, r, blobs;
  double sigma_min, sigma_max;
  int noise_kind; /* 0: noise_scale * U[0,1); 1: N(0, noise_scale^2) */
  double noise_scale;
  uint64_t seed;
  int scale_to_unit; /* divide M by its global maximum */
} mlnmf_gen_params;

const char* mlnmf_last_error(void);
int mlnmf_version(void);
void mlnmf_default_options(mlnmf_options* o);
/* Options of the per-thread default session behind the one-shot calls. */
int mlnmf_set_default_options(const mlnmf_options* o);
int mlnmf_nccl_unique_id(void* out128);

/* ---------------------------------------------------------------------------
 * One-shot, reference-shaped calls (host fp64 buffers; H2D/D2H per call).
 * ------------------------------------------------------------------------- */

/* run_configuration (proj/include/mlnmf/multilevel.hpp:43-47).  V_out (m x r)
 * and W_out (r x n) receive the factors; *trace_out a trace to free with
 * mlnmf_trace_free (may be NULL). */
int mlnmf_run_configuration(const double* M, size_t m, size_t n, size_t grid_h, size_t grid_w,
                            size_t level_count, int kind, int cycle, size_t rank, uint64_t seed,
                            int budget_mode, double budget_amount, size_t trace_every, double* V_out,
                            double* W_out, mlnmf_trace** trace_out);

/* nested_iteration / v_cycle / full_multigrid (multilevel.hpp:22-38) on the
 * hierarchy GridHierarchy::build(M, grid, hierarchy_levels) with `levels` in
 * play, from caller factors V0 (m x r), W0 (r x n).  cycle selects which. */
int mlnmf_run_cycle(const double* M, size_t m, size_t n, size_t grid_h, size_t grid_w,
                    size_t hierarchy_levels, size_t levels, const double* V0, const double* W0, size_t r,
                    int kind, int cycle, int budget_mode, double budget_amount, size_t trace_every,
                    double* V_out, double* W_out, mlnmf_trace** trace_out);

/* run_solver (proj/include/mlnmf/solvers.hpp:101-103). */
int mlnmf_run_solver(const double* M, size_t m, size_t n, const double* V0, const double* W0, size_t r,
                     int kind, int budget_mode, double budget_amount, size_t trace_every, double* V_out,
                     double* W_out, mlnmf_trace** trace_out);

/* mu_step / hals_step / anls_step (solvers.hpp:45-68); V, W updated in place.
 * degenerate: incremented per degenerate diagonal (may be NULL).
 * iter_counts: m + n exchange counts (may be NULL). */
int mlnmf_mu_step(const double* M, size_t m, size_t n, double* V, double* W, size_t r);
int mlnmf_hals_step(const double* M, size_t m, size_t n, double* V, double* W, size_t r, int* degenerate);
int mlnmf_anls_step(const double* M, size_t m, size_t n, double* V, double* W, size_t r, int* iter_counts);

/* nnls_active_set (solvers.hpp:61-63): G r x r, h and x0 length r. */
int mlnmf_nnls_active_set(const double* G, const double* h, const double* x0, size_t r, double* x,
                          int* iterations);

/* frobenius_error (matrix.hpp:99-101) */
int mlnmf_frobenius_error(const double* M, const double* V, const double* W, size_t m, size_t n, size_t r,
                          double* out);
/* random_init (matrix.hpp:106-107) */
int mlnmf_random_init(size_t m, size_t n, size_t r, uint64_t seed, double* V_out, double* W_out);
/* restrict_columns / prolong_columns (transfer.hpp:68-69) with the operators
 * build_restriction / build_prolongation(fine grid h x w) (transfer.hpp:60-66):
 * X is (h*w) x ncols (restrict) or (ceil(h/2)*ceil(w/2)) x ncols (prolong). */
int mlnmf_restrict_columns(size_t grid_h, size_t grid_w, const double* X, size_t ncols, double* Y);
int mlnmf_prolong_columns(size_t grid_h, size_t grid_w, const double* X, size_t ncols, double* Y);
/* smoothness (transfer.hpp:75-76, transfer.cpp:128-141) with R, P =
 * build_restriction / build_prolongation(grid h x w): M is (h*w) x n.
 * MLNMF_ERR_INVALID for the zero matrix. */
int mlnmf_smoothness(const double* M, size_t m, size_t n, size_t grid_h, size_t grid_w, double* out);
/* initialization_bound (transfer.hpp:85-87, transfer.cpp:143-153):
 * lhs = ||M - P(V_coarse) W||_F, rhs = s_M ||M||_F + ||P||_F ||R(M) - V_coarse W||_F;
 * V_coarse is (ceil(h/2)*ceil(w/2)) x r, W is r x n. */
int mlnmf_initialization_bound(const double* M, size_t m, size_t n, size_t grid_h, size_t grid_w,
                               const double* V_coarse, const double* W, size_t r, double* lhs, double* rhs);
/* run_bench's runs loop (proj/include/mlnmf/bench.hpp:34, proj/src/bench.cpp:28-84):
 * final_errors[i] = run_configuration(M, grid, level_count, kind, cycle, rank,
 * base_seed + i, budget, trace_every = 0).trace.final_error() for i < runs,
 * batched over `workers` concurrent device sessions (0 = 8).  opt: storage and
 * precision of the sessions (NULL = the one-shot defaults); single rank. */
int mlnmf_run_seeds(const mlnmf_options* opt, const double* M, size_t m, size_t n, size_t grid_h, size_t grid_w,
                    size_t level_count, int kind, int cycle, size_t rank, uint64_t base_seed, size_t runs,
                    int budget_mode, double budget_amount, size_t workers, double* final_errors);
/* Dry run of the host scheduler (no device work): the phase allocations,
 * steps per phase and the (work_units, level) stamps of every trace sample a
 * work-unit-budget run_configuration on an h x w grid with n columns would
 * produce (multilevel.cpp:116-132 + solvers.cpp:300-341).  Sample errors and
 * times are zero. */
int mlnmf_plan_configuration(size_t grid_h, size_t grid_w, size_t n, size_t level_count, int kind, int cycle,
                             size_t rank, double budget_amount, size_t trace_every, mlnmf_trace** trace_out);
/* iteration_cost (cost_model.hpp:36) with CostParams::with_default_sr */
double mlnmf_iteration_cost(size_t m, size_t n, size_t r, int kind);

/* ---------------------------------------------------------------------------
 * Sessions: device-resident data, fp32 storage, column sharding over ranks.
 * ------------------------------------------------------------------------- */
int mlnmf_session_create(const mlnmf_options* o, mlnmf_session** out);
/* A rank of a world > 1 problem whose collectives go through the caller
 * instead of NCCL: fn(ctx, buf, count, op) receives this rank's `count`
 * doubles in host memory and must leave there the element-wise sum (op 0) or
 * max (op 1) over all ranks; every rank issues the same sequence of calls.
 * Used to run several ranks (sessions) in one process -- e.g. on one GPU for
 * the multi-rank parity tests -- with no device-side waits between them.
 * options->nccl_id must be NULL. */
typedef int (*mlnmf_host_allreduce_fn)(void* ctx, double* buf, size_t count, int op);
int mlnmf_session_create_host_comm(const mlnmf_options* o, mlnmf_host_allreduce_fn fn, void* ctx,
                                   mlnmf_session** out);
void mlnmf_session_destroy(mlnmf_session* s);
/* M_local: m x n_local row-major host buffer (host_dtype MLNMF_F32/F64),
 * columns [col0, col0 + n_local) of an n_total-column problem.  Validated like
 * Matrix::from_data (matrix.cpp:10-22). */
int mlnmf_session_set_data(mlnmf_session* s, const void* M_local, int host_dtype, size_t m, size_t n_local,
                           size_t n_total, size_t col0, size_t grid_h, size_t grid_w);
int mlnmf_session_generate(mlnmf_session* s, const mlnmf_gen_params* g, size_t n_total, size_t col0,
                           size_t n_local);
int mlnmf_session_run_configuration(mlnmf_session* s, size_t level_count, int kind, int cycle, size_t rank,
                                    uint64_t seed, int budget_mode, double budget_amount, size_t trace_every,
                                    mlnmf_trace** trace_out);
int mlnmf_session_run_cycle(mlnmf_session* s, size_t hierarchy_levels, size_t levels, const void* V0,
                            const void* W0_local, int host_dtype, size_t r, int kind, int cycle,
                            int budget_mode, double budget_amount, size_t trace_every, mlnmf_trace** trace_out);
/* level-0 factors: V (m x r), this rank's W columns (r x n_local) */
int mlnmf_session_get_factors(mlnmf_session* s, void* V, void* W_local, int host_dtype);
int mlnmf_session_set_factors(mlnmf_session* s, const void* V, const void* W_local, int host_dtype, size_t r);
/* ---- resident per-level entries: the pieces of a multilevel cycle on the
 * session's device-resident pyramid (SURVEY 8(b) minimum), so a caller that
 * drives its own cycle (the reference's CycleRunner, multilevel.cpp:14-89, or
 * the drop-in shim's run_solver_phase) never re-uploads M. ---- */
/* GridHierarchy::build (transfer.cpp:155-174) up to level_count levels on the
 * device: R(M) restricted column-locally, no communication. */
int mlnmf_session_build_levels(mlnmf_session* s, size_t level_count);
size_t mlnmf_session_num_levels(mlnmf_session* s);
/* ImageGrid of a built level (coarsen_grid, transfer.cpp:55-59) */
int mlnmf_session_level_shape(mlnmf_session* s, size_t level, size_t* grid_h, size_t* grid_w);
/* random_init(m, n_total, r, seed) at level 0 on the device (matrix.cpp:51-60;
 * each rank draws its own W columns) */
int mlnmf_session_init_random(mlnmf_session* s, size_t r, uint64_t seed);
/* V at `level` (m_level x r) and this rank's W columns (r x n_local) */
int mlnmf_session_set_factors_level(mlnmf_session* s, size_t level, const void* V, const void* W_local,
                                    int host_dtype, size_t r);
int mlnmf_session_get_factors_level(mlnmf_session* s, size_t level, void* V, void* W_local, int host_dtype);
/* V_{level+1} = R_level V_level and V_level = P_level V_{level+1}
 * (multilevel.cpp:39,41 -- CycleRunner::nested / vcycle / fmg) */
int mlnmf_session_restrict_V(mlnmf_session* s, size_t level);
int mlnmf_session_prolong_V(mlnmf_session* s, size_t level);
/* run_solver_phase (solvers.hpp:90-92, solvers.cpp:300-341) on the resident
 * level: kind MLNMF_MU/HALS/ANLS, budget_mode MLNMF_WORK_UNITS (amount work
 * units, each step charged step_flops / unit_flops) or
 * MLNMF_WALL_CLOCK_SECONDS; samples at start, every trace_every steps and at
 * the end, stamped with *work_consumed (the run's cumulative work units,
 * advanced in place, SolveContext::work_consumed).  *leftover = the
 * unconsumed amount (the reference's return value).  The phase trace holds
 * the samples (level = level + 1, times relative to the phase start), the
 * NNLS counts, degenerate columns and the phase's step count. */
int mlnmf_session_run_phase(mlnmf_session* s, size_t level, int kind, int budget_mode, double amount,
                            double step_flops, double unit_flops, size_t trace_every, double* work_consumed,
                            double* leftover, mlnmf_trace** trace_out);
/* Enqueue n_steps solver sweeps at level 0 with no error samples (bench). */
int mlnmf_session_steps(mlnmf_session* s, int kind, size_t n_steps);
int mlnmf_session_sync(mlnmf_session* s);
int mlnmf_session_error(mlnmf_session* s, double* out); /* ||M - VW||_F at level 0, all ranks */
int mlnmf_session_norm2(mlnmf_session* s, size_t level, double* out); /* ||M_level||_F^2, all ranks */
/* Diagnostics over the resident pyramid, all ranks (transfer.cpp:128-153):
 * s_M of level `level`, and both sides of the initialization bound for
 * V_coarse (level+1 rows x r) and this rank's W columns (r x n_local).  The
 * bound call leaves V_coarse at level+1, P V_coarse at `level` and W as the
 * session's factors. */
int mlnmf_session_smoothness(mlnmf_session* s, size_t level, double* out);
int mlnmf_session_initialization_bound(mlnmf_session* s, size_t level, const void* V_coarse, const void* W_local,
                                       int host_dtype, size_t r, double* lhs, double* rhs);
/* The two M-streaming products at level 0 with the current factors, through
 * the active implementation: A = M W^T (m x r) and C = V^T M (r x n_local),
 * fp64 host buffers (either may be NULL).  Note: A is this rank's partial
 * (not allreduced). */
int mlnmf_session_products(mlnmf_session* s, double* A, double* C);
/* B = W W^T (r x r, fp64 host buffer) of this rank's W shard through the active implementation
 * (kernels::matmul_abt with X = Y = W, kernels.cpp:24-34); not allreduced. */
int mlnmf_session_gram_w(mlnmf_session* s, double* B);
/* D = V^T V (r x r, fp64 host buffer) of the level-0 V through the active implementation
 * (kernels::matmul_atb with X = V, kernels.cpp:36-46). */
int mlnmf_session_gram_v(mlnmf_session* s, double* D);
/* copy this rank's level-0 M (m x n_local) to a host buffer */
int mlnmf_session_export_data(mlnmf_session* s, void* M_local, int host_dtype);
/* copy this rank's level-`level` data R(...R(M)) (m_level x n_local; GridHierarchy::levels[level].data,
 * transfer.hpp:60-70) to a host buffer of the level's storage type: *level_dtype (0 = fp32, 1 = fp64) is
 * written first; with M_level == NULL only the type is reported.  Restricted levels of an fp32 session are
 * fp32 where the tensor path streams them and fp64 otherwise. */
int mlnmf_session_export_level(mlnmf_session* s, size_t level, void* M_level, int* level_dtype);
int mlnmf_session_set_profiling(mlnmf_session* s, int on);
int mlnmf_session_kernel_times(mlnmf_session* s, double* mwt_ms, long* mwt_n, double* vtm_ms, long* vtm_n);
/* profiled time of the per-step NCCL allreduce of [M W^T | W W^T] (world > 1;
 * 0 calls on one rank), CUDA events on the engine stream */
int mlnmf_session_comm_time(mlnmf_session* s, double* ms, long* count);
/* profiled time of each phase of the profiled solver steps, 7 entries in
 * step order: B = W W^T, A = M W^T, allreduce [A | B], V update, D = V^T V,
 * C = V^T M, W update (total ms and number of timed intervals per phase;
 * CUDA events on the engine stream).  B200 instrumentation, no reference
 * counterpart. */
#define MLNMF_NUM_PHASES 7
int mlnmf_session_phase_times(mlnmf_session* s, double* ms, long* count);
long mlnmf_session_launches(mlnmf_session* s);
void* mlnmf_session_stream(mlnmf_session* s);
/* 1 if the tcgen05 path serves the M-streaming products */
int mlnmf_session_tc_active(mlnmf_session* s);
int mlnmf_session_gram_error(mlnmf_session* s);

/* ---------------------------------------------------------------------------
 * Dataset and result I/O (proj/include/mlnmf/io.hpp), host only; the same code
 * and byte formats as the mlnmf_b200 CLI.  Errors: MLNMF_ERR_DATA with the
 * reference's message texts (file name, byte offset / row / column).
 * ------------------------------------------------------------------------- */
/* load_pgm_dir (io.hpp:46-48, io.cpp:118-144): every P5 file of `dir` in
 * byte-wise filename order as one column; *M_out (m x n, row-major, pixel
 * (i,j) of an h x w image at row j*h + i) is released with mlnmf_free */
int mlnmf_load_pgm_dir(const char* dir, double** M_out, size_t* m, size_t* n, size_t* h, size_t* w);
/* load_csv (io.hpp:50-51, io.cpp:146-187) */
int mlnmf_load_csv(const char* path, double** M_out, size_t* m, size_t* n);
/* save_matrix_csv / save_trace_csv (io.hpp:53-58): %.17g, header
 * "elapsed_s,work_units,level,error" for traces */
int mlnmf_save_matrix_csv(const double* A, size_t rows, size_t cols, const char* path);
int mlnmf_save_trace_csv(const mlnmf_trace* t, const char* path);
/* save_basis_mosaic (io.hpp:60-63): basis_kkk.pgm per column of V + mosaic.pgm */
int mlnmf_save_basis_mosaic(const double* V, size_t m, size_t r, size_t grid_h, size_t grid_w, const char* dir);
/* synth_smooth_dataset (io.hpp:69-75): M_out is (h*w) x n, caller-allocated */
int mlnmf_synth_smooth_dataset(size_t h, size_t w, size_t n, size_t blobs, uint64_t seed, double* M_out);
void mlnmf_free(void* p);

/* ---------------------------------------------------------------------------
 * Traces: RunTrace (proj/include/mlnmf/solvers.hpp:14-35).
 * ------------------------------------------------------------------------- */
size_t mlnmf_trace_num_samples(const mlnmf_trace* t);
void mlnmf_trace_samples(const mlnmf_trace* t, double* elapsed_s, double* work_units, int* level,
                         double* error);
size_t mlnmf_trace_num_allocations(const mlnmf_trace* t);
void mlnmf_trace_allocations(const mlnmf_trace* t, int* level, double* amount);
size_t mlnmf_trace_num_nnls_counts(const mlnmf_trace* t);
void mlnmf_trace_nnls_counts(const mlnmf_trace* t, int* counts);
int mlnmf_trace_degenerate(const mlnmf_trace* t);
size_t mlnmf_trace_num_phases(const mlnmf_trace* t);
void mlnmf_trace_phases(const mlnmf_trace* t, int* level, long* steps);
void mlnmf_trace_free(mlnmf_trace* t);

#ifdef __cplusplus
}
#endif
#endif /* MLNMF_B200_H_ */
