/* mlnmf_oracle.h -- TEST INFRASTRUCTURE ONLY (see mlnmf_oracle.c header).
 * Serial C restatement of the reference mlnmf solver path, used as the
 * checker for the CUDA product.  Status codes mirror the reference's
 * exception classes / CLI exit codes (proj/tools/mlnmf_main.cpp:214-233). */
#ifndef MLNMF_ORACLE_H_
#define MLNMF_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_ERUNTIME = 1, ORC_EINVAL = 2, ORC_EDATA = 3, ORC_ENNLSCAP = 4 };
/* SolverKind order as proj/include/mlnmf/cost_model.hpp:9 */
enum { ORC_ANLS = 0, ORC_MU = 1, ORC_HALS = 2 };
/* CycleKind order as proj/include/mlnmf/multilevel.hpp:11 */
enum { ORC_CYCLE_NONE = 0, ORC_CYCLE_NI = 1, ORC_CYCLE_VC = 2, ORC_CYCLE_FMG = 3 };

typedef struct {
  size_t out_dim, in_dim;
  size_t* row_ptr; /* out_dim + 1 */
  size_t* idx;
  double* wt;
} orc_op;

typedef struct {
  size_t n_samples, cap_samples;
  double* elapsed;
  double* work;
  int* level;
  double* error;
  size_t n_alloc;
  int* alloc_level;
  double* alloc_amount;
  size_t n_counts;
  int* counts;
  int hals_degenerate;
  size_t n_phases; /* not in the reference RunTrace: steps per phase */
  int* phase_level;
  long* phase_steps;
} orc_trace;

uint64_t orc_splitmix_next(uint64_t* state);
double orc_splitmix_uniform(uint64_t* state);
int orc_random_init(size_t m, size_t n, size_t r, uint64_t seed, double* V, double* W);

void orc_matmul_ab(const double* A, const double* B, double* C, size_t m, size_t k, size_t n);
void orc_matmul_abt(const double* A, const double* B, double* C, size_t m, size_t n, size_t r);
void orc_matmul_atb(const double* A, const double* B, double* C, size_t m, size_t r, size_t n);
double orc_frobenius_error(const double* M, const double* V, const double* W, size_t m, size_t n, size_t r);
double orc_frobenius_norm(const double* A, size_t count);
double orc_iteration_cost(size_t m, size_t n, size_t r, int kind);

int orc_coarsen(size_t h, size_t w, size_t* hc, size_t* wc);
orc_op* orc_build_restriction(size_t h, size_t w);
orc_op* orc_build_prolongation(size_t h, size_t w);
void orc_op_apply(const orc_op* op, const double* X, size_t ncols, double* Y);
void orc_op_free(orc_op* op);
double orc_op_frobenius_norm(const orc_op* op);
int orc_smoothness(const double* M, size_t h, size_t w, size_t n, double* out);
int orc_initialization_bound(const double* M, size_t h, size_t w, size_t n, const double* Vc,
                             const double* W, size_t r, double* lhs, double* rhs);

void orc_mu_step(const double* M, double* V, double* W, size_t m, size_t n, size_t r);
void orc_hals_step(const double* M, double* V, double* W, size_t m, size_t n, size_t r, int* degenerate);
int orc_nnls_active_set(const double* G, const double* h, const double* x0, size_t r, double* x, int* iters);
int orc_anls_step(const double* M, double* V, double* W, size_t m, size_t n, size_t r, int* counts);

int orc_run_configuration(const double* M, size_t m, size_t n, size_t h, size_t w,
                          size_t level_count, int kind, int cycle, size_t rank,
                          uint64_t seed, int mode, double amount, size_t trace_every,
                          double* V, double* W, orc_trace** out);
int orc_run_solver(const double* M, size_t m, size_t n, size_t r, double* V, double* W,
                   int kind, int mode, double amount, size_t trace_every, orc_trace** out);
int orc_run_cycle_on(const double* M, size_t m, size_t n, size_t h, size_t w,
                     size_t hierarchy_levels, size_t levels, const double* V0,
                     const double* W0, size_t r, int kind, int cycle, int mode,
                     double amount, size_t trace_every, double* V, double* W,
                     orc_trace** out);
void orc_trace_free(orc_trace* t);

/* Synthetic BASELINE.json generator (host twin of the product's device
 * generator; spec in DESIGN.md section 3).  M (m x n_cols) row-major for
 * columns [col0, col0 + n_cols) of an n_total-column dataset. */
typedef struct {
  size_t h, w, r, blobs;
  double sigma_min, sigma_max;
  int noise_kind; /* 0 = uniform noise_scale*U[0,1), 1 = gaussian N(0, noise_scale^2) */
  double noise_scale;
  uint64_t seed;
} orc_gen_params;
void orc_generate(const orc_gen_params* p, size_t n_total, size_t col0, size_t n_cols, double* M);

#ifdef __cplusplus
}
#endif
#endif
