// mlnmf_b200_shim.cpp -- the reference's solver API (namespace mlnmf) over the
// B200 C-ABI (include/mlnmf_b200.h).
//
// Drop-in recipe: compile the reference's callers and its
// non-solver sources (matrix.cpp, kernels.cpp, transfer.cpp, cost_model.cpp,
// io.cpp, bench.cpp) unchanged, replace solvers.cpp + multilevel.cpp with
// this file, and link libmlnmf_b200.so.  Every definition below has the
// signature the reference header declares:
//   proj/include/mlnmf/solvers.hpp:45-68    mu_step, hals_step, nnls_active_set, anls_step
//   proj/include/mlnmf/solvers.hpp:90-103   run_solver_phase, run_solver
//   proj/include/mlnmf/multilevel.hpp:22-47 nested_iteration, v_cycle, full_multigrid,
//                                           run_configuration
// Status codes are rethrown as the reference's exception types
// (std::invalid_argument, mlnmf::DataError, mlnmf::NnlsCapExceeded,
// std::runtime_error), so the CLI exit codes are unchanged.
//
// Precision: by default the device runs fp64 in EXACT mode (the reference's
// operation order), i.e. bit-identical results.  MLNMF_B200_FP32=1 selects fp32
// storage with the fastest product path (tcgen05 on large levels).
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "mlnmf/multilevel.hpp"
#include "mlnmf/solvers.hpp"
#include "mlnmf_b200.h"

namespace mlnmf {
namespace {

void check(int rc) {
  if (rc == MLNMF_OK) return;
  const std::string msg = mlnmf_last_error();
  switch (rc) {
    case MLNMF_ERR_INVALID: throw std::invalid_argument(msg);
    case MLNMF_ERR_DATA: throw DataError(msg);
    case MLNMF_ERR_NNLS_CAP: throw NnlsCapExceeded(msg);
    default: throw std::runtime_error(msg);
  }
}

mlnmf_options shim_options() {
  mlnmf_options o;
  mlnmf_default_options(&o);
  const char* fp32 = std::getenv("MLNMF_B200_FP32");
  const bool fast = fp32 && fp32[0] == '1';
  o.dtype = fast ? MLNMF_F32 : MLNMF_F64;
  o.exact = fast ? 0 : 1;
  if (const char* d = std::getenv("MLNMF_B200_DEVICE")) o.device = std::atoi(d);
  return o;
}

void configure_once() {
  static bool done = false;
  if (done) return;
  const mlnmf_options o = shim_options();
  check(mlnmf_set_default_options(&o));
  done = true;
}

// a session owned for one call (destroyed on every exit path)
struct SessionGuard {
  mlnmf_session* s = nullptr;
  ~SessionGuard() {
    if (s) mlnmf_session_destroy(s);
  }
};

int kind_of(SolverKind k) {
  switch (k) {
    case SolverKind::kAnls: return MLNMF_ANLS;
    case SolverKind::kMu: return MLNMF_MU;
    default: return MLNMF_HALS;
  }
}
int cycle_of(CycleKind c) {
  switch (c) {
    case CycleKind::kSingleLevel: return MLNMF_SINGLE_LEVEL;
    case CycleKind::kNestedIteration: return MLNMF_NESTED_ITERATION;
    case CycleKind::kVCycle: return MLNMF_V_CYCLE;
    default: return MLNMF_FULL_MULTIGRID;
  }
}
int mode_of(Budget::Mode m) { return m == Budget::Mode::kWorkUnits ? MLNMF_WORK_UNITS : MLNMF_WALL_CLOCK_SECONDS; }

// mlnmf_trace -> RunTrace (solvers.hpp:14-35); frees the handle
RunTrace take_trace(mlnmf_trace* t) {
  RunTrace out;
  if (!t) return out;
  const size_t ns = mlnmf_trace_num_samples(t);
  std::vector<double> el(ns), wk(ns), er(ns);
  std::vector<int> lv(ns);
  mlnmf_trace_samples(t, el.data(), wk.data(), lv.data(), er.data());
  out.samples.reserve(ns);
  for (size_t i = 0; i < ns; ++i) out.samples.push_back(TraceSample{el[i], wk[i], lv[i], er[i]});
  const size_t na = mlnmf_trace_num_allocations(t);
  std::vector<int> al(na);
  std::vector<double> aa(na);
  mlnmf_trace_allocations(t, al.data(), aa.data());
  for (size_t i = 0; i < na; ++i) out.allocations.push_back(PhaseAllocation{al[i], aa[i]});
  out.nnls_iteration_counts.resize(mlnmf_trace_num_nnls_counts(t));
  mlnmf_trace_nnls_counts(t, out.nnls_iteration_counts.data());
  out.hals_degenerate_columns = mlnmf_trace_degenerate(t);
  mlnmf_trace_free(t);
  return out;
}

void same_shape(const Matrix& M, const Matrix& V, const Matrix& W) {
  if (V.rows() != M.rows() || W.cols() != M.cols() || V.cols() != W.rows())
    throw std::invalid_argument("dimension mismatch");
}

}  // namespace

// ---------------------------------------------------------------- steps
void mu_step(const Matrix& M, Matrix& V, Matrix& W) {
  configure_once();
  same_shape(M, V, W);
  check(mlnmf_mu_step(M.data(), M.rows(), M.cols(), V.data(), W.data(), V.cols()));
}

void hals_step(const Matrix& M, Matrix& V, Matrix& W, int* degenerate) {
  configure_once();
  same_shape(M, V, W);
  check(mlnmf_hals_step(M.data(), M.rows(), M.cols(), V.data(), W.data(), V.cols(), degenerate));
}

NnlsResult nnls_active_set(const Matrix& G, std::span<const double> h, std::span<const double> x0) {
  configure_once();
  const size_t r = h.size();
  if (G.rows() != r || G.cols() != r || x0.size() != r) throw std::invalid_argument("nnls_active_set: dimension mismatch");
  NnlsResult res{std::vector<double>(r, 0.0), 0};
  check(mlnmf_nnls_active_set(G.data(), h.data(), x0.data(), r, res.x.data(), &res.iterations));
  return res;
}

void anls_step(const Matrix& M, Matrix& V, Matrix& W, std::vector<int>* iter_counts) {
  configure_once();
  same_shape(M, V, W);
  std::vector<int> counts(M.rows() + M.cols(), 0);
  check(mlnmf_anls_step(M.data(), M.rows(), M.cols(), V.data(), W.data(), V.cols(), counts.data()));
  if (iter_counts) iter_counts->insert(iter_counts->end(), counts.begin(), counts.end());
}

// ---------------------------------------------------------------- budget loop
// run_solver_phase (solvers.cpp:300-341): M is uploaded ONCE per phase into a
// device session and the whole phase -- the reference's budget loop, its
// samples every trace_every steps and at both ends, the NNLS counts -- runs
// resident through mlnmf_session_run_phase; V and W come back at the end.
// The caller's SolveContext keeps the reference's accounting: work_consumed
// advances by the phase's charges, sample times are ctx-relative, samples
// carry the caller's `level`.
double run_solver_phase(const Matrix& M, Matrix& V, Matrix& W, SolverKind kind, Budget::Mode mode, double amount,
                        double step_flops, int level, std::size_t trace_every, SolveContext& ctx) {
  configure_once();
  same_shape(M, V, W);
  const mlnmf_options o = shim_options();
  SessionGuard g;
  check(mlnmf_session_create(&o, &g.s));
  check(mlnmf_session_set_data(g.s, M.data(), MLNMF_F64, M.rows(), M.cols(), M.cols(), 0, M.rows(), 1));
  check(mlnmf_session_set_factors(g.s, V.data(), W.data(), MLNMF_F64, V.cols()));
  const double t0 = ctx.elapsed_s();
  double wc = ctx.work_consumed, left = 0.0;
  mlnmf_trace* t = nullptr;
  check(mlnmf_session_run_phase(g.s, 0, kind_of(kind), mode_of(mode), amount, step_flops, ctx.unit_flops,
                                trace_every, &wc, &left, &t));
  RunTrace ph = take_trace(t);
  check(mlnmf_session_get_factors(g.s, V.data(), W.data(), MLNMF_F64));
  for (auto& smp : ph.samples) ctx.trace.samples.push_back(TraceSample{t0 + smp.elapsed_s, smp.work_units, level,
                                                                         smp.error});
  ctx.trace.nnls_iteration_counts.insert(ctx.trace.nnls_iteration_counts.end(), ph.nnls_iteration_counts.begin(),
                                         ph.nnls_iteration_counts.end());
  ctx.trace.hals_degenerate_columns += ph.hals_degenerate_columns;
  ctx.work_consumed = wc;
  return left;
}

// ---------------------------------------------------------------- whole runs
SolveResult run_solver(const Matrix& M, const Matrix& V0, const Matrix& W0, SolverKind kind, Budget budget,
                       std::size_t trace_every) {
  configure_once();
  same_shape(M, V0, W0);
  Matrix V(V0.rows(), V0.cols()), W(W0.rows(), W0.cols());
  mlnmf_trace* t = nullptr;
  check(mlnmf_run_solver(M.data(), M.rows(), M.cols(), V0.data(), W0.data(), V0.cols(), kind_of(kind),
                         mode_of(budget.mode), budget.amount, trace_every, V.data(), W.data(), &t));
  return SolveResult{std::move(V), std::move(W), take_trace(t)};
}

#ifndef MLNMF_SHIM_PHASES_ONLY
// (MLNMF_SHIM_PHASES_ONLY: leave the multilevel entries to the reference's
// own multilevel.cpp, whose CycleRunner then drives run_solver_phase above
// -- the `make -C oracle dropin` variant acceptance_b200_phases.)
static MultilevelResult cycle_on(const GridHierarchy& h, std::size_t levels, const Matrix& V0, const Matrix& W0,
                                 SolverKind kind, CycleKind cycle, Budget budget, std::size_t trace_every) {
  configure_once();
  if (h.levels.empty() || h.restricted_data.empty()) throw std::invalid_argument("empty hierarchy");
  const Matrix& M = h.restricted_data[0];
  same_shape(M, V0, W0);
  Matrix V(V0.rows(), V0.cols()), W(W0.rows(), W0.cols());
  mlnmf_trace* t = nullptr;
  check(mlnmf_run_cycle(M.data(), M.rows(), M.cols(), h.levels[0].height, h.levels[0].width, h.levels.size(), levels,
                        V0.data(), W0.data(), V0.cols(), kind_of(kind), cycle_of(cycle), mode_of(budget.mode),
                        budget.amount, trace_every, V.data(), W.data(), &t));
  return MultilevelResult{std::move(V), std::move(W), take_trace(t)};
}

MultilevelResult nested_iteration(const GridHierarchy& h, std::size_t levels, const Matrix& V0, const Matrix& W0,
                                  SolverKind kind, Budget budget, std::size_t trace_every) {
  return cycle_on(h, levels, V0, W0, kind, CycleKind::kNestedIteration, budget, trace_every);
}
MultilevelResult v_cycle(const GridHierarchy& h, std::size_t levels, const Matrix& V0, const Matrix& W0,
                         SolverKind kind, Budget budget, std::size_t trace_every) {
  return cycle_on(h, levels, V0, W0, kind, CycleKind::kVCycle, budget, trace_every);
}
MultilevelResult full_multigrid(const GridHierarchy& h, std::size_t levels, const Matrix& V0, const Matrix& W0,
                                SolverKind kind, Budget budget, std::size_t trace_every) {
  return cycle_on(h, levels, V0, W0, kind, CycleKind::kFullMultigrid, budget, trace_every);
}

MultilevelResult run_configuration(const Matrix& M, const ImageGrid& grid, std::size_t level_count, SolverKind kind,
                                   CycleKind cycle, std::size_t rank, std::uint64_t seed, Budget budget,
                                   std::size_t trace_every) {
  configure_once();
  Matrix V(M.rows(), rank > 0 ? rank : 1), W(rank > 0 ? rank : 1, M.cols());
  mlnmf_trace* t = nullptr;
  check(mlnmf_run_configuration(M.data(), M.rows(), M.cols(), grid.height, grid.width, level_count, kind_of(kind),
                                cycle_of(cycle), rank, seed, mode_of(budget.mode), budget.amount, trace_every,
                                V.data(), W.data(), &t));
  return MultilevelResult{std::move(V), std::move(W), take_trace(t)};
}
#endif  // MLNMF_SHIM_PHASES_ONLY

}  // namespace mlnmf
