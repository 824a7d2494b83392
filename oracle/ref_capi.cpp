// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference library, compiled by
// oracle/Makefile directly from /root/reference/proj/src/*.cpp into
// oracle/_ref/libmlnmf_ref.so.  Used to pin the C restatement
// (mlnmf_oracle.c) and the CUDA product against the reference itself, to
// generate tests/golden/ fixtures, and as bench.py's `--impl reference` /
// cpu_baseline arm.  No reference source is copied here; this file only
// calls the reference's public API (proj/include/mlnmf/*.hpp).
#include <cstring>
#include <exception>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "mlnmf/cost_model.hpp"
#include "mlnmf/io.hpp"
#include "mlnmf/kernels.hpp"
#include "mlnmf/matrix.hpp"
#include "mlnmf/multilevel.hpp"
#include "mlnmf/solvers.hpp"
#include "mlnmf/transfer.hpp"

using namespace mlnmf;

namespace {

thread_local std::string g_err;

// Same status convention as the product and the C restatement.
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const NnlsCapExceeded& e) {
    g_err = e.what();
    return 4;
  } catch (const DataError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

Matrix mat(const double* p, size_t rows, size_t cols) {
  // Matrix::from_data validates (rejects negatives), like the reference's
  // own callers; zero-filled constructor + copy keeps negatives for G/h use.
  Matrix A(rows, cols);
  std::memcpy(A.data(), p, sizeof(double) * rows * cols);
  return A;
}

struct RefTrace {
  std::vector<double> elapsed, work, error, alloc_amount;
  std::vector<int> level, alloc_level, counts;
  int degenerate = 0;
};

RefTrace* to_trace(const RunTrace& t) {
  auto* o = new RefTrace;
  for (const auto& s : t.samples) {
    o->elapsed.push_back(s.elapsed_s);
    o->work.push_back(s.work_units);
    o->level.push_back(s.level);
    o->error.push_back(s.error);
  }
  for (const auto& a : t.allocations) {
    o->alloc_level.push_back(a.level);
    o->alloc_amount.push_back(a.amount);
  }
  o->counts = t.nnls_iteration_counts;
  o->degenerate = t.hals_degenerate_columns;
  return o;
}

SolverKind to_kind(int k) { return static_cast<SolverKind>(k); }
CycleKind to_cycle(int c) { return static_cast<CycleKind>(c); }
Budget budget(int mode, double amount) {
  return {mode == 0 ? Budget::Mode::kWorkUnits : Budget::Mode::kWallClockSeconds,
          amount};
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_random_init(size_t m, size_t n, size_t r, uint64_t seed, double* V,
                    double* W) {
  return guard([&] {
    auto [v, w] = random_init(m, n, r, seed);
    std::memcpy(V, v.data(), sizeof(double) * v.size());
    std::memcpy(W, w.data(), sizeof(double) * w.size());
  });
}

uint64_t ref_splitmix_first(uint64_t seed) { return Rng(seed).next_u64(); }

int ref_frobenius_error(const double* M, const double* V, const double* W,
                        size_t m, size_t n, size_t r, double* out) {
  return guard([&] {
    *out = frobenius_error(mat(M, m, n), mat(V, m, r), mat(W, r, n));
  });
}

double ref_iteration_cost(size_t m, size_t n, size_t r, int kind) {
  return iteration_cost(CostParams::with_default_sr(m, n, r), to_kind(kind));
}

// Dense operator for a grid: which = 0 restriction (coarse x fine), 1
// prolongation (fine x coarse).  out must hold out_dim*in_dim doubles.
int ref_operator_dense(size_t h, size_t w, int which, double* out) {
  return guard([&] {
    const TransferOperator op = which == 0 ? build_restriction({h, w})
                                           : build_prolongation({h, w});
    const Matrix d = op.to_dense();
    std::memcpy(out, d.data(), sizeof(double) * d.size());
  });
}

int ref_smoothness(const double* M, size_t h, size_t w, size_t n, double* out) {
  return guard([&] {
    *out = smoothness(mat(M, h * w, n), build_restriction({h, w}), build_prolongation({h, w}));
  });
}

int ref_initialization_bound(const double* M, size_t h, size_t w, size_t n, const double* Vc,
                             const double* W, size_t r, double* lhs, double* rhs) {
  return guard([&] {
    const ImageGrid c = coarsen_grid({h, w});
    const BoundCheck b = initialization_bound(mat(M, h * w, n), build_restriction({h, w}),
                                              build_prolongation({h, w}), mat(Vc, c.pixels(), r),
                                              mat(W, r, n));
    *lhs = b.lhs;
    *rhs = b.rhs;
  });
}

int ref_apply_operator(size_t h, size_t w, int which, const double* X,
                       size_t ncols, double* Y) {
  return guard([&] {
    const TransferOperator op = which == 0 ? build_restriction({h, w})
                                           : build_prolongation({h, w});
    const Matrix y = op.apply(mat(X, op.in_dim(), ncols));
    std::memcpy(Y, y.data(), sizeof(double) * y.size());
  });
}

int ref_mu_step(const double* M, double* V, double* W, size_t m, size_t n,
                size_t r) {
  return guard([&] {
    Matrix v = mat(V, m, r), w = mat(W, r, n);
    mu_step(mat(M, m, n), v, w);
    std::memcpy(V, v.data(), sizeof(double) * v.size());
    std::memcpy(W, w.data(), sizeof(double) * w.size());
  });
}

int ref_hals_step(const double* M, double* V, double* W, size_t m, size_t n,
                  size_t r, int* degenerate) {
  return guard([&] {
    Matrix v = mat(V, m, r), w = mat(W, r, n);
    hals_step(mat(M, m, n), v, w, degenerate);
    std::memcpy(V, v.data(), sizeof(double) * v.size());
    std::memcpy(W, w.data(), sizeof(double) * w.size());
  });
}

int ref_anls_step(const double* M, double* V, double* W, size_t m, size_t n,
                  size_t r, int* counts) {
  return guard([&] {
    Matrix v = mat(V, m, r), w = mat(W, r, n);
    std::vector<int> c;
    anls_step(mat(M, m, n), v, w, &c);
    std::memcpy(V, v.data(), sizeof(double) * v.size());
    std::memcpy(W, w.data(), sizeof(double) * w.size());
    if (counts) std::memcpy(counts, c.data(), sizeof(int) * c.size());
  });
}

int ref_nnls_active_set(const double* G, const double* h, const double* x0,
                        size_t r, double* x, int* iters) {
  return guard([&] {
    Matrix g(r, r);
    std::memcpy(g.data(), G, sizeof(double) * r * r);
    const NnlsResult res = nnls_active_set(
        g, std::span<const double>(h, r), std::span<const double>(x0, r));
    std::memcpy(x, res.x.data(), sizeof(double) * r);
    *iters = res.iterations;
  });
}

int ref_run_configuration(const double* M, size_t m, size_t n, size_t h,
                          size_t w, size_t level_count, int kind, int cycle,
                          size_t rank, uint64_t seed, int mode, double amount,
                          size_t trace_every, double* V, double* W,
                          void** trace_out) {
  *trace_out = nullptr;
  return guard([&] {
    const MultilevelResult res = run_configuration(
        mat(M, m, n), ImageGrid{h, w}, level_count, to_kind(kind),
        to_cycle(cycle), rank, seed, budget(mode, amount), trace_every);
    std::memcpy(V, res.V.data(), sizeof(double) * res.V.size());
    std::memcpy(W, res.W.data(), sizeof(double) * res.W.size());
    *trace_out = to_trace(res.trace);
  });
}

int ref_run_solver(const double* M, size_t m, size_t n, size_t r, double* V,
                   double* W, int kind, int mode, double amount,
                   size_t trace_every, void** trace_out) {
  *trace_out = nullptr;
  return guard([&] {
    const SolveResult res =
        run_solver(mat(M, m, n), mat(V, m, r), mat(W, r, n), to_kind(kind),
                   budget(mode, amount), trace_every);
    std::memcpy(V, res.V.data(), sizeof(double) * res.V.size());
    std::memcpy(W, res.W.data(), sizeof(double) * res.W.size());
    *trace_out = to_trace(res.trace);
  });
}

// nested_iteration / v_cycle / full_multigrid on a hierarchy of
// hierarchy_levels levels with `levels` in play (multilevel.hpp:22-38).
int ref_run_cycle_on(const double* M, size_t m, size_t n, size_t h, size_t w,
                     size_t hierarchy_levels, size_t levels, const double* V0,
                     const double* W0, size_t r, int kind, int cycle, int mode,
                     double amount, size_t trace_every, double* V, double* W,
                     void** trace_out) {
  *trace_out = nullptr;
  return guard([&] {
    const GridHierarchy hh =
        GridHierarchy::build(mat(M, m, n), ImageGrid{h, w}, hierarchy_levels);
    const Matrix v0 = mat(V0, m, r), w0 = mat(W0, r, n);
    const Budget b = budget(mode, amount);
    MultilevelResult res;
    switch (to_cycle(cycle)) {
      case CycleKind::kNestedIteration:
        res = nested_iteration(hh, levels, v0, w0, to_kind(kind), b, trace_every);
        break;
      case CycleKind::kVCycle:
        res = v_cycle(hh, levels, v0, w0, to_kind(kind), b, trace_every);
        break;
      case CycleKind::kFullMultigrid:
        res = full_multigrid(hh, levels, v0, w0, to_kind(kind), b, trace_every);
        break;
      default:
        throw std::invalid_argument("ref_run_cycle_on: cycle must be ni/vc/fmg");
    }
    std::memcpy(V, res.V.data(), sizeof(double) * res.V.size());
    std::memcpy(W, res.W.data(), sizeof(double) * res.W.size());
    *trace_out = to_trace(res.trace);
  });
}

// synth_smooth_dataset (io.cpp:297-339): only used to regenerate the
// acceptance-criterion-8 golden dataset (tests/golden/make_golden.py).
int ref_synth_smooth_dataset(size_t h, size_t w, size_t n, size_t blobs, uint64_t seed, double* M_out) {
  return guard([&] {
    const Dataset d = synth_smooth_dataset(h, w, n, blobs, seed);
    std::memcpy(M_out, d.matrix.data(), sizeof(double) * d.matrix.size());
  });
}

size_t ref_trace_n_samples(void* t) { return static_cast<RefTrace*>(t)->error.size(); }
size_t ref_trace_n_alloc(void* t) { return static_cast<RefTrace*>(t)->alloc_level.size(); }
size_t ref_trace_n_counts(void* t) { return static_cast<RefTrace*>(t)->counts.size(); }
int ref_trace_degenerate(void* t) { return static_cast<RefTrace*>(t)->degenerate; }
void ref_trace_copy(void* tp, double* elapsed, double* work, int* level,
                    double* error, int* alloc_level, double* alloc_amount,
                    int* counts) {
  const RefTrace* t = static_cast<RefTrace*>(tp);
  std::memcpy(elapsed, t->elapsed.data(), sizeof(double) * t->elapsed.size());
  std::memcpy(work, t->work.data(), sizeof(double) * t->work.size());
  std::memcpy(level, t->level.data(), sizeof(int) * t->level.size());
  std::memcpy(error, t->error.data(), sizeof(double) * t->error.size());
  std::memcpy(alloc_level, t->alloc_level.data(), sizeof(int) * t->alloc_level.size());
  std::memcpy(alloc_amount, t->alloc_amount.data(), sizeof(double) * t->alloc_amount.size());
  if (counts) std::memcpy(counts, t->counts.data(), sizeof(int) * t->counts.size());
}
void ref_trace_free(void* t) { delete static_cast<RefTrace*>(t); }

}  // extern "C"
