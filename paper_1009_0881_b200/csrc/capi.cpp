// capi.cpp -- the extern "C" boundary (include/mlnmf_b200.h) over the device
// Engine and the host scheduler.  C++ exceptions become status codes with a
// per-thread message, mirroring the reference's exception classes.
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>
#include <algorithm>
#include <thread>

#include "../../include/mlnmf_b200.h"
#include "engine.hpp"
#include "host_io.hpp"
#include "nccl_shim.hpp"
#include "scheduler.hpp"

using namespace mlb;

struct mlnmf_session {
  std::unique_ptr<Engine> e;
};
struct mlnmf_trace {
  RunTrace t;
};

namespace {

thread_local std::string g_err;
thread_local mlnmf_options g_default = {0, MLNMF_F64, 0, MLNMF_GEMM_AUTO, MLNMF_ERROR_AUTO, 1, 0, nullptr};
thread_local std::map<std::tuple<int, int, int, int, int>, std::unique_ptr<Engine>> g_sessions;

template <class F>
int guard(F&& f) {
  try {
    f();
    return MLNMF_OK;
  } catch (const NnlsCapExceeded& ex) {
    g_err = ex.what();
    return MLNMF_ERR_NNLS_CAP;
  } catch (const DataError& ex) {
    g_err = ex.what();
    return MLNMF_ERR_DATA;
  } catch (const io::DataError& ex) {  // dataset / result I/O (host_io.cpp)
    g_err = ex.what();
    return MLNMF_ERR_DATA;
  } catch (const std::invalid_argument& ex) {
    g_err = ex.what();
    return MLNMF_ERR_INVALID;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return MLNMF_ERR_RUNTIME;
  } catch (...) {
    g_err = "unknown error";
    return MLNMF_ERR_RUNTIME;
  }
}

Options to_opts(const mlnmf_options* o) {
  Options x;
  if (!o) return x;
  x.device = o->device;
  x.dtype = o->dtype;
  x.exact = o->exact;
  x.gemm = o->gemm_path;
  x.error_mode = o->error_mode;
  x.world = o->world < 1 ? 1 : o->world;
  x.rank = o->rank;
  if (o->nccl_id) {
    x.has_nccl_id = true;
    std::memcpy(x.nccl_id, o->nccl_id, 128);
  }
  return x;
}

// Per-thread default session of the one-shot calls (single rank).
Engine& default_engine() {
  const mlnmf_options& o = g_default;
  auto key = std::make_tuple(o.device, o.dtype, o.exact, o.gemm_path, o.error_mode);
  auto it = g_sessions.find(key);
  if (it != g_sessions.end()) return *it->second;
  mlnmf_options single = o;
  single.world = 1;
  single.rank = 0;
  single.nccl_id = nullptr;
  auto e = std::make_unique<Engine>(to_opts(&single));
  Engine& ref = *e;
  g_sessions.emplace(key, std::move(e));
  return ref;
}

Kind to_kind(int k) {
  if (k < 0 || k > 2) throw std::invalid_argument("unknown solver kind");
  return static_cast<Kind>(k);
}
Cycle to_cycle(int c) {
  if (c < 0 || c > 3) throw std::invalid_argument("unknown cycle kind");
  return static_cast<Cycle>(c);
}

void check_dims(size_t m, size_t n, size_t r) {
  if (m == 0 || n == 0 || r == 0) throw std::invalid_argument("Matrix: dimensions must be positive");
}

void emit_trace(RunTrace&& t, mlnmf_trace** out) {
  if (!out) return;
  auto* tr = new mlnmf_trace;
  tr->t = std::move(t);
  *out = tr;
}

}  // namespace

extern "C" {

const char* mlnmf_last_error(void) { return g_err.c_str(); }
int mlnmf_version(void) { return MLNMF_B200_VERSION; }

void mlnmf_default_options(mlnmf_options* o) {
  *o = mlnmf_options{0, MLNMF_F64, 0, MLNMF_GEMM_AUTO, MLNMF_ERROR_AUTO, 1, 0, nullptr};
}

int mlnmf_set_default_options(const mlnmf_options* o) {
  return guard([&] {
    if (!o) throw std::invalid_argument("null options");
    if (o->dtype != MLNMF_F32 && o->dtype != MLNMF_F64) throw std::invalid_argument("dtype must be F32 or F64");
    g_default = *o;
  });
}

int mlnmf_nccl_unique_id(void* out128) {
  return guard([&] {
    ncclUniqueId id;
    nccl_check(NcclApi::get().GetUniqueId(&id), "GetUniqueId");
    std::memcpy(out128, &id, 128);
  });
}

double mlnmf_iteration_cost(size_t m, size_t n, size_t r, int kind) {
  return iteration_cost(m, n, r, kind == MLNMF_ANLS ? kAnls : kMu);
}

int mlnmf_plan_configuration(size_t grid_h, size_t grid_w, size_t n, size_t level_count, int kind, int cycle,
                             size_t rank, double amount, size_t trace_every, mlnmf_trace** trace_out) {
  if (trace_out) *trace_out = nullptr;
  return guard([&] {
    if (level_count < 1) throw std::invalid_argument("run_configuration: need at least one level");
    std::vector<size_t> rows{grid_h * grid_w};
    size_t gh = grid_h, gw = grid_w;
    for (size_t l = 0; l + 1 < level_count; ++l) {
      if (gh < 2 || gw < 2) throw std::invalid_argument("coarsen_grid: grid below 2x2 cannot be coarsened");
      gh = (gh + 1) / 2;
      gw = (gw + 1) / 2;
      rows.push_back(gh * gw);
    }
    const Cycle c = to_cycle(cycle);
    const size_t hl = c == kNone ? 1 : level_count;
    rows.resize(hl);
    if (rank < 1 || rank > std::min(grid_h * grid_w, n))
      throw std::invalid_argument("random_init: rank must satisfy 1 <= r <= min(m,n)");
    RunTrace t;
    plan_cycle(rows, n, hl, rank, to_kind(kind), c, amount, trace_every, t);
    emit_trace(std::move(t), trace_out);
  });
}

int mlnmf_smoothness(const double* M, size_t m, size_t n, size_t grid_h, size_t grid_w, double* out) {
  return guard([&] {
    Engine& e = default_engine();
    check_dims(m, n, 1);
    e.set_data(M, MLNMF_F64, false, m, n, n, 0, grid_h, grid_w, false);
    *out = e.smoothness(0);
  });
}

int mlnmf_initialization_bound(const double* M, size_t m, size_t n, size_t grid_h, size_t grid_w,
                               const double* V_coarse, const double* W, size_t r, double* lhs, double* rhs) {
  return guard([&] {
    Engine& e = default_engine();
    check_dims(m, n, r);
    e.set_data(M, MLNMF_F64, false, m, n, n, 0, grid_h, grid_w, false);
    e.initialization_bound(0, V_coarse, W, MLNMF_F64, r, lhs, rhs);
  });
}

// ---------------------------------------------------------------------------
int mlnmf_run_configuration(const double* M, size_t m, size_t n, size_t grid_h, size_t grid_w, size_t level_count,
                            int kind, int cycle, size_t rank, uint64_t seed, int budget_mode, double amount,
                            size_t trace_every, double* V_out, double* W_out, mlnmf_trace** trace_out) {
  if (trace_out) *trace_out = nullptr;
  return guard([&] {
    Engine& e = default_engine();
    if (level_count < 1) throw std::invalid_argument("run_configuration: need at least one level");
    e.set_data(M, MLNMF_F64, false, m, n, n, 0, grid_h, grid_w, false);
    RunTrace t;
    run_configuration(e, level_count, to_kind(kind), to_cycle(cycle), rank, seed, budget_mode, amount, trace_every,
                      t);
    e.get_factors(0, V_out, W_out, MLNMF_F64);
    emit_trace(std::move(t), trace_out);
  });
}

int mlnmf_run_cycle(const double* M, size_t m, size_t n, size_t grid_h, size_t grid_w, size_t hierarchy_levels,
                    size_t levels, const double* V0, const double* W0, size_t r, int kind, int cycle,
                    int budget_mode, double amount, size_t trace_every, double* V_out, double* W_out,
                    mlnmf_trace** trace_out) {
  if (trace_out) *trace_out = nullptr;
  return guard([&] {
    Engine& e = default_engine();
    check_dims(m, n, r);
    e.set_data(M, MLNMF_F64, false, m, n, n, 0, grid_h, grid_w, false);
    e.ensure_levels(hierarchy_levels);
    e.set_factors(0, V0, W0, MLNMF_F64, r);
    RunTrace t;
    run_cycle(e, levels, r, to_kind(kind), to_cycle(cycle), budget_mode, amount, trace_every, t);
    e.get_factors(0, V_out, W_out, MLNMF_F64);
    emit_trace(std::move(t), trace_out);
  });
}

// run_bench's inner loop (proj/src/bench.cpp:28-84), batched: seeds
// base_seed .. base_seed + runs - 1 of run_configuration(trace_every = 0) on
// one M.  `workers` host threads each own a device session (own stream, own
// copy of M) and take seeds round-robin, so independent runs overlap on the
// GPU; every seed's result is the same as a lone run's (each run is
// deterministic and touches only its own session).
int mlnmf_run_seeds(const mlnmf_options* opt, const double* M, size_t m, size_t n, size_t grid_h, size_t grid_w,
                    size_t level_count, int kind, int cycle, size_t rank, uint64_t base_seed, size_t runs,
                    int budget_mode, double amount, size_t workers, double* final_errors) {
  return guard([&] {
    if (!M || !final_errors) throw std::invalid_argument("run_seeds: null buffer");
    if (runs < 1) throw std::invalid_argument("run_bench: runs >= 1");
    if (level_count < 1) throw std::invalid_argument("run_configuration: need at least one level");
    mlnmf_options o = opt ? *opt : g_default;
    o.world = 1;
    o.rank = 0;
    o.nccl_id = nullptr;
    const Kind k = to_kind(kind);
    const Cycle c = to_cycle(cycle);
    const size_t nw = std::max<size_t>(1, std::min(workers ? workers : 8, runs));
    std::vector<std::string> errs(nw);
    std::vector<int> codes(nw, MLNMF_OK);
    auto body = [&](size_t w) {
      codes[w] = guard([&] {
        Engine e(to_opts(&o));
        e.set_data(M, MLNMF_F64, false, m, n, n, 0, grid_h, grid_w, false);
        for (size_t i = w; i < runs; i += nw) {
          RunTrace t;
          run_configuration(e, level_count, k, c, rank, base_seed + i, budget_mode, amount, 0, t);
          final_errors[i] = t.samples.back().error;
        }
      });
      if (codes[w] != MLNMF_OK) errs[w] = g_err;
    };
    std::vector<std::thread> th;
    for (size_t w = 1; w < nw; ++w) th.emplace_back(body, w);
    body(0);
    for (auto& t : th) t.join();
    for (size_t w = 0; w < nw; ++w)
      if (codes[w] != MLNMF_OK) {
        g_err = errs[w];
        switch (codes[w]) {
          case MLNMF_ERR_INVALID: throw std::invalid_argument(errs[w]);
          case MLNMF_ERR_NNLS_CAP: throw NnlsCapExceeded(errs[w]);
          case MLNMF_ERR_DATA: throw DataError(errs[w]);
          default: throw std::runtime_error(errs[w]);
        }
      }
  });
}

// run_solver (solvers.cpp:343-355): one level, unit = one iteration on M.
int mlnmf_run_solver(const double* M, size_t m, size_t n, const double* V0, const double* W0, size_t r, int kind,
                     int budget_mode, double amount, size_t trace_every, double* V_out, double* W_out,
                     mlnmf_trace** trace_out) {
  if (trace_out) *trace_out = nullptr;
  return guard([&] {
    Engine& e = default_engine();
    check_dims(m, n, r);
    e.set_data(M, MLNMF_F64, false, m, n, n, 0, m, 1, false);
    e.set_factors(0, V0, W0, MLNMF_F64, r);
    RunTrace t;
    run_cycle(e, 1, r, to_kind(kind), kNone, budget_mode, amount, trace_every, t);
    e.get_factors(0, V_out, W_out, MLNMF_F64);
    emit_trace(std::move(t), trace_out);
  });
}

static int one_step(const double* M, size_t m, size_t n, double* V, double* W, size_t r, Kind k, int* deg,
                    int* counts) {
  return guard([&] {
    Engine& e = default_engine();
    check_dims(m, n, r);
    e.set_data(M, MLNMF_F64, false, m, n, n, 0, m, 1, false);
    e.set_factors(0, V, W, MLNMF_F64, r);
    e.mark_run_start();
    e.step(0, k);
    std::vector<int> cn;
    int d = 0;
    e.flush(nullptr, &cn, &d);
    e.get_factors(0, V, W, MLNMF_F64);
    if (deg) *deg += d;
    if (counts && !cn.empty()) std::memcpy(counts, cn.data(), cn.size() * sizeof(int));
  });
}

int mlnmf_mu_step(const double* M, size_t m, size_t n, double* V, double* W, size_t r) {
  return one_step(M, m, n, V, W, r, kMu, nullptr, nullptr);
}
int mlnmf_hals_step(const double* M, size_t m, size_t n, double* V, double* W, size_t r, int* degenerate) {
  return one_step(M, m, n, V, W, r, kHals, degenerate, nullptr);
}
int mlnmf_anls_step(const double* M, size_t m, size_t n, double* V, double* W, size_t r, int* iter_counts) {
  return one_step(M, m, n, V, W, r, kAnls, nullptr, iter_counts);
}

int mlnmf_nnls_active_set(const double* G, const double* h, const double* x0, size_t r, double* x, int* iterations) {
  return guard([&] {
    int it = 0;
    default_engine().nnls_single(G, h, x0, r, x, &it);
    if (iterations) *iterations = it;
  });
}

int mlnmf_frobenius_error(const double* M, const double* V, const double* W, size_t m, size_t n, size_t r,
                          double* out) {
  return guard([&] {
    Engine& e = default_engine();
    check_dims(m, n, r);
    e.set_data(M, MLNMF_F64, false, m, n, n, 0, m, 1, false);
    e.set_factors(0, V, W, MLNMF_F64, r);
    *out = e.frobenius_error(0);
  });
}

int mlnmf_random_init(size_t m, size_t n, size_t r, uint64_t seed, double* V_out, double* W_out) {
  return guard([&] { default_engine().random_init_host(m, n, r, seed, V_out, W_out); });
}

int mlnmf_restrict_columns(size_t grid_h, size_t grid_w, const double* X, size_t ncols, double* Y) {
  return guard([&] { default_engine().apply_transfer(grid_h, grid_w, 0, X, ncols, Y); });
}
int mlnmf_prolong_columns(size_t grid_h, size_t grid_w, const double* X, size_t ncols, double* Y) {
  return guard([&] { default_engine().apply_transfer(grid_h, grid_w, 1, X, ncols, Y); });
}

// ---------------------------------------------------------------------------
int mlnmf_session_create(const mlnmf_options* o, mlnmf_session** out) {
  *out = nullptr;
  return guard([&] {
    auto* s = new mlnmf_session;
    try {
      s->e = std::make_unique<Engine>(to_opts(o));
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

int mlnmf_session_create_host_comm(const mlnmf_options* o, mlnmf_host_allreduce_fn fn, void* ctx,
                                   mlnmf_session** out) {
  *out = nullptr;
  return guard([&] {
    if (!fn) throw std::invalid_argument("host allreduce: null function");
    if (o && o->nccl_id) throw std::invalid_argument("host allreduce: an NCCL id was given too");
    Options x = to_opts(o);
    x.host_allreduce = fn;
    x.host_allreduce_ctx = ctx;
    auto* s = new mlnmf_session;
    try {
      s->e = std::make_unique<Engine>(x);
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

void mlnmf_session_destroy(mlnmf_session* s) { delete s; }

int mlnmf_session_set_data(mlnmf_session* s, const void* M, int host_dtype, size_t m, size_t n_local, size_t n_total,
                           size_t col0, size_t grid_h, size_t grid_w) {
  return guard([&] { s->e->set_data(M, host_dtype, false, m, n_local, n_total, col0, grid_h, grid_w, true); });
}

int mlnmf_session_generate(mlnmf_session* s, const mlnmf_gen_params* g, size_t n_total, size_t col0,
                           size_t n_local) {
  return guard([&] {
    GenParams p;
    p.h = g->h, p.w = g->w, p.r = g->r, p.blobs = g->blobs;
    p.sigma_min = g->sigma_min, p.sigma_max = g->sigma_max;
    p.noise_kind = g->noise_kind, p.noise_scale = g->noise_scale, p.seed = g->seed;
    p.scale_to_unit = g->scale_to_unit;
    s->e->generate(p, n_total, col0, n_local);
  });
}

int mlnmf_session_run_configuration(mlnmf_session* s, size_t level_count, int kind, int cycle, size_t rank,
                                    uint64_t seed, int budget_mode, double amount, size_t trace_every,
                                    mlnmf_trace** trace_out) {
  if (trace_out) *trace_out = nullptr;
  return guard([&] {
    RunTrace t;
    run_configuration(*s->e, level_count, to_kind(kind), to_cycle(cycle), rank, seed, budget_mode, amount,
                      trace_every, t);
    emit_trace(std::move(t), trace_out);
  });
}

int mlnmf_session_run_cycle(mlnmf_session* s, size_t hierarchy_levels, size_t levels, const void* V0,
                            const void* W0_local, int host_dtype, size_t r, int kind, int cycle, int budget_mode,
                            double amount, size_t trace_every, mlnmf_trace** trace_out) {
  if (trace_out) *trace_out = nullptr;
  return guard([&] {
    s->e->ensure_levels(hierarchy_levels);
    s->e->set_factors(0, V0, W0_local, host_dtype, r);
    RunTrace t;
    run_cycle(*s->e, levels, r, to_kind(kind), to_cycle(cycle), budget_mode, amount, trace_every, t);
    emit_trace(std::move(t), trace_out);
  });
}

int mlnmf_session_get_factors(mlnmf_session* s, void* V, void* W_local, int host_dtype) {
  return guard([&] { s->e->get_factors(0, V, W_local, host_dtype); });
}

int mlnmf_session_set_factors(mlnmf_session* s, const void* V, const void* W_local, int host_dtype, size_t r) {
  return guard([&] { s->e->set_factors(0, V, W_local, host_dtype, r); });
}

// ---- resident per-level entries (SURVEY 8(b) minimum) ----
int mlnmf_session_build_levels(mlnmf_session* s, size_t level_count) {
  return guard([&] { s->e->ensure_levels(level_count); });
}

size_t mlnmf_session_num_levels(mlnmf_session* s) { return s->e->built_levels(); }

int mlnmf_session_level_shape(mlnmf_session* s, size_t level, size_t* grid_h, size_t* grid_w) {
  return guard([&] {
    if (level >= s->e->built_levels()) throw std::invalid_argument("level not built");
    *grid_h = s->e->grid_h(level);
    *grid_w = s->e->grid_w(level);
  });
}

int mlnmf_session_init_random(mlnmf_session* s, size_t r, uint64_t seed) {
  return guard([&] { s->e->init_random(r, seed); });
}

int mlnmf_session_set_factors_level(mlnmf_session* s, size_t level, const void* V, const void* W_local,
                                    int host_dtype, size_t r) {
  return guard([&] {
    if (level >= s->e->built_levels()) throw std::invalid_argument("level not built");
    s->e->set_factors(level, V, W_local, host_dtype, r);
  });
}

int mlnmf_session_get_factors_level(mlnmf_session* s, size_t level, void* V, void* W_local, int host_dtype) {
  return guard([&] {
    if (level >= s->e->built_levels()) throw std::invalid_argument("level not built");
    if (s->e->rank_r() == 0) throw std::invalid_argument("factors not set");
    s->e->get_factors(level, V, W_local, host_dtype);
  });
}

int mlnmf_session_restrict_V(mlnmf_session* s, size_t level) {
  return guard([&] {
    if (level + 1 >= s->e->built_levels()) throw std::invalid_argument("restrict_V: level + 1 not built");
    s->e->restrict_V(level);
  });
}

int mlnmf_session_prolong_V(mlnmf_session* s, size_t level) {
  return guard([&] {
    if (level + 1 >= s->e->built_levels()) throw std::invalid_argument("prolong_V: level + 1 not built");
    s->e->prolong_V(level);
  });
}

int mlnmf_session_run_phase(mlnmf_session* s, size_t level, int kind, int budget_mode, double amount,
                            double step_flops, double unit_flops, size_t trace_every, double* work_consumed,
                            double* leftover, mlnmf_trace** trace_out) {
  if (trace_out) *trace_out = nullptr;
  return guard([&] {
    if (s->e->rank_r() == 0) throw std::invalid_argument("run_phase: factors not set");
    RunTrace t;
    const double left = run_phase(*s->e, level, to_kind(kind), budget_mode, amount, step_flops, unit_flops,
                                  trace_every, work_consumed, t);
    if (leftover) *leftover = left;
    emit_trace(std::move(t), trace_out);
  });
}

int mlnmf_session_steps(mlnmf_session* s, int kind, size_t n_steps) {
  return guard([&] {
    const Kind k = to_kind(kind);
    for (size_t i = 0; i < n_steps; ++i) s->e->step(0, k);
  });
}

int mlnmf_session_sync(mlnmf_session* s) {
  return guard([&] { s->e->sync(); });
}

int mlnmf_session_error(mlnmf_session* s, double* out) {
  return guard([&] { *out = s->e->frobenius_error(0); });
}

int mlnmf_session_norm2(mlnmf_session* s, size_t level, double* out) {
  return guard([&] { *out = s->e->norm2(level); });
}

int mlnmf_session_smoothness(mlnmf_session* s, size_t level, double* out) {
  return guard([&] { *out = s->e->smoothness(level); });
}

int mlnmf_session_initialization_bound(mlnmf_session* s, size_t level, const void* V_coarse, const void* W_local,
                                       int host_dtype, size_t r, double* lhs, double* rhs) {
  return guard([&] { s->e->initialization_bound(level, V_coarse, W_local, host_dtype, r, lhs, rhs); });
}

int mlnmf_session_products(mlnmf_session* s, double* A, double* C) {
  return guard([&] { s->e->products(A, C); });
}

int mlnmf_session_export_data(mlnmf_session* s, void* M_local, int host_dtype) {
  return guard([&] { s->e->export_data(M_local, host_dtype); });
}

int mlnmf_session_gram_v(mlnmf_session* s, double* D) {
  return guard([&] { s->e->gram_v(D); });
}

int mlnmf_session_gram_w(mlnmf_session* s, double* B) {
  return guard([&] { s->e->gram_w(B); });
}

int mlnmf_session_export_level(mlnmf_session* s, size_t level, void* M_level, int* level_dtype) {
  return guard([&] {
    const int dt = s->e->export_level(level, M_level);
    if (level_dtype) *level_dtype = dt;
  });
}

int mlnmf_session_set_profiling(mlnmf_session* s, int on) {
  return guard([&] {
    s->e->set_profiling(on != 0);
    s->e->reset_kernel_times();
  });
}

int mlnmf_session_kernel_times(mlnmf_session* s, double* mwt_ms, long* mwt_n, double* vtm_ms, long* vtm_n) {
  return guard([&] {
    KernelTimes k = s->e->kernel_times();
    *mwt_ms = k.mwt_ms, *mwt_n = k.mwt_n, *vtm_ms = k.vtm_ms, *vtm_n = k.vtm_n;
  });
}

int mlnmf_session_comm_time(mlnmf_session* s, double* ms, long* count) {
  return guard([&] {
    KernelTimes k = s->e->kernel_times();
    *ms = k.comm_ms, *count = k.comm_n;
  });
}

int mlnmf_session_phase_times(mlnmf_session* s, double* ms, long* count) {
  return guard([&] {
    KernelTimes k = s->e->kernel_times();
    for (int i = 0; i < kNumPhases; ++i) ms[i] = k.phase_ms[i], count[i] = k.phase_n[i];
  });
}

long mlnmf_session_launches(mlnmf_session* s) { return s->e->launches(); }
void* mlnmf_session_stream(mlnmf_session* s) { return s->e->stream(); }
int mlnmf_session_tc_active(mlnmf_session* s) { return s->e->tc_active() ? 1 : 0; }
int mlnmf_session_gram_error(mlnmf_session* s) { return s->e->gram_error() ? 1 : 0; }

// ---------------------------------------------------------------------------
size_t mlnmf_trace_num_samples(const mlnmf_trace* t) { return t->t.samples.size(); }
void mlnmf_trace_samples(const mlnmf_trace* t, double* elapsed_s, double* work_units, int* level, double* error) {
  for (size_t i = 0; i < t->t.samples.size(); ++i) {
    const Sample& s = t->t.samples[i];
    if (elapsed_s) elapsed_s[i] = s.elapsed_s;
    if (work_units) work_units[i] = s.work_units;
    if (level) level[i] = s.level;
    if (error) error[i] = s.error;
  }
}
size_t mlnmf_trace_num_allocations(const mlnmf_trace* t) { return t->t.alloc_level.size(); }
void mlnmf_trace_allocations(const mlnmf_trace* t, int* level, double* amount) {
  for (size_t i = 0; i < t->t.alloc_level.size(); ++i) {
    level[i] = t->t.alloc_level[i];
    amount[i] = t->t.alloc_amount[i];
  }
}
size_t mlnmf_trace_num_nnls_counts(const mlnmf_trace* t) { return t->t.nnls_counts.size(); }
void mlnmf_trace_nnls_counts(const mlnmf_trace* t, int* counts) {
  if (!t->t.nnls_counts.empty()) std::memcpy(counts, t->t.nnls_counts.data(), t->t.nnls_counts.size() * sizeof(int));
}
int mlnmf_trace_degenerate(const mlnmf_trace* t) { return t->t.degenerate; }
size_t mlnmf_trace_num_phases(const mlnmf_trace* t) { return t->t.phase_level.size(); }
void mlnmf_trace_phases(const mlnmf_trace* t, int* level, long* steps) {
  for (size_t i = 0; i < t->t.phase_level.size(); ++i) {
    level[i] = t->t.phase_level[i];
    steps[i] = t->t.phase_steps[i];
  }
}
void mlnmf_trace_free(mlnmf_trace* t) { delete t; }

}  // extern "C"

// ---------------------------------------------------------------------------
// Dataset / result I/O (proj/include/mlnmf/io.hpp) over host_io.cpp: the same
// PGM / CSV ingestion and byte-compatible writers the CLI uses.  Buffers the
// library allocates are released with mlnmf_free.
// ---------------------------------------------------------------------------
namespace {
double* export_matrix(const io::Dense& d) {
  double* p = static_cast<double*>(std::malloc(d.v.size() * sizeof(double)));
  if (!p) throw std::runtime_error("out of host memory");
  std::memcpy(p, d.v.data(), d.v.size() * sizeof(double));
  return p;
}
}  // namespace

extern "C" {


void mlnmf_free(void* p) { std::free(p); }

int mlnmf_load_pgm_dir(const char* dir, double** M_out, size_t* m, size_t* n, size_t* h, size_t* w) {
  return guard([&] {
    const mlb::io::Dataset d = mlb::io::load_pgm_dir(dir ? dir : "");
    *m = d.M.rows, *n = d.M.cols, *h = d.grid.h, *w = d.grid.w;
    *M_out = export_matrix(d.M);
  });
}

int mlnmf_load_csv(const char* path, double** M_out, size_t* m, size_t* n) {
  return guard([&] {
    const mlb::io::Dataset d = mlb::io::load_csv(path ? path : "");
    *m = d.M.rows, *n = d.M.cols;
    *M_out = export_matrix(d.M);
  });
}

int mlnmf_save_matrix_csv(const double* A, size_t rows, size_t cols, const char* path) {
  return guard([&] { mlb::io::save_matrix_csv(A, rows, cols, path ? path : ""); });
}

int mlnmf_save_trace_csv(const mlnmf_trace* t, const char* path) {
  return guard([&] {
    if (!t) throw std::invalid_argument("save_trace_csv: null trace");
    std::vector<mlb::io::Sample> s;
    s.reserve(t->t.samples.size());
    for (const auto& x : t->t.samples) s.push_back({x.elapsed_s, x.work_units, x.level, x.error});
    mlb::io::save_trace_csv(s, path ? path : "");
  });
}

int mlnmf_save_basis_mosaic(const double* V, size_t m, size_t r, size_t grid_h, size_t grid_w, const char* dir) {
  return guard([&] { mlb::io::save_basis_mosaic(V, m, r, mlb::io::Grid{grid_h, grid_w}, dir ? dir : ""); });
}

int mlnmf_synth_smooth_dataset(size_t h, size_t w, size_t n, size_t blobs, uint64_t seed, double* M_out) {
  return guard([&] {
    const mlb::io::Dataset d = mlb::io::synth_smooth_dataset(h, w, n, blobs, seed);
    std::memcpy(M_out, d.M.v.data(), d.M.v.size() * sizeof(double));
  });
}

}  // extern "C"
