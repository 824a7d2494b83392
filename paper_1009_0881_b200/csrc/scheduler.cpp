// scheduler.cpp -- see scheduler.hpp.
#include "scheduler.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>

namespace mlb {

double iteration_cost(size_t m_, size_t n_, size_t r_, Kind kind) {
  const double m = (double)m_, n = (double)n_, r = (double)r_;
  if (kind == kAnls) {
    const double s_r = 2.0 * r;  // CostParams::with_default_sr (cost_model.hpp:20-23)
    return m * n * r + (m + n) * s_r * r * r * r;
  }
  return 2.0 * m * (n * r + r * r) + 2.0 * n * r * r;
}

namespace {

struct Runner {
  Engine* e;  // null: dry run (schedule only, no device work)
  std::vector<size_t> ms;  // rows per level
  Kind kind;
  int mode;  // 0 work units, 1 wall clock
  size_t r;
  size_t trace_every;
  RunTrace& out;
  double unit_flops = 1.0;
  double work_consumed = 0.0;

  // the cost model sees the global column count (identical on every rank)
  size_t n_total = 0;
  double step_flops(size_t cur) const { return iteration_cost(ms.at(cur), n_total, r, kind); }

  // run_solver_phase (solvers.cpp:300-341)
  double solver_phase(size_t l, double amount, double sflops) {
    const double charge = sflops / unit_flops;
    const double eps = 1e-12 * std::max(1.0, amount);
    double phase_start = 0.0;
    if (mode == 1) phase_start = e->agreed_elapsed_s();
    if (e) e->sample(l, work_consumed);
    else out.samples.push_back({0.0, work_consumed, (int)l + 1, 0.0});
    double consumed = 0.0;
    size_t steps = 0;
    auto one_step = [&]() {
      if (e) e->step(l, kind);
      consumed += charge;
      work_consumed += charge;
      ++steps;
      if (trace_every > 0 && steps % trace_every == 0) {
        if (e) e->sample(l, work_consumed);
        else out.samples.push_back({0.0, work_consumed, (int)l + 1, 0.0});
      }
    };
    if (mode == 0) {
      // work units: the step count follows from the budget arithmetic alone,
      // so every step is enqueued without a host sync
      while (consumed + charge <= amount + eps) one_step();
    } else {
      // Wall clock.  The reference checks elapsed >= amount before every
      // step (solvers.cpp:318-320).  Here the device runs ahead in batches:
      // after a sync (elapsed agreed over ranks: max), with R seconds left and
      // the last batch's per-step time tau, k = floor(R / (2 tau)) steps are
      // enqueued without a sync -- they finish by half the remaining time --
      // so batches shrink geometrically towards the deadline and the last
      // steps go one at a time: the same steps start as under a per-step
      // check, with O(log(budget / step)) syncs instead of one per step.
      double tau = -1.0;
      double now = e->agreed_elapsed_s() - phase_start;
      while (now < amount) {
        size_t k = 1;
        if (tau > 0.0) k = (size_t)std::max(1.0, std::min(4096.0, std::floor((amount - now) / (2.0 * tau))));
        for (size_t i = 0; i < k; ++i) one_step();
        const double after = e->agreed_elapsed_s() - phase_start;
        tau = e->agreed_max((after - now) / (double)k);
        now = after;
      }
    }
    if (e) e->sample(l, work_consumed);
    else out.samples.push_back({0.0, work_consumed, (int)l + 1, 0.0});
    out.phase_level.push_back((int)l + 1);
    out.phase_steps.push_back((long)steps);
    if (mode == 0) return amount - consumed;
    return std::max(0.0, amount - (e->agreed_elapsed_s() - phase_start));
  }

  // CycleRunner::phase (multilevel.cpp:28-34)
  double phase(size_t cur, double nominal, double carry) {
    out.alloc_level.push_back((int)cur + 1);
    out.alloc_amount.push_back(nominal);
    return solver_phase(cur, nominal + carry, step_flops(cur));
  }

  // CycleRunner::nested (multilevel.cpp:36-43)
  double nested(size_t cur, size_t lvls, double T, double carry) {
    if (lvls == 1) return phase(cur, T, carry);
    if (e) e->restrict_V(cur);
    const double leftover = nested(cur + 1, lvls - 1, T / 4, 0.0);
    if (e) e->prolong_V(cur);
    return phase(cur, 3 * T / 4, carry + leftover);
  }

  // CycleRunner::vcycle (multilevel.cpp:45-53)
  double vcycle(size_t cur, size_t lvls, double T, double carry) {
    if (lvls == 1) return phase(cur, T, carry);
    const double l0 = phase(cur, T / 4, 0.0);
    if (e) e->restrict_V(cur);
    const double l1 = vcycle(cur + 1, lvls - 1, T / 4, 0.0);
    if (e) e->prolong_V(cur);
    return phase(cur, T / 2, carry + l0 + l1);
  }

  // CycleRunner::fmg (multilevel.cpp:55-62)
  double fmg(size_t cur, size_t lvls, double T, double carry) {
    if (lvls == 1) return phase(cur, T, carry);
    if (e) e->restrict_V(cur);
    const double l1 = fmg(cur + 1, lvls - 1, T / 4, 0.0);
    if (e) e->prolong_V(cur);
    return vcycle(cur, lvls, 3 * T / 4, carry + l1);
  }
};

}  // namespace

static void drive(Runner& run, size_t levels, Cycle cycle, double amount) {
  run.unit_flops = run.step_flops(0);
  switch (cycle) {
    case kNone:
      run.phase(0, amount, 0.0);
      break;
    case kNested:
      run.nested(0, levels, amount, 0.0);
      break;
    case kVCycle:
      run.vcycle(0, levels, amount, 0.0);
      break;
    case kFmg:
      run.fmg(0, levels, amount, 0.0);
      break;
    default:
      throw std::invalid_argument("run_cycle: unknown cycle kind");
  }
}

void run_cycle(Engine& e, size_t levels, size_t r, Kind kind, Cycle cycle, int budget_mode, double amount,
               size_t trace_every, RunTrace& out) {
  if (levels < 1 || levels > e.built_levels()) throw std::invalid_argument("run_cycle: bad level count");
  Runner run{&e, {}, kind, budget_mode, r, trace_every, out};
  for (size_t l = 0; l < e.built_levels(); ++l) run.ms.push_back(e.m(l));
  run.n_total = e.n_total();
  e.mark_run_start();
  drive(run, levels, cycle, amount);
  e.flush(&out.samples, &out.nnls_counts, &out.degenerate);
}

double run_phase(Engine& e, size_t l, Kind kind, int budget_mode, double amount, double step_flops,
                 double unit_flops, size_t trace_every, double* work_consumed, RunTrace& out) {
  if (l >= e.built_levels()) throw std::invalid_argument("run_phase: level not built");
  if (!(unit_flops > 0.0)) throw std::invalid_argument("run_phase: unit_flops must be positive");
  Runner run{&e, {}, kind, budget_mode, e.rank_r(), trace_every, out};
  for (size_t k = 0; k < e.built_levels(); ++k) run.ms.push_back(e.m(k));
  run.n_total = e.n_total();
  run.unit_flops = unit_flops;
  run.work_consumed = work_consumed ? *work_consumed : 0.0;
  e.mark_run_start();
  const double left = run.solver_phase(l, amount, step_flops);
  e.flush(&out.samples, &out.nnls_counts, &out.degenerate);
  if (work_consumed) *work_consumed = run.work_consumed;
  return left;
}

void plan_cycle(const std::vector<size_t>& level_rows, size_t n_total, size_t levels, size_t r, Kind kind,
                Cycle cycle, double amount, size_t trace_every, RunTrace& out) {
  if (levels < 1 || levels > level_rows.size()) throw std::invalid_argument("run_cycle: bad level count");
  Runner run{nullptr, level_rows, kind, 0, r, trace_every, out};
  run.n_total = n_total;
  drive(run, levels, cycle, amount);
}

void run_configuration(Engine& e, size_t level_count, Kind kind, Cycle cycle, size_t rank, uint64_t seed,
                       int budget_mode, double amount, size_t trace_every, RunTrace& out) {
  if (level_count < 1) throw std::invalid_argument("run_configuration: need at least one level");
  if (e.built_levels() < 1) throw std::invalid_argument("run_configuration: no data");
  // feasibility check before any restriction work (multilevel.cpp:124-125)
  size_t gh = e.grid_h(0), gw = e.grid_w(0);
  for (size_t l = 0; l + 1 < level_count; ++l) {
    if (gh < 2 || gw < 2) throw std::invalid_argument("coarsen_grid: grid below 2x2 cannot be coarsened");
    gh = (gh + 1) / 2;
    gw = (gw + 1) / 2;
  }
  const size_t hl = cycle == kNone ? 1 : level_count;
  e.ensure_levels(hl);
  e.init_random(rank, seed);
  run_cycle(e, hl, rank, kind, cycle, budget_mode, amount, trace_every, out);
}

}  // namespace mlb
