// scheduler.hpp -- host restatement of the reference's budget and cycle
// control (proj/src/solvers.cpp:300-355, proj/src/multilevel.cpp:14-132) over
// the device Engine.  In work-unit mode every decision is made with the
// reference's own double arithmetic, so the level schedule and the step count
// of every phase are identical to the reference's; device work is only
// enqueued (one host sync at the end of the run).
#pragma once
#include <cstddef>
#include <cstdint>
#include <vector>

#include "engine.hpp"

namespace mlb {

struct RunTrace {
  std::vector<Sample> samples;
  std::vector<int> nnls_counts;
  std::vector<int> alloc_level;
  std::vector<double> alloc_amount;
  std::vector<int> phase_level;
  std::vector<long> phase_steps;
  int degenerate = 0;
};

// Model flops of one iteration (cost_model.cpp:8-23): MU and HALS share
// 2m(nr + r^2) + 2nr^2; ANLS is mnr + (m + n) s_r r^3 with s_r = 2r.
double iteration_cost(size_t m, size_t n, size_t r, Kind kind);

// run_cycle (multilevel.cpp:65-89) on levels [0, levels) of the engine's
// hierarchy, starting from the factors already in the engine (level-0 V, W).
void run_cycle(Engine& e, size_t levels, size_t r, Kind kind, Cycle cycle, int budget_mode, double amount,
               size_t trace_every, RunTrace& out);

// run_solver_phase (solvers.cpp:300-341) on the engine's resident level l
// (M_l, V_l and W on the device): `amount` work units (budget_mode 0,
// charging step_flops / unit_flops per step) or seconds (1), samples at
// start, every trace_every steps and end, stamped with *work_consumed (the
// run's cumulative work; advanced in place).  Returns the unconsumed amount.
// Sample times are relative to the phase start.
double run_phase(Engine& e, size_t l, Kind kind, int budget_mode, double amount, double step_flops,
                 double unit_flops, size_t trace_every, double* work_consumed, RunTrace& out);

// Dry run of the same control flow (work-unit budgets): the phase allocations,
// steps per phase and sample work/level stamps, without device work.
void plan_cycle(const std::vector<size_t>& level_rows, size_t n_total, size_t levels, size_t r, Kind kind,
                Cycle cycle, double amount, size_t trace_every, RunTrace& out);

// run_configuration (multilevel.cpp:116-132) on the engine's data: feasibility,
// hierarchy, random_init(seed) on the device, dispatch.
void run_configuration(Engine& e, size_t level_count, Kind kind, Cycle cycle, size_t rank, uint64_t seed,
                       int budget_mode, double amount, size_t trace_every, RunTrace& out);

}  // namespace mlb
