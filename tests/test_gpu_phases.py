"""GPU: the resident per-level C-ABI pieces of a multilevel cycle
(mlnmf_session_build_levels / init_random / run_phase / restrict_V /
prolong_V / get_factors_level, include/mlnmf_b200.h; SURVEY 8(b) minimum).

A Python restatement of the reference's CycleRunner (multilevel.cpp:14-62:
phase, nested, vcycle, fmg with the T/4 - 3T/4 splits and leftover carries)
driving ONLY those pieces must reproduce the session's own
run_configuration bit for bit (fp64, exact mode), for every cycle kind and
solver, and the oracle's trace.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


class PyCycleRunner:
    """multilevel.cpp:14-62 over a device session's resident levels."""

    def __init__(self, P, s, kind, r, trace_every, fixed_steps=None):
        self.P, self.s, self.kind, self.trace_every = P, s, kind, trace_every
        self.fixed = iter(fixed_steps) if fixed_steps is not None else None
        n = s.n_local
        self.rows = [s.level_grid(l).pixels() for l in range(s.num_levels)]
        self.unit = P.iteration_cost(self.rows[0], n, r, kind)
        self.flops = [P.iteration_cost(m, n, r, kind) for m in self.rows]
        self.work = 0.0
        self.samples, self.alloc, self.phases = [], [], []

    def phase(self, cur, nominal, carry):  # CycleRunner::phase (multilevel.cpp:28-34)
        self.alloc.append((cur + 1, nominal))
        amount = nominal + carry
        if self.fixed is not None:  # replay: exactly the given number of steps
            amount = next(self.fixed) * self.flops[cur] / self.unit
        left, self.work, tr = self.s.run_phase(cur, self.kind, amount, self.flops[cur], self.unit,
                                               self.trace_every, self.work)
        self.samples.append(tr)
        self.phases.append((cur + 1, int(tr.phase_steps.sum())))
        return left

    def nested(self, cur, lv, T, carry):
        if lv == 1:
            return self.phase(cur, T, carry)
        self.s.restrict_V(cur)
        left = self.nested(cur + 1, lv - 1, T / 4, 0.0)
        self.s.prolong_V(cur)
        return self.phase(cur, 3 * T / 4, carry + left)

    def vcycle(self, cur, lv, T, carry):
        if lv == 1:
            return self.phase(cur, T, carry)
        l0 = self.phase(cur, T / 4, 0.0)
        self.s.restrict_V(cur)
        l1 = self.vcycle(cur + 1, lv - 1, T / 4, 0.0)
        self.s.prolong_V(cur)
        return self.phase(cur, T / 2, carry + l0 + l1)

    def fmg(self, cur, lv, T, carry):
        if lv == 1:
            return self.phase(cur, T, carry)
        self.s.restrict_V(cur)
        l1 = self.fmg(cur + 1, lv - 1, T / 4, 0.0)
        self.s.prolong_V(cur)
        return self.vcycle(cur, lv, 3 * T / 4, carry + l1)


@pytest.mark.parametrize("kind", ["hals", "mu", "anls"])
@pytest.mark.parametrize("cycle", ["none", "ni", "vc", "fmg"])
def test_resident_pieces_reproduce_run_configuration(P, gpu, restated, kind, cycle):
    M = oracle.generate_config(0, n=240, restated=restated)
    grid, L, r, T = P.ImageGrid(32, 32), 3, 12, 16.0
    with P.Session(dtype=P.F64, exact=True) as s:
        s.set_data(M, grid)
        want = s.run_configuration(L if cycle != "none" else 1, kind, cycle, r, 0, T, 1)
        V_want, W_want = s.get_factors()
    with P.Session(dtype=P.F64, exact=True) as s:
        s.set_data(M, grid)
        s.build_levels(L if cycle != "none" else 1)
        assert s.num_levels == (L if cycle != "none" else 1)
        g = s.level_grid(s.num_levels - 1)
        assert (g.height, g.width) == ((32, 32), (16, 16), (8, 8))[s.num_levels - 1]
        s.init_random(r, 0)
        run = PyCycleRunner(P, s, kind, r, 1)
        lv = s.num_levels
        {"none": run.nested, "ni": run.nested, "vc": run.vcycle, "fmg": run.fmg}[cycle](0, lv, T, 0.0)
        V, W = s.get_factors_level(0)
    err = np.concatenate([t.error for t in run.samples])
    lev = np.concatenate([t.level for t in run.samples])
    wk = np.concatenate([t.work_units for t in run.samples])
    assert np.array_equal(err, want.error), np.max(np.abs(err - want.error))
    assert np.array_equal(lev, want.level) and np.array_equal(wk, want.work_units)
    assert [p[1] for p in run.phases] == want.phase_steps.tolist()
    assert np.array_equal(V, V_want) and np.array_equal(W, W_want)
    if kind == "anls":
        counts = np.concatenate([t.nnls_iteration_counts for t in run.samples])
        assert np.array_equal(counts, want.nnls_iteration_counts)


def test_run_phase_against_oracle_and_errors(P, gpu, restated):
    """One phase on a resident level against the oracle's run_solver
    (solvers.cpp:343-355 = one run_solver_phase), plus the boundary's error
    behaviour (unbuilt level, missing factors)."""
    M = oracle.generate_config(0, n=200, restated=restated)
    V0, W0 = restated.random_init(1024, 200, 10, 3)
    _, _, to = restated.run_solver(M, V0, W0, "hals", 12.0, 2)
    with P.Session(dtype=P.F64, exact=True) as s:
        s.set_data(M, P.ImageGrid(32, 32))
        with pytest.raises(ValueError):
            s.run_phase(0, "hals", 12.0, 1.0, 1.0, 2)       # no factors yet
        s.set_factors(V0, W0)
        with pytest.raises(ValueError):
            s.restrict_V(0)                                # level 1 not built
        unit = P.iteration_cost(1024, 200, 10, "hals")
        left, work, tr = s.run_phase(0, "hals", 12.0, unit, unit, 2)
    assert left == pytest.approx(0.0) and work == pytest.approx(12.0)
    assert np.array_equal(tr.error, to.error) and np.array_equal(tr.work_units, to.work)


@pytest.mark.parametrize("cycle", ["none", "vc", "fmg"])
def test_wall_clock_budget_structure_and_replay(P, gpu, restated, cycle):
    """Wall-clock budgets (Budget::kWallClockSeconds, solvers.cpp:318-320,340)
    run as batched device steps with O(log) host time checks
    (scheduler.cpp solver_phase).  For the realised step counts:
      * the allocations equal the oracle's (nominal T/4 - 3T/4 splits);
      * the sample structure (levels, work-unit stamps, 2 + steps/trace_every
        per phase) follows from the step counts;
      * the trajectory equals a deterministic replay of those step counts
        through the resident phases (fp64, exact: bit for bit)."""
    M = oracle.generate_config(0, n=300, restated=restated)
    L = 1 if cycle == "none" else 3
    T, te = 0.25, 2
    with P.Session(dtype=P.F64, exact=True) as s:
        s.set_data(M, P.ImageGrid(32, 32))
        tr = s.run_configuration(L, "hals", cycle, 16, 0, P.Budget(P.BudgetMode.kWallClockSeconds, T), te)
    _, _, to = restated.run_configuration(M, 32, 32, L, "hals", cycle, 16, 0, 0.05, te, mode=1)
    assert np.array_equal(tr.alloc_level, to.alloc_level)
    assert np.allclose(tr.alloc_amount / T, to.alloc_amount / 0.05, rtol=1e-12, atol=0)
    steps = tr.phase_steps.tolist()
    assert sum(steps) > 20 and tr.elapsed_s[-1] >= 0.9 * T
    assert len(tr.error) == sum(2 + k // te for k in steps)
    unit = P.iteration_cost(1024, 300, 16, "hals")
    flops = {l + 1: P.iteration_cost(m, 300, 16, "hals") for l, m in enumerate((1024, 256, 64))}
    w, k_ = [], 0.0
    for lv, n_ in zip(tr.phase_level.tolist(), steps):
        w.append(k_)
        for i in range(1, n_ + 1):
            if i % te == 0:
                w.append(k_ + i * flops[lv] / unit)
        k_ += n_ * flops[lv] / unit
        w.append(k_)
    assert np.allclose(tr.work_units, w, rtol=1e-12, atol=0)
    with P.Session(dtype=P.F64, exact=True) as s:
        s.set_data(M, P.ImageGrid(32, 32))
        s.build_levels(L)
        s.init_random(16, 0)
        run = PyCycleRunner(P, s, "hals", 16, te, fixed_steps=steps)
        {"none": run.nested, "vc": run.vcycle, "fmg": run.fmg}[cycle](0, L, T, 0.0)
    err = np.concatenate([t.error for t in run.samples])
    assert np.array_equal(err, tr.error)
