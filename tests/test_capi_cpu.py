"""CPU: the C-ABI library and the host-side logic, without a GPU.

* libmlnmf_b200.so loads and exports every entry point include/mlnmf_b200.h
  declares (the drop-in boundary; no compute call is made here);
* the host scheduler (csrc/scheduler.cpp, a restatement of CycleRunner +
  run_solver_phase, multilevel.cpp:14-89 / solvers.cpp:300-341) reproduces the
  reference's allocations and per-phase step counts: SURVEY.md Appendix B and
  the restated oracle's realised phases;
* iteration_cost KATs (cost_model.cpp:8-23, test_core.cpp:135-158);
* argument validation raises the reference's exception types;
* column sharding covers [0, n) exactly once.
"""
import os
import re

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "mlnmf_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    src = re.sub(r"//[^\n]*", "", src)
    return sorted(set(re.findall(r"\b(mlnmf_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(P):
    syms = declared_symbols()
    assert len(syms) >= 40
    missing = [s for s in syms if not hasattr(P._lib, s)]
    assert not missing, missing
    # and the library is the in-tree build
    assert os.path.realpath(P.LIB_PATH).startswith(os.path.realpath(REPO))


def test_exports_match_nm(P):
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", P.LIB_PATH], capture_output=True, text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert set(declared_symbols()) <= exported


def test_version(P):
    assert P._lib.mlnmf_version() > 0


APPENDIX_B = [
    # (h, w, n, r, L, kind, cycle, amount, [(level, steps), ...])  -- SURVEY.md Appendix B
    (32, 32, 1000, 20, 3, "hals", "ni", 100.0, [(3, 78), (2, 71), (1, 75)]),
    (32, 32, 1000, 20, 3, "hals", "vc", 100.0, [(1, 25), (2, 23), (3, 78), (2, 48), (1, 50)]),
    (32, 32, 1000, 20, 3, "hals", "fmg", 100.0,
     [(3, 78), (2, 17), (3, 58), (2, 36), (1, 18), (2, 17), (3, 58), (2, 36), (1, 38)]),
    (32, 32, 1000, 20, 3, "anls", "ni", 100.0, [(3, 12), (2, 30), (1, 75)]),
    (19, 19, 2429, 49, 2, "hals", "ni", 500.0, [(2, 345), (1, 375)]),
    (19, 19, 2429, 49, 2, "hals", "vc", 500.0, [(1, 125), (2, 345), (1, 250)]),
    (19, 19, 2429, 49, 2, "hals", "fmg", 500.0, [(2, 345), (1, 93), (2, 259), (1, 188)]),
    (19, 19, 2429, 49, 2, "anls", "ni", 500.0, [(2, 138), (1, 375)]),
    (112, 92, 400, 40, 4, "hals", "ni", 100.0, [(4, 79), (3, 71), (2, 74), (1, 75)]),
    (112, 92, 400, 40, 4, "anls", "ni", 100.0, [(4, 29), (3, 48), (2, 67), (1, 75)]),
    (243, 320, 165, 49, 5, "hals", "ni", 100.0, [(5, 84), (4, 71), (3, 74), (2, 74), (1, 75)]),
    (243, 320, 165, 49, 5, "anls", "ni", 100.0, [(5, 62), (4, 65), (3, 72), (2, 74), (1, 75)]),
    (256, 256, 262144, 64, 5, "hals", "ni", 100.0, [(5, 80), (4, 70), (3, 74), (2, 74), (1, 75)]),
    (256, 256, 262144, 64, 5, "anls", "ni", 100.0, [(5, 0), (4, 2), (3, 6), (2, 23), (1, 75)]),
]


@pytest.mark.parametrize("h,w,n,r,L,kind,cycle,amount,expect", APPENDIX_B)
def test_plan_matches_appendix_b(P, h, w, n, r, L, kind, cycle, amount, expect):
    tr = P.plan_configuration(P.ImageGrid(h, w), n, L, kind, cycle, r, amount, 1)
    assert list(zip(tr.phase_level.tolist(), tr.phase_steps.tolist())) == expect


@pytest.mark.parametrize("kind", ["mu", "hals", "anls"])
@pytest.mark.parametrize("cycle", ["none", "ni", "vc", "fmg"])
@pytest.mark.parametrize("h,w,L,amount", [(17, 17, 3, 24.0), (33, 20, 4, 37.5), (9, 9, 2, 400.0)])
def test_plan_matches_restated_oracle(P, restated, kind, cycle, h, w, L, amount):
    """The scheduler's dry run equals the oracle's realised run: same allocations,
    same steps per phase, same work/level stamp on every trace sample."""
    n, r = 11, 3
    M = np.random.default_rng(h * w + L).random((h * w, n))
    _, _, ref = restated.run_configuration(M, h, w, L, kind, cycle, r, 1, amount, 1)
    tr = P.plan_configuration(P.ImageGrid(h, w), n, L, kind, cycle, r, amount, 1)
    assert np.array_equal(tr.alloc_level, ref.alloc_level)
    assert np.array_equal(tr.alloc_amount, ref.alloc_amount)
    assert np.array_equal(tr.phase_level, ref.phase_level)
    assert np.array_equal(tr.phase_steps, ref.phase_steps)
    assert np.array_equal(tr.work_units, ref.work)
    assert np.array_equal(tr.level, ref.level)


def test_plan_trace_cadence(P):
    # trace_every = 0: only the start and end samples of each phase
    tr1 = P.plan_configuration(P.ImageGrid(32, 32), 1000, 3, "hals", "none", 20, 100.0, 1)
    tr0 = P.plan_configuration(P.ImageGrid(32, 32), 1000, 3, "hals", "none", 20, 100.0, 0)
    assert len(tr1.work_units) == 102 and int(tr1.phase_steps.sum()) == 100
    assert len(tr0.work_units) < len(tr1.work_units)
    assert tr0.work_units[-1] == tr1.work_units[-1]


def test_iteration_cost_kats(P):
    assert P.iteration_cost(1, 1, 1, "mu") == 6.0
    assert P.iteration_cost(1000, 100, 10, "mu") == 2220000.0
    assert P.iteration_cost(1000, 100, 10, "hals") == 2220000.0
    assert P.iteration_cost(1000, 100, 10, "mu") / P.iteration_cost(250, 100, 10, "mu") == \
        pytest.approx(1110000.0 / 285000.0, rel=1e-15)


def test_iteration_cost_matches_oracle(P, restated):
    rng = np.random.default_rng(0)
    for _ in range(50):
        m, n, r = (int(x) for x in rng.integers(1, 4000, 3))
        r = 1 + r % 30
        for kind in ("mu", "hals", "anls"):
            assert P.iteration_cost(m, n, r, kind) == restated.iteration_cost(m, n, r, kind)


def test_invalid_arguments_raise_reference_types(P):
    # transfer.cpp:56-57,157-167 / multilevel.cpp:121-122: std::invalid_argument
    with pytest.raises(ValueError):
        P.plan_configuration(P.ImageGrid(3, 3), 10, 4, "hals", "ni", 2, 10.0, 1)
    with pytest.raises(ValueError):
        P.plan_configuration(P.ImageGrid(8, 8), 10, 0, "hals", "ni", 2, 10.0, 1)
    with pytest.raises(ValueError):
        P.coarsen_grid(P.ImageGrid(1, 5))
    with pytest.raises(ValueError):
        P.shard_columns(10, 2, 2)


def test_coarsen_grid_chain(P):
    # the BASELINE grids
    def chain(h, w, L):
        g = [P.ImageGrid(h, w)]
        for _ in range(L - 1):
            g.append(P.coarsen_grid(g[-1]))
        return [(x.height, x.width) for x in g]
    assert chain(19, 19, 2) == [(19, 19), (10, 10)]
    assert chain(112, 92, 4) == [(112, 92), (56, 46), (28, 23), (14, 12)]
    assert chain(243, 320, 5) == [(243, 320), (122, 160), (61, 80), (31, 40), (16, 20)]
    assert P.ImageGrid(5, 7).index(2, 3) == 3 * 5 + 2


@pytest.mark.parametrize("n,world", [(262144, 1), (262144, 8), (1000, 3), (7, 4), (3, 8)])
def test_shard_columns_partition(P, n, world):
    covered = []
    prev_end = 0
    for rank in range(world):
        c0, nl = P.shard_columns(n, world, rank)
        assert c0 == prev_end and nl >= 0
        covered.extend(range(c0, c0 + nl))
        prev_end = c0 + nl
    assert covered == list(range(n))
    sizes = [P.shard_columns(n, world, k)[1] for k in range(world)]
    assert max(sizes) - min(sizes) <= 1


def test_generator_config_table_agrees(P):
    import oracle
    for k, c in P.GEN_CONFIGS.items():
        o = oracle.CONFIGS[k]
        assert (c["h"], c["w"], c["n"], c["r"], c["levels"], c["blobs"]) == \
            (o["h"], o["w"], o["n"], o["r"], o["levels"], o["blobs"])
        assert tuple(c["sigma"]) == tuple(o["sigma"]) and tuple(c["noise"]) == tuple(o["noise"])
        assert bool(c["scale_to_unit"]) == bool(o["scale_to_unit"])


def test_product_does_not_import_oracle():
    """The product path never routes through the oracle (no CPU fallback)."""
    pkg = os.path.join(REPO, "paper_1009_0881_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".hpp", ".cuh", ".h")):
                src = open(os.path.join(root, f), errors="ignore").read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "mlnmf_oracle" not in src and "libmlnmf_ref" not in src, f


def test_run_bench_skip_rules_without_device(P):
    """run_bench (bench.cpp:41-57): a single-level cycle with levels != 1 and a
    multilevel request without a pixel grid are skipped with the reference's
    notes, before any device work."""
    import numpy as np
    M = np.ones((16, 5))
    cfg = P.BenchConfig(algorithms=["hals"], cycles=["none"], level_counts=[2, 3], rank=2, runs=3, budget=10.0)
    entries = P.run_bench(M, P.ImageGrid(4, 4), cfg)
    assert [e.skipped for e in entries] == [True, True]
    assert all(e.note == "single-level runs use exactly one level" for e in entries)
    cfg = P.BenchConfig(algorithms=["mu"], cycles=["fmg"], level_counts=[2], rank=2, runs=3, budget=10.0)
    entries = P.run_bench(M, None, cfg)
    assert entries[0].skipped and entries[0].note == "dataset has no pixel grid"
    with pytest.raises(ValueError):
        P.run_bench(M, None, P.BenchConfig(runs=0))
