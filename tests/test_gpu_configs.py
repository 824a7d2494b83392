"""GPU parity at BASELINE configs 1-3: the CBCL-sized 19 x 19
(2 levels, 19x19 -> 10x10 by the odd-size rule), the paper's face-sized
(112 x 92, 4 levels: 112x92 -> 56x46 -> 28x23 -> 14x12) and large-image
(243 x 320, 5 levels: -> 122x160 -> 61x80 -> 31x40 -> 16x20) shapes, whose
pyramids exercise the odd-size coarsening and boundary-renormalised transfer
operators, with the solver kinds BASELINE.json names for them.

* fp64, exact mode: bit-identical factors, error trajectory, schedule and
  NNLS exchange counts to the C restatement of the reference (itself pinned to
  the reference by tests/test_oracle.py).
* fp32 storage (the SIMT fp64-accumulate products these sizes use): every
  trace sample within 1e-5 of the fp64 oracle fed the fp32-rounded inputs.

Budgets are a few work units so the single-threaded oracle stays in seconds.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _defaults(P):
    P.set_default_options()
    yield
    P.set_default_options()


@pytest.fixture(scope="module")
def cfg1():
    return oracle.generate_config(1)  # 361 x 2429, scaled to [0, 1]


@pytest.fixture(scope="module")
def cfg2():
    return oracle.generate_config(2)  # 10304 x 400


@pytest.fixture(scope="module")
def cfg3():
    return oracle.generate_config(3)  # 77760 x 165


def round32(a):
    return np.asarray(a, np.float32).astype(np.float64)


def rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)) / np.abs(np.asarray(b))))


def same_schedule(tg, to):
    assert len(tg.error) == len(to.error)
    assert np.array_equal(tg.level, to.level)
    assert np.array_equal(tg.work_units, to.work)
    assert np.array_equal(tg.alloc_level, to.alloc_level)
    assert np.array_equal(tg.alloc_amount, to.alloc_amount)


CASES_EXACT = [
    # (config, grid h, w, levels, kind, cycle, rank, budget)
    (1, 19, 19, 2, "hals", "fmg", 49, 20.0),
    (1, 19, 19, 2, "mu", "vc", 49, 20.0),
    (2, 112, 92, 4, "anls", "fmg", 40, 2.0),
    (2, 112, 92, 4, "hals", "vc", 40, 4.0),
    (3, 243, 320, 5, "hals", "fmg", 49, 2.0),
    (3, 243, 320, 5, "mu", "ni", 49, 2.0),
    (3, 243, 320, 1, "anls", "none", 49, 1.0),
]


@pytest.mark.parametrize("case", CASES_EXACT, ids=lambda c: f"cfg{c[0]}-{c[4]}-{c[5]}")
def test_configs_exact_bitwise(P, restated, cfg1, cfg2, cfg3, case):
    cfg, h, w, L, kind, cycle, r, budget = case
    M = {1: cfg1, 2: cfg2, 3: cfg3}[cfg]
    P.set_default_options(exact=True)
    Vo, Wo, to = restated.run_configuration(M, h, w, L, kind, cycle, r, 0, budget, 1)
    res = P.run_configuration(M, P.ImageGrid(h, w), L, kind, cycle, r, 0, budget, 1)
    same_schedule(res.trace, to)
    assert np.array_equal(res.trace.error, to.error)
    assert np.array_equal(res.V, Vo) and np.array_equal(res.W, Wo)
    if kind == "anls":
        assert np.array_equal(res.trace.nnls_iteration_counts, to.counts)


CASES_FP32 = [
    (1, 19, 19, 2, "hals", "ni", 49, 20.0),
    (2, 112, 92, 4, "hals", "ni", 40, 4.0),
    (2, 112, 92, 4, "mu", "fmg", 40, 3.0),
    (3, 243, 320, 5, "hals", "vc", 49, 2.0),
    (3, 243, 320, 5, "mu", "fmg", 49, 2.0),
]


@pytest.mark.parametrize("case", CASES_FP32, ids=lambda c: f"cfg{c[0]}-{c[4]}-{c[5]}")
def test_configs_fp32_within_1e5(P, restated, cfg1, cfg2, cfg3, case):
    cfg, h, w, L, kind, cycle, r, budget = case
    M = {1: cfg1, 2: cfg2, 3: cfg3}[cfg]
    m, n = M.shape
    M32 = M.astype(np.float32)
    V0, W0 = restated.random_init(m, n, r, 0)
    _, _, to = restated.run_cycle_on(round32(M32), h, w, L, L, round32(V0), round32(W0), kind, cycle, budget, 1)
    with P.Session(dtype=P.F32) as s:
        s.set_data(M32, P.ImageGrid(h, w))
        tg = s.run_configuration(L, kind, cycle, r, 0, budget, 1)
        assert not s.tc_active  # these sizes take the SIMT fp64-accumulate products
    same_schedule(tg, to)
    assert rel(tg.error, to.error) <= 1e-5, rel(tg.error, to.error)
