"""GPU: ranks beyond the shared-memory kernels (r > ~160): the reference
accepts any 1 <= r <= min(m, n) (matrix.cpp:53-54).  The HALS / MU sweeps
then read the Gram from global memory with the rows in a global workspace,
the batched NNLS keeps its per-warp workspace in global memory, and the
exact-order residual reads V and W directly -- same operation order, so fp64
exact runs stay bit-identical to the oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind", ["hals", "mu", "anls"])
def test_rank_200_bitwise(P, gpu, restated, kind):
    rng = np.random.default_rng(200)
    m, n, r = 400, 300, 200
    M = rng.random((m, n)) ** 2
    V0, W0 = restated.random_init(m, n, r, 1)
    steps = 1 if kind == "anls" else 3
    _, _, to = restated.run_solver(M, V0, W0, kind, float(steps), 1)
    with P.Session(dtype=P.F64, exact=True) as s:
        s.set_data(M, P.ImageGrid(20, 20))
        tr = s.run_cycle(1, 1, V0, W0, kind, "none", float(steps), 1)
    assert np.array_equal(tr.error, to.error), np.max(np.abs(tr.error - to.error) / to.error)
    if kind == "anls":
        assert np.array_equal(tr.nnls_iteration_counts, to.counts)


def test_rank_180_fp32_multilevel(P, gpu, restated):
    """fp32 storage (SIMT products: the tensor path is r <= 64), 2-level FMG."""
    rng = np.random.default_rng(180)
    M = rng.random((1024, 500))
    V0, W0 = restated.random_init(1024, 500, 180, 2)
    _, _, to = restated.run_cycle_on(M.astype(np.float32).astype(np.float64), 32, 32, 2, 2, V0, W0, "hals", "fmg",
                                     4.0, 1)
    with P.Session(dtype=P.F32) as s:
        s.set_data(M.astype(np.float32), P.ImageGrid(32, 32))
        tr = s.run_cycle(2, 2, V0, W0, "hals", "fmg", 4.0, 1)
        assert not s.tc_active
    assert np.array_equal(tr.level, to.level)
    assert np.max(np.abs(tr.error - to.error) / to.error) < 1e-5
