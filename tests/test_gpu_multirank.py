"""GPU: the sharded engine at world = 2, executed.

Two sessions (ranks) in one process on one GPU, each driven from its own
thread, exchange their [A | B] partials, error partials, norms and NNLS
counts through a HostGroup (mlnmf_session_create_host_comm: device -> host,
sum over ranks in rank order, host -> device) -- the same engine code path
as NCCL ranks (column shards, shard-local W, replicated V, the per-step
allreduce, rank-consistent tensor-path decisions), with no device-side waits
between ranks.  Against the oracle's unsharded fp64 run:
  * fp64: every error sample within 1e-10, identical levels / work units /
    phase step counts, V identical on both ranks, the W shards together = W;
  * ANLS: the NNLS exchange counts in the reference's layout (m_l V-row
    counts then all n W-column counts per step, solvers.cpp:269,296);
  * fp32 + tcgen05 products: the world-2 run equals the world-1 run to the
    products' rounding.
"""
import threading

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def run_ranks(P, world, n_total, body, **kw):
    """body(session, rank, col0, n_local) on `world` threads; results by rank."""
    grp = P.HostGroup(world)
    out, errs = [None] * world, [None] * world

    def worker(rk):
        try:
            col0, nl = P.shard_columns(n_total, world, rk)
            with P.Session(world=world, rank=rk, host_group=grp, **kw) as s:
                out[rk] = body(s, rk, col0, nl)
        except BaseException as e:  # noqa: BLE001
            errs[rk] = e
            grp.abort()

    th = [threading.Thread(target=worker, args=(rk,)) for rk in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for e in errs:
        if e is not None:
            raise e
    return out


@pytest.mark.parametrize("kind", ["hals", "mu", "anls"])
@pytest.mark.parametrize("cycle", ["none", "fmg"])
def test_world2_fp64_matches_oracle(P, gpu, restated, kind, cycle):
    cfg = oracle.CONFIGS[0]
    n = 241  # uneven shards: 121 + 120 columns
    M = oracle.generate_config(0, n=n, restated=restated)
    L = 1 if cycle == "none" else 3
    Vo, Wo, to = restated.run_configuration(M, 32, 32, L, kind, cycle, 12, 0, 12.0, 1)

    def body(s, rk, col0, nl):
        s.set_data(M[:, col0:col0 + nl], P.ImageGrid(32, 32), n_total=n, col0=col0)
        tr = s.run_configuration(L, kind, cycle, 12, 0, 12.0, 1)
        V, W = s.get_factors()
        return tr, V, W, col0

    res = run_ranks(P, 2, n, body, dtype=P.F64)
    for tr, V, W, col0 in res:
        assert np.array_equal(tr.level, to.level) and np.allclose(tr.work_units, to.work, rtol=0, atol=0)
        assert tr.phase_steps.tolist() == to.phase_steps.tolist()
        dev = np.max(np.abs(tr.error - to.error) / to.error)
        assert dev < 1e-10, dev
        assert np.max(np.abs(V - Vo)) <= 1e-9 * np.max(np.abs(Vo))
        if kind == "anls":
            assert np.array_equal(tr.nnls_iteration_counts, to.counts), \
                (len(tr.nnls_iteration_counts), len(to.counts))
    assert np.array_equal(res[0][1], res[1][1])  # V replicated bit for bit
    W = np.concatenate([res[0][2], res[1][2]], axis=1)
    assert np.max(np.abs(W - Wo)) <= 1e-9 * np.max(np.abs(Wo))


@pytest.mark.parametrize("kind", ["hals", "anls"])
def test_world2_config2_fmg(P, gpu, restated, kind):
    """Config 2's 4-level odd-size pyramid (112x92 -> 14x12), 400 columns."""
    c = oracle.CONFIGS[2]
    M = oracle.generate_config(2, restated=restated)
    n = M.shape[1]
    _, _, to = restated.run_configuration(M, c["h"], c["w"], 4, kind, "fmg", 40, 0, 6.0, 1)

    def body(s, rk, col0, nl):
        s.set_data(M[:, col0:col0 + nl], P.ImageGrid(c["h"], c["w"]), n_total=n, col0=col0)
        return s.run_configuration(4, kind, "fmg", 40, 0, 6.0, 1)

    for tr in run_ranks(P, 2, n, body, dtype=P.F64):
        assert np.array_equal(tr.level, to.level)
        assert np.max(np.abs(tr.error - to.error) / to.error) < 1e-10
        if kind == "anls":
            assert np.array_equal(tr.nnls_iteration_counts, to.counts)


def test_world2_tensor_path(P, gpu):
    """fp32 storage, tcgen05 products forced, a config-4 column slice
    (m = 65536, 2048 columns, r = 64) split 1024 + 1024: the world-2
    trajectory equals the world-1 one to the products' rounding, and both
    ranks took the tensor path."""
    n = 2048
    with P.Session(dtype=P.F32) as g:
        g.generate(4, seed=0, n_total=262144, col0=0, n_local=n)
        M = np.empty((65536, n), np.float32)
        g.export_data(M.ctypes.data)
    V0, W0 = P.random_init(65536, n, 64, 0)
    with P.Session(dtype=P.F32, gemm_path=P.GEMM_TCGEN05) as s:
        s.set_data(M, P.ImageGrid(256, 256))
        one = s.run_cycle(1, 1, V0, W0, "hals", "none", 6.0, 1)

    def body(s, rk, col0, nl):
        s.set_data(M[:, col0:col0 + nl], P.ImageGrid(256, 256), n_total=n, col0=col0)
        tr = s.run_cycle(1, 1, V0, W0[:, col0:col0 + nl], "hals", "none", 6.0, 1)
        return tr, s.tc_active

    for tr, tc in run_ranks(P, 2, n, body, dtype=P.F32, gemm_path=P.GEMM_TCGEN05):
        assert tc
        assert np.max(np.abs(tr.error - one.error) / one.error) < 1e-7


def test_world2_wall_clock_budget_agreed(P, gpu, restated):
    """Wall-clock budgets at world = 2: every time check uses the elapsed
    time agreed over the ranks (max), so both ranks realise the same step
    counts and their traces agree sample for sample."""
    n = 400
    M = oracle.generate_config(0, n=n, restated=restated)

    def body(s, rk, col0, nl):
        s.set_data(M[:, col0:col0 + nl], P.ImageGrid(32, 32), n_total=n, col0=col0)
        return s.run_configuration(3, "hals", "fmg", 12, 0, P.Budget(P.BudgetMode.kWallClockSeconds, 0.2), 1)

    a, b = run_ranks(P, 2, n, body, dtype=P.F64)
    assert a.phase_steps.tolist() == b.phase_steps.tolist() and sum(a.phase_steps) > 10
    assert np.array_equal(a.level, b.level) and np.array_equal(a.error, b.error)
