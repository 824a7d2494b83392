"""CPU, world_size 2 over gloo: the column-sharded data path.

The engine shards the columns of M over ranks; per iteration it allreduces
[A_g | B_g] = [M_g W_g^T | W_g W_g^T] (and the error partials), runs the V
sweep redundantly on every rank and the W_g sweep shard-locally.  These tests
run that decomposition with two gloo ranks in numpy and check it against the
restated oracle's single-process hals_step / mu_step / frobenius_error
(solvers.cpp:79-141, matrix.cpp:37-42), plus the per-shard generator twin and
bench.py's rank plumbing (max over ranks, id broadcast).
"""
import os
import socket

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _hals_rows(X, A, B):
    """Gauss-Seidel projected rank-1 sweeps over the rows of X (solvers.cpp:101-141)."""
    X = X.copy()
    for k in range(X.shape[1]):
        if B[k, k] <= 0:
            continue
        X[:, k] = np.maximum(0.0, (A[:, k] + X[:, k] * B[k, k] - X @ B[:, k]) / B[k, k])
    return X


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, REPO)
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_1009_0881_b200 as P
        import bench

        def allreduce(x):
            t = torch.from_numpy(np.ascontiguousarray(x))
            dist.all_reduce(t)
            return t.numpy()

        out = {}
        restated = oracle.Restated()
        n_total, r = 37, 4
        c0, nl = P.shard_columns(n_total, world, rank)
        # per-shard generation == the same columns of the full matrix
        Mg = oracle.generate_config(0, n=n_total, col0=c0, n_cols=nl, restated=restated)
        Vfull, Wfull = restated.random_init(Mg.shape[0], n_total, r, 3)
        V, Wg = Vfull.copy(), Wfull[:, c0:c0 + nl].copy()
        out["M"] = Mg
        # HALS: allreduce [A | B], V sweep everywhere, W_g sweep locally
        for _ in range(3):
            AB = allreduce(np.concatenate([Mg @ Wg.T, (Wg @ Wg.T)], axis=0))
            A, B = AB[:Mg.shape[0]], AB[Mg.shape[0]:]
            V = _hals_rows(V, A, B)
            Wg = _hals_rows(Wg.T, Mg.T @ V, V.T @ V).T
        out["hals_V"], out["hals_W"] = V, Wg
        # MU on the same shards
        V, Wg = Vfull.copy(), Wfull[:, c0:c0 + nl].copy()
        for _ in range(2):
            AB = allreduce(np.concatenate([Mg @ Wg.T, Wg @ Wg.T], axis=0))
            A, B = AB[:Mg.shape[0]], AB[Mg.shape[0]:]
            V = V * A / np.maximum(V @ B, 1e-16)
            Wg = Wg * (V.T @ Mg) / np.maximum((V.T @ V) @ Wg, 1e-16)
        out["mu_V"], out["mu_W"] = V, Wg
        # error: allreduced column partials
        e2 = allreduce(np.array([((Mg - V @ Wg) ** 2).sum()]))[0]
        out["err"] = float(np.sqrt(e2))
        out["col0"], out["nl"] = c0, nl
        # bench plumbing
        out["max"] = bench.allreduce_max(float(rank + 1) * 1.5, world)
        out["bcast"] = bench.bcast_obj(b"nccl-id-bytes" if rank == 0 else None, world)
        bench.barrier(world)
        q.put((rank, out))
    except Exception as e:  # surface the failure in the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def shards():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, 2, port, q)) for k in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for k, v in res.items():
        assert isinstance(v, dict), f"rank {k}: {v}"
    return [res[0], res[1]]


def test_sharded_generator_matches_full(shards, restated):
    import oracle
    full = oracle.generate_config(0, n=37, restated=restated)
    assert shards[0]["col0"] == 0 and shards[1]["col0"] == shards[0]["nl"]
    assert np.array_equal(np.concatenate([s["M"] for s in shards], axis=1), full)


def test_sharded_hals_matches_oracle(shards, restated):
    import oracle
    M = oracle.generate_config(0, n=37, restated=restated)
    V, W = restated.random_init(M.shape[0], 37, 4, 3)
    for _ in range(3):
        V, W, _ = restated.hals_step(M, V, W)
    for s in shards:
        assert np.allclose(s["hals_V"], V, rtol=1e-10, atol=1e-13)
    Wc = np.concatenate([s["hals_W"] for s in shards], axis=1)
    assert np.allclose(Wc, W, rtol=1e-10, atol=1e-13)
    # the redundant V sweeps agree bit for bit across ranks
    assert np.array_equal(shards[0]["hals_V"], shards[1]["hals_V"])


def test_sharded_mu_and_error_match_oracle(shards, restated):
    import oracle
    M = oracle.generate_config(0, n=37, restated=restated)
    V, W = restated.random_init(M.shape[0], 37, 4, 3)
    for _ in range(2):
        V, W = restated.mu_step(M, V, W)
    for s in shards:
        assert np.allclose(s["mu_V"], V, rtol=1e-11)
    assert np.allclose(np.concatenate([s["mu_W"] for s in shards], axis=1), W, rtol=1e-11)
    e = restated.frobenius_error(M, V, W)
    for s in shards:
        assert s["err"] == pytest.approx(e, rel=1e-10)


def test_bench_rank_plumbing(shards):
    for s in shards:
        assert s["max"] == 3.0
        assert s["bcast"] == b"nccl-id-bytes"
