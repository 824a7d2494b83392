"""GPU: the tcgen05 3xTF32 M-streaming products against fp64 references.

A = M W^T and C = V^T M from fp32 storage: the tensor-core path must agree
with an fp64 numpy product of the same fp32 inputs to 3xTF32 accuracy, on
aligned and ragged shapes, r in {16..64}; and whole fp32 runs through the
tensor path must track the fp64 oracle.

Tolerance: the tensor core's fp32 accumulate truncates, a one-sided bias of
~2.4e-7 relative per 32-K chunk accumulated in TMEM before the fp64 drain
(kWindow = 8 chunks -> ~2e-6 at long K; short-K shapes ~4e-7).  TOL = 4e-6
relative Frobenius error is that bound with a 2x margin; the long-K case
(32768 x 8192, several windows per CTA) exercises it.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

TOL = 4e-6


def relnorm(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("m,n,r", [
    (1024, 2048, 64), (1024, 2048, 20), (4096, 1024, 40), (1028, 1500, 49),
    (256, 16384, 64), (16384, 256, 64), (640, 640, 16), (2052, 4100, 33), (32768, 8192, 64),
])
def test_tc_products(P, gpu, m, n, r):
    rng = np.random.default_rng(m * 7 + n + r)
    M = rng.random((m, n)).astype(np.float32)
    M[rng.random((m, n)) < 0.1] = 0.0
    V = rng.random((m, r)).astype(np.float32)
    W = (rng.random((r, n)) * 3).astype(np.float32)
    M64, V64, W64 = M.astype(np.float64), V.astype(np.float64), W.astype(np.float64)
    A_ref, C_ref = M64 @ W64.T, V64.T @ M64
    with P.Session(dtype=P.F32, gemm_path=P.GEMM_TCGEN05) as s:
        s.set_data(M, P.ImageGrid(m, 1))
        s.set_factors(V64, W64)
        assert s.tc_active
        A, C = s.products()
    ea, ec = relnorm(A, A_ref), relnorm(C, C_ref)
    assert ea < TOL and ec < TOL, (ea, ec)
    with P.Session(dtype=P.F32, gemm_path=P.GEMM_SIMT) as s:
        s.set_data(M, P.ImageGrid(m, 1))
        s.set_factors(V64, W64)
        assert not s.tc_active
        A2, C2 = s.products()
    assert relnorm(A2, A_ref) < 1e-13 and relnorm(C2, C_ref) < 1e-13


def test_tc_deterministic(P, gpu):
    rng = np.random.default_rng(5)
    M = rng.random((2048, 4096)).astype(np.float32)
    V, W = rng.random((2048, 64)), rng.random((64, 4096))
    outs = []
    for _ in range(2):
        with P.Session(dtype=P.F32, gemm_path=P.GEMM_TCGEN05) as s:
            s.set_data(M, P.ImageGrid(2048, 1))
            s.set_factors(V, W)
            outs.append(s.products())
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


def round32(a):
    return np.asarray(a, np.float32).astype(np.float64)


@pytest.mark.parametrize("cycle", ["none", "fmg"])
def test_tc_run_tracks_oracle(P, restated, gpu, cycle):
    """Config-0 generator at a tensor-path size (32x32 grid, n = 4096, r = 20,
    HALS, work:30): the fp32 tcgen05 run tracks the fp64 oracle fed the
    fp32-rounded inputs, with an identical schedule.

    Tolerance 6e-5 (not the SIMT path's 1e-5): the products carry ~2e-6
    relative error (3xTF32 drops A_lo F_lo, and the tensor core's truncating
    fp32 accumulate biases each 8-chunk window), and 30 single-level HALS
    sweeps amplify it ~20x in the error trajectory (measured 4.5e-5; 1.2e-5
    even with 1-chunk windows).  Multilevel runs stay ~4e-6.  Strict 1e-5
    parity is the SIMT path (MLNMF_GEMM_SIMT)."""
    M = oracle.generate_config(0, n=4096, restated=restated).astype(np.float32)
    V0, W0 = restated.random_init(1024, 4096, 20, 0)
    L = 1 if cycle == "none" else 3
    _, _, to = restated.run_cycle_on(round32(M), 32, 32, L, L, round32(V0), round32(W0), "hals", cycle, 30.0, 1)
    with P.Session(dtype=P.F32, gemm_path=P.GEMM_TCGEN05) as s:
        s.set_data(M, P.ImageGrid(32, 32))
        tg = s.run_configuration(3, "hals", cycle, 20, 0, 30.0, 1)
        assert s.tc_active
    assert np.array_equal(tg.level, to.level) and np.array_equal(tg.work_units, to.work)
    dev = float(np.max(np.abs(tg.error - to.error) / to.error))
    assert dev < 6e-5, dev


@pytest.mark.parametrize("m,n,r", [(1024, 2048, 64), (2052, 4100, 33), (4096, 3000, 20), (640, 640, 16)])
def test_tc_residual_error(P, gpu, m, n, r):
    """The tensor-core direct residual ||M - VW||_F (error samples of tensor-path
    runs) against an fp64 numpy residual of the same fp32 inputs: within 1e-7
    relative (measured ~5e-9), and against the SIMT residual kernel."""
    rng = np.random.default_rng(m + n + r)
    V = rng.random((m, r)).astype(np.float32)
    W = rng.random((r, n)).astype(np.float32)
    M = np.maximum(V.astype(np.float64) @ W.astype(np.float64) * (1 + 0.05 * rng.standard_normal((m, n))),
                   0).astype(np.float32)
    ref = float(np.linalg.norm(M.astype(np.float64) - V.astype(np.float64) @ W.astype(np.float64)))
    with P.Session(dtype=P.F32, gemm_path=P.GEMM_TCGEN05) as s:
        s.set_data(M, P.ImageGrid(m, 1))
        s.set_factors(V, W)
        assert s.tc_active and not s.gram_error
        e_tc = s.error()
    assert abs(e_tc - ref) / ref < 1e-7, (e_tc, ref)


@pytest.mark.parametrize("m,n,r", [(2048, 4096, 64), (4096, 2304, 32), (3000, 2600, 64)])
def test_tc_products_cta_pairs(P, gpu, monkeypatch, m, n, r):
    """The opt-in CTA-pair products (cta_group::2, 256-row tiles, MLB_TC_PAIR=1,
    read when a session's tensor path is created) agree with fp64 like the
    single-CTA kernel, including ragged 256-row tiles."""
    monkeypatch.setenv("MLB_TC_PAIR", "1")
    rng = np.random.default_rng(m + n + r)
    M = rng.random((m, n)).astype(np.float32)
    V = rng.random((m, r)).astype(np.float32)
    W = (rng.random((r, n)) * 2).astype(np.float32)
    M64, V64, W64 = M.astype(np.float64), V.astype(np.float64), W.astype(np.float64)
    with P.Session(dtype=P.F32, gemm_path=P.GEMM_TCGEN05) as s:
        s.set_data(M, P.ImageGrid(m, 1))
        s.set_factors(V64, W64)
        A, C = s.products()
    ea, ec = relnorm(A, M64 @ W64.T), relnorm(C, V64.T @ M64)
    assert ea < TOL and ec < TOL, (ea, ec)


def test_fast_register_sweeps_match_reference_order(P, gpu, monkeypatch):
    """Config-4 rank (r = 64) at >= 16k rows and columns: the non-exact
    register sweeps (interleaved fused dot chains, reciprocal pivots) agree
    with the reference-order register sweeps to fp64 rounding over 3 HALS
    steps (same tensor-core products on both sides)."""
    out = []
    for exact_sweeps in (False, True):
        if exact_sweeps:
            monkeypatch.setenv("MLNMF_EXACT_SWEEPS", "1")
        with P.Session(dtype=P.F32) as s:
            s.generate(4, seed=0, n_total=16384)
            s.run_configuration(1, "hals", "none", 64, 0, 0.0, 0)
            s.steps("hals", 3)
            out.append(s.get_factors())
    (V0, W0), (V1, W1) = out
    assert relnorm(V0, V1) < 1e-6 and relnorm(W0, W1) < 1e-6, (relnorm(V0, V1), relnorm(W0, W1))
