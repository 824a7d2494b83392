"""GPU: the tcgen05 integer-digit M-streaming products against fp64 references.

A = M W^T and C = V^T M from fp32 M storage (ix_gemm.cu): M's fp32 entries
and the fp64 factors are rounded to per-row 31-bit fixed-point grids (M
entries within 2^7 of the row maximum exactly), split into four signed 8-bit
digits, and the digit products of the leading weight classes accumulate
EXACTLY in int32 TMEM (tcgen05.mma.kind::i8).  The error is the unbiased
grid rounding (<= 2^-31 of the row maximum), which averages out along K.
TOL = 1e-8 relative Frobenius error (the round-1 tf32 kernel needed 4e-6
and carried a one-sided ~1e-6 bias); the numpy digit model
(tests/ixmodel.py) pins the kernel's integer arithmetic to 1e-14; whole fp32
runs through the tensor path must track the fp64 oracle within the
north-star 1e-5.
"""
import numpy as np
import pytest

import oracle
import ixmodel  # tests/ixmodel.py (the digit-format model)

pytestmark = pytest.mark.gpu

TOL = 1e-8


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


@pytest.mark.parametrize("m,n,r", [(1024, 2048, 64), (1028, 1500, 49), (16384, 256, 64), (2052, 4100, 33),
                                   (640, 640, 16), (32768, 8192, 64)])
def test_tc_products_match_digit_model(P, gpu, m, n, r):
    """The kernel's integer arithmetic, pinned: A and C equal the numpy model
    of the digit format (tests/ixmodel.py: same scales, same rounding, exact
    integer digit sums) up to the fp64 rounding of the split-K sum."""
    rng = np.random.default_rng(m + 3 * n + r)
    M = (rng.random((m, n)) ** 3).astype(np.float32)
    M[rng.random((m, n)) < 0.2] = 0.0
    V = (rng.random((m, r)) * rng.random((1, r)) * 4).astype(np.float32)
    W = (rng.random((r, n)) * rng.random((r, 1)) * 9).astype(np.float32)
    with P.Session(dtype=P.F32, gemm_path=P.GEMM_TCGEN05) as s:
        s.set_data(M, P.ImageGrid(m, 1))
        s.set_factors(V, W)
        A, C = s.products()
    Am, Cm = ixmodel.product_A(M, W), ixmodel.product_C(V, M)
    np.testing.assert_allclose(A, Am, rtol=1e-14, atol=0)
    np.testing.assert_allclose(C, Cm, rtol=1e-14, atol=0)


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
    fp32-rounded inputs within the north-star 1e-5 (error trajectory), with an
    identical schedule.  The products are exact up to input rounding, so the
    remaining deviation is fp32 storage of V and W between steps."""
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
    assert dev < 1e-5, dev


@pytest.mark.parametrize("m,n,r", [(1024, 2048, 64), (2052, 4100, 33), (4096, 3000, 20), (640, 640, 16)])
def test_tc_gram_error(P, gpu, m, n, r):
    """Error samples of tensor-path runs use the Gram identity
    ||M||^2 - 2 <V^T M, W> + <V^T V, W W^T> with the tensor-path product
    C = V^T M (no residual pass).  Near a fit (5 % noise) the identity cancels
    ~400x, so C's input rounding shows, scaled down by the 31-bit grids.
    Pinned exactly by the digit model (1e-12), bounded against the fp64
    residual (2e-7)."""
    rng = np.random.default_rng(m + n + r)
    V = rng.random((m, r)).astype(np.float32)
    W = rng.random((r, n)).astype(np.float32)
    M = np.maximum(V.astype(np.float64) @ W.astype(np.float64) * (1 + 0.05 * rng.standard_normal((m, n))),
                   0).astype(np.float32)
    ref = float(np.linalg.norm(M.astype(np.float64) - V.astype(np.float64) @ W.astype(np.float64)))
    with P.Session(dtype=P.F32, gemm_path=P.GEMM_TCGEN05) as s:
        s.set_data(M, P.ImageGrid(m, 1))
        s.set_factors(V, W)
        assert s.tc_active and s.gram_error
        e_tc = s.error()
    e_model = ixmodel.gram_error(M, V, W)
    assert abs(e_tc - e_model) / e_model < 1e-12, (e_tc, e_model)
    assert abs(e_tc - ref) / ref < 2e-7, (e_tc, ref)


@pytest.mark.parametrize("m,n,r", [(1024, 2048, 64), (4096, 3000, 20)])
def test_tc_sample_tight_fit_takes_direct_residual(P, gpu, m, n, r):
    """A fit within 1 % (here 1e-4 noise: the Gram identity would cancel
    ~1e8-fold) makes the tensor path's error sample take the direct residual
    ||M - V W|| instead (gated on the device, engine.cu tc_e2): it matches the
    fp64 residual, which the Gram identity with this C could not."""
    rng = np.random.default_rng(m + 7 * n + r)
    V = rng.random((m, r)).astype(np.float32)
    W = rng.random((r, n)).astype(np.float32)
    VW = V.astype(np.float64) @ W.astype(np.float64)
    M = np.maximum(VW * (1 + 1e-4 * rng.standard_normal((m, n))), 0).astype(np.float32)
    ref = float(np.linalg.norm(M.astype(np.float64) - VW))
    with P.Session(dtype=P.F32, gemm_path=P.GEMM_TCGEN05) as s:
        s.set_data(M, P.ImageGrid(m, 1))
        s.set_factors(V, W)
        assert s.tc_active
        e_tc = s.error()
    assert abs(e_tc - ref) / ref < 1e-5, (e_tc, ref)


def test_tc_products_wide_range(P, gpu):
    """Rows of very different magnitude (per-row fixed-point scales, 24 decades
    across M's rows, 12-18 across the factors): the digit model holds exactly,
    and every entry of A and C keeps fp32-level relative accuracy against fp64
    (the sums are dominated by a few terms near the row maximum, whose grid
    step is <= 2^-21 relative)."""
    rng = np.random.default_rng(11)
    m, n, r = 1024, 4096, 64
    M = (rng.random((m, n)) * np.logspace(-12, 12, m)[:, None]).astype(np.float32)
    V = (rng.random((m, r)) * np.logspace(-6, 6, r)[None, :]).astype(np.float32)
    W = (rng.random((r, n)) * np.logspace(-9, 9, r)[:, None]).astype(np.float32)
    M64, V64, W64 = M.astype(np.float64), V.astype(np.float64), W.astype(np.float64)
    with P.Session(dtype=P.F32, gemm_path=P.GEMM_TCGEN05) as s:
        s.set_data(M, P.ImageGrid(m, 1))
        s.set_factors(V, W)
        A, C = s.products()
    np.testing.assert_allclose(A, ixmodel.product_A(M, W), rtol=1e-14, atol=0)
    np.testing.assert_allclose(C, ixmodel.product_C(V, M), rtol=1e-14, atol=0)
    A_ref, C_ref = M64 @ W64.T, V64.T @ M64
    ea = np.max(np.abs(A - A_ref) / np.abs(A_ref))
    ec = np.max(np.abs(C - C_ref) / np.abs(C_ref))
    assert ea < 5e-6 and ec < 5e-6, (ea, ec)


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


@pytest.mark.parametrize("r,n", [(64, 16384), (64, 4100), (49, 8192), (20, 2048), (7, 33002), (64, 2047)])
def test_gram_w_dmma(P, gpu, r, n):
    """B = W W^T of a wide factor on the fp64 tensor-core path (gram_dmma.cu: upper-triangle DMMA tiles,
    mirrored; ragged ranks and K ranges, an odd K taking the scalar staging path; n < 2048 the SIMT tiles)
    against fp64 numpy; exactly symmetric."""
    rng = np.random.default_rng(r * 1000 + n)
    m = 256
    M = rng.random((m, n)).astype(np.float32)
    V = rng.random((m, r))
    W = rng.random((r, n)) * (rng.random((r, n)) > 0.3)  # NMF factors are sparse
    with P.Session(dtype=P.F32) as s:
        s.set_data(M, P.ImageGrid(m, 1))
        s.set_factors(V, W)
        B = s.gram_w()
    ref = W @ W.T
    assert np.array_equal(B, B.T)
    assert np.max(np.abs(B - ref)) <= 1e-13 * np.max(np.abs(ref)) * np.sqrt(n), np.max(np.abs(B - ref))


@pytest.mark.parametrize("r", [48, 33, 16, 1])
def test_tensor_path_ranks(P, gpu, restated, r):
    """Ranks other than the benchmarked 64 on the tensor path (r = 48: the direct residual asks for exactly
    48 KB of dynamic shared memory), every sample within 1e-5 of the oracle fed the same fp32 data."""
    M = oracle.generate_config(0, n=2048, restated=restated).astype(np.float32)
    _, _, to = restated.run_configuration(M.astype(np.float64), 32, 32, 2, "hals", "fmg", r, 0, 8.0, 1)
    with P.Session(dtype=P.F32, gemm_path=P.GEMM_TCGEN05) as s:
        s.set_data(M, P.ImageGrid(32, 32))
        t = s.run_configuration(2, "hals", "fmg", r, 0, 8.0, 1)
        assert s.tc_active
    assert len(t.error) == len(to.error)
    assert np.max(np.abs(t.error - to.error) / to.error) < 1e-5


@pytest.mark.parametrize("kind", ["hals", "mu"])
@pytest.mark.parametrize("r,m,n", [(64, 4224, 4100), (49, 4100, 4228), (12, 8192, 4096), (64, 260, 4100)])
def test_dmma_sweeps_against_oracle(P, gpu, restated, kind, r, m, n):
    """One HALS / MU step of an fp32 non-exact session whose sweeps run on the fp64 tensor cores
    (hals_dmma.cu: blocked HALS sweeps, MU products; ranks below 64 zero-padded, ragged last warps) with
    fp64-accumulated SIMT products, against the oracle's step on the same fp32 data: the sweeps only reorder
    fp64 sums."""
    rng = np.random.default_rng(m + n + r)
    M = rng.random((m, n)).astype(np.float32)
    V0 = rng.random((m, r))
    W0 = rng.random((r, n)) * (rng.random((r, n)) > 0.25)
    step = restated.hals_step if kind == "hals" else restated.mu_step
    Vo, Wo = step(M.astype(np.float64), V0, W0)[:2]
    with P.Session(dtype=P.F32, gemm_path=P.GEMM_SIMT) as s:
        s.set_data(M, P.ImageGrid(m, 1))
        s.set_factors(V0, W0)
        s.steps(kind, 1)
        V, W = s.get_factors()
    assert relnorm(V, Vo) < 1e-11 and relnorm(W, Wo) < 1e-11, (relnorm(V, Vo), relnorm(W, Wo))


@pytest.mark.parametrize("r,m", [(64, 16384), (49, 4100), (20, 2048), (7, 33001), (64, 2047)])
def test_gram_v_dmma(P, gpu, r, m):
    """D = V^T V of a tall factor on the fp64 tensor-core path (gram_dmma.cu over V's K-major layout; an odd
    rank takes the scalar staging path, m < 2048 the SIMT tiles) against fp64 numpy; exactly symmetric."""
    rng = np.random.default_rng(r * 1000 + m)
    n = 128
    M = rng.random((m, n)).astype(np.float32)
    V = rng.random((m, r)) * (rng.random((m, r)) > 0.3)
    W = rng.random((r, n))
    with P.Session(dtype=P.F32) as s:
        s.set_data(M, P.ImageGrid(m, 1))
        s.set_factors(V, W)
        D = s.gram_v()
    ref = V.T @ V
    assert np.array_equal(D, D.T)
    assert np.max(np.abs(D - ref)) <= 1e-13 * np.max(np.abs(ref)) * np.sqrt(m), np.max(np.abs(D - ref))
