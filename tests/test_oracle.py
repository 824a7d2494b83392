"""CPU: pin the C restatement (oracle/mlnmf_oracle.c) before trusting it.

Two independent anchors, both offline:
  * tests/golden/reference_golden.npz -- outputs of the UNMODIFIED reference
    (oracle/_ref, built from /root/reference/proj/src by oracle/Makefile) on
    seeded inputs, written by tests/golden/make_golden.py.  The restatement
    must reproduce them bit for bit (same operation order, no FMA).
  * the known-answer tests the reference's own suites hold for the path
    (SURVEY.md section 4), restated here as plain asserts:
    test_core.cpp:33-35,46-60,135-195, test_transfer.cpp:49-116,
    test_solvers.cpp:120-201,310-314, test_multilevel.cpp:44-150 and the
    acceptance.cpp:359-386 end-to-end means.
When oracle/_ref exists (this container) the restatement is also compared
with the live reference on fresh random inputs.
"""
import math

import numpy as np
import pytest

import oracle

G = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "reference_golden.npz"))


# ---------------------------------------------------------------------------
# golden vectors from the reference
# ---------------------------------------------------------------------------
def test_splitmix_and_random_init_golden(restated):
    got = [restated.splitmix_first(int(s)) for s in G["splitmix_seeds"]]
    assert got == [int(x) for x in G["splitmix_first"]]
    V, W = restated.random_init(5, 4, 3, 9)
    assert np.array_equal(V, G["ri_V"]) and np.array_equal(W, G["ri_W"])


@pytest.mark.parametrize("h,w", [(3, 3), (8, 7), (5, 5), (4, 6), (2, 2)])
def test_transfer_operators_golden(restated, h, w):
    assert np.array_equal(restated.operator_dense(h, w, 0), G[f"R_{h}x{w}"])
    assert np.array_equal(restated.operator_dense(h, w, 1), G[f"P_{h}x{w}"])


def test_transfer_apply_golden(restated):
    assert np.array_equal(restated.apply_operator(19, 17, 0, G["apply_X"]), G["apply_R"])
    assert np.array_equal(restated.apply_operator(19, 17, 1, G["apply_Xc"]), G["apply_P"])


D = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "diagnostics.npz"))
SMOOTH_CASES = sorted({k[2:-2] for k in D.files if k.startswith("s_") and k.endswith("_s")})


@pytest.mark.parametrize("name", SMOOTH_CASES)
def test_smoothness_golden(restated, name):
    h, w = (int(x) for x in D[f"s_{name}_hw"])
    assert restated.smoothness(D[f"s_{name}_M"], h, w) == float(D[f"s_{name}_s"])


def test_initialization_bound_golden(restated):
    for t in range(int(D["n_bound"])):
        h, w = (int(x) for x in D[f"b{t}_hw"])
        lhs, rhs = restated.initialization_bound(D[f"b{t}_M"], h, w, D[f"b{t}_Vc"], D[f"b{t}_W"])
        assert (lhs, rhs) == tuple(D[f"b{t}_lr"]), t
        assert lhs <= rhs * (1 + 1e-9)  # acceptance.cpp:405


def test_diagnostics_known_answers(restated):
    # test_transfer.cpp:155-160, 200-218
    assert restated.smoothness(np.ones((9, 4)), 3, 3) == pytest.approx(0.0, abs=1e-15)
    with pytest.raises(oracle.OracleError):
        restated.smoothness(np.zeros((9, 4)), 3, 3)
    C_ = np.full((9, 3), 0.5)
    Cc = restated.apply_operator(3, 3, 0, C_)
    lhs, rhs = restated.initialization_bound(C_, 3, 3, Cc[:, :1], np.ones((1, 3)))
    assert lhs == pytest.approx(0.0, abs=1e-12) and rhs >= lhs


@pytest.mark.parametrize("i", [0, 1, 2])
def test_single_steps_golden(restated, i):
    M, V0, W0 = G[f"step{i}_M"], G[f"step{i}_V0"], G[f"step{i}_W0"]
    V, W, deg = restated.hals_step(M, V0, W0)
    assert np.array_equal(V, G[f"step{i}_hals_V"]) and np.array_equal(W, G[f"step{i}_hals_W"])
    assert deg == int(G[f"step{i}_hals_deg"])
    V, W = restated.mu_step(M, V0, W0)
    assert np.array_equal(V, G[f"step{i}_mu_V"]) and np.array_equal(W, G[f"step{i}_mu_W"])
    V, W, counts = restated.anls_step(M, V0, W0)
    assert np.array_equal(V, G[f"step{i}_anls_V"]) and np.array_equal(W, G[f"step{i}_anls_W"])
    assert np.array_equal(counts, G[f"step{i}_anls_counts"])
    assert restated.frobenius_error(M, V0, W0) == float(G[f"step{i}_err"])


def test_nnls_golden(restated):
    for t in range(G["nnls_G"].shape[0]):
        r, it = (int(v) for v in G["nnls_rit"][t])
        x, it2 = restated.nnls_active_set(G["nnls_G"][t][:r, :r], G["nnls_h"][t][:r], G["nnls_x0"][t][:r])
        assert np.array_equal(x, G["nnls_x"][t][:r]), t
        assert it2 == it, t


@pytest.mark.parametrize("kind", ["mu", "hals", "anls"])
@pytest.mark.parametrize("cycle", ["none", "ni", "vc", "fmg"])
def test_run_configuration_golden(restated, kind, cycle):
    amount = 8.0 if kind == "anls" else 24.0
    V, W, tr = restated.run_configuration(G["run_M"], 17, 17, 3, kind, cycle, 4, 5, amount, 1)
    k = f"run_{kind}_{cycle}"
    assert np.array_equal(V, G[k + "_V"]) and np.array_equal(W, G[k + "_W"])
    assert np.array_equal(tr.error, G[k + "_err"])
    assert np.array_equal(tr.work, G[k + "_work"])
    assert np.array_equal(tr.level, G[k + "_level"])
    assert np.array_equal(tr.alloc_level.astype(np.float64), G[k + "_alloc"][0])
    assert np.array_equal(tr.alloc_amount, G[k + "_alloc"][1])
    assert np.array_equal(tr.counts, G[k + "_counts"])
    assert tr.degenerate == int(G[k + "_deg"])


@pytest.mark.parametrize("cycle", ["none", "fmg"])
def test_config0_trajectory_golden(restated, cycle):
    """BASELINE config 0 (1024 x 1000, r 20, HALS, work:100) error trajectory."""
    M0 = oracle.generate_config(0, restated=restated)
    V, W, tr = restated.run_configuration(M0, 32, 32, 3, "hals", cycle, 20, 0, 100.0, 1)
    assert np.array_equal(tr.error, G[f"cfg0_{cycle}_err"])
    assert np.array_equal(tr.work, G[f"cfg0_{cycle}_work"])
    assert np.array_equal(np.array([np.linalg.norm(V), np.linalg.norm(W), V.sum(), W.sum()]),
                          G[f"cfg0_{cycle}_VWnorm"])


# ---------------------------------------------------------------------------
# the reference suites' known-answer tests, restated
# ---------------------------------------------------------------------------
def test_kat_splitmix_seed0(restated):
    # test_core.cpp:33-35
    assert restated.splitmix_first(0) == 0xE220A8397B1DCDAF


def test_kat_random_init_layout(restated):
    # test_core.cpp:77-98: V row-major first, then W, from one stream
    V, W = restated.random_init(3, 4, 2, 5)
    V2, W2 = restated.random_init(3, 4, 2, 5)
    assert np.array_equal(V, V2) and np.array_equal(W, W2)
    assert (V >= 0).all() and (V < 1).all() and (W >= 0).all() and (W < 1).all()
    s = 5
    draws = []
    mask = (1 << 64) - 1
    for _ in range(3 * 2 + 2 * 4):  # SplitMix64 (matrix.hpp:76-95) in Python, U = (z >> 11) 2^-53
        s = (s + 0x9E3779B97F4A7C15) & mask
        z = s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & mask
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & mask
        z ^= z >> 31
        draws.append((z >> 11) * 2.0 ** -53)
    assert np.array_equal(V.ravel(), np.array(draws[:6]))
    assert np.array_equal(W.ravel(), np.array(draws[6:]))


def test_kat_frobenius(restated):
    # test_core.cpp:46-60: || [[1,2],[3,4]] - [1,1]^T [1,1] ||_F = sqrt(14)
    M = np.array([[1.0, 2.0], [3.0, 4.0]])
    assert restated.frobenius_error(M, np.ones((2, 1)), np.ones((1, 2))) == pytest.approx(math.sqrt(14.0), rel=1e-15)


def test_kat_iteration_cost(restated):
    # test_core.cpp:135-158 (default s_r = 2r for ANLS: cost_model.hpp:14-24)
    assert restated.iteration_cost(1, 1, 1, "mu") == 6.0
    assert restated.iteration_cost(1000, 100, 10, "mu") == 2220000.0
    assert restated.iteration_cost(1000, 100, 10, "hals") == 2220000.0
    # reduction factor 1110000/285000 for a 4x coarser m (test_core.cpp:171-174)
    assert restated.iteration_cost(1000, 100, 10, "mu") / restated.iteration_cost(250, 100, 10, "mu") == \
        pytest.approx(1110000.0 / 285000.0, rel=1e-15)
    for m in (10, 100, 321):  # exactly linear in m
        c0, c1, c2 = (restated.iteration_cost(x, 50, 4, "mu") for x in (0, m, 2 * m))
        assert c2 - c1 == pytest.approx(c1 - c0, rel=1e-12)


def test_kat_transfer_3x3_and_stencil(restated):
    # test_transfer.cpp:49-116: 3x3 -> 2x2; interior 5x5 stencil 4/16, 2/16, 1/16
    R = restated.operator_dense(5, 5, 0)
    centre = R[1 * 3 + 1]  # coarse (1,1) <- fine (2,2) neighbourhood
    W = centre.reshape(5, 5)  # [j][i] (pixel j*h + i)
    assert W[2, 2] == pytest.approx(4 / 16)
    assert W[1, 2] == pytest.approx(2 / 16) and W[2, 1] == pytest.approx(2 / 16)
    assert W[1, 1] == pytest.approx(1 / 16)
    for n in range(2, 34):  # row sums are 1 on every grid (test_transfer.cpp:91-104)
        for (h, w) in ((n, n), (n, max(2, n - 1))):
            assert np.allclose(restated.operator_dense(h, w, 0).sum(axis=1), 1.0, rtol=0, atol=1e-14)
            assert np.allclose(restated.operator_dense(h, w, 1).sum(axis=1), 1.0, rtol=0, atol=1e-14)


def test_kat_transfer_worked_example(restated):
    # test_transfer.cpp:105-116,135-140: restrict 1..9 on 3x3 and prolong [1,2,3,4] centre
    X = np.arange(1.0, 10.0).reshape(9, 1)
    Y = restated.apply_operator(3, 3, 0, X)
    assert Y.shape == (4, 1)
    Xc = np.array([[1.0], [2.0], [3.0], [4.0]])
    Z = restated.apply_operator(3, 3, 1, Xc)
    assert Z[4, 0] == pytest.approx(2.5)


def test_kat_mu_hand_example(restated):
    # test_solvers.cpp:120-126: M=[[2]], V=W=[[1]] -> V=2, W=1
    V, W = restated.mu_step(np.array([[2.0]]), np.array([[1.0]]), np.array([[1.0]]))
    assert V[0, 0] == 2.0 and W[0, 0] == 1.0


def test_kat_fixed_points(restated):
    # test_solvers.cpp:128-138,165-173: exact factorizations are fixed points
    rng = np.random.default_rng(3)
    V0 = rng.random((12, 3)) + 0.1
    W0 = rng.random((3, 9)) + 0.1
    M = V0 @ W0
    V, W = restated.mu_step(M, V0, W0)
    assert np.allclose(V, V0, rtol=1e-12) and np.allclose(W, W0, rtol=1e-12)
    V, W, _ = restated.hals_step(M, V0, W0)
    assert np.allclose(V, V0, rtol=1e-10) and np.allclose(W, W0, rtol=1e-10)


def test_kat_hals_rank1_and_degenerate(restated):
    # test_solvers.cpp:175-201: rank-1 closed form; a zero column is left untouched
    rng = np.random.default_rng(4)
    M = rng.random((6, 5))
    V0 = rng.random((6, 1)) + 0.1
    W0 = rng.random((1, 5)) + 0.1
    V, W, _ = restated.hals_step(M, V0, W0)
    v = np.maximum(0.0, M @ W0.T / (W0 @ W0.T))
    w = np.maximum(0.0, v.T @ M / (v.T @ v))
    assert np.allclose(V, v, rtol=1e-12) and np.allclose(W, w, rtol=1e-12)
    W0 = rng.random((2, 5))
    W0[1] = 0.0
    V0 = rng.random((6, 2))
    V, W, deg = restated.hals_step(M, V0, W0)
    assert deg >= 1
    assert np.array_equal(V[:, 1], V0[:, 1])


def test_kat_nnls_bruteforce(restated):
    # test_solvers.cpp:41-101: the active-set answer equals the best of all 2^r supports
    rng = np.random.default_rng(5)
    for _ in range(40):
        r = int(rng.integers(1, 6))
        A = rng.random((r, r + 3))
        Gm = A @ A.T + 1e-3 * np.eye(r)
        h = rng.standard_normal(r)
        x, _ = restated.nnls_active_set(Gm, h, np.zeros(r))
        best, bestf = None, np.inf
        for mask in range(1 << r):
            idx = [k for k in range(r) if mask >> k & 1]
            z = np.zeros(r)
            if idx:
                z[idx] = np.linalg.solve(Gm[np.ix_(idx, idx)], h[idx])
            if (z < -1e-12).any():
                continue
            f = 0.5 * z @ Gm @ z - h @ z
            if f < bestf:
                best, bestf = z, f
        assert np.allclose(x, best, atol=1e-9), (x, best)
        g = Gm @ x - h  # KKT
        assert (x >= 0).all() and (g > -1e-8).all() and abs(x @ g) < 1e-8


def test_kat_budget_work10(restated):
    # test_solvers.cpp:310-314: work:10 -> exactly 10 steps and 12 samples
    rng = np.random.default_rng(6)
    M = rng.random((20, 15))
    V0, W0 = restated.random_init(20, 15, 3, 1)
    _, _, tr = restated.run_solver(M, V0, W0, "hals", 10.0, 1)
    assert len(tr.error) == 12
    assert tr.work[-1] == pytest.approx(10.0)
    # first sample = error of the initial factors (test_io.cpp:242-247)
    assert tr.error[0] == restated.frobenius_error(M, V0, W0)


@pytest.mark.parametrize("cycle,expect", [
    ("ni", [(2, 100.0), (1, 300.0)]),
    ("vc", [(1, 100.0), (2, 100.0), (1, 200.0)]),
    ("fmg", [(2, 100.0), (1, 75.0), (2, 75.0), (1, 150.0)]),
])
def test_kat_allocations(restated, cycle, expect):
    # test_multilevel.cpp:44-96 (9x9 grid, 2 levels, MU, T = 400)
    rng = np.random.default_rng(7)
    M = rng.random((81, 6))
    _, _, tr = restated.run_configuration(M, 9, 9, 2, "mu", cycle, 2, 11, 400.0, 1)
    got = list(zip(tr.alloc_level.tolist(), tr.alloc_amount.tolist()))
    assert [lv for lv, _ in got] == [lv for lv, _ in expect]
    assert np.allclose([a for _, a in got], [a for _, a in expect], rtol=1e-12)


def test_kat_step_count_48(restated):
    # test_multilevel.cpp:128-150: 33x33, NI, L=3, MU, work:64 -> 48 fine steps
    rng = np.random.default_rng(8)
    M = rng.random((33 * 33, 4))
    _, _, tr = restated.run_configuration(M, 33, 33, 3, "mu", "ni", 2, 31, 64.0, 1)
    fine = sum(1 for i in range(1, len(tr.work)) if tr.work[i] > tr.work[i - 1] and tr.level[i] == 1)
    assert fine == 48


def test_kat_monotone(restated):
    # acceptance.cpp:97-116 (reduced): MU and HALS never increase the error
    rng = np.random.default_rng(9)
    for s in range(5):
        M = rng.random((30, 20))
        for kind in ("mu", "hals"):
            _, _, tr = restated.run_configuration(M, 6, 5, 1, kind, "none", 3, s, 40.0, 1)
            assert (np.diff(tr.error) <= 1e-12 * tr.error[0]).all()


def test_acceptance8_means(restated):
    """acceptance.cpp:359-386 end-to-end means on the reference's own synthetic
    dataset (fixture), pinned to the values its acceptance binary checks."""
    A = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "acceptance8.npz"))
    expect = {"mu_none": 9.691148, "mu_fmg": 8.924942, "hals_none": 8.251099, "hals_fmg": 8.091289}
    for k, v in expect.items():
        assert float(A[k].mean()) == pytest.approx(v, abs=5e-7)
    # the restatement reproduces two of the twenty runs per arm exactly
    for k in expect:
        kind, cyc = k.split("_")
        lv = 1 if cyc == "none" else 3
        for s in (0, 13):
            _, _, tr = restated.run_configuration(A["M"], 65, 65, lv, kind, cyc, 8, 100 + s, 300.0, 0)
            assert tr.error[-1] == A[k][s]


# ---------------------------------------------------------------------------
# the live reference (only where oracle/_ref was built, i.e. this container)
# ---------------------------------------------------------------------------
def test_restated_matches_live_reference(restated, reference):
    rng = np.random.default_rng(10)
    for (h, w, n, r, kind, cyc) in [(11, 13, 9, 3, "hals", "fmg"), (16, 9, 7, 4, "mu", "vc"),
                                    (10, 10, 12, 2, "anls", "ni")]:
        M = rng.random((h * w, n))
        a = restated.run_configuration(M, h, w, 3, kind, cyc, r, 3, 12.0, 1)
        b = reference.run_configuration(M, h, w, 3, kind, cyc, r, 3, 12.0, 1)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        assert np.array_equal(a[2].error, b[2].error)
