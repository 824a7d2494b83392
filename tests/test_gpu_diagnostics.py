"""GPU parity of the multigrid diagnostics (transfer.cpp:128-153): smoothness
s_M = ||M - P R M||_F / ||M||_F and both sides of the coarse-initialization
bound, computed on the device (k_csr_residual + the resident pyramid) and
checked against the reference's golden values (tests/golden/diagnostics.npz,
from oracle/_ref) and the C restatement on larger grids.

Tolerance: fp64 sessions 1e-12 relative (the device sums in a different, fixed
order); fp32 sessions 1e-6 relative (M and R M stored in fp32).
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

D = np.load(os.path.join(os.path.dirname(__file__), "golden", "diagnostics.npz"))
SMOOTH_CASES = sorted({k[2:-2] for k in D.files if k.startswith("s_") and k.endswith("_s")})


@pytest.fixture(autouse=True)
def _defaults(P, gpu):
    P.set_default_options()
    yield
    P.set_default_options()


@pytest.mark.parametrize("name", SMOOTH_CASES)
def test_smoothness_golden(P, name):
    h, w = (int(x) for x in D[f"s_{name}_hw"])
    want = float(D[f"s_{name}_s"])
    got = P.smoothness(D[f"s_{name}_M"], P.ImageGrid(h, w))
    assert abs(got - want) <= 1e-12 * max(want, 1e-3), (got, want)


def test_smoothness_zero_matrix_raises(P):
    # test_transfer.cpp:160
    with pytest.raises(ValueError, match="zero matrix"):
        P.smoothness(np.zeros((9, 4)), P.ImageGrid(3, 3))


def test_initialization_bound_golden(P):
    for t in range(int(D["n_bound"])):
        h, w = (int(x) for x in D[f"b{t}_hw"])
        lhs, rhs = P.initialization_bound(D[f"b{t}_M"], P.ImageGrid(h, w), D[f"b{t}_Vc"], D[f"b{t}_W"])
        wl, wr = D[f"b{t}_lr"]
        assert abs(lhs - wl) <= 1e-12 * wl and abs(rhs - wr) <= 1e-12 * wr, (t, lhs, wl, rhs, wr)
        assert lhs <= rhs * (1 + 1e-9)  # acceptance.cpp:405


def test_initialization_bound_known_answers(P, restated):
    # test_transfer.cpp:200-218: exact coarse factorisation of constant data -> lhs = 0
    Cm = np.full((9, 3), 0.5)
    Cc = restated.apply_operator(3, 3, 0, Cm)
    lhs, rhs = P.initialization_bound(Cm, P.ImageGrid(3, 3), Cc[:, :1], np.ones((1, 3)))
    assert lhs == pytest.approx(0.0, abs=1e-12) and rhs >= lhs


@pytest.mark.parametrize("dtype,tol", [("f64", 1e-12), ("f32", 1e-6)])
def test_session_diagnostics_pyramid(P, restated, dtype, tol):
    """Session path on a 129 x 96 grid, 700 columns: s_M at levels 0 and 1 and
    the bound at level 1, against the restatement on the same (restricted) data."""
    rng = np.random.default_rng(7)
    h, w, n, r = 129, 96, 700, 6
    yy, xx = np.meshgrid(np.linspace(0, 1, h), np.linspace(0, 1, w), indexing="ij")  # (h, w)
    base = np.stack([np.exp(-((xx - rng.random()) ** 2 + (yy - rng.random()) ** 2) / 0.05).T.reshape(-1)
                     for _ in range(r)], 1)  # column-major pixels (ImageGrid::index)
    M = base @ rng.random((r, n)) + 0.05 * rng.random((h * w, n))
    dt = np.float64 if dtype == "f64" else np.float32
    Md = M.astype(dt).astype(np.float64)
    M1 = restated.apply_operator(h, w, 0, Md)
    h1, w1 = (h + 1) // 2, (w + 1) // 2
    with P.Session(dtype=P.F64 if dtype == "f64" else P.F32) as s:
        s.set_data(M.astype(dt), P.ImageGrid(h, w))
        s0 = s.smoothness(0)
        s1 = s.smoothness(1)
        Vc = rng.random(((h1 + 1) // 2 * ((w1 + 1) // 2), r))
        W = rng.random((r, n))
        lhs, rhs = s.initialization_bound(Vc, W, level=1)
    want0 = restated.smoothness(Md, h, w)
    want1 = restated.smoothness(M1.astype(dt).astype(np.float64), h1, w1)
    wl, wr = restated.initialization_bound(M1.astype(dt).astype(np.float64), h1, w1, Vc.astype(dt), W.astype(dt))
    assert abs(s0 - want0) <= tol * want0, (s0, want0)
    assert abs(s1 - want1) <= tol * want1, (s1, want1)
    assert abs(lhs - wl) <= tol * wl and abs(rhs - wr) <= tol * wr, (lhs, wl, rhs, wr)
    assert lhs <= rhs
    # smooth data: the pyramid loses little (test_io.cpp:203 uses < 0.1 on its synthetic set)
    assert s0 < 0.1
