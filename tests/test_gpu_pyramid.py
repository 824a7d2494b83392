"""GPU parity of the resident pyramid R(...R(M)) (GridHierarchy::build,
transfer.cpp:155-174) against the oracle's restriction, level by level.

Covers both restriction kernels: the TMA-pipelined stream (restrict_tma.cu:
rows of at least 2048 bytes, 16-byte aligned) and the cp.async slab kernel
(narrow or unaligned matrices), on even, odd and mixed grids whose strips of
8 coarse pixel rows are ragged, with column counts that leave a ragged last
512-byte slab.  fp64 sessions and exact mode are bit-identical to the oracle
(the reference's unfused fp64 sum in entry order); fp32 non-exact levels use
fp32 FMA in the same order (within a few ulp).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RNG = np.random.default_rng(77)

# (h, w, n): n * 8 >= 2048 and n % 2 == 0 take the TMA stream in fp64; 165 and 251 take the slab kernel
GRIDS = [(32, 32, 1000), (19, 19, 300), (112, 92, 400), (37, 50, 258), (243, 320, 256), (21, 18, 165), (16, 9, 251),
         (2, 2, 512), (5, 3, 640)]


def oracle_pyramid(restated, M, h, w, levels):
    out = [M]
    for _ in range(levels - 1):
        out.append(restated.apply_operator(h, w, 0, out[-1]))
        h, w = (h + 1) // 2, (w + 1) // 2
        if h < 2 or w < 2:
            break
    return out


def n_levels(h, w, cap=5):
    L = 1
    while L < cap and h >= 2 and w >= 2:
        h, w, L = (h + 1) // 2, (w + 1) // 2, L + 1
    return L


@pytest.mark.parametrize("h,w,n", GRIDS)
@pytest.mark.parametrize("exact", [False, True])
def test_pyramid_fp64_bitwise(P, gpu, restated, h, w, n, exact):
    M = RNG.random((h * w, n))
    L = n_levels(h, w)
    ref = oracle_pyramid(restated, M, h, w, L)
    with P.Session(dtype=P.F64, exact=exact) as s:
        s.set_data(M, P.ImageGrid(h, w))
        s.build_levels(len(ref))
        for l in range(1, len(ref)):
            got = s.export_level(l)
            assert got.dtype == np.float64 and got.shape == ref[l].shape
            assert np.array_equal(got, ref[l]), (l, float(np.max(np.abs(got - ref[l]))))
            # the level norms feed every error sample
            assert s.norm2(l) == pytest.approx(float(np.sum(ref[l] * ref[l])), rel=1e-13)


@pytest.mark.parametrize("h,w,n", [(32, 32, 1000), (112, 92, 576), (37, 50, 516), (21, 18, 165)])
def test_pyramid_fp32_storage(P, gpu, restated, h, w, n):
    """fp32 sessions: restricted levels are fp64 (restricted from the fp32 data in the reference's fp64
    arithmetic: bit-identical to the oracle fed the same fp32 M) unless the tensor path streams them."""
    M = RNG.random((h * w, n)).astype(np.float32)
    L = n_levels(h, w, 4)
    ref = oracle_pyramid(restated, M.astype(np.float64), h, w, L)
    with P.Session(dtype=P.F32) as s:
        s.set_data(M, P.ImageGrid(h, w))
        s.build_levels(len(ref))
        for l in range(1, len(ref)):
            got = s.export_level(l)
            assert got.dtype == np.float64
            assert np.array_equal(got, ref[l]), l


@pytest.mark.parametrize("exact", [False, True])
def test_pyramid_fp32_levels_tensor_path(P, gpu, restated, exact):
    """Levels the tensor path streams stay fp32 (its input format): the fp32 -> fp32 restriction, exact mode
    in the reference's fp64 arithmetic rounded once, otherwise fp32 FMA in the same order."""
    h, w, n = 64, 48, 1536
    M = RNG.random((h * w, n)).astype(np.float32)
    ref = oracle_pyramid(restated, M.astype(np.float64), h, w, 3)
    with P.Session(dtype=P.F32, gemm_path=P.GEMM_TCGEN05, exact=exact) as s:
        s.set_data(M, P.ImageGrid(h, w))
        s.build_levels(3)
        got1 = s.export_level(1)
        if got1.dtype == np.float32:  # streamed by the tensor path
            if exact:
                assert np.array_equal(got1, ref[1].astype(np.float32))
            else:
                assert np.max(np.abs(got1 - ref[1]) / np.maximum(ref[1], 1e-30)) < 5e-7
            # the maxima pass also sums ||M_1||^2
            assert s.norm2(1) == pytest.approx(float(np.sum(got1.astype(np.float64) ** 2)), rel=1e-12)
        else:
            assert np.array_equal(got1, ref[1])
