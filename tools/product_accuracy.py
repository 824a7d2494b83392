"""Tensor-path product accuracy: A = M W^T and C = V^T M (r = 64) against fp64
numpy products of the same fp32 inputs, at three aligned shapes."""
import sys; sys.path.insert(0, '.')
import numpy as np, paper_1009_0881_b200 as P
for (m, n) in [(1024, 2048), (2048, 4096), (4096, 8192)]:
    rng = np.random.default_rng(m + n)
    M = rng.random((m, n)).astype(np.float32); M[rng.random((m, n)) < 0.1] = 0
    V = rng.random((m, 64)).astype(np.float32); W = (rng.random((64, n)) * 3).astype(np.float32)
    M64, V64, W64 = M.astype(np.float64), V.astype(np.float64), W.astype(np.float64)
    with P.Session(dtype=P.F32, gemm_path=P.GEMM_TCGEN05) as s:
        s.set_data(M, P.ImageGrid(m, 1)); s.set_factors(V64, W64)
        A, C = s.products()
    ea = np.linalg.norm(A - M64 @ W64.T) / np.linalg.norm(M64 @ W64.T)
    ec = np.linalg.norm(C - V64.T @ M64) / np.linalg.norm(V64.T @ M64)
    print(m, n, "rel err A %.2e C %.2e" % (ea, ec))
