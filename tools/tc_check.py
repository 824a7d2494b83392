"""Quick correctness sweep of the tcgen05 products (one process per shape)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1009_0881_b200 as P
m, n, r = (int(x) for x in sys.argv[1:4])
rng = np.random.default_rng(1)
M = rng.random((m, n)).astype(np.float32)
V = rng.random((m, r)); W = rng.random((r, n))
with P.Session(dtype=P.F32, gemm_path=P.GEMM_TCGEN05) as s:
    s.set_data(M, P.ImageGrid(m, 1)); s.set_factors(V, W)
    A, C = s.products()
M64 = M.astype(np.float64); V32 = V.astype(np.float32).astype(np.float64); W32 = W.astype(np.float32).astype(np.float64)
ea = np.linalg.norm(A - M64 @ W32.T) / np.linalg.norm(M64 @ W32.T)
ec = np.linalg.norm(C - V32.T @ M64) / np.linalg.norm(V32.T @ M64)
print(f"{m}x{n} r={r}: relerr A {ea:.2e} C {ec:.2e}", "OK" if max(ea, ec) < 2e-6 else "BAD")
