"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
the tensor-path products and a Gram-identity sample, fp32 and fp64 HALS /
MU / ANLS single-level and FMG runs, a tight-fit direct-residual sample and
the resident phase API, all at small shapes.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1009_0881_b200 as P  # noqa: E402

rng = np.random.default_rng(0)
M = rng.random((1024, 2048)).astype(np.float32)
V = rng.random((1024, 64))
W = rng.random((64, 2048))
with P.Session(dtype=P.F32, gemm_path=P.GEMM_TCGEN05) as s:
    s.set_data(M, P.ImageGrid(32, 32))
    s.set_factors(V, W)
    A, C = s.products()
    e = s.error()
    tr = s.run_configuration(3, "hals", "fmg", 64, 0, 4.0, 1)
print("tc products", A.shape, C.shape, e, tr.error[-1])
Mt = (V[:, :8] @ W[:8]).astype(np.float32)
with P.Session(dtype=P.F32, gemm_path=P.GEMM_TCGEN05) as s:
    s.set_data(Mt, P.ImageGrid(32, 32))
    s.set_factors(V[:, :8], W[:8])
    print("tight-fit sample", s.error())
for dt in (P.F32, P.F64):
    for kind in ("hals", "mu", "anls"):
        with P.Session(dtype=dt) as s:
            s.set_data(M[:, :300], P.ImageGrid(32, 32))
            t1 = s.run_configuration(1, kind, "none", 10, 0, 3.0, 1)
            t2 = s.run_configuration(3, kind, "fmg", 10, 0, 3.0, 1)
        print(dt, kind, t1.error[-1], t2.error[-1])
with P.Session(dtype=P.F64, exact=True) as s:
    s.set_data(M[:, :200], P.ImageGrid(32, 32))
    s.build_levels(2)
    s.init_random(8, 1)
    s.restrict_V(0)
    left, work, tr = s.run_phase(1, "hals", 2.0, 1.0, 1.0, 1)
    s.prolong_V(0)
    print("phase", left, work, tr.error[-1])
print("sanitize_run ok")
