"""Trajectory deviation of a tensor-path fp32 run (config-0 generator at n = 4096,
r = 20, HALS work:30, none and 3-level FMG) from the fp64 oracle fed the
fp32-rounded inputs (the quantity tests/test_gpu_tc.py bounds by 6e-5)."""
import sys; sys.path.insert(0, '.')
import numpy as np, oracle, paper_1009_0881_b200 as P
o = oracle.Restated()
M = oracle.generate_config(0, n=4096, restated=o).astype(np.float32)
V0, W0 = o.random_init(1024, 4096, 20, 0)
r32 = lambda a: np.asarray(a, np.float32).astype(np.float64)
for cycle in ("none", "fmg"):
    L = 1 if cycle == "none" else 3
    _, _, to = o.run_cycle_on(r32(M), 32, 32, L, L, r32(V0), r32(W0), "hals", cycle, 30.0, 1)
    with P.Session(dtype=P.F32, gemm_path=P.GEMM_TCGEN05) as s:
        s.set_data(M, P.ImageGrid(32, 32))
        tg = s.run_configuration(3, "hals", cycle, 20, 0, 30.0, 1)
    print(cycle, "max rel dev %.2e" % float(np.max(np.abs(tg.error - to.error) / to.error)))
