"""Config-4 pyramid build (GridHierarchy::build on the device, transfer.cpp:
155-174): time of build_levels(5) on the generated 64 GiB M, and the
restriction kernels' achieved bandwidth (bytes = sum over levels of
(m_l + m_(l+1)) n 4: read the finer level, write the coarser)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1009_0881_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
for rep in range(2):
    with P.Session(dtype=P.F32) as s:
        s.generate(4, seed=0, n_total=n)
        s.sync()
        t0 = time.perf_counter()
        s.build_levels(5)
        s.sync()
        dt = time.perf_counter() - t0
        ms = [s.level_grid(l).pixels() for l in range(5)]
    byts = sum((ms[l] + ms[l + 1]) * n * 4 for l in range(4))
    print(f"n={n} levels {ms}: build {dt * 1e3:.1f} ms, {byts / 1e9:.1f} GB moved, {byts / dt / 1e9:.0f} GB/s")
