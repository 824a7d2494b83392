"""Golden error trajectories of the BENCHMARKED path's configuration, from the
UNMODIFIED reference (oracle/_ref, built by `make -C oracle ref`):

    python tests/golden/make_tc_trajectory.py      (~5 min on 8 cores)

Input: a column slice of BASELINE config 4 -- the config-4 generator
(256x256 grid, m = 65536, r = 64, 3 blobs, sigma in [4, 20], seed 0) with
n_total = 262144, columns [0, 4096) -- rounded to fp32, and random_init(m,
4096, 64, seed 0) rounded to fp32.  The reference runs in fp64 on those
fp32-rounded inputs (SURVEY 8(c) "fp32 parity"):
  * none: run_solver(M, V0, W0, HALS, work:20, trace_every=1)
          (proj/src/solvers.cpp:343-355)
  * fmg:  full_multigrid over the 5-level hierarchy (multilevel.hpp:22-38,
          multilevel.cpp:93-114), HALS, work:20, trace_every=1.
tests/test_gpu_tc_config4.py runs the same inputs through the tcgen05 path
(GEMM_TCGEN05 forced) and compares every sample.  The fixture stores the
trajectories and a digest of the fp32 M (the GPU test regenerates M on the
device and checks the digest: the device generator must reproduce it bit
for bit).
"""
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402

N_TOTAL, N_SLICE, R, LEVELS, WORK = 262144, 4096, 64, 5, 20.0


def main():
    ref, restated = oracle.Reference(), oracle.Restated()
    t0 = time.time()
    M = oracle.generate_config(4, n=N_TOTAL, col0=0, n_cols=N_SLICE, restated=restated)
    M32 = M.astype(np.float32)
    V0, W0 = ref.random_init(M32.shape[0], N_SLICE, R, 0)
    V32, W32 = V0.astype(np.float32), W0.astype(np.float32)
    M64, V64, W64 = M32.astype(np.float64), V32.astype(np.float64), W32.astype(np.float64)
    out = {"m_digest": np.frombuffer(hashlib.sha256(M32.tobytes()).digest(), np.uint8),
           "shape": np.array(M32.shape), "rank": np.array(R), "work": np.array(WORK),
           "norm": np.array(np.sqrt((M64 * M64).sum()))}
    _, _, t = ref.run_solver(M64, V64, W64, "hals", WORK, 1)
    print(f"none: {len(t.error)} samples, final rel {t.error[-1] / out['norm']:.6f} ({time.time() - t0:.0f} s)",
          flush=True)
    out.update(none_error=t.error, none_level=t.level, none_work=t.work)
    _, _, t = ref.run_cycle_on(M64, 256, 256, LEVELS, LEVELS, V64, W64, "hals", "fmg", WORK, 1)
    print(f"fmg: {len(t.error)} samples, final rel {t.error[-1] / out['norm']:.6f} ({time.time() - t0:.0f} s)",
          flush=True)
    out.update(fmg_error=t.error, fmg_level=t.level, fmg_work=t.work)
    np.savez_compressed(os.path.join(HERE, "tc_trajectory_config4.npz"), **out)


if __name__ == "__main__":
    main()
