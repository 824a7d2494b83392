"""Trajectory deviation on the config-4 golden slice (tests/golden/
tc_trajectory_config4.npz) for several storage / product paths, to separate
the tensor-path product error from the fp32 storage of the factors.

    python tools/config4_deviation.py
"""
import hashlib
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_1009_0881_b200 as P  # noqa: E402

g = np.load(os.path.join(REPO, "tests", "golden", "tc_trajectory_config4.npz"))
m, n = (int(x) for x in g["shape"])
with P.Session(dtype=P.F32) as s:
    s.generate(4, seed=0, n_total=262144, col0=0, n_local=n)
    M32 = np.empty((m, n), np.float32)
    s.export_data(M32.ctypes.data)
assert hashlib.sha256(M32.tobytes()).digest() == g["m_digest"].tobytes()
V0, W0 = P.random_init(m, n, int(g["rank"]), 0)
V0, W0 = V0.astype(np.float32).astype(np.float64), W0.astype(np.float32).astype(np.float64)
variants = [("f32 tc", P.F32, P.GEMM_TCGEN05), ("f32 simt", P.F32, P.GEMM_SIMT), ("f64 simt", P.F64, P.GEMM_SIMT)]
for name, dt, gemm in variants:
    for cycle in ("none", "fmg"):
        L = 1 if cycle == "none" else 5
        with P.Session(dtype=dt, gemm_path=gemm) as s:
            s.set_data(M32 if dt == P.F32 else M32.astype(np.float64), P.ImageGrid(256, 256))
            tr = s.run_cycle(L, L, V0, W0, "hals", cycle, float(g["work"]), 1)
        err, lev = g[f"{cycle}_error"], g[f"{cycle}_level"]
        dev = np.abs(tr.error - err) / err
        per = {int(l): float(dev[lev == l].max()) for l in np.unique(lev)}
        print(f"{name:9s} {cycle:4s} max {dev.max():.2e}  per level " +
              " ".join(f"L{k}:{v:.1e}" for k, v in per.items()) + f"  first>1e-5 at sample "
              f"{int(np.argmax(dev > 1e-5)) if (dev > 1e-5).any() else -1} of {len(dev)}", flush=True)

# evaluation vs trajectory: the tensor path with its error samples taken by
# the direct residual (ERROR_DIRECT) instead of the Gram identity
for cycle in ("none", "fmg"):
    L = 1 if cycle == "none" else 5
    with P.Session(dtype=P.F32, gemm_path=P.GEMM_TCGEN05, error_mode=P.ERROR_DIRECT) as s:
        s.set_data(M32, P.ImageGrid(256, 256))
        tr = s.run_cycle(L, L, V0, W0, "hals", cycle, float(g["work"]), 1)
    err, lev = g[f"{cycle}_error"], g[f"{cycle}_level"]
    dev = np.abs(tr.error - err) / err
    print(f"tc+direct {cycle:4s} max {dev.max():.2e}  per level " +
          " ".join(f"L{int(l)}:{float(dev[lev == l].max()):.1e}" for l in np.unique(lev)), flush=True)
    nrm = float(g["norm"])
    if cycle == "fmg":
        print("rel errors (golden) per level min:", {int(l): float((err[lev == l]).min()) for l in np.unique(lev)})
        print("dev trace:", " ".join(f"{l}:{d:.1e}" for l, d in zip(lev[:80], dev[:80])))
