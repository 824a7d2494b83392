"""Sweeps/s of every solver kind (MU / HALS / ANLS) on BASELINE configs 0-3
through the session API: single level, work:W (exactly W sweeps),
trace_every=0, device data, fp32 storage; next to the reference's own step
(oracle/_ref, fp64, OpenMP on all host cores) on the same data when
available.  ANLS counts its NNLS exchanges (warm starts make late sweeps cheap,
so the first sweeps are timed separately)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1009_0881_b200 as P

ref = None
try:
    import oracle
    if oracle.Reference.available():
        ref, restated = oracle.Reference(), oracle.Restated()
except Exception:
    pass

for cfg in (0, 1, 2, 3):
    c = P.GEN_CONFIGS[cfg]
    for kind in ("mu", "hals", "anls"):
        for work in (5.0, 50.0):
            with P.Session(dtype=P.F32) as s:
                s.generate(cfg, seed=0)
                s.run_configuration(1, kind, "none", c["r"], 0, 2.0, 0)  # warm-up
                s.sync()
                t = time.perf_counter()
                tr = s.run_configuration(1, kind, "none", c["r"], 0, work, 0)
                s.sync()
                dt = time.perf_counter() - t
            steps = int(tr.phase_steps.sum())
            line = f"cfg{cfg} {kind:4s} work:{int(work):3d}: {dt / steps * 1e3:8.3f} ms/sweep"
            if ref is not None and work == 5.0:
                M = oracle.generate_config(cfg, restated=restated)
                V, W = ref.random_init(M.shape[0], M.shape[1], c["r"], 0)
                step = {"mu": ref.mu_step, "hals": ref.hals_step, "anls": ref.anls_step}[kind]
                ts = []
                for _ in range(2):
                    t0 = time.perf_counter()
                    out = step(M, V, W)
                    ts.append(time.perf_counter() - t0)
                    V, W = out[0], out[1]
                line += f"   reference (first sweeps) {np.median(ts) * 1e3:9.2f} ms/sweep"
            print(line, flush=True)
