"""Iterations/s on BASELINE configs 0-3 (L2-resident shapes) through the session
API: HALS single-level work:100 (exactly 100 sweeps), trace_every=0, device
data; fp32 storage (SIMT fp64-accumulating products) and fp64."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1009_0881_b200 as P

for cfg in (0, 1, 2, 3):
    c = P.GEN_CONFIGS[cfg]
    for dt, name in ((P.F32, "f32"), (P.F64, "f64")):
        with P.Session(dtype=dt) as s:
            s.generate(cfg, seed=0)
            s.run_configuration(1, "hals", "none", c["r"], 0, 5.0, 0)  # warm-up
            s.sync()
            t = time.perf_counter()
            tr = s.run_configuration(1, "hals", "none", c["r"], 0, 100.0, 0)
            s.sync()
            dt_s = time.perf_counter() - t
            steps = int(tr.phase_steps.sum())
            print(f"cfg{cfg} {name}: {steps} sweeps in {dt_s*1e3:.1f} ms -> {steps/dt_s:.0f} it/s "
                  f"({dt_s/steps*1e3:.3f} ms/step), launches/step {s.launches/ max(steps,1):.1f}")
