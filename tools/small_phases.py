"""Per-phase event times of one solver step on BASELINE configs 0-3 (fp32
storage, device data, profiled eager steps) next to the graph-replayed step
time -- where the small shapes spend their sweep."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1009_0881_b200 as P  # noqa: E402

for cfg, kinds in ((0, ("hals",)), (1, ("mu", "hals")), (2, ("anls", "hals")), (3, ("hals", "mu", "anls"))):
    c = P.GEN_CONFIGS[cfg]
    for kind in kinds:
        with P.Session(dtype=P.F32) as s:
            s.generate(cfg, seed=0)
            s.run_configuration(1, kind, "none", c["r"], 0, 3.0, 0)
            s.sync()
            t = time.perf_counter()
            n = 20 if kind == "anls" else 200
            s.steps(kind, n)
            s.sync()
            dt = (time.perf_counter() - t) / n
            s.set_profiling(True)
            s.steps(kind, 5)
            ph = s.phase_times()
            s.set_profiling(False)
        print(f"config {cfg} {kind}: step {dt * 1e3:.4f} ms; phases (ms) " +
              ", ".join(f"{k} {v:.4f}" for k, v in ph.items()), flush=True)
