"""Config-4 HALS step time per pyramid level (resident phases, CUDA events),
next to the level's two-pass HBM time: python tools/level_steps.py [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1009_0881_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
with P.Session(dtype=P.F32) as s:
    s.generate(4, seed=0, n_total=n)
    s.build_levels(5)
    s.init_random(64, 0)
    for l in range(4):
        s.restrict_V(l)
    ext = torch.cuda.ExternalStream(s.stream)
    for l in range(5):
        m = s.level_grid(l).pixels()
        s.run_phase(l, "hals", 3.0, 1.0, 1.0, 0)  # warm-up: level norm and statistics, graph capture
        s.sync()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(ext)
        s.run_phase(l, "hals", 10.0, 1.0, 1.0, 0)
        b.record(ext)
        b.synchronize()
        ms = a.elapsed_time(b) / 10
        ideal = 2 * m * n * 4 / 6.5e12 * 1e3
        print(f"level {l}: m={m} step {ms:.3f} ms; two passes at 6.5 TB/s {ideal:.3f} ms ({ideal / ms:.2f})", flush=True)
    # per-phase event times of profiled (eager) steps at each level
    for l in range(5):
        s.set_profiling(True)
        s.run_phase(l, "hals", 5.0, 1.0, 1.0, 0)
        ph = s.phase_times()
        s.set_profiling(False)
        print(f"level {l} phases (ms): " + ", ".join(f"{k} {v:.3f}" for k, v in ph.items()), flush=True)
