"""Config-4 HALS step time: CUDA-graph replay vs eager launches (set
MLNMF_NO_GRAPHS=1 for eager), whole steps timed with events on the engine
stream, next to the per-phase event breakdown of profiled (eager) steps."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1009_0881_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
with P.Session(dtype=P.F32) as s:
    s.generate(4, seed=0, n_total=n)
    s.run_configuration(1, "hals", "none", 64, 0, 0.0, 0)
    ext = torch.cuda.ExternalStream(s.stream)
    s.steps("hals", 3)
    s.sync()
    for rep in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(ext)
        s.steps("hals", 10)
        b.record(ext)
        b.synchronize()
        print(f"{'eager' if os.environ.get('MLNMF_NO_GRAPHS') else 'graph'} steps: {a.elapsed_time(b) / 10:.3f} ms/step")
    s.set_profiling(True)
    s.steps("hals", 5)
    ph = s.phase_times()
    s.set_profiling(False)
    print("profiled phases (ms):", {k: round(v, 3) for k, v in ph.items()}, "sum", round(sum(ph.values()), 3))
