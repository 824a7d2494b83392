"""Step time of one solver kind on one BASELINE small config (0-3), CUDA-event
timed over repeated batches of graph-replayed (or, with MLNMF_NO_GRAPHS=1,
eager) steps: python tools/small_steps.py CFG KIND [STEPS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1009_0881_b200 as P  # noqa: E402

cfg, kind = int(sys.argv[1]), sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 200
c = P.GEN_CONFIGS[cfg]
with P.Session(dtype=P.F32) as s:
    s.generate(cfg, seed=0)
    s.run_configuration(1, kind, "none", c["r"], 0, 3.0, 0)
    ext = torch.cuda.ExternalStream(s.stream)
    s.steps(kind, 5)
    s.sync()
    out = []
    for rep in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(ext)
        s.steps(kind, n)
        b.record(ext)
        b.synchronize()
        out.append(a.elapsed_time(b) / n)
    mode = "eager" if os.environ.get("MLNMF_NO_GRAPHS") else "graph"
    print(f"config {cfg} {kind} {mode}: " + " ".join(f"{x * 1e3:.1f}" for x in out) + " us/step")
