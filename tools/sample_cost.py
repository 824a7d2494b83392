"""Per-step cost with and without an error sample every step (trace_every 1
vs 0) on BASELINE configs 0-3, fp32 storage, device data: the sampling
overhead the time-to-target runs pay."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1009_0881_b200 as P  # noqa: E402

for cfg, kind in ((0, "hals"), (1, "mu"), (2, "hals"), (3, "hals")):
    c = P.GEN_CONFIGS[cfg]
    with P.Session(dtype=P.F32) as s:
        s.generate(cfg, seed=0)
        s.run_configuration(1, kind, "none", c["r"], 0, 5.0, 1)
        out = []
        for te in (0, 1):
            s.sync()
            t = time.perf_counter()
            tr = s.run_configuration(1, kind, "none", c["r"], 0, 100.0, te)
            s.sync()
            out.append((time.perf_counter() - t) / 100)
    print(f"config {cfg} {kind}: {out[0] * 1e3:.4f} ms/step untraced, {out[1] * 1e3:.4f} ms/step traced "
          f"(sample {1e3 * (out[1] - out[0]):.4f} ms)", flush=True)
