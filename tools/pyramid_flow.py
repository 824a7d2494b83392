import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1009_0881_b200 as P
for rep in range(2):
    with P.Session(dtype=P.F32) as s:
        s.generate(4, seed=0)
        norm = float(np.sqrt(s.norm2(0)))
        if rep == 0:
            r = s.run_configuration(1, "hals", "none", 64, 0, 4.0, 2)
        s.sync()
        t0 = time.perf_counter(); s.build_levels(2); s.sync(); t1 = time.perf_counter()
        s.build_levels(5); s.sync(); t2 = time.perf_counter()
        print(f"rep {rep}: level1 {1e3*(t1-t0):.1f} ms, levels 2-4 {1e3*(t2-t1):.1f} ms")
