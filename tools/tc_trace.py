"""Summarise an MLB_TC_TRACE=1 event trace of the tcgen05 product kernel (CTA 0).

events per chunk g: 0 M TMA issued, 1 converter saw mfull, 2 converter got its
staging slot (sdone of g-4), 3 converter arrived ready, 4 MMA saw ready,
5 MMA issued + committed, 6 factor-slice TMA issued.
"""
import sys
import numpy as np

t = np.fromfile(sys.argv[1], dtype=np.int64).reshape(8, -1)
n = int((t[5] > 0).sum())
lo, hi = 200, min(n, 3800)  # steady state
g = np.arange(lo, hi)
T = t[:, lo:hi].astype(np.float64)
per_chunk = np.diff(t[5, lo:hi]).mean()
print(f"chunks traced {n}; steady-state cycles/chunk (MMA issue cadence): {per_chunk:.0f}")
def stat(name, d):
    print(f"  {name:42s} mean {d.mean():8.0f}  p50 {np.median(d):8.0f}  p90 {np.percentile(d, 90):8.0f}")
stat("M TMA issue -> converter sees data", T[1] - T[0])
stat("converter: data -> slot free (sdone)", T[2] - T[1])
stat("converter: slot free -> ready arrive", T[3] - T[2])
stat("ready arrive -> MMA sees ready", T[4] - T[3])
stat("MMA: ready -> issued+committed", T[5] - T[4])
stat("B TMA issue -> MMA sees ready", T[4] - T[6])
# completion latency proxy: MMA commit of chunk g -> converter of chunk g+4 gets slot
c = t[2, lo + 4:hi + 4].astype(np.float64) - t[5, lo:hi]
stat("MMA commit(g) -> slot(g+4) granted", c[:len(g)])
stat("converter(g+4) waiting for slot", (t[2, lo + 4:hi + 4] - t[1, lo + 4:hi + 4]).astype(np.float64))
stat("MMA issue gap between consecutive chunks", np.diff(t[5, lo:hi]).astype(np.float64))
