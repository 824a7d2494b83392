"""Profiling driver: the two M-streaming products at config-4 shape on a
column slice (m = 65536, r = 64, n = --n), through the active path.

    python tools/profile_products.py --n 32768 --reps 3 [--gemm tc|simt]

Prints per-product device times (CUDA events) and achieved HBM GB/s.
Intended to be wrapped by ncu (-k regex:k_ix_product).
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--gemm", default="tc", choices=["tc", "simt", "auto"])
    ap.add_argument("--steps", type=int, default=0, help="also time full HALS steps")
    ap.add_argument("--r", type=int, default=64, help="rank (the factor digit planes scale with it)")
    ap.add_argument("--residual", type=int, default=0, help="also time this many error samples (||M - VW||_F)")
    a = ap.parse_args()
    import paper_1009_0881_b200 as P
    gemm = {"tc": P.GEMM_TCGEN05, "simt": P.GEMM_SIMT, "auto": P.GEMM_AUTO}[a.gemm]
    with P.Session(dtype=P.F32, gemm_path=gemm) as s:
        s.generate(4, seed=0, n_total=a.n)
        s.run_configuration(1, "hals", "none", a.r, 0, 0.0, 0)  # random_init
        s.products()  # warm-up (buffer allocation)
        s.set_profiling(True)
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from bench import ClockSampler
        with ClockSampler(0) as clk:
            for _ in range(a.reps):
                s.products()
            s.sync()
        kt = s.kernel_times()
        print("clocks during the products:", clk.summary())
        mb = 65536 * a.n * 4
        mw, vt = kt["mwt_ms"] / kt["mwt_n"], kt["vtm_ms"] / kt["vtm_n"]
        print(f"n={a.n} tc={s.tc_active} A=MW^T {mw:.3f} ms ({mb / mw / 1e6:.0f} GB/s)  "
              f"C=V^TM {vt:.3f} ms ({mb / vt / 1e6:.0f} GB/s)")
        if a.residual:
            import time
            e0 = s.error()  # warm-up (split buffers, tensor maps)
            s.sync()
            t = time.perf_counter()
            for _ in range(a.residual):
                e = s.error()
            dt = (time.perf_counter() - t) / a.residual
            print(f"residual {dt * 1e3:.3f} ms ({mb / dt / 1e9:.0f} GB/s)  error {e:.10g} (first {e0:.10g})")
        if a.steps:
            s.set_profiling(False)
            import time
            s.sync()
            t = time.perf_counter()
            s.steps("hals", a.steps)
            s.sync()
            print(f"hals step {1e3 * (time.perf_counter() - t) / a.steps:.3f} ms")


if __name__ == "__main__":
    main()
