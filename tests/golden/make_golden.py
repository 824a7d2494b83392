"""Regenerate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref,
built by `make -C oracle ref` from /root/reference/proj/src).

    python tests/golden/make_golden.py

The fixtures pin the C restatement (oracle/mlnmf_oracle.c) offline -- on the
GPU box and in the driver's CPU test run, /root/reference does not exist --
and are small: seeded inputs plus the reference's outputs on them.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import ctypes as C  # noqa: E402

import oracle  # noqa: E402


def main():
    ref = oracle.Reference()
    rng = np.random.default_rng(20261019)
    out = {}

    # --- SplitMix64 / random_init (matrix.hpp:76-95, matrix.cpp:51-60)
    out["splitmix_seeds"] = np.array([0, 1, 42, 12345, 2**63 + 7], np.uint64)
    out["splitmix_first"] = np.array([ref.splitmix_first(int(s)) for s in out["splitmix_seeds"]], np.uint64)
    V, W = ref.random_init(5, 4, 3, 9)
    out["ri_V"], out["ri_W"] = V, W

    # --- transfer operators (transfer.cpp:61-118)
    for (h, w) in [(3, 3), (8, 7), (5, 5), (4, 6), (2, 2)]:
        out[f"R_{h}x{w}"] = ref.operator_dense(h, w, 0)
        out[f"P_{h}x{w}"] = ref.operator_dense(h, w, 1)
    X = rng.random((19 * 17, 3))
    out["apply_X"] = X
    out["apply_R"] = ref.apply_operator(19, 17, 0, X)
    Xc = rng.random((10 * 9, 2))
    out["apply_Xc"] = Xc
    out["apply_P"] = ref.apply_operator(19, 17, 1, Xc)

    # --- single steps (solvers.cpp:79-298)
    for i, (m, n, r) in enumerate([(10, 8, 3), (30, 20, 5), (64, 50, 8)]):
        M = rng.random((m, n))
        V0, W0 = ref.random_init(m, n, r, 100 + i)
        out[f"step{i}_M"], out[f"step{i}_V0"], out[f"step{i}_W0"] = M, V0, W0
        out[f"step{i}_hals_V"], out[f"step{i}_hals_W"], deg = ref.hals_step(M, V0, W0)
        out[f"step{i}_hals_deg"] = np.array(deg)
        out[f"step{i}_mu_V"], out[f"step{i}_mu_W"] = ref.mu_step(M, V0, W0)
        out[f"step{i}_anls_V"], out[f"step{i}_anls_W"], out[f"step{i}_anls_counts"] = ref.anls_step(M, V0, W0)
        out[f"step{i}_err"] = np.array(ref.frobenius_error(M, V0, W0))

    # --- NNLS (solvers.cpp:143-243)
    Gs, hs, x0s, xs, its = [], [], [], [], []
    for t in range(60):
        r = [1, 2, 3, 5, 8][t % 5]
        A = rng.random((r, r + 2))
        G = A @ A.T + 0.1 * np.eye(r)
        h = 2.0 * rng.random(r) - 1.0
        x0 = np.where(rng.random(r) < 0.5, rng.random(r), 0.0)
        x, it = ref.nnls_active_set(G, h, x0)
        pad = lambda a, s: np.pad(a, [(0, 8 - d) for d in a.shape]) if s else a
        Gs.append(np.pad(G, ((0, 8 - r), (0, 8 - r))))
        hs.append(np.pad(h, (0, 8 - r)))
        x0s.append(np.pad(x0, (0, 8 - r)))
        xs.append(np.pad(x, (0, 8 - r)))
        its.append([r, it])
    out["nnls_G"], out["nnls_h"], out["nnls_x0"] = np.array(Gs), np.array(hs), np.array(x0s)
    out["nnls_x"], out["nnls_rit"] = np.array(xs), np.array(its)

    # --- whole runs on a 17x17 grid (multilevel.cpp:116-132)
    M = rng.random((17 * 17, 30))
    out["run_M"] = M
    for kind in ("mu", "hals", "anls"):
        for cyc in ("none", "ni", "vc", "fmg"):
            amount = 8.0 if kind == "anls" else 24.0
            V, W, tr = ref.run_configuration(M, 17, 17, 3, kind, cyc, 4, 5, amount, 1)
            k = f"run_{kind}_{cyc}"
            out[k + "_V"], out[k + "_W"] = V, W
            out[k + "_err"], out[k + "_work"], out[k + "_level"] = tr.error, tr.work, tr.level
            out[k + "_alloc"] = np.stack([tr.alloc_level.astype(np.float64), tr.alloc_amount])
            out[k + "_counts"], out[k + "_deg"] = tr.counts, np.array(tr.degenerate)

    # --- config 0 (BASELINE.json), HALS work:100: error trajectories
    M0 = oracle.generate_config(0)
    for cyc in ("none", "fmg"):
        V, W, tr = ref.run_configuration(M0, 32, 32, 3, "hals", cyc, 20, 0, 100.0, 1)
        out[f"cfg0_{cyc}_err"], out[f"cfg0_{cyc}_work"] = tr.error, tr.work
        out[f"cfg0_{cyc}_VWnorm"] = np.array([np.linalg.norm(V), np.linalg.norm(W), V.sum(), W.sum()])

    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)

    # --- acceptance criterion 8 dataset (acceptance.cpp:359-386):
    # synth_smooth_dataset(65, 65, 40, 3, 7), r = 8, work:300, seeds 100..119
    Md = np.zeros(65 * 65 * 40)
    rc = ref.lib.ref_synth_smooth_dataset(C.c_size_t(65), C.c_size_t(65), C.c_size_t(40), C.c_size_t(3),
                                          C.c_uint64(7), Md.ctypes.data_as(C.POINTER(C.c_double)))
    assert rc == 0
    Md = Md.reshape(65 * 65, 40)
    finals = {}
    for kind in ("mu", "hals"):
        for (lv, cyc) in ((1, "none"), (3, "fmg")):
            finals[f"{kind}_{cyc}"] = np.array([
                ref.run_configuration(Md, 65, 65, lv, kind, cyc, 8, 100 + s, 300.0, 0)[2].error[-1]
                for s in range(20)])
    np.savez_compressed(os.path.join(HERE, "acceptance8.npz"), M=Md, **finals)
    print({k: float(v.mean()) for k, v in finals.items()})


def diagnostics():
    """smoothness / initialization_bound (transfer.cpp:128-153) on the
    reference's own test shapes (test_transfer.cpp:155-220, acceptance.cpp:390-408)
    plus larger odd grids; -> tests/golden/diagnostics.npz."""
    ref = oracle.Reference()
    rng = np.random.default_rng(1009)
    out = {}
    cb = np.array([[(i + j) % 2 for j in range(3)] for i in range(3)], np.float64)
    cases = [("ones", 3, 3, np.ones((9, 4))), ("checker", 3, 3, cb.T.reshape(9, 1))]
    for (h, w, n) in [(8, 7, 5), (19, 17, 3), (64, 64, 16), (33, 65, 7), (2, 2, 1)]:
        cases.append((f"rand_{h}x{w}", h, w, rng.random((h * w, n))))
    for name, h, w, M in cases:
        out[f"s_{name}_M"] = M
        out[f"s_{name}_hw"] = np.array([h, w])
        out[f"s_{name}_s"] = np.array(ref.smoothness(M, h, w))
    # acceptance criterion 9 shape draws: h, w in [2, 13], n in [1, 6], r in [1, 3]
    for t in range(40):
        h, w = int(rng.integers(2, 14)), int(rng.integers(2, 14))
        n, r = int(rng.integers(1, 7)), int(rng.integers(1, 4))
        hc, wc = (h + 1) // 2, (w + 1) // 2
        M, Vc, W = rng.random((h * w, n)), rng.random((hc * wc, r)), rng.random((r, n))
        out[f"b{t}_M"], out[f"b{t}_Vc"], out[f"b{t}_W"], out[f"b{t}_hw"] = M, Vc, W, np.array([h, w])
        out[f"b{t}_lr"] = np.array(ref.initialization_bound(M, h, w, Vc, W))
    out["n_bound"] = np.array(40)
    np.savez_compressed(os.path.join(HERE, "diagnostics.npz"), **out)


if __name__ == "__main__":
    if "diagnostics" not in sys.argv[1:]:
        main()
    diagnostics()
