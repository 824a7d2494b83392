"""CPU tests of the dataset / result I/O on the C-ABI and its Python mirror
(load_pgm_dir, load_csv, save_matrix_csv, save_trace_csv, save_basis_mosaic,
synth_smooth_dataset; proj/include/mlnmf/io.hpp): host-only code in the
library, the same bytes as the CLI (tests/test_cli_cpu.py) and the reference.
"""
import json
import os

import numpy as np
import pytest

from test_cli_cpu import CLI, GOLDEN, run, tree_digest


def test_synth_and_pgm_round_trip(P, tmp_path):
    d = P.synth_smooth_dataset(20, 17, 5, 3, 0)
    assert d.matrix.shape == (340, 5) and d.grid.height == 20 and d.grid.width == 17
    assert d.matrix.min() >= 0.0 and d.matrix.max() <= 1.0
    # the reference writes this dataset as PGMs whose digest is committed
    with open(GOLDEN) as f:
        golden = json.load(f)["synth"]["20x17_n5_b3_s0"]
    out = tmp_path / "imgs"
    out.mkdir()
    assert run(CLI, "synth", "--out", out / "s", "--height", 20, "--width", 17, "--n", 5, "--seed", 0)[0] == 0
    assert tree_digest(out / "s") == golden
    # loading the PGMs back gives the 8-bit quantised matrix
    L = P.load_pgm_dir(out / "s")
    assert L.matrix.shape == (340, 5) and (L.grid.height, L.grid.width) == (20, 17) and L.name == "s"
    assert np.max(np.abs(L.matrix - np.round(d.matrix * 255) / 255)) < 1e-12


def test_csv_round_trip_and_errors(P, tmp_path):
    M = np.random.default_rng(0).random((7, 5))
    p = tmp_path / "m.csv"
    P.save_matrix_csv(M, p)
    text = p.read_text().splitlines()
    assert text[0] == ",".join("%.17g" % v for v in M[0])
    D = P.load_csv(p)
    assert D.grid is None and D.name == "m" and np.array_equal(D.matrix, M)
    bad = tmp_path / "bad.csv"
    bad.write_text("1,2\n3\n")
    with pytest.raises(P.DataError, match="ragged row 2"):
        P.load_csv(bad)
    with pytest.raises(P.DataError, match="is not a directory"):
        P.load_pgm_dir(tmp_path / "nope")


def test_trace_and_basis_writers(P, tmp_path):
    tr = P.plan_configuration(P.ImageGrid(8, 8), 10, 2, "hals", "fmg", 3, 4.0, 1)
    P.save_trace_csv(tr, tmp_path / "t.csv")
    lines = (tmp_path / "t.csv").read_text().splitlines()
    assert lines[0] == "elapsed_s,work_units,level,error" and len(lines) == len(tr.error) + 1
    V = np.random.default_rng(1).random((64, 3))
    V[:, 2] = 0.0
    P.save_basis_mosaic(V, P.ImageGrid(8, 8), tmp_path / "b")
    names = sorted(os.listdir(tmp_path / "b"))
    assert names == ["basis_000.pgm", "basis_001.pgm", "basis_002.pgm", "mosaic.pgm"]
    assert (tmp_path / "b" / "basis_002.pgm").read_bytes().endswith(bytes(64))  # zero column stays black
