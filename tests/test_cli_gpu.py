"""GPU tests of the `mlnmf_b200` CLI: every file and stdout line of
factorize / bench / transfer-check against the reference library's own
writers run on the same inputs (oracle/_ref/mlnmf_ref_cli, oracle/ref_cli.cpp,
prebuilt -- /root/reference is not read at run time).

Default precision (fp64, the reference's operation order): V.csv, W.csv, the
basis PGMs, the bench summaries and the stdout lines are byte-identical; the
trace CSV is identical except its elapsed_s column (wall time).
transfer-check's s_M is a device reduction (1e-12 relative, test_gpu_diagnostics)
and is compared numerically.
"""
import csv
import os
import re

import pytest

from test_cli_cpu import CLI, REF, run

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not (os.path.exists(CLI) and os.path.exists(REF)),
                                                  reason="CLI or reference driver not built")]


@pytest.fixture(scope="module")
def data(tmp_path_factory):
    root = tmp_path_factory.mktemp("cli")
    rc, _, err = run(CLI, "synth", "--out", root / "imgs", "--height", "24", "--width", "20", "--n", "36",
                     "--blobs", "3", "--seed", "4")
    assert rc == 0, err
    # a CSV dataset (no grid): 40 x 30 smooth nonnegative matrix
    with open(root / "m.csv", "w") as f:
        for i in range(40):
            f.write(",".join(f"{((i * 7 + j * 3) % 11) / 10 + 0.05 * ((i + j) % 3):.6g}" for j in range(30)) + "\n")
    return root


def both(tmp, sub, *args):
    """Run the subcommand through both CLIs, each writing under its own prefix."""
    res = {}
    for name, exe in (("b200", CLI), ("ref", REF)):
        rc, out, err = run(exe, sub, *args, "--out", tmp / name) if sub != "transfer-check" else run(exe, sub, *args)
        assert rc == 0, (name, err)
        res[name] = out
    return res


def read(p):
    with open(p, "rb") as f:
        return f.read()


def trace_rows(p):
    with open(p) as f:
        rows = list(csv.reader(f))
    return rows[0], [r[1:] for r in rows[1:]]  # drop elapsed_s


@pytest.mark.parametrize("args", [
    ["--algo", "hals", "--cycle", "fmg", "--levels", "3", "--rank", "5", "--budget", "work:12"],
    ["--algo", "mu", "--cycle", "vc", "--levels", "2", "--rank", "4", "--budget", "work:8", "--trace-every", "3"],
    ["--algo", "anls", "--cycle", "ni", "--levels", "3", "--rank", "3", "--budget", "work:5", "--seed", "9"],
    ["--algo", "hals", "--rank", "6", "--budget", "work:10", "--trace-every", "0"],
], ids=["hals-fmg", "mu-vc", "anls-ni", "hals-none"])
def test_factorize_pgm_identical(tmp_path, data, args):
    out = both(tmp_path, "factorize", "--data", data / "imgs", *args)
    assert out["b200"].replace(str(tmp_path / "b200"), "P") == out["ref"].replace(str(tmp_path / "ref"), "P")
    for suf in (".V.csv", ".W.csv"):
        assert read(f"{tmp_path / 'b200'}{suf}") == read(f"{tmp_path / 'ref'}{suf}"), suf
    assert trace_rows(f"{tmp_path / 'b200'}.trace.csv") == trace_rows(f"{tmp_path / 'ref'}.trace.csv")
    bd, rd = f"{tmp_path / 'b200'}.basis", f"{tmp_path / 'ref'}.basis"
    assert sorted(os.listdir(bd)) == sorted(os.listdir(rd))
    for name in os.listdir(rd):
        assert read(os.path.join(bd, name)) == read(os.path.join(rd, name)), name


def test_factorize_csv_identical(tmp_path, data):
    args = ["--data", data / "m.csv", "--format", "csv", "--algo", "mu", "--rank", "4", "--budget", "work:15"]
    out = both(tmp_path, "factorize", *args)
    assert out["b200"].replace("b200", "X") == out["ref"].replace("ref", "X")
    for suf in (".V.csv", ".W.csv"):
        assert read(f"{tmp_path / 'b200'}{suf}") == read(f"{tmp_path / 'ref'}{suf}")
    assert not os.path.exists(f"{tmp_path / 'b200'}.basis")  # no grid, no basis images
    # a grid given on the command line makes it multilevel-capable
    args2 = ["--data", data / "m.csv", "--format", "csv", "--grid-height", "8", "--grid-width", "5", "--algo", "hals",
             "--cycle", "fmg", "--levels", "2", "--rank", "3", "--budget", "work:6"]
    os.makedirs(tmp_path / "g")
    both(tmp_path / "g", "factorize", *args2)
    for suf in (".V.csv", ".W.csv"):
        assert read(f"{tmp_path / 'g' / 'b200'}{suf}") == read(f"{tmp_path / 'g' / 'ref'}{suf}")


def test_factorize_errors(tmp_path, data):
    # rank > min(m, n): random_init's invalid_argument -> exit 2 in both
    for exe in (CLI, REF):
        rc, _, err = run(exe, "factorize", "--data", data / "imgs", "--rank", "37", "--budget", "work:1",
                         "--out", tmp_path / "o")
        assert rc == 2 and "random_init: rank must satisfy" in err, err
    # multilevel cycle on grid-less data: usage error
    rc, _, _ = run(CLI, "factorize", "--data", data / "m.csv", "--format", "csv", "--cycle", "fmg", "--levels", "2",
                   "--rank", "2", "--budget", "work:1", "--out", tmp_path / "o")
    assert rc == 2


def test_bench_identical(tmp_path, data):
    args = ["--data", data / "imgs", "--algos", "mu,hals", "--cycles", "none,fmg", "--levels", "1,3",
            "--rank", "4", "--runs", "3", "--budget", "work:6", "--seed", "2"]
    out = both(tmp_path, "bench", *args)
    assert out["b200"] == out["ref"]
    for suf in (".summary.csv", ".summary.txt"):
        assert read(f"{tmp_path / 'b200'}{suf}") == read(f"{tmp_path / 'ref'}{suf}"), suf
    # skipped rows (single level with levels != 1; a too-deep pyramid -> the
    # invalid_argument text as the note)
    args = ["--data", data / "imgs", "--algos", "hals", "--cycles", "none,ni", "--levels", "2,7",
            "--rank", "3", "--runs", "2", "--budget", "work:3"]
    os.makedirs(tmp_path / "s")
    out = both(tmp_path / "s", "bench", *args)
    assert out["b200"] == out["ref"]
    assert read(f"{tmp_path / 's' / 'b200'}.summary.csv") == read(f"{tmp_path / 's' / 'ref'}.summary.csv")


def test_bench_fp32_close(tmp_path, data):
    """--precision fp32 (fp32 storage on the device): same table layout, errors
    within 1e-4 of the fp64 reference."""
    args = ["--data", data / "imgs", "--algos", "hals", "--cycles", "fmg", "--levels", "3",
            "--rank", "4", "--runs", "2", "--budget", "work:6"]
    rc, out32, err = run(CLI, "bench", *args, "--precision", "fp32", "--out", tmp_path / "f32")
    assert rc == 0, err
    rc, outr, _ = run(REF, "bench", *args, "--out", tmp_path / "ref")
    with open(f"{tmp_path / 'f32'}.summary.csv") as f:
        a = list(csv.DictReader(f))
    with open(f"{tmp_path / 'ref'}.summary.csv") as f:
        b = list(csv.DictReader(f))
    for x, y in zip(a, b):
        assert abs(float(x["mean_error"]) - float(y["mean_error"])) <= 1e-4 * float(y["mean_error"])


def test_transfer_check(tmp_path, data):
    out = both(tmp_path, "transfer-check", "--data", data / "imgs", "--levels", "4")
    num = re.compile(r"s_M = ([0-9.eE+-]+)")
    a, b = out["b200"].splitlines(), out["ref"].splitlines()
    assert len(a) == len(b) == 3
    for x, y in zip(a, b):
        assert num.sub("", x) == num.sub("", y)
        sa, sb = float(num.search(x).group(1)), float(num.search(y).group(1))
        assert abs(sa - sb) <= 1e-5 * sb  # %.6g printing
