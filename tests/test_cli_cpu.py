"""CPU tests of the `mlnmf_b200` CLI (paper_1009_0881_b200/csrc/cli_main.cpp,
host_io.cpp) against the reference CLI's behaviour (proj/tools/mlnmf_main.cpp,
proj/src/io.cpp, proj/src/bench.cpp).

Everything here runs without a GPU: usage errors, dataset ingestion and its
error texts (data errors are raised before any device call), the synthetic
PGM writer, and `transfer-check --levels 1` (no pyramid, no device work).
The comparison target is `oracle/_ref/mlnmf_ref_cli` (the reference library's
own loaders and writers, oracle/ref_cli.cpp) when it is built, and the
committed digests in tests/golden/cli_golden.json (tests/golden/make_cli_golden.py)
always.
"""
import hashlib
import json
import os
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(REPO, "paper_1009_0881_b200", "_lib", "mlnmf_b200")
REF = os.path.join(REPO, "oracle", "_ref", "mlnmf_ref_cli")
GOLDEN = os.path.join(REPO, "tests", "golden", "cli_golden.json")

pytestmark = pytest.mark.skipif(not os.path.exists(CLI), reason="CLI not built (python __graft_entry__.py)")


def run(exe, *args, cwd=None):
    p = subprocess.run([exe, *map(str, args)], capture_output=True, text=True, cwd=cwd, timeout=120)
    return p.returncode, p.stdout, p.stderr


def have_ref():
    return os.path.exists(REF)


def tree_digest(d):
    h = hashlib.sha256()
    for name in sorted(os.listdir(d)):
        h.update(name.encode())
        with open(os.path.join(d, name), "rb") as f:
            h.update(f.read())
    return h.hexdigest()


def pgm(path, w, h, maxval=255, data=None, header=None):
    bpp = 1 if maxval == 255 else 2
    if data is None:
        data = bytes((i * 7) % 256 for i in range(w * h * bpp))
    hdr = header if header is not None else f"P5\n{w} {h}\n{maxval}\n".encode()
    with open(path, "wb") as f:
        f.write(hdr + data)


# --------------------------------------------------------------------------
# usage and exit codes (mlnmf_main.cpp:137-143, 221-233)
# --------------------------------------------------------------------------
def test_usage_exit_codes(tmp_path):
    assert run(CLI, "--help")[0] == 0
    assert run(CLI)[0] == 2                                        # subcommand required
    assert run(CLI, "frobnicate")[0] == 2
    assert run(CLI, "factorize", "--rank", "2")[0] == 2            # --data/--budget/--out required
    assert run(CLI, "factorize", "--data", tmp_path, "--rank", "x", "--budget", "work:1", "--out", "o")[0] == 2
    assert run(CLI, "synth", "--out", tmp_path / "s", "--bogus", "1")[0] == 2
    for spec in ["work", "work:abc", "work:0", "work:-1", "days:3"]:
        rc, _, err = run(CLI, "factorize", "--data", tmp_path / "nodir", "--rank", "2", "--budget", spec, "--out", "o",
                         "--format", "csv")
        # data is loaded first (a missing file is a data error), as in the reference
        assert rc == 3, (spec, err)
    d = tmp_path / "imgs"
    d.mkdir()
    pgm(d / "a.pgm", 4, 4)
    pgm(d / "b.pgm", 4, 4)
    for extra in (["--budget", "work"], ["--budget", "work:0"], ["--budget", "days:3"], ["--algo", "svd"],
                  ["--cycle", "w"], ["--format", "tiff"]):
        args = ["factorize", "--data", d, "--rank", "2", "--budget", "work:1", "--out", tmp_path / "o"] + extra
        assert run(CLI, *args)[0] == 2, extra


def test_equals_syntax_and_synth_defaults(tmp_path):
    rc, out, _ = run(CLI, "synth", f"--out={tmp_path / 's'}", "--n=3", "--height=9", "--width=7")
    assert rc == 0 and out == f"wrote 3 images (9x7) to {tmp_path / 's'}\n"
    assert sorted(os.listdir(tmp_path / "s")) == ["img_0000.pgm", "img_0001.pgm", "img_0002.pgm"]


# --------------------------------------------------------------------------
# synth (io.cpp:311-366): byte-identical PGM sets
# --------------------------------------------------------------------------
SYNTH_CASES = [dict(height=20, width=17, n=5, blobs=3, seed=0), dict(height=32, width=32, n=12, blobs=5, seed=7),
               dict(height=9, width=31, n=4, blobs=1, seed=123)]


@pytest.mark.parametrize("case", SYNTH_CASES, ids=lambda c: f"{c['height']}x{c['width']}s{c['seed']}")
def test_synth_matches_reference(tmp_path, case):
    args = [x for k, v in case.items() for x in (f"--{k}", v)]
    rc, out, _ = run(CLI, "synth", "--out", tmp_path / "b200", *args)
    assert rc == 0
    dig = tree_digest(tmp_path / "b200")
    with open(GOLDEN) as f:
        golden = json.load(f)["synth"]
    key = "{height}x{width}_n{n}_b{blobs}_s{seed}".format(**case)
    assert dig == golden[key]
    if have_ref():
        rc2, out2, _ = run(REF, "synth", "--out", tmp_path / "ref", *args)
        assert rc2 == 0 and tree_digest(tmp_path / "ref") == dig
        assert out.replace("b200", "ref") == out2


def test_synth_blobs_zero_is_invalid(tmp_path):
    rc, _, err = run(CLI, "synth", "--out", tmp_path / "s", "--blobs", "0")
    assert rc == 2 and "synth_smooth_dataset: blobs >= 1" in err


# --------------------------------------------------------------------------
# ingestion errors (io.cpp:65-187): exit 3 with the reference's message
# --------------------------------------------------------------------------
def _bad_pgm_dirs(root):
    """(name, directory) pairs, each holding one malformed PGM case."""
    cases = []

    def mk(name, **kw):
        d = root / name
        d.mkdir()
        pgm(d / "x.pgm", kw.pop("w", 4), kw.pop("h", 3), **kw)
        cases.append((name, d))

    mk("truncated", data=b"\x01\x02")
    mk("maxval", maxval=255, header=b"P5\n4 3\n1000\n")
    mk("zero", header=b"P5\n0 3\n255\n")
    mk("notint", header=b"P5\n4x 3\n255\n")
    mk("nows", header=b"P5\n4 3\n255#c\n")
    mk("eof", header=b"P5\n4 3", data=b"")
    mk("comment_eof", header=b"P5 # only a comment", data=b"")
    # mismatched sizes across files
    d = root / "mismatch"
    d.mkdir()
    pgm(d / "a.pgm", 4, 3)
    pgm(d / "b.pgm", 3, 4)
    cases.append(("mismatch", d))
    e = root / "empty"
    e.mkdir()
    (e / "readme.txt").write_text("P2 not binary")
    cases.append(("empty", e))
    cases.append(("missing", root / "does_not_exist"))
    return cases


def test_pgm_errors_match_reference(tmp_path):
    for name, d in _bad_pgm_dirs(tmp_path):
        rc, out, err = run(CLI, "transfer-check", "--data", d)
        assert rc == 3, (name, rc, err)
        assert err.startswith("data error: "), (name, err)
        if have_ref():
            rc2, _, err2 = run(REF, "transfer-check", "--data", d)
            assert (rc2, err2) == (rc, err), name


def _csv_cases(root):
    cases = {
        "ragged": "1,2,3\n4,5\n",
        "negative": "1,2\n3,-4\n",
        "text": "1,2\nfoo,3\n",
        "trailing_junk": "1,2x\n",
        "empty": "\n\n",
        "inf": "1,inf\n",
        "empty_cell": "1,,2\n",
        "underflow": "1,1e-320\n",
    }
    out = {}
    for k, v in cases.items():
        p = root / f"{k}.csv"
        p.write_text(v)
        out[k] = p
    return out


def test_csv_errors_match_reference(tmp_path):
    for name, p in _csv_cases(tmp_path).items():
        rc, _, err = run(CLI, "factorize", "--data", p, "--format", "csv", "--rank", "1", "--budget", "work:1",
                         "--out", tmp_path / "o")
        assert rc == 3, (name, err)
        if have_ref():
            rc2, _, err2 = run(REF, "factorize", "--data", p, "--format", "csv", "--rank", "1", "--budget", "work:1",
                               "--out", tmp_path / "o")
            assert (rc2, err2) == (rc, err), name


def test_loads_that_succeed(tmp_path):
    """Accepted inputs: comments in the header, 16-bit big-endian pixels, CRLF
    CSV with blank lines, '-0' -- transfer-check at one level stops right after
    loading (no device work)."""
    d = tmp_path / "ok"
    d.mkdir()
    pgm(d / "a.pgm", 5, 4, header=b"P5 # comment\n5 # w\n4\n255\n")
    pgm(d / "b.pgm", 5, 4, maxval=65535)
    (d / "c.txt").write_text("not an image")
    assert run(CLI, "transfer-check", "--data", d)[0] == 0
    c = tmp_path / "m.csv"
    c.write_bytes(b"1,2,3\r\n\r\n4,-0,6\r\n")
    assert run(CLI, "transfer-check", "--data", c, "--format", "csv", "--grid-height", "2", "--grid-width", "1")[0] == 0
    rc, _, err = run(CLI, "transfer-check", "--data", c, "--format", "csv")
    assert rc == 3 and "transfer-check needs a pixel grid" in err
    rc, _, err = run(CLI, "transfer-check", "--data", c, "--format", "csv", "--grid-height", "3", "--grid-width", "1")
    assert rc == 3 and "grid dimensions do not match matrix rows" in err
    rc, _, err = run(CLI, "transfer-check", "--data", d, "--levels", "4")
    assert rc == 2 and "GridHierarchy: too many levels for this grid" in err
