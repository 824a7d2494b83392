"""Generate tests/golden/cli_golden.json: sha256 digests of the reference's
synthetic PGM sets (`mlnmf synth`, proj/src/io.cpp:311-366), written by the
UNMODIFIED reference library through oracle/_ref/mlnmf_ref_cli
(make -C oracle refcli).  Run here, where /root/reference exists:

    python tests/golden/make_cli_golden.py
"""
import json
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from test_cli_cpu import REF, SYNTH_CASES, tree_digest  # noqa: E402

out = {"generator": "oracle/_ref/mlnmf_ref_cli synth (reference io.cpp)", "synth": {}}
for c in SYNTH_CASES:
    with tempfile.TemporaryDirectory() as t:
        args = [x for k, v in c.items() for x in (f"--{k}", str(v))]
        subprocess.run([REF, "synth", "--out", os.path.join(t, "s")] + args, check=True, capture_output=True)
        out["synth"]["{height}x{width}_n{n}_b{blobs}_s{seed}".format(**c)] = tree_digest(os.path.join(t, "s"))
with open(os.path.join(HERE, "cli_golden.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out, indent=1))
