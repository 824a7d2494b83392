"""GPU: the reference's own acceptance binary through the drop-in boundary.

oracle/_ref/acceptance_b200 is proj/tests/acceptance.cpp compiled UNCHANGED
with the reference's non-solver sources, with solvers.cpp + multilevel.cpp
replaced by integration/mlnmf_b200_shim.cpp over libmlnmf_b200.so
(`make -C oracle dropin`, run by __graft_entry__.build() where the reference
sources exist).  Every solver call the acceptance criteria make -- mu/hals/
anls steps, nnls_active_set, nested_iteration / v_cycle / full_multigrid,
run_configuration -- runs on the B200 (fp64, exact mode), and the binary must
pass all its criteria and print the reference's end-to-end means
(acceptance.cpp:359-386) to the printed precision.
"""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(REPO, "oracle", "_ref", "acceptance_b200")
MEANS = "mu: single 9.691148  fmg 8.924942 | hals: single 8.251099  fmg 8.091289"


def test_reference_acceptance_through_b200(gpu, tmp_path):
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/acceptance_b200 not built (needs the reference sources at build time)")
    p = subprocess.run([BIN], cwd=tmp_path, capture_output=True, text=True, timeout=1200)
    out = p.stdout + p.stderr
    assert p.returncode == 0, out[-4000:]
    assert "all criteria passed" in out, out[-4000:]
    assert MEANS in out, out[-4000:]
    assert "[FAIL]" not in out


def test_reference_cycle_runner_over_resident_phases(gpu, tmp_path):
    """The reference's own multilevel.cpp (CycleRunner, multilevel.cpp:14-89)
    compiled unchanged, calling the shim's run_solver_phase: every phase runs
    device-resident through mlnmf_session_run_phase (one upload of the
    level's M per phase, not per step).  Same criteria and means."""
    binp = os.path.join(REPO, "oracle", "_ref", "acceptance_b200_phases")
    if not os.path.exists(binp):
        pytest.skip("oracle/_ref/acceptance_b200_phases not built (needs the reference sources at build time)")
    p = subprocess.run([binp], cwd=tmp_path, capture_output=True, text=True, timeout=1200)
    out = p.stdout + p.stderr
    assert p.returncode == 0, out[-4000:]
    assert "all criteria passed" in out, out[-4000:]
    assert MEANS in out, out[-4000:]
    assert "[FAIL]" not in out
