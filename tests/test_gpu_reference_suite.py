"""The REFERENCE's own test suite (138 tests of /root/reference/pkg/tests,
vendored verbatim in tests/ref_suite/) run against this package through a
`schurpd` module alias (tools/reference_suite.py).

Deselected, with the reason:
  * test_harness.py::test_cli_* (3): the reference CLI is out of scope;
  * test_solver.py::test_inner_loop_keeps_x1_bitwise_frozen,
    ::test_early_exit_skips_remaining_outer_passes: they spy on the Python
    function collision.detect being called per pass; detection runs inside the
    device frame here. Their invariants (x1 frozen across inner passes, the
    early exit) are checked on the device instead:
    tests/test_gpu_parity.py::test_inner_keeps_x1_frozen_and_rhs_maintenance
    and tests/test_gpu_early_exit.py (outer passes counted by the device,
    states bitwise equal to the shortened frame).
Everything else must pass (133 tests, incl. acceptance criteria 1-9)."""

import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
SUITE = ROOT / "tests" / "ref_suite"

DESELECT = [
    "test_harness.py::test_cli_run_and_errors",
    "test_harness.py::test_cli_compare",
    "test_harness.py::test_cli_solver_and_iteration_overrides",
    "test_solver.py::test_inner_loop_keeps_x1_bitwise_frozen",
    "test_solver.py::test_early_exit_skips_remaining_outer_passes",
]


def test_reference_suite_passes():
    assert (SUITE / "test_solver.py").exists(), "tests/ref_suite (vendored reference suite) is missing"
    args = [sys.executable, str(ROOT / "tools" / "reference_suite.py"), "-q", "-p", "no:randomly"]
    for d in DESELECT:
        args += ["--deselect", d]
    r = subprocess.run(args, capture_output=True, text=True, timeout=1500)
    tail = "\n".join(r.stdout.splitlines()[-15:])
    assert r.returncode == 0, tail
    assert " passed" in tail and "failed" not in tail, tail
