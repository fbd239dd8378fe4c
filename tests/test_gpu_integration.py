"""Drop-in evidence: the reference's OWN acceptance suite
(/root/reference/proj/tests/acceptance.cpp, unmodified: 11 criteria incl.
exact-solver agreement, HCM convergence, published sweep counts, FHCM/FMSM
error ratios, upper bounds) linked against integration/eikonal_b200_dropin.cpp
-- the reference's solver signatures implemented over the C-ABI -- so every
fmm/fsm/hcm/fhcm/fmsm call of the suite runs on the B200.  The binary is
built here by oracle/Makefile (target `dropin`) and travels to the GPU box."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")


@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/acceptance_b200 not built")
def test_reference_acceptance_suite_on_b200():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
    assert r.stdout.count("[PASS]") == 11
