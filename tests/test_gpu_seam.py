"""The compiled drop-in seam: integration/control_gpu.cpp is compiled
against the REAL pdeopt headers (with the Eigen-API shim for Eigen) and linked with the
reference's own objects and libfetigpu.so (integration/Makefile).  integration/seam_check
runs the reference's solve_range_space (CPU FETI-DP) and solve_range_space_gpu on the same
pdeopt::ControlProblem / FactorSolverConfig and requires y, u, lambda to 1e-8 and the
iteration counts to +-2 (north_star), plus ContractError for phi <= 0 from both."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "integration", "_build", "seam_check")


@pytest.mark.parametrize("n,s,phi,target,augment", [
    (64, 4, 1e-4, "sine", 0),       # BASELINE config 1
    (32, 4, 1e-4, "thermal", 1),    # the reference's own problem (y_c != 0), augment = true (its default)
    (128, 4, 1e-6, "sine", 0),      # config 2's subdomain shape, config 3's phi
])
def test_seam_matches_reference(fetigpu, n, s, phi, target, augment):
    if not os.path.exists(BIN):
        pytest.skip("integration/_build/seam_check not built (needs the reference headers at build time)")
    out = subprocess.run([BIN, str(n), str(s), repr(phi), target, str(augment)], capture_output=True, text=True,
                         timeout=600)
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert out.returncode == 0 and line["ok"], (line, out.stderr[-2000:])
