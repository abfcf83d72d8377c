"""The reference's own release gate (proj/tests/acceptance.cpp, criteria
1..11) linked against the C++ drop-in shim instead of the reference's
estimators.cpp / compensation.cpp: every estimation, refinement and
prediction call runs on the GPU.  The binary is built in the build container
(paper_1002_1168_b200/shim/Makefile) and travels with the repository."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_1002_1168_b200", "shim", "build", "acceptance_b200")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN), reason="drop-in acceptance binary not built")
@pytest.mark.parametrize("criterion", range(1, 12))
def test_reference_acceptance_on_gpu(me_gpu, criterion):
    r = subprocess.run([BIN, str(criterion)], capture_output=True, text=True, timeout=300)
    line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else ""
    assert line.startswith("PASS"), f"{line}\n{r.stderr}"
