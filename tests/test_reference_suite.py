"""The reference's own test files, unmodified, against the GPU package.

tests/refshim/stabsim re-exports ``paper_2505_03307_b200`` under the reference's module names (plus
a state-vector checker for the tests that need one), so ``from stabsim.stabilizer import flatten``
in the reference's test_stabilizer.py reaches the CUDA path.  Needs BOTH a GPU and the reference's
test files: /root/reference/pkg/tests (the build container, which has no GPU) or a staged copy under
tests/_refsuite (tools/run_reference_suite.sh stages it for one gpurun call and removes it again;
the log of that run is kept under profiles/).  Skipped where either is missing.  test_cli.py is not
run: the CLI is outside the accelerated path."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
CANDIDATES = ("/root/reference/pkg/tests", os.path.join(HERE, "_refsuite"))
FILES = ("test_stabilizer.py", "test_engine.py", "test_measure.py", "test_acceptance.py", "test_lut.py",
         "test_circuit.py", "test_pauli.py", "test_oracle.py")


def test_reference_tests_pass_on_the_gpu_package():
    src = next((d for d in CANDIDATES if os.path.exists(os.path.join(d, "test_stabilizer.py"))), None)
    if src is None:
        pytest.skip("the reference's test files are not on this machine")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(HERE, "refshim"), os.path.dirname(HERE), env.get("PYTHONPATH", "")])
    files = [os.path.join(src, f) for f in FILES if os.path.exists(os.path.join(src, f))]
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-o", "addopts=",
                          "--rootdir", src,
                          # monkeypatches an internal of the reference engine (its per-generator flatten call)
                          "--deselect", "test_engine.py::TestCollapseGuard::test_degenerate_flatten_raises", *files], env=env, capture_output=True, text=True, cwd=src)
    tail = "\n".join(out.stdout.splitlines()[-30:])
    assert out.returncode == 0, tail
