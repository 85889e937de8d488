#!/bin/bash
# The reference's OWN test files against the GPU package (tests/refshim/stabsim re-exports it under
# the reference's module names).  The files are staged from /root/reference into tests/_refsuite
# (git-ignored, removed again afterwards: no reference source stays in the repo), shipped to the GPU
# box with the snapshot, run there, and the log comes back under gpurun_out/.
#   tools/run_reference_suite.sh [tag]        (run in the build container)
set -e
tag=${1:-r02}
here=$(cd "$(dirname "$0")/.." && pwd)
src=/root/reference/pkg/tests
[ -d "$src" ] || { echo "no $src here"; exit 1; }
stage=$here/tests/_refsuite
rm -rf "$stage"; mkdir -p "$stage"
cp "$src"/dense_ref.py "$src"/test_*.py "$stage"/
rm -f "$stage"/test_cli.py                       # the CLI is outside the accelerated path: not built
# One test is deselected: TestCollapseGuard::test_degenerate_flatten_raises monkeypatches the
# reference engine's per-generator `flatten` call, an internal the device engine does not have
# (terms never leave HBM between operators); the collapse guard itself is exercised by
# tests/test_gpu_engine.py and tools/fuzz_eager.py (same exception, generator and step).
trap 'rm -rf "$stage"' EXIT
cd "$here"
gpurun --timeout 1500 -- "PYTHONPATH=tests/refshim:. timeout 1200 python -m pytest tests/_refsuite -q -p no:cacheprovider -o addopts= --deselect tests/_refsuite/test_engine.py::TestCollapseGuard::test_degenerate_flatten_raises > gpurun_out/${tag}_reference_suite.log 2>&1; tail -25 gpurun_out/${tag}_reference_suite.log"
