"""`stabsim` as the reference's own tests import it, answered by the B200 package.

TEST INFRASTRUCTURE.  Points the reference's unit / acceptance tests (written against the CPU
package under /root/reference/pkg/src/stabsim) at ``paper_2505_03307_b200`` unmodified: put this
directory's parent first on PYTHONPATH and run the reference's test files (tools/run_reference_suite.sh,
tests/test_reference_suite.py).  Every submodule re-exports the product's module of the same name;
``oracle`` (the dense state-vector checker) is not part of the accelerated path and is provided
here, for the tests only; ``cli`` does not exist (test_cli.py is not run).
"""

from paper_2505_03307_b200 import *  # noqa: F401,F403
from paper_2505_03307_b200 import __version__  # noqa: F401

from .oracle import compare, sv_expectation, sv_prob_z, sv_run  # noqa: F401
from .pauli import Axis  # noqa: F401
