from paper_2505_03307_b200.measure import *  # noqa: F401,F403
from paper_2505_03307_b200.measure import (  # noqa: F401
    DEFAULT_TERM_BUDGET, DENSITY_MAX_QUBITS, PauliExpansion, density_expansion, expectation, prob_z,
)
