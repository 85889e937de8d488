"""B200-native extended-stabilizer hot path behind the reference's ``stabsim`` API.

The names below are the reference's (``stabsim/__init__.py:16-53``) for the hot
path: gate list in, ``run(instructions, n, mode)`` with v1/v2/v3 selection,
``RunReport`` out, ``prob_z`` / ``expectation`` / ``density_expansion`` read-out.
Importing the package does not load the CUDA library; the first compute call does,
and raises ``NativeError`` if ``lib/libqimax_b200.so`` or a CUDA device is missing
(there is no CPU fallback).
"""

from .circuit import CircuitParseError, Instruction, divide_instruction, parse_circuit, serialize_circuit
from .engine import AgreementReport, Mode, RunReport, compare_reports, run, run_all_modes
from .errors import ConsistencyError, NativeError, NumericalCollapseError, ResourceLimitError
from .measure import PauliExpansion, density_expansion, expectation, expectation_heisenberg, prob_z
from .pauli import Axis
from .stabilizer import (
    DenseComplexGenerator,
    GeneratorSet,
    RaggedComplexGenerator,
    generator_set_to_dict,
    SimpleGenerator,
    apply_1q,
    apply_cx,
    canonicalize,
    flatten,
    init_z,
    rank_stats,
    sub,
)
from .workloads import gen_ghz, gen_graph, gen_random, gen_xyz_chain, near_clifford, ring_edges

__version__ = "0.1.0"

__all__ = [
    "AgreementReport", "Axis", "CircuitParseError", "DenseComplexGenerator", "RaggedComplexGenerator", "ConsistencyError", "GeneratorSet", "Instruction", "Mode", "NativeError",
    "NumericalCollapseError", "PauliExpansion", "ResourceLimitError", "RunReport", "SimpleGenerator",
    "apply_1q", "apply_cx", "canonicalize", "compare_reports", "density_expansion",
    "divide_instruction", "expectation", "expectation_heisenberg", "flatten", "gen_ghz", "gen_graph",
    "gen_random", "gen_xyz_chain", "generator_set_to_dict", "init_z", "near_clifford", "parse_circuit", "prob_z", "rank_stats", "ring_edges",
    "run", "run_all_modes", "serialize_circuit", "sub",
]
