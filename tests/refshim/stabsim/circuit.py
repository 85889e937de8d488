from paper_2505_03307_b200.circuit import *  # noqa: F401,F403
from paper_2505_03307_b200.circuit import (  # noqa: F401
    ALL_GATES, GATES_1Q, GATES_2Q, PARAMETRIC_GATES, CircuitParseError, Instruction, OperatorPartition,
    create_chain, cx, divide_instruction, h, parse_circuit, rx, ry, rz, s, serialize_circuit, sx, x,
)
from paper_2505_03307_b200.workloads import gen_ghz, gen_graph, gen_random, gen_xyz_chain, ring_edges  # noqa: F401
