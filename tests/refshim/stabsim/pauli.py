from paper_2505_03307_b200.pauli import *  # noqa: F401,F403
from paper_2505_03307_b200.pauli import (  # noqa: F401
    AXIS_CHARS, AXIS_PRODUCT, PHASE_EXP, PHASE_VALUES, PHASE_VALUES_NP, Axis, axis_mul, axis_to_index,
    axis_to_weight, index_to_axis, index_to_word, phase_value, str_to_word, weight_to_axis, word_mul,
    word_to_index, word_to_str,
)
