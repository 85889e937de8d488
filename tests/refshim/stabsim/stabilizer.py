from paper_2505_03307_b200.stabilizer import *  # noqa: F401,F403
from paper_2505_03307_b200.stabilizer import (  # noqa: F401
    DEFAULT_EPS, DENSE_FLATTEN_BUDGET, DenseComplexGenerator, GeneratorSet, RaggedComplexGenerator,
    SimpleGenerator, apply_cx, branch_counts, canonicalize, digits_to_indices, flatten,
    generator_set_to_dict, index_dtype, indices_to_digits, init_z, make_index_array, rank_stats, sub,
    to_dense, to_ragged,
)
