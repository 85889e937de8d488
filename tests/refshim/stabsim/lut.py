from paper_2505_03307_b200.lut import *  # noqa: F401,F403
from paper_2505_03307_b200.lut import (  # noqa: F401
    LUT_C, LUT_SIGN, LUT_T, axis_map, conjugate_axis, create_lut_1q, cx_lookup, lut_to_json,
)
