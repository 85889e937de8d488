from paper_2505_03307_b200.errors import *  # noqa: F401,F403
from paper_2505_03307_b200.errors import ConsistencyError, NumericalCollapseError, ResourceLimitError  # noqa: F401
