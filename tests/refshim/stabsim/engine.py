from paper_2505_03307_b200.engine import *  # noqa: F401,F403
from paper_2505_03307_b200.engine import AgreementReport, Mode, RunReport, compare_reports, run, run_all_modes  # noqa: F401
