"""morphreg.objective -> paper_2106_08817_b200.objective (shim)."""
from paper_2106_08817_b200.objective import *  # noqa: F401,F403
