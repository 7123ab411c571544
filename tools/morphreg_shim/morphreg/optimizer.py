"""morphreg.optimizer -> paper_2106_08817_b200.optimizer (shim)."""
from paper_2106_08817_b200.optimizer import *  # noqa: F401,F403
