"""morphreg.kernel -> paper_2106_08817_b200.kernel (shim)."""
from paper_2106_08817_b200.kernel import *  # noqa: F401,F403
