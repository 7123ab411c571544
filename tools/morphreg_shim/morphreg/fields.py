"""morphreg.fields -> paper_2106_08817_b200.fields (shim)."""
from paper_2106_08817_b200.fields import *  # noqa: F401,F403
from paper_2106_08817_b200.fields import identity_coords  # noqa: F401
