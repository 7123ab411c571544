"""morphreg.synthetic -> paper_2106_08817_b200.shapes (shim)."""
from paper_2106_08817_b200.shapes import *  # noqa: F401,F403
