"""morphreg.image_io -> paper_2106_08817_b200.image_io (shim)."""
from paper_2106_08817_b200.image_io import *  # noqa: F401,F403
