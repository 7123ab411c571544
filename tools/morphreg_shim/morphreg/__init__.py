"""`morphreg` compatibility shim over the B200 facade (test harness, fp64 mode).

Lets the reference's own test suite (`/root/reference/pkg/tests`, run by
`tools/run_reference_suite.sh`) import `morphreg` and exercise
`paper_2106_08817_b200` unchanged: every name resolves to the facade, and
ShootingConfig defaults to the float64 device instantiation (the reference's
finite-difference tests need float64).  Array-level operators
already run in float64 for numpy inputs.  Not part of the product.
"""

from paper_2106_08817_b200 import *  # noqa: F401,F403
from paper_2106_08817_b200 import __all__ as _facade_all

from .integrator import ShootingConfig  # noqa: F401  (float64 default)

__version__ = "0.1.0"
__all__ = list(_facade_all)
