"""morphreg.integrator -> paper_2106_08817_b200.integrator, float64 ShootingConfig (shim)."""
from dataclasses import dataclass, field

import torch

from paper_2106_08817_b200 import integrator as _integrator
from paper_2106_08817_b200.integrator import *  # noqa: F401,F403


@dataclass(frozen=True)
class ShootingConfig(_integrator.ShootingConfig):
    dtype: torch.dtype = field(default=torch.float64, compare=False)
