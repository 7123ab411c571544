"""Truncated Gaussian RKHS kernel (kernel.py:17-33) and its device smoothing.

The weights are computed on the host in float64 exactly as the reference does;
the separable replicate-border convolution and its transpose run in the
sm_100a FIR engine (mr_smooth / mr_velocity / mr_velocity_adjoint).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import engine
from .errors import FieldError
from .fields import ScalarField, VectorField

__all__ = ["GaussianKernel", "smooth_scalar", "smooth_vector", "smooth_scalar_adjoint", "v_norm_sq"]


class GaussianKernel:
    """Normalized, truncated Gaussian; immutable after construction (kernel.py:17-33)."""

    def __init__(self, sigma: float, radius: int | None = None):
        if sigma <= 0:
            raise FieldError(f"kernel sigma must be positive, got {sigma}")
        self.sigma = float(sigma)
        self.radius = int(math.ceil(4 * sigma)) if radius is None else int(radius)
        if self.radius < 1:
            raise FieldError(f"kernel radius must be >= 1, got {self.radius}")
        x = np.arange(-self.radius, self.radius + 1, dtype=np.float64)
        w = np.exp(-0.5 * (x / self.sigma) ** 2)
        self.weights = w / np.sum(w)
        self.weights.flags.writeable = False

    def __repr__(self) -> str:
        return f"GaussianKernel(sigma={self.sigma}, radius={self.radius})"


def _device(dtype=torch.float32):
    return torch.device("cuda", torch.cuda.current_device()), dtype


def smooth_scalar(kernel: GaussianKernel, f: ScalarField, dtype=torch.float32) -> ScalarField:
    """smooth_scalar (kernel.py:95-96) on the device."""
    dev, dt = _device(dtype)
    a = f.tensor.to(dev, dt).unsqueeze(0).contiguous()
    out = engine.smooth(a, kernel.weights)[0]
    return ScalarField(f.geometry, out, _trusted=True)


def smooth_scalar_adjoint(kernel: GaussianKernel, f: ScalarField, dtype=torch.float32) -> ScalarField:
    """smooth_adjoint_arr (kernel.py:76-79) on the device."""
    dev, dt = _device(dtype)
    a = f.tensor.to(dev, dt).unsqueeze(0).contiguous()
    out = engine.smooth(a, kernel.weights, adjoint=True)[0]
    return ScalarField(f.geometry, out, _trusted=True)


def smooth_vector(kernel: GaussianKernel, v: VectorField, dtype=torch.float32) -> VectorField:
    """smooth_vector (kernel.py:99-100): component-wise smoothing."""
    dev, dt = _device(dtype)
    a = v.tensor.to(dev, dt).contiguous()  # [d, *shape] = a batch of d scalars
    out = engine.smooth(a, kernel.weights)
    return VectorField(v.geometry, out, channel_first=True, _trusted=True)


def v_norm_sq(kernel: GaussianKernel, m: VectorField, dtype=torch.float32) -> float:
    """<m, K m> summed over components (kernel.py:103-112)."""
    dev, dt = _device(dtype)
    a = m.tensor.to(dev, dt).contiguous()
    km = engine.smooth(a, kernel.weights)
    return float((a.double() * km.double()).sum())
