"""Truncated Gaussian RKHS kernel (kernel.py:17-33) and its device smoothing.

The weights are computed on the host in float64 exactly as the reference does;
the separable replicate-border convolution and its transpose run on the device:
the sm_100a FIR engine for 2D scalar batches (mr_smooth), the direct 1D FIR
(mr_conv1d) for single axes and for 3D.  Array-level functions follow the
reference's layout and dtype rules (numpy in -> float64 on the device -> numpy
out; torch in -> same dtype and device out, see ``fields._to_dev``).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import engine
from .errors import FieldError
from .fields import ScalarField, VectorField, _back, _first_to_last, _last_to_first, _to_dev

__all__ = [
    "GaussianKernel",
    "conv1d_replicate",
    "conv1d_replicate_adjoint",
    "smooth_arr",
    "smooth_adjoint_arr",
    "smooth_vec_arr",
    "smooth_adjoint_vec_arr",
    "smooth_scalar",
    "smooth_scalar_adjoint",
    "smooth_vector",
    "v_norm_sq_arr",
    "v_norm_sq",
]


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


def _smooth_batch(t: torch.Tensor, weights, adjoint: bool = False) -> torch.Tensor:
    """Separable smoothing of a scalar batch [B, *shape] on the device.

    Forward: last axis first (kernel.py:71-73, axis 1 then axis 0 in 2D);
    transpose: axis 0 first (kernel.py:76-79)."""
    d = t.dim() - 1
    if d == 2 and t.shape[-1] >= 2 and t.shape[-2] >= 2:
        return engine.smooth(t.contiguous(), weights, adjoint=adjoint)
    axes = range(d) if adjoint else reversed(range(d))
    for ax in axes:
        t = engine.conv1d(t.contiguous(), weights, ax, adjoint=adjoint)
    return t


def conv1d_replicate(a, weights, axis: int):
    """1D convolution along `axis` with replicate borders (kernel.py:36-45)."""
    t, np_in = _to_dev(a)
    return _back(engine.conv1d(t[None], np.asarray(weights), axis)[0], np_in)


def conv1d_replicate_adjoint(gbar, weights, axis: int):
    """Exact transpose of conv1d_replicate (kernel.py:48-68)."""
    t, np_in = _to_dev(gbar)
    return _back(engine.conv1d(t[None], np.asarray(weights), axis, adjoint=True)[0], np_in)


def smooth_arr(kernel: GaussianKernel, a):
    """kernel.py:71-73."""
    t, np_in = _to_dev(a)
    return _back(_smooth_batch(t[None], kernel.weights)[0], np_in)


def smooth_adjoint_arr(kernel: GaussianKernel, gbar):
    """kernel.py:76-79."""
    t, np_in = _to_dev(gbar)
    return _back(_smooth_batch(t[None], kernel.weights, adjoint=True)[0], np_in)


def smooth_vec_arr(kernel: GaussianKernel, v):
    """kernel.py:82-85: component-wise on [*shape, d]."""
    t, np_in = _to_dev(v)
    return _back(_first_to_last(_smooth_batch(_last_to_first(t), kernel.weights)), np_in)


def smooth_adjoint_vec_arr(kernel: GaussianKernel, gbar):
    """kernel.py:88-92."""
    t, np_in = _to_dev(gbar)
    out = _smooth_batch(_last_to_first(t), kernel.weights, adjoint=True)
    return _back(_first_to_last(out), np_in)


def _field_tensor(f, dtype):
    dev = torch.device("cuda", torch.cuda.current_device())
    t = f.tensor
    return t.to(dev, dtype if dtype is not None else t.dtype).contiguous()


def smooth_scalar(kernel: GaussianKernel, f: ScalarField, dtype=None) -> ScalarField:
    """kernel.py:95-96 (dtype: device precision; default the field's own)."""
    out = _smooth_batch(_field_tensor(f, dtype)[None], kernel.weights)[0]
    return ScalarField(f.geometry, out, _trusted=True)


def smooth_scalar_adjoint(kernel: GaussianKernel, f: ScalarField, dtype=None) -> ScalarField:
    """smooth_adjoint_arr (kernel.py:76-79) on a field."""
    out = _smooth_batch(_field_tensor(f, dtype)[None], kernel.weights, adjoint=True)[0]
    return ScalarField(f.geometry, out, _trusted=True)


def smooth_vector(kernel: GaussianKernel, v: VectorField, dtype=None) -> VectorField:
    """kernel.py:99-100: component-wise smoothing ([d, *shape] = a batch of d scalars)."""
    out = _smooth_batch(_field_tensor(v, dtype), kernel.weights)
    return VectorField(v.geometry, out, channel_first=True, _trusted=True)


def _v_norm_sq_dev(m: torch.Tensor, weights) -> float:
    """sum_c <m_c, K m_c> (kernel.py:103-108) for a channel-first [d, *shape] tensor."""
    km = _smooth_batch(m, weights)
    per = engine.reduce(m, km, engine.REDUCE_DOT)  # fp64, one value per component
    total = 0.0
    for x in per.cpu().numpy():  # accumulated in component order, as the reference
        total += float(x)
    return total


def v_norm_sq_arr(kernel: GaussianKernel, m) -> float:
    """Squared velocity-space norm of a raw momentum field [*shape, d] (kernel.py:103-108)."""
    t, _ = _to_dev(m)
    return _v_norm_sq_dev(_last_to_first(t), kernel.weights)


def v_norm_sq(kernel: GaussianKernel, m: VectorField, dtype=None) -> float:
    """kernel.py:111-112."""
    return _v_norm_sq_dev(_field_tensor(m, dtype), kernel.weights)
