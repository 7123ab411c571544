"""Synthetic imagery of the reference's experiments (synthetic.py:14-144): disks,
annuli, the open 'C' ring and smooth random fields, plus the two named presets.

Host-side set-up code, not on the hot path; the anti-alias blur runs through the
device smoothing (kernel.smooth_arr -> mr_smooth)."""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

from .errors import FieldError
from .fields import GridGeometry, ScalarField, VectorField
from .kernel import GaussianKernel, smooth_arr

__all__ = ["ShapeKind", "ShapeSpec", "render", "smooth_random_field", "smooth_random_vec",
           "PRESETS", "preset_pair"]


class ShapeKind(Enum):
    DISK = "disk"
    ANNULUS = "annulus"
    C_OPENING = "c"


@dataclass(frozen=True)
class ShapeSpec:
    """A shape in pixel units (synthetic.py:20-46).  ``orientation``: direction the C
    opening faces, degrees counter-clockwise from +column; unused otherwise."""

    kind: ShapeKind
    center: tuple
    outer: float
    inner: float = 0.0
    opening_angle: float = 70.0
    orientation: float = 0.0
    intensity: float = 1.0
    smoothing_sigma: float = 0.0

    def __post_init__(self) -> None:
        if min(self.inner, self.outer) < 0:
            raise FieldError("shape radii must be non-negative")
        if self.kind is not ShapeKind.DISK and not self.inner < self.outer:
            raise FieldError("annular shapes need inner < outer")
        if not (0.0 <= self.intensity <= 1.0):
            raise FieldError(f"intensity must lie in [0,1], got {self.intensity}")
        if self.smoothing_sigma < 0:
            raise FieldError("smoothing_sigma must be >= 0")


def _indicator(spec: ShapeSpec, shape) -> np.ndarray:
    rows = np.arange(shape[0], dtype=np.float64)[:, None] - spec.center[0]
    cols = np.arange(shape[1], dtype=np.float64)[None, :] - spec.center[1]
    radius = np.hypot(rows, cols)
    inside = radius < spec.outer
    if spec.kind is ShapeKind.DISK:
        return inside
    ring = inside & (radius >= spec.inner)
    if spec.kind is ShapeKind.ANNULUS:
        return ring
    # C ring: drop the sector of half-width opening_angle / 2 around `orientation`
    # (image rows grow downwards, hence -rows)
    bearing = np.degrees(np.arctan2(-rows, cols))
    off_axis = (bearing - spec.orientation + 180.0) % 360.0 - 180.0
    return ring & (np.abs(off_axis) > 0.5 * spec.opening_angle)


def render(spec: ShapeSpec, geometry: GridGeometry) -> ScalarField:
    """Rasterise the indicator scaled by the intensity; blur when asked (synthetic.py:49-75)."""
    img = spec.intensity * _indicator(spec, geometry.shape).astype(np.float64)
    if spec.smoothing_sigma > 0:
        img = smooth_arr(GaussianKernel(spec.smoothing_sigma), img)
    return ScalarField(geometry, img)


def _noise(geometry: GridGeometry, seed: int, trailing=()):
    return np.random.default_rng(seed).standard_normal(geometry.shape + tuple(trailing))


def smooth_random_field(geometry: GridGeometry, sigma: float, seed: int) -> ScalarField:
    """Gaussian-smoothed white noise, a function of the seed only (synthetic.py:78-84)."""
    return ScalarField(geometry, smooth_arr(GaussianKernel(sigma), _noise(geometry, seed)))


def smooth_random_vec(geometry: GridGeometry, sigma: float, seed: int) -> VectorField:
    """Two smoothed noise components drawn as one [H, W, 2] block (synthetic.py:87-95)."""
    white = _noise(geometry, seed, (2,))
    kern = GaussianKernel(sigma)
    comps = [np.asarray(smooth_arr(kern, np.ascontiguousarray(white[..., c]))) for c in range(2)]
    return VectorField(geometry, np.stack(comps, axis=-1))


# Presets are laid out on a 200 x 200 grid and scale with `size` (synthetic.py:98-144).
PRESETS = ("c2disk", "disk2c")


def preset_pair(name: str, size: int = 200):
    """(source, target) of a named preset: ``c2disk`` = C ring -> the same ring plus a
    detached small disk to its right; ``disk2c`` = filled disk -> C ring."""
    if name not in PRESETS:
        raise FieldError(f"unknown preset {name!r}; choose from {PRESETS}")
    geometry = GridGeometry(size, size)
    unit = size / 200.0
    mid = 0.5 * (size - 1)
    blur = max(1.0, 1.5 * unit)

    def shape(kind, outer, inner=0.0, dx=0.0):
        return render(ShapeSpec(kind=kind, center=(mid, mid + dx * unit), outer=outer * unit,
                                inner=inner * unit, smoothing_sigma=blur), geometry)

    ring = shape(ShapeKind.C_OPENING, 60.0, 35.0)
    if name == "disk2c":
        return shape(ShapeKind.DISK, 50.0), ring
    satellite = shape(ShapeKind.DISK, 15.0, dx=80.0)
    return ring, ScalarField(geometry, np.maximum(ring.values, satellite.values))
