"""Grid value types of the reference API (fields.py:20-128), backed by torch tensors.

Drop-in behaviour: ``ScalarField(geometry, values)`` accepts the reference's
numpy arrays (or torch tensors, possibly on the GPU); ``.values`` returns a
read-only float64 numpy array in the reference layout ([H, W] / [H, W, 2]),
``.tensor`` the stored tensor (vector fields channel-first, [d, *shape]).
Construction checks shape and finiteness like ``_frozen_array``
(fields.py:41-48); no per-step copies are made on the device path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .errors import FieldError

__all__ = [
    "FieldError",
    "GridGeometry",
    "ScalarField",
    "VectorField",
    "SampleGrid",
    "identity_coords",
    "dot",
    "ssd",
]


@dataclass(frozen=True)
class GridGeometry:
    """Rectangular grid (fields.py:20-38); ``depth`` set makes it 3D [D, H, W]."""

    height: int
    width: int
    spacing: float = 1.0
    depth: int | None = None

    def __post_init__(self) -> None:
        if self.height < 2 or self.width < 2 or (self.depth is not None and self.depth < 2):
            dims = f"{self.height}x{self.width}" if self.depth is None else (
                f"{self.depth}x{self.height}x{self.width}")
            raise FieldError(f"grid must be at least 2x2, got {dims}")
        if self.spacing <= 0:
            raise FieldError(f"grid spacing must be positive, got {self.spacing}")

    @property
    def shape(self) -> tuple:
        if self.depth is None:
            return (self.height, self.width)
        return (self.depth, self.height, self.width)

    @property
    def ndim(self) -> int:
        return len(self.shape)

    @classmethod
    def from_shape(cls, shape) -> "GridGeometry":
        shape = tuple(int(s) for s in shape)
        if len(shape) == 2:
            return cls(shape[0], shape[1])
        if len(shape) == 3:
            return cls(shape[1], shape[2], depth=shape[0])
        raise FieldError(f"expected a 2d or 3d grid, got shape {shape}")


def _as_tensor(values) -> torch.Tensor:
    if isinstance(values, torch.Tensor):
        t = values.detach()
        if not t.is_floating_point():
            t = t.to(torch.float64)
        return t
    return torch.from_numpy(np.array(values, dtype=np.float64, order="C"))


def _check(t: torch.Tensor, shape, what: str) -> torch.Tensor:
    if tuple(t.shape) != tuple(shape):
        raise FieldError(f"{what}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
    if not bool(torch.isfinite(t).all()):
        raise FieldError(f"{what}: non-finite values")
    return t.contiguous()


def _readonly(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    a.flags.writeable = False
    return a


class ScalarField:
    """Real-valued function sampled on the grid (fields.py:51-75)."""

    __slots__ = ("geometry", "_t", "_np")

    def __init__(self, geometry: GridGeometry, values, _trusted: bool = False):
        t = _as_tensor(values)
        self.geometry = geometry
        self._t = t.contiguous() if _trusted else _check(t, geometry.shape, "ScalarField")
        self._np = None

    @property
    def tensor(self) -> torch.Tensor:
        return self._t

    @property
    def values(self) -> np.ndarray:
        if self._np is None:
            self._np = _readonly(self._t.detach().to("cpu", torch.float64).numpy())
        return self._np

    @classmethod
    def from_array(cls, values) -> "ScalarField":
        t = _as_tensor(values)
        if t.ndim not in (2, 3):
            raise FieldError(f"ScalarField: expected 2d or 3d array, got {t.ndim}d")
        return cls(GridGeometry.from_shape(t.shape), t)

    @classmethod
    def zeros(cls, geometry: GridGeometry) -> "ScalarField":
        return cls(geometry, torch.zeros(geometry.shape, dtype=torch.float64), _trusted=True)

    def __repr__(self) -> str:
        return f"ScalarField({self.geometry}, device={self._t.device}, dtype={self._t.dtype})"


class VectorField:
    """d-component field (fields.py:78-101).

    Accepts the reference layout [*shape, d] (numpy or torch) or, with
    ``channel_first=True``, the device layout [d, *shape].  ``.values`` is
    always the reference layout.
    """

    __slots__ = ("geometry", "_t", "_np")
    _what = "VectorField"

    def __init__(self, geometry: GridGeometry, values, channel_first: bool = False,
                 _trusted: bool = False):
        t = _as_tensor(values)
        d = geometry.ndim
        self.geometry = geometry
        if not channel_first:
            t = _check(t, geometry.shape + (d,), self._what) if not _trusted else t
            t = torch.movedim(t, -1, 0).contiguous()
        else:
            t = _check(t, (d,) + geometry.shape, self._what) if not _trusted else t.contiguous()
        self._t = t
        self._np = None

    @property
    def tensor(self) -> torch.Tensor:
        """Channel-first [d, *shape]."""
        return self._t

    @property
    def values(self) -> np.ndarray:
        if self._np is None:
            a = self._t.detach().to("cpu", torch.float64).numpy()
            self._np = _readonly(np.moveaxis(a, 0, -1))
        return self._np

    @classmethod
    def from_array(cls, values) -> "VectorField":
        t = _as_tensor(values)
        if t.ndim not in (3, 4) or t.shape[-1] != t.ndim - 1:
            raise FieldError(f"{cls._what}: expected [*shape, d] array, got {tuple(t.shape)}")
        return cls(GridGeometry.from_shape(t.shape[:-1]), t)

    @classmethod
    def zeros(cls, geometry: GridGeometry):
        return cls(geometry, torch.zeros((geometry.ndim,) + geometry.shape, dtype=torch.float64),
                   channel_first=True, _trusted=True)


class SampleGrid(VectorField):
    """Per-pixel sample positions (fields.py:104-119); ``.coords`` is the reference layout."""

    _what = "SampleGrid"

    @property
    def coords(self) -> np.ndarray:
        return self.values

    @classmethod
    def identity(cls, geometry: GridGeometry) -> "SampleGrid":
        return cls(geometry, torch.from_numpy(identity_coords(geometry.shape)))


def identity_coords(shape) -> np.ndarray:
    """fields.py:114-120 (reference layout [*shape, d])."""
    grids = np.meshgrid(*[np.arange(n, dtype=np.float64) for n in shape], indexing="ij")
    return np.stack(grids, axis=-1)


def _require_same_geometry(a, b) -> None:
    if a.geometry != b.geometry:
        raise FieldError(f"geometry mismatch: {a.geometry} vs {b.geometry}")


def dot(f: ScalarField, g: ScalarField) -> float:
    """L2 inner product (fields.py:285-288)."""
    _require_same_geometry(f, g)
    return float(np.sum(f.values * g.values))


def ssd(f: ScalarField, g: ScalarField) -> float:
    """Half the sum of squared differences (fields.py:291-295)."""
    _require_same_geometry(f, g)
    diff = f.values - g.values
    return 0.5 * float(np.sum(diff * diff))
