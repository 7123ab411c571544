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

from . import engine
from .errors import FieldError

__all__ = [
    "FieldError",
    "GridGeometry",
    "ScalarField",
    "VectorField",
    "SampleGrid",
    "identity_coords",
    "axis_diff",
    "axis_diff_adjoint",
    "gradient_arr",
    "gradient_adjoint_arr",
    "divergence_arr",
    "divergence_adjoint_arr",
    "gradient",
    "divergence",
    "BilinearPlan",
    "bilinear_plan",
    "bilinear_apply",
    "bilinear_adjoint_values",
    "bilinear_coord_grad",
    "interpolate",
    "interpolate_vec",
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


# ---- array-level operators (fields.py:144-262) on the device ----------------------
#
# Same names, arguments and array layout as the reference (channel-last vector
# arrays [*shape, d]).  A numpy operand runs in float64 on the current CUDA device
# and returns numpy; a torch operand keeps its dtype (float32 / float64) and
# device and returns torch.  All arithmetic runs in libmorphreg_sm100.so
# (mr_ops.cu); there is no CPU fallback.


def _cuda_device():
    return torch.device("cuda", torch.cuda.current_device())


def _to_dev(a, dtype=None):
    """(CUDA tensor, is_numpy) for an array-level operand."""
    if isinstance(a, torch.Tensor):
        t = a.detach()
        if not t.is_floating_point():
            t = t.to(torch.float64)
        if dtype is not None:
            t = t.to(dtype)
        if not t.is_cuda:
            t = t.to(_cuda_device())
        return t.contiguous(), False
    t = torch.from_numpy(np.array(a, dtype=np.float64, order="C"))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(_cuda_device()), True


def _back(t: torch.Tensor, as_numpy: bool):
    return t.cpu().numpy() if as_numpy else t


def _last_to_first(t: torch.Tensor) -> torch.Tensor:
    return torch.movedim(t, -1, 0).contiguous()


def _first_to_last(t: torch.Tensor) -> torch.Tensor:
    return torch.movedim(t, 0, -1).contiguous()


def axis_diff(a, axis: int):
    """np.gradient along `axis` (fields.py:144-145)."""
    t, np_in = _to_dev(a)
    return _back(engine.axis_diff(t[None], axis)[0], np_in)


def axis_diff_adjoint(gbar, axis: int):
    """Exact transpose of axis_diff (fields.py:148-158)."""
    t, np_in = _to_dev(gbar)
    return _back(engine.axis_diff(t[None], axis, adjoint=True)[0], np_in)


def gradient_arr(f):
    """fields.py:161-162: [*shape] -> [*shape, d]."""
    t, np_in = _to_dev(f)
    return _back(_first_to_last(engine.gradient(t[None])[0]), np_in)


def gradient_adjoint_arr(gbar):
    """fields.py:165-166: [*shape, d] -> [*shape]."""
    t, np_in = _to_dev(gbar)
    return _back(engine.gradient_adjoint(_last_to_first(t)[None])[0], np_in)


def divergence_arr(v):
    """fields.py:169-170: [*shape, d] -> [*shape]."""
    t, np_in = _to_dev(v)
    return _back(engine.divergence(_last_to_first(t)[None])[0], np_in)


def divergence_adjoint_arr(dbar):
    """fields.py:173-176: [*shape] -> [*shape, d] (axis_diff_adjoint per axis)."""
    t, np_in = _to_dev(dbar)
    out = torch.stack([engine.axis_diff(t[None], ax, adjoint=True)[0] for ax in range(t.ndim)])
    return _back(_first_to_last(out), np_in)


def gradient(f: ScalarField) -> VectorField:
    """Discrete spatial gradient (fields.py:179-181)."""
    g = engine.gradient(f.tensor.to(_cuda_device())[None].contiguous())[0]
    return VectorField(f.geometry, g, channel_first=True, _trusted=True)


def divergence(v: VectorField) -> ScalarField:
    """Discrete divergence (fields.py:184-186)."""
    d = engine.divergence(v.tensor.to(_cuda_device())[None].contiguous())[0]
    return ScalarField(v.geometry, d, _trusted=True)


class BilinearPlan:
    """fields.py:196-204.  The device plan is the sample coordinates themselves
    (channel-first [d, *sample_shape] on the GPU): corner indices, fractions and the
    strict inside masks are formed in registers by every kernel that uses the
    plan (mr_interpolate*, mr_ops.cu), exactly as bilinear_plan defines them.
    ``shape`` is the shape of the sampled array; the sample positions may form any
    other grid (the kernels take one sample per array cell, so other sample counts
    run as ceil(M / N) array-shaped batches, padded with samples that are dropped)."""

    __slots__ = ("coords", "shape", "sample_shape")

    def __init__(self, coords: torch.Tensor, shape):
        self.coords = coords
        self.shape = tuple(int(n) for n in shape)
        self.sample_shape = tuple(coords.shape[1:])

    def __repr__(self) -> str:
        return (f"BilinearPlan(shape={self.shape}, samples={self.sample_shape}, "
                f"device={self.coords.device})")


def bilinear_plan(coords, shape) -> BilinearPlan:
    """fields.py:207-224: coords [..., d] (reference layout, any sample grid) -> plan."""
    t, _ = _to_dev(coords)
    shape = tuple(int(n) for n in shape)
    if t.ndim < 2 or t.shape[-1] != len(shape):
        raise FieldError(f"sample coordinates: expected [..., {len(shape)}], got {tuple(t.shape)}")
    if not bool(torch.isfinite(t).all()):
        raise FieldError("sample coordinates contain non-finite values")
    return BilinearPlan(_last_to_first(t), shape)


def _plan_coords(p: BilinearPlan, like: torch.Tensor) -> torch.Tensor:
    """[nb, d, *shape] coordinate batches of the plan (nb = 1 when the sample grid is
    the array grid)."""
    c = p.coords.to(device=like.device, dtype=like.dtype)
    if p.sample_shape == p.shape:
        return c.contiguous()[None]
    d, n = len(p.shape), int(np.prod(p.shape))
    m = int(np.prod(p.sample_shape))
    nb = max(1, -(-m // n))
    flat = torch.zeros((d, nb * n), dtype=c.dtype, device=c.device)
    flat[:, :m] = c.reshape(d, m)
    return flat.view((d, nb) + p.shape).transpose(0, 1).contiguous()


def _to_samples(p: BilinearPlan, out: torch.Tensor) -> torch.Tensor:
    """[nb, *shape] kernel output -> [*sample_shape]."""
    if p.sample_shape == p.shape:
        return out[0]
    m = int(np.prod(p.sample_shape))
    return out.reshape(-1)[:m].view(p.sample_shape)


def bilinear_apply(arr, p: BilinearPlan):
    """fields.py:235-240 (same term order, bitwise-exact at nodes in float64)."""
    t, np_in = _to_dev(arr)
    c = _plan_coords(p, t)
    a = t[None, None].expand((c.shape[0], 1) + tuple(t.shape)).contiguous()
    return _back(_to_samples(p, engine.interpolate(c, a)[:, 0]), np_in)


def bilinear_adjoint_values(p: BilinearPlan, gbar, shape):
    """fields.py:243-254: transpose of bilinear_apply w.r.t. the sampled array."""
    t, np_in = _to_dev(gbar)
    if tuple(shape) != p.shape:
        raise FieldError(f"geometry mismatch: {tuple(shape)} vs {p.shape}")
    c = _plan_coords(p, t)
    if p.sample_shape == p.shape:
        g = t[None]
    else:
        g = torch.zeros((c.shape[0] * int(np.prod(p.shape)),), dtype=t.dtype, device=t.device)
        g[:t.numel()] = t.reshape(-1)
        g = g.view((c.shape[0],) + p.shape)
    return _back(engine.interpolate_adjoint(c, g.contiguous()).sum(dim=0), np_in)


def bilinear_coord_grad(arr, p: BilinearPlan):
    """fields.py:257-262: per-axis derivative of the interpolated value (tuple)."""
    t, np_in = _to_dev(arr)
    c = _plan_coords(p, t)
    a = t[None].expand((c.shape[0],) + tuple(t.shape)).contiguous()
    out = engine.interpolate_coord_grad(c, a)
    return tuple(_back(_to_samples(p, out[:, ax]), np_in) for ax in range(out.shape[1]))


def interpolate(f: ScalarField, at: SampleGrid) -> ScalarField:
    """Bilinear interpolation of f at the sample positions, clamped (fields.py:265-269)."""
    _require_same_geometry(f, at)
    dev = _cuda_device()
    a = f.tensor.to(dev)
    c = at.tensor.to(dev, a.dtype)
    out = engine.interpolate(c[None].contiguous(), a[None, None].contiguous())[0, 0]
    return ScalarField(f.geometry, out, _trusted=True)


def interpolate_vec(v: VectorField, at: SampleGrid) -> VectorField:
    """Component-wise bilinear interpolation (fields.py:272-280)."""
    _require_same_geometry(v, at)
    dev = _cuda_device()
    a = v.tensor.to(dev)
    c = at.tensor.to(dev, a.dtype)
    out = engine.interpolate(c[None].contiguous(), a[None].contiguous())[0]
    return VectorField(v.geometry, out, channel_first=True, _trusted=True)


def _pair_reduce(f, g, op) -> float:
    dev = _cuda_device()
    a = f.tensor.to(dev)
    b = g.tensor.to(dev, a.dtype)
    return float(engine.reduce(a[None].contiguous(), b[None].contiguous(), op)[0].item())


def dot(f: ScalarField, g: ScalarField) -> float:
    """L2 inner product (fields.py:285-288), fp64 device reduction."""
    _require_same_geometry(f, g)
    return _pair_reduce(f, g, engine.REDUCE_DOT)


def ssd(f: ScalarField, g: ScalarField) -> float:
    """Half the sum of squared differences (fields.py:291-295), fp64 device reduction."""
    _require_same_geometry(f, g)
    return _pair_reduce(f, g, engine.REDUCE_SSD)
