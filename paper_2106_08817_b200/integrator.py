"""Geodesic shooting with the reference's signatures (integrator.py:48-219).

``shoot(i0, z0, cfg)`` runs the whole T-step loop on the device through one
``mr_shoot_forward_scheme`` call, then checks the device guard once and raises
``IntegrationDiverged(step, what)`` with the reference's text
(integrator.py:113-118).  All three schemes run on the device: the
semi-Lagrangian hot path (TMA-staged kernels, 2D and 3D) and the Eulerian /
Hybrid stencil steps (integrator.py:97-106, 2D as in the reference).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum

import torch

from . import engine
from .errors import FieldError, IntegrationDiverged
from .fields import GridGeometry, SampleGrid, ScalarField, VectorField
from .kernel import GaussianKernel

MAGNITUDE_GUARD = 1e6  # integrator.py:36

__all__ = [
    "MAGNITUDE_GUARD",
    "IntegrationDiverged",
    "Scheme",
    "ShootingConfig",
    "GeodesicState",
    "GeodesicTrajectory",
    "velocity_from_momentum",
    "advect_image_euler",
    "advect_image_sl",
    "continuity_euler",
    "continuity_sl",
    "shoot",
    "shoot_lddmm",
    "path_energy",
]


class Scheme(str, Enum):
    EULERIAN = "eulerian"
    SEMI_LAGRANGIAN = "semi-lagrangian"
    HYBRID = "hybrid"


@dataclass(frozen=True)
class ShootingConfig:
    """integrator.py:54-69.  ``dtype`` selects the device precision (float32
    default); ``deterministic`` makes grad() bitwise reproducible run to run
    (fixed-point adjoint scatters, MR_OPT_DETERMINISTIC -- the reference's replay
    promise, optimizer.py:5-7); the batched engine defaults to the faster
    atomic scatters."""

    scheme: Scheme
    n_steps: int
    mu: float
    kernel: GaussianKernel
    dtype: torch.dtype = field(default=torch.float32, compare=False)
    deterministic: bool = field(default=True, compare=False)

    def __post_init__(self) -> None:
        if self.n_steps < 1:
            raise FieldError(f"n_steps must be >= 1, got {self.n_steps}")
        if self.mu < 0:
            raise FieldError(f"mu must be >= 0, got {self.mu}")

    @property
    def dt(self) -> float:
        return 1.0 / self.n_steps


@dataclass(frozen=True)
class GeodesicState:
    t: float
    image: ScalarField
    momentum: ScalarField
    velocity: VectorField


@dataclass(frozen=True)
class GeodesicTrajectory:
    states: list
    deformation: SampleGrid
    device: engine.DeviceTrajectory | None = None

    @property
    def final_image(self) -> ScalarField:
        return self.states[-1].image


def _to_device(f, dtype=None) -> torch.Tensor:
    """A field's tensor on the current CUDA device (dtype None: the field's own)."""
    dev = torch.device("cuda", torch.cuda.current_device())
    t = f.tensor
    return t.to(dev, dtype if dtype is not None else t.dtype).contiguous()


def velocity_from_momentum(z: ScalarField, image: ScalarField, kernel: GaussianKernel,
                           dtype=None) -> VectorField:
    """v = -K * (z grad I) (integrator.py:124-130)."""
    if z.geometry != image.geometry:
        raise FieldError("momentum/image geometry mismatch")
    I = _to_device(image, dtype).unsqueeze(0)
    zz = _to_device(z, I.dtype).unsqueeze(0)
    if len(z.geometry.shape) == 2:
        v = engine.velocity(I, zz, kernel.weights)[0]
    else:  # 3D: one-state shoot of the whole-loop entry point (velocity at step 0)
        traj = engine.allocate_trajectory(1, z.geometry.shape, 1, I.dtype, I.device)
        traj.I[0].copy_(I)
        traj.z[0].copy_(zz)
        engine.shoot_forward(traj, 0.0, kernel.weights)
        v = traj.v[0, 0]
    return VectorField(z.geometry, v, channel_first=True, _trusted=True)


def _single_step(scheme: Scheme, image: ScalarField, v: VectorField, z: ScalarField,
                 mu: float, dt: float):
    if not (image.geometry == v.geometry == z.geometry):
        raise FieldError("image/velocity/momentum geometry mismatch")
    I = _to_device(image).unsqueeze(0)
    zz = _to_device(z, I.dtype).unsqueeze(0)
    vv = _to_device(v, I.dtype).unsqueeze(0)
    In, zn, _ = engine.scheme_step(I, zz, vv, dt, mu, scheme=scheme.value)
    return In[0], zn[0]


def advect_image_euler(image: ScalarField, v: VectorField, z: ScalarField, mu: float,
                       dt: float) -> ScalarField:
    """I + dt(-(grad I . v) + mu z) (integrator.py:133-138)."""
    In, _ = _single_step(Scheme.EULERIAN, image, v, z, mu, dt)
    return ScalarField(image.geometry, In, _trusted=True)


def advect_image_sl(image: ScalarField, v: VectorField, z: ScalarField, mu: float,
                    dt: float) -> ScalarField:
    """B(I) + dt mu z at the feet Id - dt v (integrator.py:141-146)."""
    In, _ = _single_step(Scheme.SEMI_LAGRANGIAN, image, v, z, mu, dt)
    return ScalarField(image.geometry, In, _trusted=True)


def continuity_euler(z: ScalarField, v: VectorField, dt: float) -> ScalarField:
    """z - dt div(z v) (integrator.py:149-150)."""
    _, zn = _single_step(Scheme.EULERIAN, z, v, z, 0.0, dt)
    return ScalarField(z.geometry, zn, _trusted=True)


def continuity_sl(z: ScalarField, v: VectorField, dt: float) -> ScalarField:
    """B(z)(1 - dt div v) at the feet Id - dt v (integrator.py:153-159)."""
    _, zn = _single_step(Scheme.SEMI_LAGRANGIAN, z, v, z, 0.0, dt)
    return ScalarField(z.geometry, zn, _trusted=True)


def _run(i0: ScalarField, z0: ScalarField, cfg: ShootingConfig, mu: float) -> GeodesicTrajectory:
    if i0.geometry != z0.geometry:
        raise FieldError("image/momentum geometry mismatch")
    geom = i0.geometry
    traj = engine.allocate_trajectory(1, geom.shape, cfg.n_steps, cfg.dtype, with_phi=True)
    traj.I[0, 0].copy_(_to_device(i0, cfg.dtype))
    traj.z[0, 0].copy_(_to_device(z0, cfg.dtype))
    engine.shoot_forward(traj, mu, cfg.kernel.weights, scheme=cfg.scheme.value)
    engine.raise_on_guard(traj)
    dt = cfg.dt
    states = []
    for k in range(cfg.n_steps + 1):
        states.append(
            GeodesicState(
                t=(k * dt if k < cfg.n_steps else 1.0),
                image=ScalarField(geom, traj.I[k, 0], _trusted=True),
                momentum=ScalarField(geom, traj.z[k, 0], _trusted=True),
                velocity=VectorField(geom, traj.v[k, 0], channel_first=True, _trusted=True),
            )
        )
    phi = SampleGrid(geom, traj.phi[0, 0], channel_first=True, _trusted=True)
    return GeodesicTrajectory(states=states, deformation=phi, device=traj)


def shoot(i0: ScalarField, z0: ScalarField, cfg: ShootingConfig) -> GeodesicTrajectory:
    """Integrate the geodesic system from (i0, z0) over unit time (integrator.py:163-219)."""
    return _run(i0, z0, cfg, cfg.mu)


def shoot_lddmm(i0: ScalarField, z0: ScalarField, cfg: ShootingConfig) -> GeodesicTrajectory:
    """Deformation-only shooting (integrator.py:222-277): the mu = 0 path of the
    same kernels, so ``shoot`` with mu = 0 reproduces it bit for bit."""
    return _run(i0, z0, cfg, 0.0)


def path_energy(traj: GeodesicTrajectory, kernel: GaussianKernel, rho: float) -> list:
    """Per-state ||v_t||_V^2 + rho ||z_t||^2 with v built from ``kernel``
    (integrator.py:280-289): m_t = z_t grad I_t, ||v_t||_V^2 = <m_t, K m_t>.

    All T+1 states run as one batch on the device: the velocity kernels give
    K m_t = -v_t for the requested kernel and mr_cost_terms reduces
    -<m_t, v_t> and |z_t|^2 in fp64."""
    if traj.device is not None:
        I = traj.device.I
        z = traj.device.z
        T1, B = I.shape[0], I.shape[1]
        I = I.reshape((T1 * B,) + tuple(I.shape[2:]))
        z = z.reshape((T1 * B,) + tuple(z.shape[2:]))
    else:
        I = torch.stack([_to_device(s.image) for s in traj.states])
        z = torch.stack([_to_device(s.momentum, I.dtype) for s in traj.states])
        T1, B = I.shape[0], 1
    shape = tuple(I.shape[1:])
    if len(shape) == 2:
        v = engine.velocity(I.contiguous(), z.contiguous(), kernel.weights)
    else:
        tr = engine.allocate_trajectory(T1 * B, shape, 1, I.dtype, I.device)
        tr.I[0].copy_(I)
        tr.z[0].copy_(z)
        engine.shoot_forward(tr, 0.0, kernel.weights)
        v = tr.v[0]
    terms = engine.cost_terms(I.contiguous(), z.contiguous(), v, I.contiguous(), I.contiguous(),
                              1.0, rho).cpu().numpy()
    per = [float(t[2] + rho * t[3]) for t in terms]  # v_norm + rho * z_norm
    if B == 1:
        return per
    return [per[k * B:(k + 1) * B] for k in range(T1)]
