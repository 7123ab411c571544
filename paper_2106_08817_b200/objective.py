"""Inexact-matching cost and its exact discrete gradient (objective.py:39-174).

``grad(problem, z0)`` = one ``mr_shoot_forward`` + one ``mr_shoot_adjoint``
(the hand-built reverse accumulation of the reference, as explicit sm_100a
kernels).  ``ShootingCost`` wraps the same pair as a ``torch.autograd.Function``
over a batch: forward = shoot + cost terms, backward = the adjoint sweep.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import engine
from .errors import FieldError
from .fields import ScalarField
from .integrator import GeodesicTrajectory, ShootingConfig, _require_sl, _to_device

__all__ = ["RegistrationProblem", "CostReport", "cost", "grad", "ShootingCost", "cost_and_grad_batch"]


@dataclass(frozen=True)
class RegistrationProblem:
    source: ScalarField
    target: ScalarField
    lam: float
    rho: float
    cfg: ShootingConfig

    def __post_init__(self) -> None:
        if self.source.geometry != self.target.geometry:
            raise FieldError("source/target geometry mismatch")
        if self.lam <= 0:
            raise FieldError(f"lambda must be positive, got {self.lam}")
        if self.rho < 0:
            raise FieldError(f"rho must be >= 0, got {self.rho}")


@dataclass(frozen=True)
class CostReport:
    total: float
    data_term: float
    v_norm: float
    z_norm: float


def _report(row) -> CostReport:
    return CostReport(total=float(row[0]), data_term=float(row[1]), v_norm=float(row[2]),
                      z_norm=float(row[3]))


def cost(problem: RegistrationProblem, z0: ScalarField,
         trajectory: GeodesicTrajectory | None = None) -> CostReport:
    """objective.py:71-88: data + lam * (||v0||_V^2 + rho ||z0||^2)."""
    if z0.geometry != problem.source.geometry:
        raise FieldError("initial momentum geometry mismatch")
    cfg = problem.cfg
    _require_sl(cfg)
    if trajectory is None or trajectory.device is None:
        traj = engine.allocate_trajectory(1, z0.geometry.shape, cfg.n_steps, cfg.dtype)
        traj.I[0, 0].copy_(_to_device(problem.source, cfg.dtype))
        traj.z[0, 0].copy_(_to_device(z0, cfg.dtype))
        engine.shoot_forward(traj, cfg.mu, cfg.kernel.weights)
        engine.raise_on_guard(traj)
    else:
        traj = trajectory.device
    J = _to_device(problem.target, traj.I.dtype).unsqueeze(0)
    terms = engine.cost_terms(traj.I[0], traj.z[0], traj.v[0], traj.I[-1], J, problem.lam,
                              problem.rho)
    return _report(terms[0].cpu().numpy())


def grad(problem: RegistrationProblem, z0: ScalarField) -> ScalarField:
    """Gradient of the discrete cost w.r.t. every entry of z0 (objective.py:91-174)."""
    if z0.geometry != problem.source.geometry:
        raise FieldError("initial momentum geometry mismatch")
    cfg = problem.cfg
    _require_sl(cfg)
    traj = engine.allocate_trajectory(1, z0.geometry.shape, cfg.n_steps, cfg.dtype)
    traj.I[0, 0].copy_(_to_device(problem.source, cfg.dtype))
    traj.z[0, 0].copy_(_to_device(z0, cfg.dtype))
    engine.shoot_forward(traj, cfg.mu, cfg.kernel.weights)
    engine.raise_on_guard(traj)
    J = _to_device(problem.target, cfg.dtype).unsqueeze(0)
    bufs = engine.shoot_adjoint(traj, J, problem.lam, problem.rho, cfg.mu, cfg.kernel.weights)
    if int(bufs.flags[0].item()) != 0:  # objective.py:171-173
        bad = torch.nonzero(~torch.isfinite(bufs.zbar[0]))[0].tolist()
        raise FieldError(f"non-finite gradient entry at pixel {tuple(bad)}")
    return ScalarField(z0.geometry, bufs.zbar[0], _trusted=True)


class ShootingCost(torch.autograd.Function):
    """Batched cost H(z0) per pair with the explicit adjoint as backward.

    forward(z0 [B,*shape], source [B,*shape], target [B,*shape], cfg, lam, rho)
      -> totals [B] (float64); the full CostReport rows are in ``ctx``-free
      form via :func:`cost_and_grad_batch`.
    """

    @staticmethod
    def forward(ctx, z0, source, target, cfg: ShootingConfig, lam: float, rho: float):
        _require_sl(cfg)
        B = z0.shape[0]
        shape = tuple(z0.shape[1:])
        traj = engine.allocate_trajectory(B, shape, cfg.n_steps, z0.dtype, z0.device)
        traj.I[0].copy_(source)
        traj.z[0].copy_(z0)
        engine.shoot_forward(traj, cfg.mu, cfg.kernel.weights)
        engine.raise_on_guard(traj)
        tgt = target.contiguous()
        terms = engine.cost_terms(traj.I[0], traj.z[0], traj.v[0], traj.I[-1], tgt, lam, rho)
        ctx.traj = traj
        ctx.target = tgt
        ctx.params = (cfg, float(lam), float(rho))
        return terms[:, 0].clone()

    @staticmethod
    def backward(ctx, grad_out):
        cfg, lam, rho = ctx.params
        bufs = engine.shoot_adjoint(ctx.traj, ctx.target, lam, rho, cfg.mu, cfg.kernel.weights)
        scale = grad_out.to(bufs.zbar.dtype).view((-1,) + (1,) * (bufs.zbar.ndim - 1))
        ctx.traj = None
        return bufs.zbar * scale, None, None, None, None, None


def cost_and_grad_batch(source: torch.Tensor, target: torch.Tensor, z0: torch.Tensor,
                        cfg: ShootingConfig, lam: float, rho: float, raise_on_divergence=True):
    """One grad() per pair of a device batch -> (zbar [B,*shape], terms [B,4] fp64, guard [B,T+1])."""
    _require_sl(cfg)
    B = z0.shape[0]
    shape = tuple(z0.shape[1:])
    traj = engine.allocate_trajectory(B, shape, cfg.n_steps, z0.dtype, z0.device)
    traj.I[0].copy_(source)
    traj.z[0].copy_(z0)
    engine.shoot_forward(traj, cfg.mu, cfg.kernel.weights)
    bufs = engine.shoot_adjoint(traj, target.contiguous(), lam, rho, cfg.mu, cfg.kernel.weights)
    if raise_on_divergence:
        engine.raise_on_guard(traj)
    return bufs.zbar, bufs.terms, traj.guard
