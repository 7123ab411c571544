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
from .integrator import GeodesicTrajectory, ShootingConfig, _to_device

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
    if trajectory is None or trajectory.device is None:
        traj = engine.allocate_trajectory(1, z0.geometry.shape, cfg.n_steps, cfg.dtype)
        traj.I[0, 0].copy_(_to_device(problem.source, cfg.dtype))
        traj.z[0, 0].copy_(_to_device(z0, cfg.dtype))
        engine.shoot_forward(traj, cfg.mu, cfg.kernel.weights, scheme=cfg.scheme.value)
        engine.raise_on_guard(traj)
    else:
        traj = trajectory.device
    J = _to_device(problem.target, traj.I.dtype).unsqueeze(0)
    terms = engine.cost_terms(traj.I[0], traj.z[0], traj.v[0], traj.I[-1], J, problem.lam,
                              problem.rho)
    return _report(terms[0].cpu().numpy())


def _shoot_device(problem: RegistrationProblem, z0: ScalarField) -> engine.DeviceTrajectory:
    """The forward sweep of cost()/grad() on the device (raises IntegrationDiverged)."""
    if z0.geometry != problem.source.geometry:
        raise FieldError("initial momentum geometry mismatch")
    cfg = problem.cfg
    traj = engine.allocate_trajectory(1, z0.geometry.shape, cfg.n_steps, cfg.dtype)
    traj.I[0, 0].copy_(_to_device(problem.source, cfg.dtype))
    traj.z[0, 0].copy_(_to_device(z0, cfg.dtype))
    engine.shoot_forward(traj, cfg.mu, cfg.kernel.weights, scheme=cfg.scheme.value)
    engine.raise_on_guard(traj)
    return traj


def _cost_and_trajectory(problem: RegistrationProblem, z0: ScalarField):
    """cost() that also returns the device trajectory it shot, so a caller that
    needs grad() at the same z0 can skip the forward."""
    traj = _shoot_device(problem, z0)
    J = _to_device(problem.target, traj.I.dtype).unsqueeze(0)
    terms = engine.cost_terms(traj.I[0], traj.z[0], traj.v[0], traj.I[-1], J, problem.lam,
                              problem.rho)
    return _report(terms[0].cpu().numpy()), traj


def grad(problem: RegistrationProblem, z0: ScalarField) -> ScalarField:
    """Gradient of the discrete cost w.r.t. every entry of z0 (objective.py:91-174)."""
    return _grad_on(problem, z0, _shoot_device(problem, z0))


def _grad_on(problem: RegistrationProblem, z0: ScalarField,
             traj: engine.DeviceTrajectory) -> ScalarField:
    """grad() over an existing forward trajectory of z0 (the reverse sweep only).
    The forward is deterministic, so this equals grad(problem, z0) exactly."""
    if z0.geometry != problem.source.geometry:
        raise FieldError("initial momentum geometry mismatch")
    cfg = problem.cfg
    J = _to_device(problem.target, cfg.dtype).unsqueeze(0)
    bufs = engine.shoot_adjoint(traj, J, problem.lam, problem.rho, cfg.mu, cfg.kernel.weights,
                                scheme=cfg.scheme.value, deterministic=cfg.deterministic)
    flag = int(bufs.flags[0].item())
    if flag & 1:  # objective.py:171-173
        bad = torch.nonzero(~torch.isfinite(bufs.zbar[0]))[0].tolist()
        raise FieldError(f"non-finite gradient entry at pixel {tuple(bad)}")
    if flag & 2:
        raise FieldError("deterministic adjoint: contribution outside the fixed-point range "
                         "(non-finite adjoint state)")
    return ScalarField(z0.geometry, bufs.zbar[0], _trusted=True)


class ShootingCost(torch.autograd.Function):
    """Batched cost H(z0) per pair with the explicit adjoint as backward.

    forward(z0 [B,*shape], source [B,*shape], target [B,*shape], cfg, lam, rho)
      -> totals [B] (float64); the full CostReport rows are in ``ctx``-free
      form via :func:`cost_and_grad_batch`.
    """

    @staticmethod
    def forward(ctx, z0, source, target, cfg: ShootingConfig, lam: float, rho: float):
        B = z0.shape[0]
        shape = tuple(z0.shape[1:])
        traj = engine.allocate_trajectory(B, shape, cfg.n_steps, z0.dtype, z0.device)
        traj.I[0].copy_(source)
        traj.z[0].copy_(z0)
        engine.shoot_forward(traj, cfg.mu, cfg.kernel.weights, scheme=cfg.scheme.value)
        engine.raise_on_guard(traj)
        tgt = target.to(device=z0.device, dtype=z0.dtype).contiguous()
        terms = engine.cost_terms(traj.I[0], traj.z[0], traj.v[0], traj.I[-1], tgt, lam, rho)
        ctx.traj = traj
        ctx.target = tgt
        ctx.params = (cfg, float(lam), float(rho))
        return terms[:, 0].clone()

    @staticmethod
    def backward(ctx, grad_out):
        cfg, lam, rho = ctx.params
        bufs = engine.shoot_adjoint(ctx.traj, ctx.target, lam, rho, cfg.mu, cfg.kernel.weights,
                                    scheme=cfg.scheme.value, deterministic=cfg.deterministic)
        scale = grad_out.to(bufs.zbar.dtype).view((-1,) + (1,) * (bufs.zbar.ndim - 1))
        ctx.traj = None
        return bufs.zbar * scale, None, None, None, None, None


def cost_and_grad_batch(source: torch.Tensor, target: torch.Tensor, z0: torch.Tensor,
                        cfg: ShootingConfig, lam: float, rho: float, raise_on_divergence=True,
                        chunks: int | None = None):
    """One grad() per pair of a batch -> (zbar [B,*shape], terms [B,4] fp64, guard [B,T+1]).

    Device tensors in -> device tensors out, stream-ordered on the current stream.
    Host tensors in -> host tensors out: the batch is pipelined in ``chunks``
    groups of pairs (see :func:`_host_pipeline`), so the host<->device copies
    overlap the shooting of the other groups.
    """
    if not z0.is_cuda:
        return _host_pipeline(source, target, z0, cfg, lam, rho, raise_on_divergence, chunks)
    B = z0.shape[0]
    shape = tuple(z0.shape[1:])
    traj = engine.allocate_trajectory(B, shape, cfg.n_steps, z0.dtype, z0.device)
    traj.I[0].copy_(source)
    traj.z[0].copy_(z0)
    engine.shoot_forward(traj, cfg.mu, cfg.kernel.weights, scheme=cfg.scheme.value)
    tgt = target.to(device=z0.device, dtype=z0.dtype).contiguous()
    bufs = engine.shoot_adjoint(traj, tgt, lam, rho, cfg.mu, cfg.kernel.weights,
                                scheme=cfg.scheme.value, deterministic=cfg.deterministic)
    if raise_on_divergence:
        engine.raise_on_guard(traj)
    return bufs.zbar, bufs.terms, traj.guard


_PIPE_STREAMS: dict = {}


def _pipe_streams(device, n: int):
    """Persistent streams of the host pipeline (one upload stream + n pair groups), so
    the caching allocator reuses each group's trajectory across calls."""
    key = (device.index, n)
    if key not in _PIPE_STREAMS:
        _PIPE_STREAMS[key] = (torch.cuda.Stream(device), [torch.cuda.Stream(device) for _ in range(n)])
    return _PIPE_STREAMS[key]


def _host_pipeline(source, target, z0, cfg, lam, rho, raise_on_divergence, chunks):
    """Host-buffer grad() of a batch with the PCIe transfers hidden behind compute.

    The pairs are split into ``chunks`` groups, each with its own trajectory and
    stream.  One upload stream copies every group's (I0, z0) first, then every
    group's target J (needed only by the adjoint, after the forward sweep).  Group
    g's forward waits for its (I0, z0) event, its adjoint for its J event, and its
    dH/dz0, cost rows and guard go back to pinned host memory on its own stream
    while the other groups still compute.  The groups' kernels run concurrently,
    so the device sees the whole batch; per pair the result is the same as a
    device-tensor call.
    """
    B = z0.shape[0]
    shape = tuple(z0.shape[1:])
    if tuple(source.shape) != tuple(z0.shape) or tuple(target.shape) != tuple(z0.shape):
        raise FieldError("source/target/z0 batch shapes differ")
    if chunks is None:
        chunks = 4 if B >= 16 else (2 if B >= 2 else 1)
    if isinstance(chunks, (list, tuple)):  # explicit group sizes (sum = B)
        sizes = [int(n) for n in chunks]
        if sum(sizes) != B or min(sizes) < 1:
            raise FieldError(f"chunk sizes {sizes} do not partition the batch of {B}")
    else:
        chunks = max(1, min(int(chunks), B))
        sizes = [B * (g + 1) // chunks - B * g // chunks for g in range(chunks)]
    chunks = len(sizes)
    dtype = cfg.dtype if z0.dtype not in (torch.float32, torch.float64) else z0.dtype
    device = torch.device("cuda", torch.cuda.current_device())

    def pinned(t):
        t = t.to(dtype).contiguous()
        return t if t.is_pinned() else t.pin_memory()

    src_h, tgt_h, z0_h = pinned(source), pinned(target), pinned(z0)
    zbar_h = torch.empty((B,) + shape, dtype=dtype, pin_memory=True)
    terms_h = torch.empty((B, 4), dtype=torch.float64, pin_memory=True)
    guard_h = torch.empty((B, cfg.n_steps + 1), dtype=torch.int32, pin_memory=True)
    up, streams = _pipe_streams(device, chunks)
    up.wait_stream(torch.cuda.current_stream(device))
    edges = [0]
    for n in sizes:
        edges.append(edges[-1] + n)
    bounds = list(zip(edges[:-1], edges[1:]))

    trajs, tgts, ev_in, ev_J = [], [], [], []
    for g, (a, b) in enumerate(bounds):
        with torch.cuda.stream(streams[g]):
            trajs.append(engine.allocate_trajectory(b - a, shape, cfg.n_steps, dtype, device))
            tgts.append(torch.empty((b - a,) + shape, dtype=dtype, device=device))
    with torch.cuda.stream(up):
        for g, (a, b) in enumerate(bounds):
            trajs[g].I[0].copy_(src_h[a:b], non_blocking=True)
            trajs[g].z[0].copy_(z0_h[a:b], non_blocking=True)
            ev_in.append(up.record_event())
        for g, (a, b) in enumerate(bounds):
            tgts[g].copy_(tgt_h[a:b], non_blocking=True)
            ev_J.append(up.record_event())
    w = cfg.kernel.weights
    keep = []
    for g, (a, b) in enumerate(bounds):
        s = streams[g]
        with torch.cuda.stream(s):  # every allocation and launch of group g is on s
            s.wait_event(ev_in[g])
            engine.shoot_forward(trajs[g], cfg.mu, w, stream=s, scheme=cfg.scheme.value)
            s.wait_event(ev_J[g])
            bufs = engine.shoot_adjoint(trajs[g], tgts[g], lam, rho, cfg.mu, w, stream=s,
                                        scheme=cfg.scheme.value,
                                        deterministic=cfg.deterministic)
            keep.append(bufs)
            zbar_h[a:b].copy_(bufs.zbar, non_blocking=True)
            terms_h[a:b].copy_(bufs.terms, non_blocking=True)
            guard_h[a:b].copy_(trajs[g].guard, non_blocking=True)
            # the upload stream wrote into this group's buffers
            for t in (trajs[g].I, trajs[g].z, tgts[g]):
                t.record_stream(up)
    for s in streams:
        s.synchronize()
    if raise_on_divergence:
        rep = engine.guard_report(guard_h)
        if rep is not None:
            from .errors import IntegrationDiverged

            raise IntegrationDiverged(rep[1], rep[2])
    return zbar_h, terms_h, guard_h
