"""Batched device engine: the reference's shoot / cost / grad over a batch of
independent pairs, on device tensors, through the C-ABI (include/morphreg_sm100.h).

Layouts (SoA, C-contiguous, one CUDA device):
  scalar batch  [B, *shape]          vector batch  [B, d, *shape]
  trajectory    I, z: [T+1, B, *shape];  v: [T+1, B, d, *shape]

This module is the native-backed core the reference-API facade
(``integrator.py`` / ``objective.py`` of this package) and ``bench.py`` call.
Everything numeric happens in libmorphreg_sm100.so; torch only allocates.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import FieldError, IntegrationDiverged

MAGNITUDE_GUARD = 1e6  # integrator.py:36


def _check_field(t: torch.Tensor, shape, what: str):
    if tuple(t.shape) != tuple(shape):
        raise FieldError(f"{what}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
    if not t.is_cuda:
        raise FieldError(f"{what}: expected a CUDA tensor")
    if not t.is_contiguous():
        raise FieldError(f"{what}: expected a contiguous tensor")


@dataclass
class DeviceTrajectory:
    """All T+1 states of a batched shoot (GeodesicTrajectory, integrator.py:72-87)."""

    I: torch.Tensor      # [T+1, B, *shape]
    z: torch.Tensor      # [T+1, B, *shape]
    v: torch.Tensor      # [T+1, B, d, *shape]
    guard: torch.Tensor  # int32 [B, T+1]
    phi: torch.Tensor | None = None  # [B, d, *shape] (first half of a 2x buffer)
    workspace: torch.Tensor | None = None  # forward scratch (3D smoothing)

    @property
    def n_steps(self) -> int:
        return self.I.shape[0] - 1

    @property
    def batch(self) -> int:
        return self.I.shape[1]

    @property
    def shape(self):
        return tuple(self.I.shape[2:])


def allocate_trajectory(batch, shape, n_steps, dtype=torch.float32, device=None,
                        with_phi=False) -> DeviceTrajectory:
    device = device or torch.device("cuda", torch.cuda.current_device())
    d = len(shape)
    I = torch.empty((n_steps + 1, batch) + tuple(shape), dtype=dtype, device=device)
    z = torch.empty_like(I)
    v = torch.empty((n_steps + 1, batch, d) + tuple(shape), dtype=dtype, device=device)
    guard = torch.empty((batch, n_steps + 1), dtype=torch.int32, device=device)
    phi = None
    if with_phi:
        phi = torch.empty((2, batch, d) + tuple(shape), dtype=dtype, device=device)
    lib = _lib.load_library()
    nbytes = lib.mr_forward_workspace_bytes(_lib.dtype_code(dtype), _lib.make_grid(batch, shape))
    ws = None
    if nbytes:
        ws = torch.empty(nbytes // (torch.finfo(dtype).bits // 8), dtype=dtype, device=device)
    return DeviceTrajectory(I, z, v, guard, phi, ws)


def shoot_forward(traj: DeviceTrajectory, mu: float, weights, stream=None,
                  scheme: str = "semi-lagrangian") -> DeviceTrajectory:
    """Run the forward sweep in place; traj.I[0], traj.z[0] hold I0, z0.

    One mr_shoot_forward_scheme call (scheme = a Scheme value) launches the
    whole sweep.  Does not synchronise; call :func:`raise_on_guard` to surface
    divergence.
    """
    lib = _lib.load_library()
    kern = _lib.KernelHandle(weights)
    dt = _lib.dtype_code(traj.I.dtype)
    g = _lib.make_grid(traj.batch, traj.shape)
    rc = lib.mr_shoot_forward_scheme(
        dt, g, kern.struct, _lib.SCHEME_CODES[str(scheme)], float(mu), int(traj.n_steps),
        _lib.ptr(traj.I), _lib.ptr(traj.z),
        _lib.ptr(traj.v), _lib.ptr(traj.phi), _lib.ptr(traj.guard), _lib.ptr(traj.workspace),
        _lib.stream_ptr(stream),
    )
    _lib.check(rc)
    return traj


def guard_report(guard: torch.Tensor):
    """First (pair, step, what) flagged by the device guard, else None (host sync)."""
    g = guard.cpu().numpy()
    nz = np.argwhere(g != 0)
    if nz.size == 0:
        return None
    # first pair with a flag, then its first step; lowest bit = reference order
    b = int(nz[0, 0])
    steps = np.nonzero(g[b])[0]
    k = int(steps[0])
    bits = int(g[b, k])
    for bit, what in _lib.GUARD_BITS:
        if bits & bit:
            return b, k, what
    return b, k, "unknown"


def diverged_pairs(guard: torch.Tensor) -> np.ndarray:
    """Boolean mask [B] of pairs whose shoot tripped the guard (host sync)."""
    return (guard.cpu().numpy() != 0).any(axis=1)


def raise_on_guard(traj: DeviceTrajectory) -> None:
    rep = guard_report(traj.guard)
    if rep is not None:
        _, k, what = rep
        raise IntegrationDiverged(k, what)


class AdjointBuffers:
    """Reusable device buffers of one reverse sweep."""

    def __init__(self, batch, shape, dtype=torch.float32, device=None):
        device = device or torch.device("cuda", torch.cuda.current_device())
        lib = _lib.load_library()
        g = _lib.make_grid(batch, shape)
        nbytes = lib.mr_adjoint_workspace_bytes(_lib.dtype_code(dtype), g)
        if nbytes == 0:
            raise FieldError(lib.mr_last_error().decode())
        esize = torch.finfo(dtype).bits // 8
        self.workspace = torch.empty(nbytes // esize, dtype=dtype, device=device)
        self.zbar = torch.empty((batch,) + tuple(shape), dtype=dtype, device=device)
        self.terms = torch.empty((batch, 4), dtype=torch.float64, device=device)
        self.flags = torch.empty((batch,), dtype=torch.int32, device=device)


def shoot_adjoint(traj: DeviceTrajectory, target: torch.Tensor, lam: float, rho: float, mu: float,
                  weights, bufs: AdjointBuffers | None = None, stream=None,
                  scheme: str = "semi-lagrangian") -> AdjointBuffers:
    """Reverse sweep of grad() (objective.py:91-174) over a forward trajectory.

    Returns the buffers: .zbar = dH/dz0 [B, *shape], .terms = CostReport rows
    {total, data_term, v_norm, z_norm} [B, 4] (fp64), .flags = non-finite flag [B].
    """
    lib = _lib.load_library()
    _check_field(target, (traj.batch,) + traj.shape, "target")
    if bufs is None:
        bufs = AdjointBuffers(traj.batch, traj.shape, traj.I.dtype, traj.I.device)
    kern = _lib.KernelHandle(weights)
    g = _lib.make_grid(traj.batch, traj.shape)
    rc = lib.mr_shoot_adjoint_scheme(
        _lib.dtype_code(traj.I.dtype), g, kern.struct, _lib.SCHEME_CODES[str(scheme)], float(mu),
        int(traj.n_steps), float(lam),
        float(rho), _lib.ptr(traj.I), _lib.ptr(traj.z), _lib.ptr(traj.v), _lib.ptr(target),
        _lib.ptr(bufs.zbar), _lib.ptr(bufs.terms), _lib.ptr(bufs.flags), _lib.ptr(bufs.workspace),
        _lib.stream_ptr(stream),
    )
    _lib.check(rc)
    return bufs


def cost_terms(I0, z0, v0, IT, J, lam, rho, stream=None) -> torch.Tensor:
    """CostReport rows [B, 4] = {total, data, v_norm, z_norm} (objective.py:71-88)."""
    lib = _lib.load_library()
    B = I0.shape[0]
    shape = tuple(I0.shape[1:])
    terms = torch.empty((B, 4), dtype=torch.float64, device=I0.device)
    g = _lib.make_grid(B, shape)
    rc = lib.mr_cost_terms(
        _lib.dtype_code(I0.dtype), g, float(lam), float(rho), _lib.ptr(I0), _lib.ptr(z0),
        _lib.ptr(v0), _lib.ptr(IT), _lib.ptr(J), _lib.ptr(terms), None, _lib.stream_ptr(stream),
    )
    _lib.check(rc)
    return terms


def _split_workspace(I: torch.Tensor, split: bool):
    """2 scalars per pixel of scratch for the split (two-kernel) 2D FIR paths."""
    if not split or I.dim() != 3:
        return None
    return torch.empty((I.shape[0], 2) + tuple(I.shape[1:]), dtype=I.dtype, device=I.device)


def velocity(I: torch.Tensor, z: torch.Tensor, weights, guard=None, stream=None,
             split: bool = True) -> torch.Tensor:
    """v = -K*(z grad I) for a batch [B, *shape] -> [B, d, *shape] (integrator.py:93-94).

    split=True passes a workspace so the fp32 path runs the same two kernels as
    mr_shoot_forward; split=False runs the single-kernel variant."""
    lib = _lib.load_library()
    B = I.shape[0]
    shape = tuple(I.shape[1:])
    _check_field(z, I.shape, "momentum")
    v = torch.empty((B, len(shape)) + shape, dtype=I.dtype, device=I.device)
    kern = _lib.KernelHandle(weights)
    rc = lib.mr_velocity(_lib.dtype_code(I.dtype), _lib.make_grid(B, shape), kern.struct,
                         _lib.ptr(I), _lib.ptr(z), _lib.ptr(v), _lib.ptr(guard),
                         _lib.ptr(_split_workspace(I, split)), _lib.stream_ptr(stream))
    _lib.check(rc)
    return v


def sl_step(I, z, v, dt, mu, phi=None, stream=None):
    """One SL step (integrator.py:193-205) -> (I', z', phi' or None)."""
    lib = _lib.load_library()
    B = I.shape[0]
    shape = tuple(I.shape[1:])
    In = torch.empty_like(I)
    zn = torch.empty_like(z)
    phn = torch.empty_like(phi) if phi is not None else None
    rc = lib.mr_sl_step(_lib.dtype_code(I.dtype), _lib.make_grid(B, shape), float(dt), float(mu),
                        _lib.ptr(I), _lib.ptr(z), _lib.ptr(v), _lib.ptr(In), _lib.ptr(zn),
                        _lib.ptr(phi), _lib.ptr(phn), _lib.stream_ptr(stream))
    _lib.check(rc)
    return In, zn, phn


def sl_step_adjoint(I, z, v, ibar, zbar, dt, mu, stream=None):
    """Adjoint of one SL step -> (ib_acc, zb_acc, vbar) (objective.py:118-147)."""
    lib = _lib.load_library()
    B = I.shape[0]
    shape = tuple(I.shape[1:])
    ib = torch.zeros_like(I)
    zb = torch.zeros_like(I)
    vbar = torch.empty_like(v)
    rc = lib.mr_sl_step_adjoint(_lib.dtype_code(I.dtype), _lib.make_grid(B, shape), float(dt),
                                float(mu), _lib.ptr(I), _lib.ptr(z), _lib.ptr(v), _lib.ptr(ibar),
                                _lib.ptr(zbar), _lib.ptr(ib), _lib.ptr(zb), _lib.ptr(vbar),
                                _lib.stream_ptr(stream))
    _lib.check(rc)
    return ib, zb, vbar


def velocity_adjoint(I, z, vbar, ib, zb, weights, stream=None, split: bool = True):
    """In place: zb += mbar.grad I, ib += G^T(mbar z), mbar = -K^T vbar (objective.py:157-161).

    split as in velocity(): True runs the kernels mr_shoot_adjoint runs."""
    lib = _lib.load_library()
    B = I.shape[0]
    shape = tuple(I.shape[1:])
    kern = _lib.KernelHandle(weights)
    rc = lib.mr_velocity_adjoint(_lib.dtype_code(I.dtype), _lib.make_grid(B, shape), kern.struct,
                                 _lib.ptr(I), _lib.ptr(z), _lib.ptr(vbar), _lib.ptr(ib),
                                 _lib.ptr(zb), _lib.ptr(_split_workspace(I, split)),
                                 _lib.stream_ptr(stream))
    _lib.check(rc)
    return ib, zb


def smooth(a: torch.Tensor, weights, adjoint: bool = False, stream=None) -> torch.Tensor:
    """smooth_arr / smooth_adjoint_arr on a scalar batch [B, *shape] (kernel.py:71-79)."""
    lib = _lib.load_library()
    B = a.shape[0]
    shape = tuple(a.shape[1:])
    out = torch.empty_like(a)
    kern = _lib.KernelHandle(weights)
    rc = lib.mr_smooth(_lib.dtype_code(a.dtype), _lib.make_grid(B, shape), kern.struct,
                       _lib.ptr(a), _lib.ptr(out), int(bool(adjoint)), _lib.stream_ptr(stream))
    _lib.check(rc)
    return out


class BatchGrad:
    """Preallocated forward + adjoint for a fixed (B, shape, T) problem.

    ``run()`` = one grad() per pair: mr_shoot_forward + mr_shoot_adjoint, all
    on device, no host sync.  Inputs live in ``traj.I[0]``, ``traj.z[0]`` and
    ``target``; results in ``bufs.zbar`` / ``bufs.terms``.
    """

    def __init__(self, batch, shape, n_steps, mu, weights, lam, rho, dtype=torch.float32,
                 device=None, scheme: str = "semi-lagrangian"):
        self.scheme = str(scheme)
        self.traj = allocate_trajectory(batch, shape, n_steps, dtype, device)
        self.target = torch.empty((batch,) + tuple(shape), dtype=dtype,
                                  device=self.traj.I.device)
        self.bufs = AdjointBuffers(batch, shape, dtype, self.traj.I.device)
        self.mu, self.lam, self.rho = float(mu), float(lam), float(rho)
        self.weights = np.asarray(weights, dtype=np.float64)
        self.n_steps = n_steps

    def load(self, source, target, z0):
        self.traj.I[0].copy_(source)
        self.traj.z[0].copy_(z0)
        self.target.copy_(target)

    def run(self, stream=None):
        shoot_forward(self.traj, self.mu, self.weights, stream, scheme=self.scheme)
        shoot_adjoint(self.traj, self.target, self.lam, self.rho, self.mu, self.weights,
                      self.bufs, stream, scheme=self.scheme)
        return self.bufs

    def capture_graph(self):
        """Capture one run() (all forward and adjoint launches) in a CUDA graph.

        Buffers and tensor maps are fixed at capture time, so replays read the
        current contents of traj.I[0], traj.z[0] and target.  Warm up first so
        the one-time kernel attribute setup happens outside the capture.
        """
        self.run()
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.run()
        torch.cuda.synchronize()
        return self.graph

    def replay(self):
        self.graph.replay()
        return self.bufs

    def launches_per_run(self) -> int:
        """Kernels of ours per run() (memsets excluded)."""
        T = self.n_steps
        if len(self.traj.shape) == 2:
            H, W = self.traj.shape
            f32 = self.traj.I.dtype == torch.float32 and W % 4 == 0
            # forward: T+1 velocities (2 kernels when split: 64x32 tiles fill the GPU
            # twice, mr_capi.cu shoot_forward) + T steps; adjoint: cost + finalize +
            # T x (transport adjoint + velocity adjoint, 2 kernels when split)
            tiles = ((W + 63) // 64) * ((H + 31) // 32) * self.traj.batch
            vel = 2 if f32 and tiles >= 2 * 148 else 1
            vadj = 2 if f32 else 1
            return (vel * (T + 1) + T) + (2 + (1 + vadj) * T)
        # 3D: velocity = 3 kernels, step 1; adjoint: 2 + (2 + 2 FIR + 1) per step
        return (3 * (T + 1) + T) + (2 + 5 * T)


class GroupedBatchGrad:
    """A batch run as G concurrent pair groups, one stream each (one CUDA graph).

    Pairs are independent, so a grad() of the whole batch is G grad() calls on
    disjoint pair ranges.  Issued on separate streams, the FP32-bound smoothing
    kernels of one group overlap the HBM-bound transport kernels of another
    (measured on B200 at cfg2: 13.82 -> 13.30 ms for G = 2).
    """

    def __init__(self, batch, shape, n_steps, mu, weights, lam, rho, dtype=torch.float32,
                 device=None, scheme: str = "semi-lagrangian", groups: int = 2):
        groups = max(1, min(int(groups), batch))
        bounds = [batch * g // groups for g in range(groups + 1)]
        self.bounds = list(zip(bounds[:-1], bounds[1:]))
        self.parts = [BatchGrad(b1 - b0, shape, n_steps, mu, weights, lam, rho, dtype, device,
                                scheme) for b0, b1 in self.bounds]
        self.streams = [torch.cuda.Stream(device=device) for _ in self.parts]
        self.mu = float(mu)
        self.n_steps = n_steps

    def load(self, source, target, z0):
        for (b0, b1), p in zip(self.bounds, self.parts):
            p.load(source[b0:b1], target[b0:b1], z0[b0:b1])

    def run(self, stream=None):
        main = torch.cuda.current_stream() if stream is None else stream
        for s, p in zip(self.streams, self.parts):
            s.wait_stream(main)
            with torch.cuda.stream(s):
                p.run(stream=s)
        for s in self.streams:
            main.wait_stream(s)

    def capture_graph(self):
        self.run()
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.run()
        torch.cuda.synchronize()
        return self.graph

    def replay(self):
        self.graph.replay()

    @property
    def terms(self) -> torch.Tensor:
        return torch.cat([p.bufs.terms for p in self.parts])

    @property
    def guard(self) -> torch.Tensor:
        return torch.cat([p.traj.guard for p in self.parts])

    @property
    def zbar(self) -> torch.Tensor:
        return torch.cat([p.bufs.zbar for p in self.parts])

    def trajectory_bytes(self) -> int:
        return sum(p.traj.I.numel() * p.traj.I.element_size() * (2 + len(p.traj.shape))
                   for p in self.parts)

    def launches_per_run(self) -> int:
        return sum(p.launches_per_run() for p in self.parts)
