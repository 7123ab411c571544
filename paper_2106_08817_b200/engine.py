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


def _check_field(t: torch.Tensor, shape, what: str, like: torch.Tensor | None = None):
    """Shape, CUDA, contiguity and -- against `like` -- dtype and device: the
    kernels read raw pointers, so a float64 operand next to float32 ones (or a
    tensor on another GPU) would otherwise be misread silently."""
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise FieldError(f"{what}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
    if not t.is_cuda:
        raise FieldError(f"{what}: expected a CUDA tensor")
    if not t.is_contiguous():
        raise FieldError(f"{what}: expected a contiguous tensor")
    if like is not None and (t.dtype != like.dtype or t.device != like.device):
        raise FieldError(f"{what}: expected {like.dtype} on {like.device}, got {t.dtype} on {t.device}")


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
    with torch.cuda.device(traj.I.device):
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
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=device)
        self.zbar = torch.empty((batch,) + tuple(shape), dtype=dtype, device=device)
        self.terms = torch.empty((batch, 4), dtype=torch.float64, device=device)
        self.flags = torch.empty((batch,), dtype=torch.int32, device=device)


def shoot_adjoint(traj: DeviceTrajectory, target: torch.Tensor, lam: float, rho: float, mu: float,
                  weights, bufs: AdjointBuffers | None = None, stream=None,
                  scheme: str = "semi-lagrangian", deterministic: bool = False) -> AdjointBuffers:
    """Reverse sweep of grad() (objective.py:91-174) over a forward trajectory.

    Returns the buffers: .zbar = dH/dz0 [B, *shape], .terms = CostReport rows
    {total, data_term, v_norm, z_norm} [B, 4] (fp64), .flags [B] (bit 0: non-finite
    gradient entry; bit 1: deterministic-mode fixed-point range exceeded).
    ``deterministic`` selects MR_OPT_DETERMINISTIC: fixed-point scatters, so
    repeated calls give bitwise-identical results (optimizer.py:5-7).
    """
    lib = _lib.load_library()
    _check_field(target, (traj.batch,) + traj.shape, "target", like=traj.I)
    if bufs is None:
        bufs = AdjointBuffers(traj.batch, traj.shape, traj.I.dtype, traj.I.device)
    kern = _lib.KernelHandle(weights)
    g = _lib.make_grid(traj.batch, traj.shape)
    with torch.cuda.device(traj.I.device):
        rc = lib.mr_shoot_adjoint_ex(
            _lib.dtype_code(traj.I.dtype), g, kern.struct, _lib.SCHEME_CODES[str(scheme)],
            float(mu), int(traj.n_steps), float(lam),
            float(rho), _lib.ptr(traj.I), _lib.ptr(traj.z), _lib.ptr(traj.v), _lib.ptr(target),
            _lib.ptr(bufs.zbar), _lib.ptr(bufs.terms), _lib.ptr(bufs.flags),
            _lib.ptr(bufs.workspace), _lib.MR_OPT_DETERMINISTIC if deterministic else 0,
            _lib.stream_ptr(stream),
        )
    _lib.check(rc)
    return bufs


def cost_terms(I0, z0, v0, IT, J, lam, rho, stream=None) -> torch.Tensor:
    """CostReport rows [B, 4] = {total, data, v_norm, z_norm} (objective.py:71-88)."""
    lib = _lib.load_library()
    B = I0.shape[0]
    shape = tuple(I0.shape[1:])
    _check_field(I0, None, "I0")
    for t, what in ((z0, "z0"), (IT, "I_T"), (J, "target")):
        _check_field(t, I0.shape, what, like=I0)
    _check_field(v0, (B, len(shape)) + shape, "v0", like=I0)
    terms = torch.empty((B, 4), dtype=torch.float64, device=I0.device)
    g = _lib.make_grid(B, shape)
    code = _lib.dtype_code(I0.dtype)
    part = torch.empty((lib.mr_cost_workspace_bytes(code, g) // 8,), dtype=torch.float64,
                       device=I0.device)
    with torch.cuda.device(I0.device):
        rc = lib.mr_cost_terms(
            code, g, float(lam), float(rho), _lib.ptr(I0), _lib.ptr(z0),
            _lib.ptr(v0), _lib.ptr(IT), _lib.ptr(J), _lib.ptr(terms), None, _lib.ptr(part),
            _lib.stream_ptr(stream),
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
    _check_field(I, None, "image")
    _check_field(z, I.shape, "momentum", like=I)
    v = torch.empty((B, len(shape)) + shape, dtype=I.dtype, device=I.device)
    kern = _lib.KernelHandle(weights)
    with torch.cuda.device(I.device):
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
    _check_field(I, None, "image")
    _check_field(z, I.shape, "momentum", like=I)
    _check_field(v, (B, len(shape)) + shape, "velocity", like=I)
    if phi is not None:
        _check_field(phi, (B, len(shape)) + shape, "phi", like=I)
    In = torch.empty_like(I)
    zn = torch.empty_like(z)
    phn = torch.empty_like(phi) if phi is not None else None
    with torch.cuda.device(I.device):
        rc = lib.mr_sl_step(_lib.dtype_code(I.dtype), _lib.make_grid(B, shape), float(dt),
                            float(mu), _lib.ptr(I), _lib.ptr(z), _lib.ptr(v), _lib.ptr(In),
                            _lib.ptr(zn), _lib.ptr(phi), _lib.ptr(phn), _lib.stream_ptr(stream))
    _lib.check(rc)
    return In, zn, phn


def sl_step_adjoint(I, z, v, ibar, zbar, dt, mu, stream=None):
    """Adjoint of one SL step -> (ib_acc, zb_acc, vbar) (objective.py:118-147)."""
    lib = _lib.load_library()
    B = I.shape[0]
    shape = tuple(I.shape[1:])
    _check_field(I, None, "image")
    for t, what in ((z, "momentum"), (ibar, "ibar"), (zbar, "zbar")):
        _check_field(t, I.shape, what, like=I)
    _check_field(v, (B, len(shape)) + shape, "velocity", like=I)
    ib = torch.zeros_like(I)
    zb = torch.zeros_like(I)
    vbar = torch.empty_like(v)
    with torch.cuda.device(I.device):
        rc = lib.mr_sl_step_adjoint(_lib.dtype_code(I.dtype), _lib.make_grid(B, shape),
                                    float(dt), float(mu), _lib.ptr(I), _lib.ptr(z), _lib.ptr(v),
                                    _lib.ptr(ibar), _lib.ptr(zbar), _lib.ptr(ib), _lib.ptr(zb),
                                    _lib.ptr(vbar), _lib.stream_ptr(stream))
    _lib.check(rc)
    return ib, zb, vbar


def velocity_adjoint(I, z, vbar, ib, zb, weights, stream=None, split: bool = True):
    """In place: zb += mbar.grad I, ib += G^T(mbar z), mbar = -K^T vbar (objective.py:157-161).

    split as in velocity(): True runs the kernels mr_shoot_adjoint runs."""
    lib = _lib.load_library()
    B = I.shape[0]
    shape = tuple(I.shape[1:])
    _check_field(I, None, "image")
    for t, what in ((z, "momentum"), (ib, "ib"), (zb, "zb")):
        _check_field(t, I.shape, what, like=I)
    _check_field(vbar, (B, len(shape)) + shape, "vbar", like=I)
    kern = _lib.KernelHandle(weights)
    with torch.cuda.device(I.device):
        rc = lib.mr_velocity_adjoint(_lib.dtype_code(I.dtype), _lib.make_grid(B, shape),
                                     kern.struct, _lib.ptr(I), _lib.ptr(z), _lib.ptr(vbar),
                                     _lib.ptr(ib), _lib.ptr(zb),
                                     _lib.ptr(_split_workspace(I, split)), _lib.stream_ptr(stream))
    _lib.check(rc)
    return ib, zb


def smooth(a: torch.Tensor, weights, adjoint: bool = False, stream=None) -> torch.Tensor:
    """smooth_arr / smooth_adjoint_arr on a scalar batch [B, *shape] (kernel.py:71-79)."""
    lib = _lib.load_library()
    B = a.shape[0]
    shape = tuple(a.shape[1:])
    _check_field(a, None, "field")
    out = torch.empty_like(a)
    kern = _lib.KernelHandle(weights)
    with torch.cuda.device(a.device):
        rc = lib.mr_smooth(_lib.dtype_code(a.dtype), _lib.make_grid(B, shape), kern.struct,
                           _lib.ptr(a), _lib.ptr(out), int(bool(adjoint)),
                           _lib.stream_ptr(stream))
    _lib.check(rc)
    return out


class BatchGrad:
    """Preallocated forward + adjoint for a fixed (B, shape, T) problem.

    ``run()`` = one grad() per pair: mr_shoot_forward + mr_shoot_adjoint, all
    on device, no host sync.  Inputs live in ``traj.I[0]``, ``traj.z[0]`` and
    ``target``; results in ``bufs.zbar`` / ``bufs.terms``.
    """

    def __init__(self, batch, shape, n_steps, mu, weights, lam, rho, dtype=torch.float32,
                 device=None, scheme: str = "semi-lagrangian", deterministic: bool = False):
        self.scheme = str(scheme)
        self.deterministic = bool(deterministic)
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
                      self.bufs, stream, scheme=self.scheme, deterministic=self.deterministic)
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
                 device=None, scheme: str = "semi-lagrangian", groups: int = 2,
                 deterministic: bool = False):
        groups = max(1, min(int(groups), batch))
        bounds = [batch * g // groups for g in range(groups + 1)]
        self.bounds = list(zip(bounds[:-1], bounds[1:]))
        self.parts = [BatchGrad(b1 - b0, shape, n_steps, mu, weights, lam, rho, dtype, device,
                                scheme, deterministic) for b0, b1 in self.bounds]
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


# ---- array-level operators (mr_ops.cu; fields.py:144-262, kernel.py:36-68) ----------
# Scalar batch [B, *shape], vector batch [B, d, *shape]; any device / dtype the
# library supports; results on the same device and dtype.


def _grid_of(a: torch.Tensor, vector: bool = False, allow_1d: bool = False):
    shape = tuple(a.shape[2:]) if vector else tuple(a.shape[1:])
    if len(shape) not in ((1, 2, 3) if allow_1d else (2, 3)):
        raise FieldError(f"expected a {'1d, ' if allow_1d else ''}2d or 3d grid, got shape {shape}")
    if vector and a.shape[1] != len(shape):
        raise FieldError(f"vector batch needs {len(shape)} components, got {a.shape[1]}")
    return _lib.make_grid(a.shape[0], shape), shape


def _prep(*ts):
    """Check every operand is a contiguous CUDA tensor of one dtype and device."""
    ref = ts[0]
    for t in ts:
        if not t.is_cuda:
            raise FieldError("expected CUDA tensors")
        if t.dtype != ref.dtype or t.device != ref.device:
            raise FieldError(f"operand mismatch: {t.dtype}@{t.device} vs {ref.dtype}@{ref.device}")
        if not t.is_contiguous():
            raise FieldError("expected contiguous tensors")
    return _lib.dtype_code(ref.dtype)


def axis_diff(a: torch.Tensor, axis: int, adjoint: bool = False, stream=None) -> torch.Tensor:
    """np.gradient along grid axis `axis` (fields.py:144-145) or its exact
    transpose (axis_diff_adjoint, fields.py:148-158)."""
    lib = _lib.load_library()
    dt = _prep(a)
    g, _ = _grid_of(a, allow_1d=True)
    out = torch.empty_like(a)
    with torch.cuda.device(a.device):
        _lib.check(lib.mr_axis_diff(dt, g, int(axis), _lib.ptr(a), _lib.ptr(out),
                                    int(bool(adjoint)), _lib.stream_ptr(stream)))
    return out


def gradient(f: torch.Tensor, stream=None) -> torch.Tensor:
    """gradient_arr (fields.py:161-162): [B, *shape] -> [B, d, *shape]."""
    lib = _lib.load_library()
    dt = _prep(f)
    g, shape = _grid_of(f)
    out = torch.empty((f.shape[0], len(shape)) + shape, dtype=f.dtype, device=f.device)
    with torch.cuda.device(f.device):
        _lib.check(lib.mr_gradient(dt, g, _lib.ptr(f), _lib.ptr(out), 0, _lib.stream_ptr(stream)))
    return out


def gradient_adjoint(gbar: torch.Tensor, stream=None) -> torch.Tensor:
    """gradient_adjoint_arr (fields.py:165-166): [B, d, *shape] -> [B, *shape]."""
    lib = _lib.load_library()
    dt = _prep(gbar)
    g, shape = _grid_of(gbar, vector=True)
    out = torch.empty((gbar.shape[0],) + shape, dtype=gbar.dtype, device=gbar.device)
    with torch.cuda.device(gbar.device):
        _lib.check(lib.mr_gradient(dt, g, _lib.ptr(gbar), _lib.ptr(out), 1,
                                   _lib.stream_ptr(stream)))
    return out


def divergence(v: torch.Tensor, stream=None) -> torch.Tensor:
    """divergence_arr (fields.py:169-170): [B, d, *shape] -> [B, *shape]."""
    lib = _lib.load_library()
    dt = _prep(v)
    g, shape = _grid_of(v, vector=True)
    out = torch.empty((v.shape[0],) + shape, dtype=v.dtype, device=v.device)
    with torch.cuda.device(v.device):
        _lib.check(lib.mr_divergence(dt, g, _lib.ptr(v), _lib.ptr(out), _lib.stream_ptr(stream)))
    return out


def conv1d(a: torch.Tensor, weights, axis: int, adjoint: bool = False, stream=None) -> torch.Tensor:
    """conv1d_replicate (kernel.py:36-45) along grid axis `axis`, or its exact
    transpose conv1d_replicate_adjoint (kernel.py:48-68)."""
    lib = _lib.load_library()
    dt = _prep(a)
    g, _ = _grid_of(a, allow_1d=True)
    kern = _lib.KernelHandle(weights)
    out = torch.empty_like(a)
    with torch.cuda.device(a.device):
        _lib.check(lib.mr_conv1d(dt, g, kern.struct, int(axis), _lib.ptr(a), _lib.ptr(out),
                                 int(bool(adjoint)), _lib.stream_ptr(stream)))
    return out


def _bad_flag(device):
    return torch.zeros((1,), dtype=torch.int32, device=device)


def _raise_bad(bad):
    if int(bad.item()) != 0:
        raise FieldError("sample coordinates contain non-finite values")  # fields.py:208-209


def interpolate(coords: torch.Tensor, a: torch.Tensor, stream=None) -> torch.Tensor:
    """bilinear_plan + bilinear_apply (fields.py:207-240; trilinear in 3D) of a
    [B, C, *shape] at absolute coordinates [B, d, *shape] -> [B, C, *shape]."""
    lib = _lib.load_library()
    dt = _prep(coords, a)
    g, shape = _grid_of(coords, vector=True)
    if tuple(a.shape[2:]) != shape or a.shape[0] != coords.shape[0]:
        raise FieldError("interpolated array and sample grid shapes differ")
    out = torch.empty_like(a)
    bad = _bad_flag(a.device)
    with torch.cuda.device(a.device):
        _lib.check(lib.mr_interpolate(dt, g, _lib.ptr(coords), _lib.ptr(a), _lib.ptr(out),
                                      int(a.shape[1]), _lib.ptr(bad), _lib.stream_ptr(stream)))
    _raise_bad(bad)
    return out


def interpolate_adjoint(coords: torch.Tensor, gbar: torch.Tensor, stream=None) -> torch.Tensor:
    """bilinear_adjoint_values (fields.py:243-254): [B, *shape] -> [B, *shape]."""
    lib = _lib.load_library()
    dt = _prep(coords, gbar)
    g, shape = _grid_of(coords, vector=True)
    out = torch.empty_like(gbar)
    bad = _bad_flag(gbar.device)
    with torch.cuda.device(gbar.device):
        _lib.check(lib.mr_interpolate_adjoint(dt, g, _lib.ptr(coords), _lib.ptr(gbar),
                                              _lib.ptr(out), _lib.ptr(bad),
                                              _lib.stream_ptr(stream)))
    _raise_bad(bad)
    return out


def interpolate_coord_grad(coords: torch.Tensor, a: torch.Tensor, stream=None) -> torch.Tensor:
    """bilinear_coord_grad (fields.py:257-262): [B, *shape] -> [B, d, *shape]."""
    lib = _lib.load_library()
    dt = _prep(coords, a)
    g, shape = _grid_of(coords, vector=True)
    out = torch.empty_like(coords)
    bad = _bad_flag(a.device)
    with torch.cuda.device(a.device):
        _lib.check(lib.mr_interpolate_coord_grad(dt, g, _lib.ptr(coords), _lib.ptr(a),
                                                 _lib.ptr(out), _lib.ptr(bad),
                                                 _lib.stream_ptr(stream)))
    _raise_bad(bad)
    return out


def scheme_step(I, z, v, dt, mu, scheme: str = "semi-lagrangian", phi=None, stream=None):
    """One transport step of any scheme with an explicit dt -> (I', z', phi' or None)
    (advect_image_* / continuity_*, integrator.py:133-159)."""
    lib = _lib.load_library()
    code = _prep(I, z, v)
    g, shape = _grid_of(I)
    In = torch.empty_like(I)
    zn = torch.empty_like(z)
    phn = torch.empty_like(phi) if phi is not None else None
    with torch.cuda.device(I.device):
        _lib.check(lib.mr_scheme_step(code, g, _lib.SCHEME_CODES[str(scheme)], float(dt),
                                      float(mu), _lib.ptr(I), _lib.ptr(z), _lib.ptr(v),
                                      _lib.ptr(In), _lib.ptr(zn), _lib.ptr(phi), _lib.ptr(phn),
                                      _lib.stream_ptr(stream)))
    return In, zn, phn


REDUCE_DOT, REDUCE_SSD, REDUCE_SUMSQ = 0, 1, 2


def reduce(a: torch.Tensor, b: torch.Tensor | None, op: int, stream=None) -> torch.Tensor:
    """Per-pair dot / ssd / sum of squares (fields.py:285-295) -> float64 [B]."""
    lib = _lib.load_library()
    code = _prep(a) if b is None else _prep(a, b)
    g, _ = _grid_of(a, allow_1d=True)
    out = torch.empty((a.shape[0],), dtype=torch.float64, device=a.device)
    with torch.cuda.device(a.device):
        _lib.check(lib.mr_reduce(code, g, int(op), _lib.ptr(a), _lib.ptr(b), _lib.ptr(out),
                                 _lib.stream_ptr(stream)))
    return out
