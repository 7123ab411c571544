"""Momentum calibration against the divergence guard.

The configs' nominal per-step back-trace offsets (1 vox for configs 3-4,
3 vox for config 5) can make a metamorphic shoot run away (max|z| > 1e6,
integrator.py:113-118).  As the survey prescribes, each pair's momentum is
scaled down by a fixed geometric sequence until its forward shoot completes
without the guard firing -- and, so the run is not sitting on the edge of a
blow-up, with bounded momentum growth max_t max|z_t| <= GROWTH * max|z_0| --
and the achieved offset is recorded.  The check is
the device forward itself (its guard is parity-tested against the oracle's on
reduced grids); input preparation only, not part of the timed path.
"""

from __future__ import annotations

import numpy as np
import torch

from . import engine

FACTORS = tuple(0.8 ** k for k in range(25))
GROWTH = 10.0


def calibrate_no_divergence(c, dtype=torch.float32, check_fp64: bool = True,
                            scheme: str = "semi-lagrangian"):
    """Scale ``c.z0`` in place, pair by pair, until no shoot diverges.

    Returns the per-pair scale factors (also stored in ``c.manifest``).
    """
    B = c.batch
    w = c.weights()
    scale = np.ones(B)
    dev = torch.device("cuda", torch.cuda.current_device())
    z_base = c.z0.copy()
    dtypes = (dtype, torch.float64) if check_fp64 and dtype != torch.float64 else (dtype,)
    for dt in dtypes:
        traj = engine.allocate_trajectory(B, c.shape, c.n_steps, dt, dev)
        traj.I[0].copy_(torch.as_tensor(c.source, dtype=dt))
        idx = np.zeros(B, dtype=int)  # position in FACTORS per pair
        idx[:] = [FACTORS.index(s) if s in FACTORS else 0 for s in scale]
        while True:
            z = z_base * np.array([FACTORS[i] for i in idx]).reshape((-1,) + (1,) * len(c.shape))
            traj.z[0].copy_(torch.as_tensor(z, dtype=dt))
            engine.shoot_forward(traj, c.mu, w, scheme=scheme)
            bad = engine.diverged_pairs(traj.guard)
            zmax = traj.z.abs().flatten(2).amax(dim=2)  # [T+1, B]
            growth = (zmax.amax(dim=0) / zmax[0].clamp_min(1e-30)).cpu().numpy()
            bad = bad | ~(growth <= GROWTH)
            if not bad.any():
                break
            if np.any(idx[bad] >= len(FACTORS) - 1):
                raise RuntimeError("momentum calibration failed to avoid divergence")
            idx[bad] += 1
        scale = np.array([FACTORS[i] for i in idx])
        del traj
    c.z0 = z_base * scale.reshape((-1,) + (1,) * len(c.shape))
    offset = c.manifest.get("offset_nominal")
    c.manifest["momentum_scale"] = [float(s) for s in scale]
    if offset is not None:
        c.manifest["offset_achieved"] = [float(offset * s) for s in scale]
    torch.cuda.empty_cache()
    return scale
