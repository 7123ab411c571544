"""Calibration study (debug aid, GPU): for configs 3-5, how the fp32 device shoot
behaves as the momentum scale grows towards the nominal per-step offset --
guard status, momentum growth max_t|z_t| / |z_0| and the achieved offset, and
fp32-vs-fp64 final-image agreement.  Output: one JSON line per (config, scale)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_08817_b200 import engine  # noqa: E402
from paper_2106_08817_b200.synthetic import make_config  # noqa: E402


def shoot(c, scale, dtype):
    traj = engine.allocate_trajectory(1, c.shape, c.n_steps, dtype)
    traj.I[0].copy_(torch.as_tensor(c.source[:1], dtype=dtype))
    traj.z[0].copy_(torch.as_tensor(c.z0[:1] * scale, dtype=dtype))
    engine.shoot_forward(traj, c.mu, c.weights())
    rep = engine.guard_report(traj.guard)
    zmax = traj.z.abs().flatten(2).amax(dim=2)[:, 0]
    growth = float(zmax.max() / zmax[0].clamp_min(1e-30))
    off = float(traj.v[0].abs().max()) / c.n_steps
    IT = traj.I[-1, 0].double().cpu()
    del traj
    torch.cuda.empty_cache()
    return rep, growth, off, IT


for cfg in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "3,4,5").split(",")]:
    c = make_config(cfg, batch=1)
    mus = [c.mu, 0.0] if cfg == 5 else [c.mu]
    for mu in mus:
        c.mu = mu
        for k in range(0, 16):
            scale = 0.8 ** k
            rep, growth, off, IT32 = shoot(c, scale, torch.float32)
            row = {"config": cfg, "mu": mu, "scale": scale, "guard": rep, "growth": growth,
                   "offset_vox": off}
            if rep is None:
                rep64, g64, _, IT64 = shoot(c, scale, torch.float64)
                row["fp64_guard"] = rep64
                if rep64 is None:
                    row["fp32_vs_fp64_final_image_rel_l2"] = float(
                        (IT32 - IT64).norm() / IT64.norm())
            print(json.dumps(row), flush=True)
            if rep is None and row.get("fp32_vs_fp64_final_image_rel_l2", 1) < 1e-4 and growth < 3:
                break
