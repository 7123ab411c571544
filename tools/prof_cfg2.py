"""Profiling driver: N grad() runs of the cfg-2 batch (for ncu; not a benchmark)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2106_08817_b200 import engine  # noqa: E402
from paper_2106_08817_b200.synthetic import make_config  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", type=int, default=2)
p.add_argument("--batch", type=int, default=None)
p.add_argument("--iters", type=int, default=2)
a = p.parse_args()
c = make_config(a.config, batch=a.batch)
if a.config in (3, 4, 5):  # as bench.py: scale z0 until the shoot stays below the guard
    from paper_2106_08817_b200.calibrate import calibrate_no_divergence

    calibrate_no_divergence(c)
bg = engine.BatchGrad(c.batch, c.shape, c.n_steps, c.mu, c.weights(), c.lam, c.rho)
dt = torch.float32
bg.load(torch.as_tensor(c.source, dtype=dt), torch.as_tensor(c.target, dtype=dt),
        torch.as_tensor(c.z0, dtype=dt))
for _ in range(a.iters):
    bg.run()
torch.cuda.synchronize()
print("ok", c.name, "launches/run", bg.launches_per_run())
