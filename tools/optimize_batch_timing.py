"""Iteration time of the batched line search (optimize_batch) on a BASELINE config:
B independent Armijo descents as batched device sweeps."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2106_08817_b200 as mr  # noqa: E402
from paper_2106_08817_b200.synthetic import make_config  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", type=int, default=2)
p.add_argument("--batch", type=int, default=None)
p.add_argument("--iters", type=int, default=3)
p.add_argument("--init-step", type=float, default=1.0)
a = p.parse_args()
c = make_config(a.config, batch=a.batch)
cfg = mr.ShootingConfig(mr.Scheme.SEMI_LAGRANGIAN, c.n_steps, c.mu, mr.GaussianKernel(c.sigma, c.radius),
                        deterministic=False)
src = torch.as_tensor(c.source, dtype=torch.float32).cuda()
tgt = torch.as_tensor(c.target, dtype=torch.float32).cuda()
z0 = torch.zeros_like(src)  # default_init: zero momentum
ocfg = mr.OptimizeConfig(max_iters=a.iters, init_step=a.init_step)
mr.optimize_batch(src, tgt, z0, cfg, c.lam, c.rho, mr.OptimizeConfig(max_iters=1, init_step=a.init_step))
torch.cuda.synchronize()
t0 = time.perf_counter()
res = mr.optimize_batch(src, tgt, z0, cfg, c.lam, c.rho, ocfg)
torch.cuda.synchronize()
sec = time.perf_counter() - t0
nit = max(len(h) - 1 for h in res.histories)
first = np.array([h[0].total for h in res.histories])
last = np.array([h[-1].total for h in res.histories])
print(json.dumps({
    "workload": c.name, "pairs": int(src.shape[0]), "outer_iterations": nit,
    "forward_rounds": res.rounds, "pair_shoots": res.pair_shoots, "grad_sweeps": res.grad_sweeps,
    "seconds": sec, "ms_per_outer_iteration": 1e3 * sec / max(nit, 1),
    "ms_per_round": 1e3 * sec / (res.rounds + res.grad_sweeps),
    "mean_cost_first": float(first.mean()), "mean_cost_last": float(last.mean()),
    "terminations": sorted({t.value for t in res.terminations}),
}))
