"""Run each kernel once in isolation with a sync after it (debug aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2106_08817_b200 import engine
w = np.exp(-0.5 * (np.arange(-4, 5) / 1.0) ** 2); w /= w.sum()
for shape in [(16, 16), (64, 64), (13, 21)]:
    for dt in (torch.float32, torch.float64):
        I = torch.rand((2,) + shape, dtype=dt, device="cuda")
        z = torch.rand((2,) + shape, dtype=dt, device="cuda")
        try:
            v = engine.velocity(I, z, w); torch.cuda.synchronize(); print(shape, dt, "velocity ok", flush=True)
            ib = torch.zeros_like(I); zb = torch.zeros_like(I)
            engine.velocity_adjoint(I, z, v, ib, zb, w); torch.cuda.synchronize(); print(shape, dt, "veladj ok", flush=True)
        except Exception as e:
            print(shape, dt, "FAIL", e, flush=True); raise
