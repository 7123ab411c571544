"""Debug aid: velocity / velocity adjoint fast path vs the classic kernels on one shape."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2106_08817_b200 import engine
B, H, W, R = [int(x) for x in sys.argv[1:5]]
x = np.arange(-R, R + 1) / max(R / 3.0, 1e-9)
w = np.exp(-0.5 * x * x); w /= w.sum()
g = torch.Generator(device="cuda").manual_seed(1)
I = torch.rand(B, H, W, device="cuda", generator=g); z = torch.randn(B, H, W, device="cuda", generator=g)
vbar = torch.randn(B, 2, H, W, device="cuda", generator=g)
ib0 = torch.randn(B, H, W, device="cuda", generator=g); zb0 = torch.randn(B, H, W, device="cuda", generator=g)
def rel(a, b): return float((a.double() - b.double()).norm() / b.double().norm())
which = sys.argv[5] if len(sys.argv) > 5 else "both"
if which in ("both", "vel"):
    v1 = engine.velocity(I, z, w, split=True); torch.cuda.synchronize(); print("vel fast ok")
    v0 = engine.velocity(I.double(), z.double(), w, split=False); torch.cuda.synchronize()
    print("velocity rel", rel(v1, v0))
if which in ("both", "adj"):
    ib1, zb1 = engine.velocity_adjoint(I, z, vbar, ib0.clone(), zb0.clone(), w, split=True); torch.cuda.synchronize(); print("adj fast ok")
    ib2, zb2 = engine.velocity_adjoint(I.double(), z.double(), vbar.double(), ib0.double(), zb0.double(), w, split=False); torch.cuda.synchronize()
    print("veladj ib rel", rel(ib1, ib2), "zb rel", rel(zb1, zb2))
