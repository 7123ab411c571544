"""Small cases for compute-sanitizer (memcheck / racecheck): every kernel family of the
hot path once -- 2D TMA and non-TMA widths, fp32 and fp64, Eulerian / Hybrid schemes,
deterministic scatters, 3D, and the single-step operators."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_08817_b200 import engine  # noqa: E402


def taps(r):
    x = np.arange(-r, r + 1) / (r / 3.0)
    w = np.exp(-0.5 * x * x)
    return w / w.sum()


def run(shape, B, T, r, dtype, mu=0.3, scheme="semi-lagrangian", det=False):
    g = torch.Generator(device="cuda").manual_seed(7)
    traj = engine.allocate_trajectory(B, shape, T, dtype)
    traj.I[0].copy_(torch.rand((B,) + shape, device="cuda", generator=g, dtype=dtype))
    traj.z[0].copy_(0.3 * torch.randn((B,) + shape, device="cuda", generator=g, dtype=dtype))
    J = torch.rand((B,) + shape, device="cuda", generator=g, dtype=dtype)
    w = taps(r)
    engine.shoot_forward(traj, mu, w, scheme=scheme)
    bufs = engine.shoot_adjoint(traj, J, 1e-3, 1.0, mu, w, scheme=scheme, deterministic=det)
    torch.cuda.synchronize()
    print("ok", shape, B, T, r, dtype, scheme, "det" if det else "", float(bufs.terms[0, 0]))


run((40, 56), 2, 3, 5, torch.float32)            # TMA path, fast velocity kernels
run((130, 72), 1, 2, 24, torch.float32)          # several tiles along y, radius 24
run((41, 57), 2, 2, 4, torch.float32)            # width not 16-byte describable: cp.async / generic path
run((24, 32), 1, 2, 3, torch.float64)            # fp64 instantiation
run((40, 56), 1, 2, 3, torch.float32, scheme="eulerian", mu=0.0)
run((40, 56), 1, 2, 3, torch.float32, scheme="hybrid")
run((40, 56), 2, 2, 3, torch.float32, det=True)  # fixed-point scatters
run((12, 20, 24), 2, 2, 3, torch.float32)        # 3D
run((12, 20, 24), 1, 2, 3, torch.float32, det=True)
run((10, 12, 16), 1, 2, 2, torch.float64)
# single-step operators of the boundary
a = torch.rand(2, 33, 48, device="cuda")
engine.smooth(a, taps(4))
engine.smooth(a, taps(4), adjoint=True)
engine.gradient(a)
engine.divergence(torch.rand(2, 2, 33, 48, device="cuda"))
torch.cuda.synchronize()
print("ops ok")
