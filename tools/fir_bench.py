"""Microbenchmark (builder aid, not a bench value): mr_velocity / mr_velocity_adjoint at the
cfg2 group size (32 x 512^2, R = 24), rotating over buffer sets larger than L2."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_08817_b200 import _lib  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--batch", type=int, default=32)
p.add_argument("--size", type=int, default=512)
p.add_argument("--radius", type=int, default=24)
p.add_argument("--iters", type=int, default=20)
p.add_argument("--sets", type=int, default=4)
p.add_argument("--only", default="both")
a = p.parse_args()
lib = _lib.load_library()
B, H, W, R = a.batch, a.size, a.size, a.radius
x = np.arange(-R, R + 1) / (R / 4.0)
w = np.exp(-0.5 * x * x)
w /= w.sum()
kern = _lib.KernelHandle(w)
g = _lib.make_grid(B, (H, W))
dev = "cuda"
sets = []
for s in range(a.sets):
    sets.append(dict(I=torch.rand(B, H, W, device=dev), z=torch.randn(B, H, W, device=dev),
                     v=torch.empty(B, 2, H, W, device=dev), vbar=torch.randn(B, 2, H, W, device=dev),
                     ib=torch.randn(B, H, W, device=dev), zb=torch.randn(B, H, W, device=dev)))
ws = torch.empty(B, 2, H, W, device=dev)
st = _lib.stream_ptr(None)
code = _lib.dtype_code(torch.float32)


def vel(s):
    _lib.check(lib.mr_velocity(code, g, kern.struct, _lib.ptr(s["I"]), _lib.ptr(s["z"]),
                               _lib.ptr(s["v"]), None, _lib.ptr(ws), st))


def adj(s):
    _lib.check(lib.mr_velocity_adjoint(code, g, kern.struct, _lib.ptr(s["I"]), _lib.ptr(s["z"]),
                                       _lib.ptr(s["vbar"]), _lib.ptr(s["ib"]), _lib.ptr(s["zb"]),
                                       _lib.ptr(ws), st))


for name, fn in (("velocity", vel), ("velocity_adjoint", adj)):
    if a.only not in ("both", name[:3], name):
        continue
    for s in sets:
        fn(s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(a.iters):
        fn(sets[i % a.sets])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.iters
    fl = 2.0 * 2 * 2 * (2 * R + 1) * B * H * W
    print(f"{name}: {ms * 1e3:.1f} us  ({fl / ms / 1e9:.1f} TFLOP/s FIR)")
