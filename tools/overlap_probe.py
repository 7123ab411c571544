"""Probe (builder aid): do an FP32-bound FIR operation and an HBM-bound transport
operation overlap when issued on two streams?  t(A), t(B), t(A || B) at the cfg2 group size."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_08817_b200 import _lib  # noqa: E402

lib = _lib.load_library()
B, H, W, R = 32, 512, 512, 24
x = np.arange(-R, R + 1) / 6.0
w = np.exp(-0.5 * x * x)
w /= w.sum()
kern = _lib.KernelHandle(w)
g = _lib.make_grid(B, (H, W))
code = _lib.dtype_code(torch.float32)
P = _lib.ptr


def bufs():
    return dict(I=torch.rand(B, H, W, device="cuda"), z=torch.randn(B, H, W, device="cuda"),
                v=torch.randn(B, 2, H, W, device="cuda"), vout=torch.empty(B, 2, H, W, device="cuda"),
                ib=torch.randn(B, H, W, device="cuda"), zb=torch.randn(B, H, W, device="cuda"),
                a1=torch.zeros(B, H, W, device="cuda"), a2=torch.zeros(B, H, W, device="cuda"),
                vbar=torch.empty(B, 2, H, W, device="cuda"), ws=torch.empty(B, 2, H, W, device="cuda"),
                In=torch.empty(B, H, W, device="cuda"), zn=torch.empty(B, H, W, device="cuda"))


X, Y = bufs(), bufs()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def vel(d, s):
    _lib.check(lib.mr_velocity(code, g, kern.struct, P(d["I"]), P(d["z"]), P(d["vout"]), None, P(d["ws"]),
                               _lib.stream_ptr(s)))


def vadj(d, s):
    _lib.check(lib.mr_velocity_adjoint(code, g, kern.struct, P(d["I"]), P(d["z"]), P(d["v"]), P(d["ib"]),
                                       P(d["zb"]), P(d["ws"]), _lib.stream_ptr(s)))


def step(d, s):
    _lib.check(lib.mr_sl_step(code, g, 0.05, 0.0, P(d["I"]), P(d["z"]), P(d["v"]), P(d["In"]), P(d["zn"]),
                              None, None, _lib.stream_ptr(s)))


def sadj(d, s):
    _lib.check(lib.mr_sl_step_adjoint(code, g, 0.05, 0.0, P(d["I"]), P(d["z"]), P(d["v"]), P(d["ib"]),
                                      P(d["zb"]), P(d["a1"]), P(d["a2"]), P(d["vbar"]), _lib.stream_ptr(s)))


def timeit(fa, fb, n=20):
    for _ in range(3):
        if fa: fa(X, s1)
        if fb: fb(Y, s2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s1.wait_event(e0)
    s2.wait_event(e0)
    for _ in range(n):
        if fa: fa(X, s1)
        if fb: fb(Y, s2)
    cur = torch.cuda.current_stream()
    cur.wait_stream(s1)
    cur.wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


ops = {"velocity": vel, "velocity_adjoint": vadj, "sl_step": step, "sl_adjoint": sadj}
alone = {k: timeit(f, None) for k, f in ops.items()}
print("alone (us):", {k: round(v, 1) for k, v in alone.items()})
for a in ("velocity", "velocity_adjoint"):
    for b in ("sl_step", "sl_adjoint", "velocity"):
        t = timeit(ops[a], ops[b])
        print(f"{a} || {b}: {t:.1f} us  (sum {alone[a] + alone[b]:.1f}, max {max(alone[a], alone[b]):.1f})")
