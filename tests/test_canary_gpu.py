"""Out-of-bounds write check without compute-sanitizer (closed on this pool,
profiles/r02/compute_sanitizer_closed.log): every buffer the C-ABI writes is carved
out of one slab with poisoned gaps on both sides; after a forward + adjoint sweep
the gaps must be untouched and the results must equal a run on ordinary buffers."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GAP = 4096  # bytes of canary on each side of every buffer (keeps 256-byte alignment)
POISON = 0x5A


class Slab:
    def __init__(self, nbytes):
        self.buf = torch.full((nbytes,), POISON, dtype=torch.uint8, device="cuda")
        self.off = 0
        self.gaps = []

    def _gap(self):
        self.gaps.append((self.off, self.off + GAP))
        self.off += GAP

    def take(self, shape, dtype):
        n = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
        self._gap()
        view = self.buf[self.off:self.off + n].view(dtype).view(shape)
        self.off += (n + 255) // 256 * 256
        self._gap()
        return view

    def check(self):
        for lo, hi in self.gaps:
            assert bool((self.buf[lo:hi] == POISON).all()), f"canary [{lo}, {hi}) was overwritten"


def taps(r):
    x = np.arange(-r, r + 1) / (r / 3.0)
    w = np.exp(-0.5 * x * x)
    return w / w.sum()


@pytest.mark.parametrize("shape,B,T,r,dtype,scheme,det", [
    ((40, 56), 2, 3, 5, torch.float32, "semi-lagrangian", False),   # TMA path, k_vel_a / k_vel_b
    ((130, 72), 1, 2, 24, torch.float32, "semi-lagrangian", False),  # several tiles, radius 24
    ((41, 57), 2, 2, 4, torch.float32, "semi-lagrangian", False),   # not TMA-describable
    ((24, 32), 1, 2, 3, torch.float64, "semi-lagrangian", False),
    ((40, 56), 1, 2, 3, torch.float32, "eulerian", False),
    ((40, 56), 1, 2, 3, torch.float32, "hybrid", False),
    ((40, 56), 2, 2, 3, torch.float32, "semi-lagrangian", True),    # fixed-point scatters
    ((12, 20, 24), 2, 2, 3, torch.float32, "semi-lagrangian", False),
    ((12, 20, 24), 1, 2, 3, torch.float32, "semi-lagrangian", True),
    ((10, 12, 16), 1, 2, 2, torch.float64, "semi-lagrangian", False),
])
def test_no_write_outside_the_buffers(shape, B, T, r, dtype, scheme, det):
    from paper_2106_08817_b200 import _lib, engine

    lib = _lib.load_library()
    d = len(shape)
    mu = 0.0 if scheme == "eulerian" else 0.3
    w = taps(r)
    g = torch.Generator(device="cuda").manual_seed(11)
    I0 = torch.rand((B,) + shape, device="cuda", generator=g, dtype=dtype)
    z0 = 0.3 * torch.randn((B,) + shape, device="cuda", generator=g, dtype=dtype)
    J = torch.rand((B,) + shape, device="cuda", generator=g, dtype=dtype)

    # ordinary buffers
    ref = engine.allocate_trajectory(B, shape, T, dtype)
    ref.I[0].copy_(I0)
    ref.z[0].copy_(z0)
    engine.shoot_forward(ref, mu, w, scheme=scheme)
    rb = engine.shoot_adjoint(ref, J, 1e-3, 1.0, mu, w, scheme=scheme, deterministic=det)

    # the same sweep on slab views with canaries
    grid = _lib.make_grid(B, shape)
    code = _lib.dtype_code(dtype)
    es = torch.empty((), dtype=dtype).element_size()
    fw = lib.mr_forward_workspace_bytes(code, grid)
    aw = lib.mr_adjoint_workspace_bytes(code, grid)
    n = int(np.prod(shape))
    total = (2 * (T + 1) * B * n + (T + 1) * B * d * n + B * n) * es + fw + aw + 64 * GAP + (1 << 16)
    slab = Slab(total)
    I = slab.take((T + 1, B) + shape, dtype)
    z = slab.take((T + 1, B) + shape, dtype)
    v = slab.take((T + 1, B, d) + shape, dtype)
    guard = slab.take((B, T + 1), torch.int32)
    ws = slab.take((fw // es,), dtype) if fw else None
    traj = engine.DeviceTrajectory(I, z, v, guard, None, ws)
    traj.I[0].copy_(I0)
    traj.z[0].copy_(z0)
    engine.shoot_forward(traj, mu, w, scheme=scheme)
    bufs = engine.AdjointBuffers.__new__(engine.AdjointBuffers)
    bufs.workspace = slab.take((aw,), torch.uint8)
    bufs.zbar = slab.take((B,) + shape, dtype)
    bufs.terms = slab.take((B, 4), torch.float64)
    bufs.flags = slab.take((B,), torch.int32)
    engine.shoot_adjoint(traj, J, 1e-3, 1.0, mu, w, bufs=bufs, scheme=scheme, deterministic=det)
    torch.cuda.synchronize()
    slab.check()
    assert torch.equal(traj.I, ref.I) and torch.equal(traj.z, ref.z) and torch.equal(traj.v, ref.v)
    assert torch.equal(traj.guard, ref.guard)
    if det:
        assert torch.equal(bufs.zbar, rb.zbar) and torch.equal(bufs.terms, rb.terms)
    else:
        torch.testing.assert_close(bufs.zbar, rb.zbar, rtol=1e-4, atol=1e-5)
