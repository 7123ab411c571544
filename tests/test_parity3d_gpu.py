"""3D parity of the CUDA path (BASELINE configs 3-5).

No 3D reference exists; the N-D oracle is pinned by extrusion to
the 2D reference goldens (tests/test_oracle.py).  Here the device path is
checked (a) by the same extrusion directly against the 2D reference goldens,
(b) against the oracle on small volumes and on reduced-size config recipes,
and (c) at full BASELINE sizes through size-independent properties
(directional derivative = central difference of the cost, fp64).
"""

import numpy as np
import pytest
import torch

from conftest import load_golden, rel_l2

pytestmark = pytest.mark.gpu


def _eng():
    from paper_2106_08817_b200 import engine

    return engine


def _dev(a, dtype):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device="cuda")


def _run(src, tgt, z0, T, mu, w, lam, rho, dtype, with_phi=False):
    eng = _eng()
    B = src.shape[0]
    traj = eng.allocate_trajectory(B, src.shape[1:], T, dtype, with_phi=with_phi)
    traj.I[0].copy_(_dev(src, dtype))
    traj.z[0].copy_(_dev(z0, dtype))
    eng.shoot_forward(traj, mu, w)
    bufs = eng.shoot_adjoint(traj, _dev(tgt, dtype), lam, rho, mu, w)
    torch.cuda.synchronize()
    return traj, bufs


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64], ids=["fp32", "fp64"])
@pytest.mark.parametrize("case", ["shoot_A_16sq.npz", "shoot_B_13x21.npz", "shoot_E_40x33.npz"])
def test_3d_extrusion_matches_2d_reference(case, dtype):
    """A volume constant along axis 0 reproduces the 2D reference slice by slice;
    the axis-0 mean of the 3D gradient equals the 2D reference gradient."""
    g = load_golden(case)
    D = 4
    T, mu = int(g["n_steps"]), float(g["mu"])
    ext = lambda a: np.repeat(a[None, None], D, axis=1)  # noqa: E731  [1, D, H, W]
    traj, bufs = _run(ext(g["source"]), ext(g["target"]), ext(g["z0"]), T, mu, g["weights"],
                      float(g["lam"]), float(g["rho"]), dtype, with_phi=True)
    assert _eng().guard_report(traj.guard) is None
    tol = 1e-12 if dtype == torch.float64 else 1e-5
    for k in range(T + 1):
        Ik = traj.I[k, 0].cpu().numpy()
        for s in range(D):
            assert rel_l2(Ik[s], g["I"][k]) < tol, (k, s)
        v = traj.v[k, 0].cpu().numpy()
        assert np.abs(v[0]).max() == 0.0  # no motion along the extruded axis
        assert rel_l2(v[1:, 1], g["v"][k]) < tol
    assert rel_l2(traj.phi[0, 0, 1:, 1].cpu(), g["phi"]) < tol
    gr = bufs.zbar[0].cpu().numpy()
    assert rel_l2(gr.mean(axis=0), g["grad"]) < (1e-11 if dtype == torch.float64 else 1e-4)
    c = bufs.terms[0].cpu().numpy()
    assert np.allclose(c, D * g["cost"], rtol=1e-11 if dtype == torch.float64 else 1e-5)


def _random_case(shape, seed, amp, B=1):
    from oracle import morphreg_oracle as O

    rng = np.random.default_rng(seed)
    w1 = O.gaussian_weights(1.0)
    win = np.zeros(shape)
    win[tuple(slice(1, n - 1) for n in shape)] = 1.0
    src = np.stack([np.abs(O.smooth(rng.standard_normal(shape), w1)) * win for _ in range(B)])
    tgt = np.stack([np.abs(O.smooth(rng.standard_normal(shape), w1)) * win for _ in range(B)])
    z0 = np.stack([amp * O.smooth(rng.standard_normal(shape), w1) * win for _ in range(B)])
    return src, tgt, z0


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64], ids=["fp32", "fp64"])
@pytest.mark.parametrize("shape,sigma,radius,T,mu,amp", [
    ((10, 12, 14), 1.5, None, 3, 0.3, 2.0),
    ((6, 7, 9), 3.0, None, 2, 0.1, 1.0),      # radius 12 > every extent
    ((20, 17, 24), 2.0, 6, 4, 0.0, 60.0),     # ~1 vox per-step back-trace
    ((2, 5, 4), 1.0, None, 2, 0.2, 0.5),      # 2-sample axis
])
def test_3d_matches_oracle(shape, sigma, radius, T, mu, amp, dtype):
    from oracle import morphreg_oracle as O

    src, tgt, z0 = _random_case(shape, 3, amp, B=2)
    w = O.gaussian_weights(sigma, radius)
    lam, rho = 1e-3, 0.5
    traj, bufs = _run(src, tgt, z0, T, mu, w, lam, rho, dtype, with_phi=True)
    assert _eng().guard_report(traj.guard) is None
    step_tol = 1e-11 if dtype == torch.float64 else 1e-4
    fin_tol = 1e-10 if dtype == torch.float64 else 1e-3
    for b in range(2):
        I, z, v, phi = O.shoot(src[b], z0[b], T, mu, w)
        for k in range(T + 1):
            assert rel_l2(traj.I[k, b].cpu(), I[k]) < step_tol, ("I", b, k)
            assert rel_l2(traj.z[k, b].cpu(), z[k]) < step_tol, ("z", b, k)
            assert rel_l2(traj.v[k, b].cpu(), v[k]) < step_tol, ("v", b, k)
        assert rel_l2(traj.phi[0, b].cpu(), phi) < step_tol
        gr = O.grad(src[b], tgt[b], z0[b], lam, rho, T, mu, w)
        assert rel_l2(bufs.zbar[b].cpu(), gr) < fin_tol
        c = O.cost(src[b], tgt[b], z0[b], lam, rho, T, mu, w)
        assert np.allclose(bufs.terms[b].cpu().numpy(), c, rtol=fin_tol)


@pytest.mark.parametrize("cfg,shape,T,amp", [(3, (40, 48, 40), 5, 1.0), (4, (32, 32, 32), 4, 1.0),
                                             (5, (48, 48, 48), 6, 1.0), (5, (48, 48, 48), 4, 0.5)])
def test_config_recipes_reduced_match_oracle(cfg, shape, T, amp):
    """The config 3-5 recipes (phantoms, warps, calibrated momenta, radii, mu) at
    reduced grids against the oracle, fp32 device path.  Where the oracle's
    guard fires (integrator.py:113-118) the device must report the same step
    and check."""
    from oracle import morphreg_oracle as O
    from paper_2106_08817_b200.synthetic import CONFIGS, make_config

    c = make_config(cfg, batch=1, shape=shape)
    # keep the full-size geometry: per-step offset scaled with the grid, fewer steps
    scale = shape[1] / CONFIGS[cfg]["shape"][1]
    c.z0 = c.z0 * (T / c.n_steps) * scale * amp
    w = c.weights()
    try:
        I, z, v, _ = O.shoot(c.source[0], c.z0[0], T, c.mu, w, with_phi=False)
    except O.OracleDiverged as e:
        eng = _eng()
        traj = eng.allocate_trajectory(1, c.shape, T, torch.float32)
        traj.I[0].copy_(_dev(c.source, torch.float32))
        traj.z[0].copy_(_dev(c.z0, torch.float32))
        eng.shoot_forward(traj, c.mu, w)
        assert eng.guard_report(traj.guard) == (0, e.step, e.what)
        return
    traj, bufs = _run(c.source, c.target, c.z0, T, c.mu, w, c.lam, c.rho, torch.float32)
    assert _eng().guard_report(traj.guard) is None
    for k in range(T + 1):
        assert rel_l2(traj.I[k, 0].cpu(), I[k]) < 1e-4, k
        assert rel_l2(traj.z[k, 0].cpu(), z[k]) < 1e-4, k
        assert rel_l2(traj.v[k, 0].cpu(), v[k]) < 1e-4, k
    gr = O.grad(c.source[0], c.target[0], c.z0[0], c.lam, c.rho, T, c.mu, w)
    assert rel_l2(bufs.zbar[0].cpu(), gr) < 1e-3


def _dir_deriv_check(c, T, dtype=torch.float64):
    eng = _eng()
    w = c.weights()
    B = c.batch
    traj = eng.allocate_trajectory(B, c.shape, T, dtype)
    src, tgt, z0 = _dev(c.source, dtype), _dev(c.target, dtype), _dev(c.z0, dtype)
    rng = np.random.default_rng(0)
    d = _dev(rng.standard_normal(c.z0.shape), dtype)
    d = d / d.flatten(1).norm(dim=1).view((-1,) + (1,) * len(c.shape))

    def total(zz):
        traj.I[0].copy_(src)
        traj.z[0].copy_(zz)
        eng.shoot_forward(traj, c.mu, w)
        return eng.cost_terms(traj.I[0], traj.z[0], traj.v[0], traj.I[-1], tgt, c.lam, c.rho)[:, 0]

    traj.I[0].copy_(src)
    traj.z[0].copy_(z0)
    eng.shoot_forward(traj, c.mu, w)
    assert eng.guard_report(traj.guard) is None
    bufs = eng.shoot_adjoint(traj, tgt, c.lam, c.rho, c.mu, w)
    an = (bufs.zbar * d).flatten(1).sum(1)
    # fp64: eps small enough that the O(eps^2) truncation is below the tolerance
    eps = 1e-6 * float(z0.abs().max())
    fd = (total(z0 + eps * d) - total(z0 - eps * d)) / (2 * eps)
    # same tolerance as the reference's directional-derivative test (test_objective.py:129)
    assert torch.allclose(an, fd, rtol=1e-4, atol=0), (an, fd)


def _calibrated(cfg, **kw):
    from paper_2106_08817_b200.calibrate import calibrate_no_divergence
    from paper_2106_08817_b200.synthetic import make_config

    c = make_config(cfg, **kw)
    calibrate_no_divergence(c)
    print(cfg, "momentum scale", c.manifest["momentum_scale"], "offset",
          c.manifest.get("offset_achieved"))
    return c


def test_config3_full_size_directional_derivative():
    _dir_deriv_check(_calibrated(3), 20)


def test_config4_full_size_directional_derivative():
    _dir_deriv_check(_calibrated(4, batch=2), 15)


def test_config5_full_size_stress():
    """256^3, T=50, r=24, ~3 vox per-step back-trace: the fp32 forward stays
    finite, fp32 and fp64 agree on the final image, and the fp64 gradient
    passes the directional-derivative check."""
    eng = _eng()
    c = _calibrated(5)
    w = c.weights()
    out = {}
    for dtype in (torch.float32, torch.float64):
        traj = eng.allocate_trajectory(1, c.shape, c.n_steps, dtype)
        traj.I[0].copy_(_dev(c.source, dtype))
        traj.z[0].copy_(_dev(c.z0, dtype))
        eng.shoot_forward(traj, c.mu, w)
        assert eng.guard_report(traj.guard) is None
        out[dtype] = traj.I[-1, 0].double().cpu()
        if dtype == torch.float32:  # per-step offset as calibrated (nominal 3 vox)
            off = float(traj.v[0].abs().max()) / c.n_steps
            assert 0.1 < off < 4.0, off
        del traj
        torch.cuda.empty_cache()
    assert rel_l2(out[torch.float32], out[torch.float64]) < 1e-3
    _dir_deriv_check(c, c.n_steps)
