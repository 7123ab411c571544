"""Parity of the CUDA path (through the C-ABI) against the reference goldens and
the CPU oracle.

Tolerances (BASELINE.json north_star): fp32 per-step images, momenta and
velocities within 1e-4 relative L2; final image and cost gradient within 1e-3.
The fp64 instantiation of the same kernels must agree to ~1e-10.
"""

import numpy as np
import pytest
import torch

from conftest import load_golden, rel_l2, scheme_cases, shoot_cases

pytestmark = pytest.mark.gpu

TOL = {torch.float32: dict(step=1e-4, final=1e-3, cost=1e-4),
       torch.float64: dict(step=1e-10, final=1e-9, cost=1e-11)}


def _eng():
    from paper_2106_08817_b200 import engine

    return engine


def _dev(a, dtype):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device="cuda")


_SENS = {}


def _fp32_sensitivity(case, g):
    """Conditioning of a case: the oracle's own error when only its INPUTS are
    rounded to fp32 (computed in fp64).  Per step (I, z, v) and for the grad."""
    if case in _SENS:
        return _SENS[case]
    from oracle import morphreg_oracle as O

    T, mu = int(g["n_steps"]), float(g["mu"])
    sch = str(g["scheme"])
    r = lambda a: np.asarray(a, np.float32).astype(np.float64)  # noqa: E731
    I, z, v, _ = O.shoot(r(g["source"]), r(g["z0"]), T, mu, g["weights"], with_phi=False,
                         scheme=sch)
    gr = O.grad(r(g["source"]), r(g["target"]), r(g["z0"]), float(g["lam"]), float(g["rho"]), T, mu,
                g["weights"], scheme=sch)
    ref = lambda name, k: g[name][k] if name in g else g[f"{name}{k}"]  # noqa: E731
    steps = range(T + 1) if "I" in g else (0, T)
    s = {k: max(rel_l2(I[k], ref("I", k)), rel_l2(z[k], ref("z", k)), rel_l2(v[k], ref("v", k)))
         for k in steps}
    s["grad"] = rel_l2(gr, g["grad"])
    _SENS[case] = s
    return s


def _run_case(g, dtype, batch_copies=1):
    eng = _eng()
    T, mu = int(g["n_steps"]), float(g["mu"])
    shape = g["source"].shape
    traj = eng.allocate_trajectory(batch_copies, shape, T, dtype, with_phi=True)
    for b in range(batch_copies):
        traj.I[0, b].copy_(_dev(g["source"], dtype))
        traj.z[0, b].copy_(_dev(g["z0"], dtype))
    sch = str(g["scheme"])
    eng.shoot_forward(traj, mu, g["weights"], scheme=sch)
    J = _dev(np.repeat(g["target"][None], batch_copies, 0), dtype)
    bufs = eng.shoot_adjoint(traj, J, float(g["lam"]), float(g["rho"]), mu, g["weights"],
                             scheme=sch)
    torch.cuda.synchronize()
    return traj, bufs


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64], ids=["fp32", "fp64"])
@pytest.mark.parametrize("case", shoot_cases() + scheme_cases())
def test_shoot_and_grad_match_reference(case, dtype):
    g = load_golden(case)
    tol = TOL[dtype]
    traj, bufs = _run_case(g, dtype)
    T = int(g["n_steps"])
    assert _eng().guard_report(traj.guard) is None
    steps = range(T + 1) if "I" in g else (0, T)
    # fp32: the north_star tolerances, widened only where the case itself is
    # ill-conditioned (10x the error that rounding its inputs to fp32 causes)
    sens = _fp32_sensitivity(case, g) if dtype == torch.float32 else {}
    errs = []
    for k in steps:
        Ik = g["I"][k] if "I" in g else g[f"I{k}"]
        zk = g["z"][k] if "z" in g else g[f"z{k}"]
        vk = g["v"][k] if "v" in g else g[f"v{k}"]
        e = (rel_l2(traj.I[k, 0].cpu(), Ik), rel_l2(traj.z[k, 0].cpu(), zk),
             rel_l2(traj.v[k, 0].cpu(), vk))
        errs.append(e)
        t = max(tol["step"], 10 * sens.get(k, 0.0))
        assert max(e) < t, (k, e, t)
    print(case, dtype, "per-step max rel L2", [f"{max(e):.1e}" for e in errs])
    t_final = max(tol["final"], 10 * sens.get("grad", 0.0))
    terms = bufs.terms[0].cpu().numpy()
    assert np.allclose(terms, g["cost"], rtol=max(tol["cost"], 10 * sens.get(T, 0.0)), atol=1e-300)
    assert rel_l2(traj.phi[0, 0].cpu(), g["phi"]) < max(tol["step"], 10 * sens.get(T, 0.0))
    eg = rel_l2(bufs.zbar[0].cpu(), g["grad"])
    print(case, dtype, "grad rel L2", f"{eg:.1e}", "sensitivity", sens.get("grad"))
    assert eg < t_final
    assert int(bufs.flags[0]) == 0


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64], ids=["fp32", "fp64"])
def test_batched_pairs_equal_single_pair_runs(dtype):
    """Pairs of a batch are independent: batch results equal per-pair results."""
    eng = _eng()
    g = load_golden("shoot_H_100x90_r9.npz")
    T, mu, w = int(g["n_steps"]), float(g["mu"]), g["weights"]
    scales = [1.0, -0.5, 2.0]
    B = len(scales)
    traj = eng.allocate_trajectory(B, g["source"].shape, T, dtype)
    for b, s in enumerate(scales):
        traj.I[0, b].copy_(_dev(g["source"], dtype))
        traj.z[0, b].copy_(_dev(s * g["z0"], dtype))
    J = _dev(np.repeat(g["target"][None], B, 0), dtype)
    eng.shoot_forward(traj, mu, w)
    bufs = eng.shoot_adjoint(traj, J, float(g["lam"]), float(g["rho"]), mu, w)
    for b, s in enumerate(scales):
        one = eng.allocate_trajectory(1, g["source"].shape, T, dtype)
        one.I[0, 0].copy_(traj.I[0, b])
        one.z[0, 0].copy_(traj.z[0, b])
        eng.shoot_forward(one, mu, w)
        ob = eng.shoot_adjoint(one, J[b:b + 1].contiguous(), float(g["lam"]), float(g["rho"]), mu, w)
        # forward is deterministic per pair: bitwise
        assert torch.equal(one.I[:, 0], traj.I[:, b])
        assert torch.equal(one.v[:, 0], traj.v[:, b])
        # the adjoint scatter uses float atomics: order-dependent rounding only
        assert rel_l2(ob.zbar[0].cpu(), bufs.zbar[b].cpu()) < (1e-5 if dtype == torch.float32 else 1e-13)


def test_forward_is_bitwise_deterministic():
    eng = _eng()
    g = load_golden("shoot_E_40x33.npz")
    a, _ = _run_case(g, torch.float32)
    b, _ = _run_case(g, torch.float32)
    assert torch.equal(a.I, b.I) and torch.equal(a.z, b.z) and torch.equal(a.v, b.v)


def test_guard_reports_reference_step_and_check():
    import paper_2106_08817_b200 as mr

    g = load_golden("guard.npz")
    for dtype in (torch.float32, torch.float64):
        cfg = mr.ShootingConfig(mr.Scheme.SEMI_LAGRANGIAN, int(g["n_steps"]), float(g["mu"]),
                                mr.GaussianKernel(float(g["sigma"])), dtype=dtype)
        with pytest.raises(mr.IntegrationDiverged) as e:
            mr.shoot(mr.ScalarField.from_array(g["source"]), mr.ScalarField.from_array(g["z0"]), cfg)
        assert e.value.step == int(g["step"])
        assert e.value.what == str(g["what"])


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64], ids=["fp32", "fp64"])
def test_zero_momentum_is_bitwise_identity(dtype):
    import paper_2106_08817_b200 as mr

    g = load_golden("shoot_H_100x90_r9.npz")
    src = mr.ScalarField.from_array(g["source"])
    cfg = mr.ShootingConfig(mr.Scheme.SEMI_LAGRANGIAN, 5, 0.3, mr.GaussianKernel(3.0, 9), dtype=dtype)
    traj = mr.shoot(src, mr.ScalarField.zeros(src.geometry), cfg)
    ref = torch.as_tensor(g["source"], dtype=dtype)
    for s in traj.states:
        assert torch.equal(s.image.tensor.cpu(), ref)
        assert not bool(s.momentum.tensor.any())
        assert not bool(s.velocity.tensor.any())
    ident = np.stack(np.meshgrid(np.arange(100.0), np.arange(90.0), indexing="ij"), axis=-1)
    assert np.array_equal(traj.deformation.coords, ident)


@pytest.mark.parametrize("dtype,tol", [(torch.float64, 1e-13), (torch.float32, 1e-5)], ids=["fp64", "fp32"])
def test_shoot_lddmm_matches_the_references_separate_lddmm_path(dtype, tol):
    """shoot_lddmm against the golden of the REFERENCE's own deformation-only routine
    (integrator.py:222-277, a code path of its own there), run on a config whose mu is
    non-zero: mu must be ignored.  The device shoot(mu = 0) must then equal
    shoot_lddmm bitwise, as the reference's two paths do (its acceptance criterion 2)."""
    import paper_2106_08817_b200 as mr

    g = load_golden("lddmm_path.npz")
    assert bool(g["reference_paths_bitwise_equal"])
    kern = mr.GaussianKernel(float(g["sigma"]))
    assert np.array_equal(kern.weights, g["weights"])
    src, z0 = mr.ScalarField.from_array(g["source"]), mr.ScalarField.from_array(g["z0"])
    T = int(g["n_steps"])
    b = mr.shoot_lddmm(src, z0, mr.ShootingConfig(mr.Scheme.SEMI_LAGRANGIAN, T,
                                                 float(g["mu_in_config"]), kern, dtype=dtype))
    for k, st in enumerate(b.states):
        assert rel_l2(st.image.values, g["I"][k]) < tol
        assert rel_l2(st.momentum.values, g["z"][k]) < tol
        assert rel_l2(np.moveaxis(st.velocity.values, -1, 0), g["v"][k]) < tol
    assert rel_l2(np.moveaxis(b.deformation.coords, -1, 0), g["phi"]) < tol
    a = mr.shoot(src, z0, mr.ShootingConfig(mr.Scheme.SEMI_LAGRANGIAN, T, 0.0, kern, dtype=dtype))
    for sa, sb in zip(a.states, b.states):
        assert sa.image.values.tobytes() == sb.image.values.tobytes()
        assert sa.momentum.values.tobytes() == sb.momentum.values.tobytes()
        assert sa.velocity.values.tobytes() == sb.velocity.values.tobytes()


@pytest.mark.parametrize("n,sigma", [(3, 1.0), (8, 1.0), (16, 2.0), (5, 3.0), (40, 2.5)])
def test_device_smoothing_and_transpose_match_reference(n, sigma):
    eng = _eng()
    g = load_golden("ops.npz")
    key = f"conv_{n}_{sigma}"
    a = _dev(g[key + "_in"][None], torch.float64)
    w = g[key + "_w"]
    assert rel_l2(eng.smooth(a, w)[0].cpu(), g[key + "_smooth"]) < 1e-13
    assert rel_l2(eng.smooth(a, w, adjoint=True)[0].cpu(), g[key + "_smoothT"]) < 1e-13
    a32 = a.float()
    assert rel_l2(eng.smooth(a32, w)[0].cpu(), g[key + "_smooth"]) < 1e-6
    assert rel_l2(eng.smooth(a32, w, adjoint=True)[0].cpu(), g[key + "_smoothT"]) < 1e-6


@pytest.mark.parametrize("R", [1, 5, 12, 24, 32])
def test_device_smoothing_transpose_identity_multi_tile(R):
    """<K f, g> == <f, K^T g> on grids spanning several tiles, every radius class."""
    eng = _eng()
    rng = np.random.default_rng(R)
    w = np.exp(-0.5 * (np.arange(-R, R + 1) / (R / 3.0 + 0.5)) ** 2)
    w /= w.sum()
    f = _dev(rng.standard_normal((2, 97, 150)), torch.float64)
    h = _dev(rng.standard_normal((2, 97, 150)), torch.float64)
    lhs = float((eng.smooth(f, w) * h).sum())
    rhs = float((f * eng.smooth(h, w, adjoint=True)).sum())
    assert lhs == pytest.approx(rhs, rel=1e-12)


def test_config1_full_size_matches_reference():
    import paper_2106_08817_b200 as mr

    g = load_golden("config1.npz")
    from paper_2106_08817_b200.synthetic import make_config

    c = make_config(1)
    geom = mr.GridGeometry(200, 200)
    cfg = mr.ShootingConfig(mr.Scheme.SEMI_LAGRANGIAN, c.n_steps, c.mu, mr.GaussianKernel(c.sigma, c.radius))
    prob = mr.RegistrationProblem(mr.ScalarField(geom, g["source"]), mr.ScalarField(geom, g["target"]),
                                  c.lam, c.rho, cfg)
    z0 = mr.ScalarField(geom, g["z0"])
    traj = mr.shoot(prob.source, z0, cfg)
    assert rel_l2(traj.final_image.values, g["IT"]) < 1e-4
    assert rel_l2(traj.states[-1].momentum.values, g["zT"]) < 1e-4
    rep = mr.cost(prob, z0)
    assert rep.total == pytest.approx(float(g["cost"][0]), rel=1e-4)
    assert rel_l2(mr.grad(prob, z0).values, g["grad"]) < 1e-3
    # the config's 20 fixed-step gradient-descent iterations
    z, hist = mr.fixed_step_descent(prob, z0, 20, 1e-2)
    totals = np.array([h.total for h in hist])
    assert np.allclose(totals, g["gd_history"][:, 0], rtol=1e-3)
    assert rel_l2(z.values, g["gd_final_z"]) < 1e-3


def test_config2_pair_full_size_matches_oracle():
    """One cfg-2 pair at full size (512^2, T=20, r=24) against the fp64 oracle."""
    from oracle import morphreg_oracle as O
    from paper_2106_08817_b200.synthetic import make_config

    eng = _eng()
    c = make_config(2, batch=1)
    w = c.weights()
    src, tgt, z0 = c.source[0], c.target[0], c.z0[0]
    I, z, v, _ = O.shoot(src, z0, c.n_steps, c.mu, w, with_phi=False)
    gr = O.grad(src, tgt, z0, c.lam, c.rho, c.n_steps, c.mu, w)
    traj = eng.allocate_trajectory(1, src.shape, c.n_steps, torch.float32)
    traj.I[0, 0].copy_(_dev(src, torch.float32))
    traj.z[0, 0].copy_(_dev(z0, torch.float32))
    eng.shoot_forward(traj, c.mu, w)
    bufs = eng.shoot_adjoint(traj, _dev(tgt[None], torch.float32), c.lam, c.rho, c.mu, w)
    for k in range(c.n_steps + 1):
        assert rel_l2(traj.I[k, 0].cpu(), I[k]) < 1e-4, k
        assert rel_l2(traj.z[k, 0].cpu(), z[k]) < 1e-4, k
        assert rel_l2(traj.v[k, 0].cpu(), v[k]) < 1e-4, k
    assert rel_l2(bufs.zbar[0].cpu(), gr) < 1e-3
    # the calibrated momentum really moves: max per-step back-trace ~1 px
    assert 0.5 < float(np.abs(v[0]).max()) / c.n_steps < 1.5


def test_config2_batch_directional_derivative_fp64():
    """Size-independent property at BASELINE size: <grad, d> equals the central
    difference of the cost along d (4 pairs x 512^2, T=20, fp64 kernels)."""
    from paper_2106_08817_b200.synthetic import make_config

    eng = _eng()
    c = make_config(2, batch=4)
    w = c.weights()
    dt = torch.float64
    B = c.batch
    traj = eng.allocate_trajectory(B, c.shape, c.n_steps, dt)
    src, tgt, z0 = _dev(c.source, dt), _dev(c.target, dt), _dev(c.z0, dt)
    rng = np.random.default_rng(0)
    d = _dev(rng.standard_normal(c.z0.shape), dt)
    d = d / d.flatten(1).norm(dim=1).view(-1, 1, 1)

    def total(zz):
        traj.I[0].copy_(src)
        traj.z[0].copy_(zz)
        eng.shoot_forward(traj, c.mu, w)
        return eng.cost_terms(traj.I[0], traj.z[0], traj.v[0], traj.I[-1], tgt, c.lam, c.rho)[:, 0]

    traj.I[0].copy_(src)
    traj.z[0].copy_(z0)
    eng.shoot_forward(traj, c.mu, w)
    bufs = eng.shoot_adjoint(traj, tgt, c.lam, c.rho, c.mu, w)
    an = (bufs.zbar * d).flatten(1).sum(1)
    eps = 1e-4 * float(z0.abs().max())
    fd = (total(z0 + eps * d) - total(z0 - eps * d)) / (2 * eps)
    assert torch.allclose(an, fd, rtol=1e-5, atol=0)


def test_autograd_function_matches_engine():
    import paper_2106_08817_b200 as mr

    g = load_golden("shoot_K_60x44_border.npz")
    cfg = mr.ShootingConfig(mr.Scheme.SEMI_LAGRANGIAN, int(g["n_steps"]), float(g["mu"]),
                            mr.GaussianKernel(float(g["sigma"])))
    z0 = _dev(g["z0"][None], torch.float32).requires_grad_(True)
    src = _dev(g["source"][None], torch.float32)
    tgt = _dev(g["target"][None], torch.float32)
    tot = mr.ShootingCost.apply(z0, src, tgt, cfg, float(g["lam"]), float(g["rho"]))
    assert float(tot[0]) == pytest.approx(float(g["cost"][0]), rel=1e-4)
    (2.0 * tot.sum()).backward()
    assert rel_l2(z0.grad[0].cpu() / 2.0, g["grad"]) < 1e-3


@pytest.mark.parametrize("scheme", ["semi-lagrangian", "eulerian", "hybrid"])
def test_facade_directional_derivative_fp64_like_reference_suite(scheme):
    """test_objective.py:117-129 / test_acceptance.py:75-90 (all schemes) restated
    through the device kernels (fp64)."""
    import paper_2106_08817_b200 as mr

    g = load_golden("shoot_A_16sq.npz")
    cfg = mr.ShootingConfig(mr.Scheme(scheme), 6, 0.05, mr.GaussianKernel(1.0), dtype=torch.float64)
    geom = mr.GridGeometry(16, 16)
    prob = mr.RegistrationProblem(mr.ScalarField(geom, g["source"]), mr.ScalarField(geom, g["target"]),
                                  1e-3, 0.5, cfg)
    z0 = g["z0"]
    d = np.random.default_rng(17).standard_normal(z0.shape)
    d /= np.linalg.norm(d)
    eps = 1e-4
    plus = mr.cost(prob, mr.ScalarField(geom, z0 + eps * d)).total
    minus = mr.cost(prob, mr.ScalarField(geom, z0 - eps * d)).total
    fd = (plus - minus) / (2 * eps)
    an = float(np.sum(mr.grad(prob, mr.ScalarField(geom, z0)).values * d))
    assert an == pytest.approx(fd, rel=1e-4)


@pytest.mark.parametrize("chunks", [1, 3, 4])
def test_host_pipeline_matches_device_call(chunks):
    """cost_and_grad_batch with pinned HOST tensors (pair groups on their own streams,
    copies overlapped) returns what the device-tensor call returns, and matches the
    oracle per pair."""
    import paper_2106_08817_b200 as mr
    from oracle import morphreg_oracle as O

    rng = np.random.default_rng(7)
    B, H, W, T, mu, lam, rho = 7, 48, 40, 5, 0.25, 1e-3, 1.0
    sig = 2.0
    w = O.gaussian_weights(sig)
    win = np.zeros((H, W))
    win[6:-6, 6:-6] = 1.0
    src = np.stack([np.abs(O.smooth(rng.standard_normal((H, W)), O.gaussian_weights(1.0))) * win
                    for _ in range(B)])
    tgt = np.stack([np.abs(O.smooth(rng.standard_normal((H, W)), O.gaussian_weights(1.0))) * win
                    for _ in range(B)])
    z0 = np.stack([2.0 * O.smooth(rng.standard_normal((H, W)), O.gaussian_weights(1.0)) * win
                   for _ in range(B)])
    cfg = mr.ShootingConfig(mr.Scheme.SEMI_LAGRANGIAN, T, mu, mr.GaussianKernel(sig))
    f32 = torch.float32
    hs, ht, hz = (torch.as_tensor(a, dtype=f32) for a in (src, tgt, z0))
    zb_h, terms_h, guard_h = mr.cost_and_grad_batch(hs, ht, hz, cfg, lam, rho, chunks=chunks)
    assert not zb_h.is_cuda and zb_h.shape == (B, H, W)
    zb_d, terms_d, guard_d = mr.cost_and_grad_batch(_dev(src, f32), _dev(tgt, f32), _dev(z0, f32),
                                                    cfg, lam, rho)
    torch.cuda.synchronize()
    assert torch.equal(guard_h, guard_d.cpu())
    # adjoint scatters use fp32 atomics: equal up to summation order
    assert rel_l2(zb_h, zb_d.cpu().numpy()) < 1e-6
    assert np.allclose(terms_h.numpy(), terms_d.cpu().numpy(), rtol=1e-6)
    for b in (0, B - 1):
        g = O.grad(src[b], tgt[b], z0[b], lam, rho, T, mu, w)
        assert rel_l2(zb_h[b], g) < 1e-3


@pytest.mark.parametrize("split", [True, False], ids=["split", "single"])
@pytest.mark.parametrize("B,H,W,R", [(1, 40, 56, 3), (2, 97, 152, 12), (3, 64, 128, 24),
                                     (1, 20, 24, 24), (2, 130, 200, 9)])
def test_velocity_operators_match_oracle(B, H, W, R, split):
    """mr_velocity / mr_velocity_adjoint, both kernel structures (split = product +
    axis-1 tile pass, then whole-column axis-0 pass) against the oracle:
    v = -K(z grad I) (integrator.py:93-94) and its adjoint (objective.py:157-161)."""
    from oracle import morphreg_oracle as O

    eng = _eng()
    rng = np.random.default_rng(1000 * R + H)
    w = O.gaussian_weights(R / 3.0, R)
    I = rng.random((B, H, W))
    z = rng.standard_normal((B, H, W))
    vbar = rng.standard_normal((B, 2, H, W))
    ib0 = rng.standard_normal((B, H, W))
    zb0 = rng.standard_normal((B, H, W))
    for dtype, tol in ((torch.float32, 1e-5), (torch.float64, 1e-12)):
        v = eng.velocity(_dev(I, dtype), _dev(z, dtype), w, split=split).cpu().numpy()
        ib, zb = _dev(ib0, dtype), _dev(zb0, dtype)
        eng.velocity_adjoint(_dev(I, dtype), _dev(z, dtype), _dev(vbar, dtype), ib, zb, w,
                             split=split)
        for b in range(B):
            assert rel_l2(v[b], O.velocity(z[b], O.gradient(I[b]), w)) < tol
            mbar = -np.stack([O.smooth_adjoint(vbar[b, c], w) for c in range(2)])
            gi = O.gradient(I[b])
            assert rel_l2(zb[b].cpu().numpy(), zb0[b] + (mbar * gi).sum(0)) < tol
            assert rel_l2(ib[b].cpu().numpy(), ib0[b] + O.gradient_adjoint(mbar * z[b])) < tol


def test_schemes_are_2d_only_and_validated():
    """Eulerian / Hybrid exist in 2D only (as in the reference); bad codes are FieldError."""
    from paper_2106_08817_b200 import _lib
    from paper_2106_08817_b200.errors import FieldError

    eng = _eng()
    traj = eng.allocate_trajectory(1, (8, 8, 8), 2, torch.float32)
    with pytest.raises(FieldError):
        eng.shoot_forward(traj, 0.1, np.array([0.25, 0.5, 0.25]), scheme="eulerian")
    lib = _lib.load_library()
    rc = lib.mr_shoot_forward_scheme(0, _lib.make_grid(1, (8, 8)),
                                     _lib.KernelHandle(np.ones(3) / 3).struct, 7, 0.0, 2,
                                     None, None, None, None, None, None, None)
    assert rc == 1 and b"unknown scheme" in lib.mr_last_error()


def test_optimize_reuses_trajectories_with_reference_iterates(monkeypatch):
    """optimize() (optimizer.py:65-113) shoots once per cost evaluation only: the
    gradient at an accepted point runs over that point's kept trajectory.  Its
    iterates equal a plain loop over the public cost()/grad() (fp64)."""
    import paper_2106_08817_b200 as mr
    from paper_2106_08817_b200 import engine, optimizer

    g = load_golden("shoot_E_40x33.npz")
    cfg = mr.ShootingConfig(mr.Scheme.SEMI_LAGRANGIAN, int(g["n_steps"]), float(g["mu"]),
                            mr.GaussianKernel(float(g["sigma"]), int(g["radius"])),
                            dtype=torch.float64)
    geom = mr.GridGeometry(*g["source"].shape)
    prob = mr.RegistrationProblem(mr.ScalarField(geom, g["source"]),
                                  mr.ScalarField(geom, g["target"]), float(g["lam"]),
                                  float(g["rho"]), cfg)
    ocfg = mr.OptimizeConfig(max_iters=4)
    calls = {"n": 0}
    real = engine.shoot_forward

    def counting(*a, **k):
        calls["n"] += 1
        return real(*a, **k)

    monkeypatch.setattr(engine, "shoot_forward", counting)
    res = optimizer.optimize(prob, mr.ScalarField(geom, g["z0"]), ocfg)
    n_opt = calls["n"]
    # the reference algorithm over the public API (one extra shoot per gradient)
    z = mr.ScalarField(geom, g["z0"])
    rep = mr.cost(prob, z)
    totals, step = [rep.total], ocfg.init_step
    for it in range(len(res.history) - 1):
        gr = mr.grad(prob, z).values
        gn = float(np.sum(gr * gr))
        step = step / ocfg.backtrack_factor if it > 0 else ocfg.init_step
        while True:
            trial = mr.ScalarField(geom, z.values - step * gr)
            tr = mr.cost(prob, trial)
            if tr.total <= rep.total - ocfg.sufficient_decrease * step * gn:
                break
            step *= ocfg.backtrack_factor
        z, rep = trial, tr
        totals.append(rep.total)
    assert [h.total for h in res.history] == pytest.approx(totals, rel=1e-12)
    assert np.allclose(res.z0.values, z.values, rtol=1e-10, atol=1e-14)
    n_evals = len(res.history) - 1
    assert n_opt == calls["n"] - n_opt - n_evals  # the reference loop shot n_evals more times
