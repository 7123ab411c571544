"""Deterministic mode (MR_OPT_DETERMINISTIC): bitwise run-to-run reproducible
gradients and optimiser histories -- the reference's replay promise
(optimizer.py:5-7, pinned by test_optimizer.py:82-89).  The fixed-point scatter
must also still match the oracle at the north_star tolerances."""

import numpy as np
import pytest
import torch

from conftest import load_golden, rel_l2

pytestmark = pytest.mark.gpu


def _run(src, tgt, z0, T, mu, w, lam, rho, dtype, scheme, det):
    from paper_2106_08817_b200 import engine

    traj = engine.allocate_trajectory(src.shape[0], src.shape[1:], T, dtype)
    traj.I[0].copy_(torch.as_tensor(src, dtype=dtype))
    traj.z[0].copy_(torch.as_tensor(z0, dtype=dtype))
    engine.shoot_forward(traj, mu, w, scheme=scheme)
    J = torch.as_tensor(tgt, dtype=dtype, device="cuda")
    bufs = engine.shoot_adjoint(traj, J, lam, rho, mu, w, scheme=scheme, deterministic=det)
    torch.cuda.synchronize()
    assert int(bufs.flags.max()) == 0
    return bufs.zbar.cpu().numpy().copy(), bufs.terms.cpu().numpy().copy()


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64], ids=["fp32", "fp64"])
@pytest.mark.parametrize("case,scheme", [("shoot_J_48sq_bigdisp.npz", "semi-lagrangian"),
                                         ("shoot_E_40x33.npz", "semi-lagrangian"),
                                         ("scheme_hy_C_48sq_bigdisp.npz", "hybrid"),
                                         ("scheme_eu_B_13x21.npz", "eulerian")])
def test_deterministic_grad_is_bitwise_reproducible_2d(case, scheme, dtype):
    g = load_golden(case)
    T, mu, lam, rho = int(g["n_steps"]), float(g["mu"]), float(g["lam"]), float(g["rho"])
    B = 4  # a batch: the same pair repeated, each copy must give the same bits too
    rep = lambda a: np.repeat(a[None], B, axis=0)  # noqa: E731
    args = (rep(g["source"]), rep(g["target"]), rep(g["z0"]), T, mu, g["weights"], lam, rho,
            dtype, scheme)
    g1, t1 = _run(*args, det=True)
    g2, t2 = _run(*args, det=True)
    assert g1.tobytes() == g2.tobytes()
    assert t1.tobytes() == t2.tobytes()
    for b in range(1, B):
        assert g1[b].tobytes() == g1[0].tobytes()
    # same numbers as the atomic path and the reference golden
    ga, _ = _run(*args, det=False)
    tol = 1e-12 if dtype == torch.float64 else 1e-5
    assert rel_l2(g1[0], ga[0]) < tol
    ref_tol = 1e-10 if dtype == torch.float64 else (4e-3 if "bigdisp" in case else 1e-3)
    assert rel_l2(g1[0], g["grad"]) < ref_tol


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64], ids=["fp32", "fp64"])
def test_deterministic_grad_is_bitwise_reproducible_3d(dtype):
    from oracle import morphreg_oracle as O

    rng = np.random.default_rng(4)
    shape = (12, 14, 10)
    w1 = O.gaussian_weights(1.0)
    win = np.zeros(shape)
    win[1:-1, 1:-1, 1:-1] = 1.0
    src = np.abs(O.smooth(rng.standard_normal(shape), w1)) * win
    tgt = np.abs(O.smooth(rng.standard_normal(shape), w1)) * win
    z0 = 40.0 * O.smooth(rng.standard_normal(shape), w1) * win
    w = O.gaussian_weights(2.0, 5)
    T, mu, lam, rho = 4, 0.2, 1e-3, 0.5
    args = (src[None], tgt[None], z0[None], T, mu, w, lam, rho, dtype, "semi-lagrangian")
    g1, t1 = _run(*args, det=True)
    g2, t2 = _run(*args, det=True)
    assert g1.tobytes() == g2.tobytes() and t1.tobytes() == t2.tobytes()
    ref = O.grad(src, tgt, z0, lam, rho, T, mu, w)
    assert rel_l2(g1[0], ref) < (1e-10 if dtype == torch.float64 else 1e-3)


def test_cost_terms_are_deterministic():
    """The cost reduction has no floating-point atomics (fixed block order)."""
    from paper_2106_08817_b200 import engine

    g = load_golden("shoot_E_40x33.npz")
    B = 8
    rep = lambda a: torch.as_tensor(np.repeat(a[None], B, axis=0), device="cuda")  # noqa: E731
    I0, z0 = rep(g["source"]), rep(g["z0"])
    v0 = engine.velocity(I0, z0, g["weights"])
    a = engine.cost_terms(I0, z0, v0, I0 * 0.5, rep(g["target"]), 1e-3, 0.5).cpu().numpy()
    b = engine.cost_terms(I0, z0, v0, I0 * 0.5, rep(g["target"]), 1e-3, 0.5).cpu().numpy()
    assert a.tobytes() == b.tobytes()
    assert all(a[k].tobytes() == a[0].tobytes() for k in range(B))


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64], ids=["fp32", "fp64"])
def test_optimize_replays_bit_for_bit(dtype):
    """test_optimizer.py:82-89 analogue: two optimize() runs from the same inputs
    give identical histories, step sizes and final momenta."""
    import paper_2106_08817_b200 as mr

    g = load_golden("shoot_E_40x33.npz")
    k = mr.GaussianKernel(float(g["sigma"]), int(g["radius"]))
    cfg = mr.ShootingConfig(mr.Scheme.SEMI_LAGRANGIAN, int(g["n_steps"]), float(g["mu"]), k,
                            dtype=dtype)
    assert cfg.deterministic
    prob = mr.RegistrationProblem(mr.ScalarField.from_array(g["source"]),
                                  mr.ScalarField.from_array(g["target"]), float(g["lam"]),
                                  float(g["rho"]), cfg)
    oc = mr.OptimizeConfig(max_iters=6, init_step=1.0)
    r1 = mr.optimize(prob, mr.default_init(prob), oc)
    r2 = mr.optimize(prob, mr.default_init(prob), oc)
    assert [h.total for h in r1.history] == [h.total for h in r2.history]
    assert r1.step_sizes == r2.step_sizes
    assert r1.termination == r2.termination
    assert r1.z0.values.tobytes() == r2.z0.values.tobytes()
    assert r1.history[-1].total < r1.history[0].total
