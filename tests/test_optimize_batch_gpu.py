"""optimize_batch: B independent Armijo descents (optimizer.py:65-113) as batched
device sweeps.  Per pair the iterates, step sizes, histories and terminations must be
those of optimize() on that pair alone."""

import numpy as np
import pytest
import torch

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _problem_set(B, dtype):
    import paper_2106_08817_b200 as mr

    g = load_golden("shoot_E_40x33.npz")
    cfg = mr.ShootingConfig(mr.Scheme.SEMI_LAGRANGIAN, int(g["n_steps"]), float(g["mu"]),
                            mr.GaussianKernel(float(g["sigma"]), int(g["radius"])), dtype=dtype)
    rng = np.random.default_rng(5)
    H, W = g["source"].shape
    src = np.stack([g["source"]] * B)
    tgt = np.stack([g["target"]] * B)
    z0 = np.stack([g["z0"]] * B)
    # make the pairs different (pair 0 is the golden): shifted targets, scaled starting
    # momenta, and image contrasts 1, 3, 0.3, 6, 1.5 -- the gradient scales with the
    # contrast squared, so the accepted Armijo steps differ from pair to pair
    contrast = [1.0, 3.0, 0.3, 6.0, 1.5]
    for b in range(1, B):
        tgt[b] = np.clip(np.roll(g["target"], (b % 3 - 1, b - 2), axis=(0, 1)) * (1.0 - 0.07 * b), 0, 1)
        z0[b] = g["z0"] * (0.4 * b) + 0.02 * rng.standard_normal((H, W)) * (b % 2)
        src[b] *= contrast[b % 5]
        tgt[b] *= contrast[b % 5]
    return mr, cfg, float(g["lam"]), float(g["rho"]), src, tgt, z0


def test_batched_line_search_equals_per_pair_optimize_fp64():
    B = 5
    mr, cfg, lam, rho, src, tgt, z0 = _problem_set(B, torch.float64)
    ocfg = mr.OptimizeConfig(max_iters=5, init_step=400.0)  # large enough that pairs backtrack
    res = mr.optimize_batch(torch.as_tensor(src), torch.as_tensor(tgt), torch.as_tensor(z0), cfg,
                            lam, rho, ocfg)
    geom = mr.GridGeometry(*src.shape[1:])
    n_backtracks = set()
    for b in range(B):
        prob = mr.RegistrationProblem(mr.ScalarField(geom, src[b]), mr.ScalarField(geom, tgt[b]),
                                      lam, rho, cfg)
        one = mr.optimize(prob, mr.ScalarField(geom, z0[b]), ocfg)
        assert res.terminations[b] == one.termination
        assert [h.total for h in res.histories[b]] == pytest.approx([h.total for h in one.history],
                                                                    rel=1e-12)
        assert res.step_sizes[b] == pytest.approx(one.step_sizes, rel=0, abs=0)
        assert np.allclose(res.z0[b].cpu().numpy(), one.z0.values, rtol=1e-10, atol=1e-14)
        n_backtracks.add(tuple(one.step_sizes))
    assert len(n_backtracks) > 1  # the pairs really took different step-size paths
    # compaction: fewer pair-shoots than rounds x B once pairs accept at different rounds
    assert res.pair_shoots < res.rounds * B
    assert res.grad_sweeps <= ocfg.max_iters


def test_batched_line_search_fp32_decreases_every_cost_and_stays_on_device():
    B = 4
    mr, cfg, lam, rho, src, tgt, z0 = _problem_set(B, torch.float32)
    res = mr.optimize_batch(torch.as_tensor(src), torch.as_tensor(tgt), torch.as_tensor(z0), cfg,
                            lam, rho, mr.OptimizeConfig(max_iters=3))
    assert res.z0.is_cuda and res.z0.dtype == torch.float32
    for b in range(B):
        totals = [h.total for h in res.histories[b]]
        assert all(t1 < t0 for t0, t1 in zip(totals, totals[1:]))
        assert len(res.step_sizes[b]) == len(totals)


def test_initial_divergence_raises_like_the_reference():
    mr, cfg, lam, rho, src, tgt, z0 = _problem_set(2, torch.float64)
    z0[1] *= 1e9
    with pytest.raises(mr.IntegrationDiverged):
        mr.optimize_batch(torch.as_tensor(src), torch.as_tensor(tgt), torch.as_tensor(z0), cfg, lam,
                          rho, mr.OptimizeConfig(max_iters=1))


def test_host_pipeline_with_explicit_group_sizes_equals_the_device_call():
    """cost_and_grad_batch on host tensors, pair groups given as sizes (objective._host_pipeline)."""
    mr, cfg, lam, rho, src, tgt, z0 = _problem_set(4, torch.float64)
    args = [torch.as_tensor(a) for a in (src, tgt, z0)]
    zb_h, terms_h, guard_h = mr.cost_and_grad_batch(*args, cfg, lam, rho, chunks=[1, 3])
    zb_d, terms_d, guard_d = mr.cost_and_grad_batch(*[a.cuda() for a in args], cfg, lam, rho)
    assert not zb_h.is_cuda
    assert torch.equal(zb_h, zb_d.cpu()) and torch.equal(terms_h, terms_d.cpu())
    assert torch.equal(guard_h, guard_d.cpu())
    with pytest.raises(mr.FieldError):
        mr.cost_and_grad_batch(*args, cfg, lam, rho, chunks=[2, 3])


def test_batched_line_search_runs_in_3d_and_matches_single_pair_runs():
    """optimize_batch is dimension-agnostic: two 3D pairs, each equal to its own run."""
    import paper_2106_08817_b200 as mr

    rng = np.random.default_rng(9)
    shape = (12, 16, 20)
    kern = mr.GaussianKernel(1.5)
    cfg = mr.ShootingConfig(mr.Scheme.SEMI_LAGRANGIAN, 3, 0.2, kern, dtype=torch.float64)

    src = rng.random((2,) + shape)
    tgt = np.clip(src + 0.1 * rng.standard_normal((2,) + shape), 0, 1)
    tgt[1] *= 2.0  # different contrast: different accepted steps
    src[1] *= 2.0
    z0 = np.zeros((2,) + shape)
    ocfg = mr.OptimizeConfig(max_iters=3, init_step=50.0)
    both = mr.optimize_batch(torch.as_tensor(src), torch.as_tensor(tgt), torch.as_tensor(z0), cfg,
                             1e-2, 1.0, ocfg)
    for b in range(2):
        one = mr.optimize_batch(torch.as_tensor(src[b:b + 1]), torch.as_tensor(tgt[b:b + 1]),
                                torch.as_tensor(z0[b:b + 1]), cfg, 1e-2, 1.0, ocfg)
        assert both.terminations[b] == one.terminations[0]
        assert both.step_sizes[b] == one.step_sizes[0]
        assert [h.total for h in both.histories[b]] == pytest.approx(
            [h.total for h in one.histories[0]], rel=1e-12)
        assert torch.allclose(both.z0[b], one.z0[0], rtol=1e-10, atol=1e-14)
        totals = [h.total for h in both.histories[b]]
        assert len(totals) >= 2 and totals[-1] < totals[0]
