"""Array-level operators of the reference API on the device (mr_ops.cu through
the C-ABI) against the oracle restatement of fields.py / kernel.py, plus the
field-level facade functions the reference re-exports (gradient, divergence,
interpolate, interpolate_vec, dot, ssd, single-step transport, path_energy)."""

import numpy as np
import pytest
import torch

from conftest import load_golden, rel_l2

pytestmark = pytest.mark.gpu

SHAPES = [(9, 7), (2, 5), (6, 5, 4), (2, 3, 7), (11,), (2,)]


def _O():
    from oracle import morphreg_oracle as O

    return O


def _rng(seed=0):
    return np.random.default_rng(seed)


@pytest.mark.parametrize("shape", SHAPES, ids=str)
def test_axis_diff_and_transpose(shape):
    from paper_2106_08817_b200 import fields as F

    O = _O()
    a = _rng(1).standard_normal(shape)
    for ax in range(len(shape)):
        # forward np.gradient: bitwise in float64 (same formula, same rounding)
        assert np.array_equal(F.axis_diff(a, ax), O.axis_diff(a, ax))
        assert rel_l2(F.axis_diff_adjoint(a, ax), O.axis_diff_adjoint(a, ax)) < 1e-15
        # float32 torch operands stay float32 on the device
        t = torch.as_tensor(a, dtype=torch.float32, device="cuda")
        r = F.axis_diff(t, ax)
        assert r.dtype == torch.float32 and r.is_cuda
        assert rel_l2(r.cpu(), O.axis_diff(a, ax)) < 1e-6


def test_axis_diff_adjoint_is_dense_transpose():
    """test_fields.py:125-135 analogue: <D e_i, e_j> matrix transposed."""
    from paper_2106_08817_b200 import fields as F

    n, m = 6, 4
    for ax in (0, 1):
        mat = np.zeros((n * m, n * m))
        for i in range(n * m):
            e = np.zeros(n * m)
            e[i] = 1.0
            mat[:, i] = F.axis_diff(e.reshape(n, m), ax).ravel()
        g = _rng(2).standard_normal((n, m))
        assert np.allclose(F.axis_diff_adjoint(g, ax).ravel(), mat.T @ g.ravel(), atol=1e-14)


@pytest.mark.parametrize("shape", SHAPES[:4], ids=str)
def test_gradient_divergence_and_adjoints(shape):
    from paper_2106_08817_b200 import fields as F

    O = _O()
    d = len(shape)
    f = _rng(3).standard_normal(shape)
    v = _rng(4).standard_normal(shape + (d,))
    assert np.array_equal(F.gradient_arr(f), np.moveaxis(O.gradient(f), 0, -1))
    assert np.array_equal(F.divergence_arr(v), O.divergence(np.moveaxis(v, -1, 0)))
    assert rel_l2(F.gradient_adjoint_arr(v), O.gradient_adjoint(np.moveaxis(v, -1, 0))) < 1e-15
    da = F.divergence_adjoint_arr(f)
    for ax in range(d):
        assert rel_l2(da[..., ax], O.axis_diff_adjoint(f, ax)) < 1e-15


def test_field_gradient_divergence_match_reference_goldens():
    """gradient / divergence of the reference (fields.py:179-186) on golden data."""
    import paper_2106_08817_b200 as mr

    O = _O()
    g = load_golden("shoot_E_40x33.npz")
    f = mr.ScalarField.from_array(g["source"])
    gr = mr.gradient(f)
    assert np.array_equal(gr.values, np.moveaxis(O.gradient(g["source"]), 0, -1))
    dv = mr.divergence(gr)
    assert np.array_equal(dv.values, O.divergence(O.gradient(g["source"])))


@pytest.mark.parametrize("shape,sigma,radius", [((12, 9), 1.5, None), ((5, 7), 2.0, 9),
                                                ((6, 5, 8), 1.0, 3), ((2, 3), 1.0, 4),
                                                ((16,), 2.0, None), ((3,), 1.0, None)], ids=str)
def test_conv1d_and_transpose(shape, sigma, radius):
    from paper_2106_08817_b200 import kernel as K

    O = _O()
    w = O.gaussian_weights(sigma, radius)
    a = _rng(5).standard_normal(shape)
    for ax in range(len(shape)):
        # forward: the reference's tap loop order with separately rounded products
        assert np.array_equal(K.conv1d_replicate(a, w, ax), O.conv1d_replicate(a, w, ax))
        assert rel_l2(K.conv1d_replicate_adjoint(a, w, ax),
                      O.conv1d_replicate_adjoint(a, w, ax)) < 1e-14


def test_conv1d_adjoint_is_dense_transpose():
    """test_kernel.py:98-109 analogue, radius larger than the axis."""
    from paper_2106_08817_b200 import kernel as K

    O = _O()
    w = O.gaussian_weights(2.0, 9)
    n = 7
    mat = np.zeros((n, n))
    for i in range(n):
        e = np.zeros((n, 3))
        e[i] = 1.0
        mat[:, i] = K.conv1d_replicate(e, w, 0)[:, 0]
    g = _rng(6).standard_normal((n, 3))
    assert np.allclose(K.conv1d_replicate_adjoint(g, w, 0), mat.T @ g, atol=1e-14)


@pytest.mark.parametrize("shape", [(16, 12), (7, 9, 6)], ids=str)
def test_smoothing_arrays_match_oracle(shape):
    from paper_2106_08817_b200 import kernel as K

    O = _O()
    k = K.GaussianKernel(1.5)
    a = _rng(7).standard_normal(shape)
    assert rel_l2(K.smooth_arr(k, a), O.smooth(a, k.weights)) < 1e-14
    assert rel_l2(K.smooth_adjoint_arr(k, a), O.smooth_adjoint(a, k.weights)) < 1e-14
    m = _rng(8).standard_normal(shape + (len(shape),))
    vn = K.v_norm_sq_arr(k, m)
    assert vn == pytest.approx(O.v_norm_sq(np.moveaxis(m, -1, 0), k.weights), rel=1e-13)


@pytest.mark.parametrize("shape", [(9, 7), (5, 6, 4)], ids=str)
def test_interpolation_operators_match_oracle(shape):
    from paper_2106_08817_b200 import fields as F

    O = _O()
    d = len(shape)
    rng = _rng(9)
    a = rng.standard_normal(shape)
    # feet inside, outside (clamped) and exactly on nodes / borders
    coords = O.identity_coords(shape) + rng.uniform(-2.5, 2.5, (d,) + shape)
    coords[:, 0] = np.round(coords[:, 0])
    coords[0, -1] = shape[0] - 1
    p_ref = O.Plan(coords, shape)
    p = F.bilinear_plan(np.moveaxis(coords, 0, -1), shape)
    assert np.array_equal(F.bilinear_apply(a, p), O.interp_apply(a, p_ref))
    g = rng.standard_normal(shape)
    assert rel_l2(F.bilinear_adjoint_values(p, g, shape), O.interp_adjoint(p_ref, g)) < 1e-14
    cg = F.bilinear_coord_grad(a, p)
    ref = O.interp_coord_grad(a, p_ref)
    for ax in range(d):
        assert np.array_equal(cg[ax], ref[ax]), ax


def test_interpolate_identity_bitwise_and_nonfinite_rejected():
    """test_fields.py:139-143; bilinear_plan's FieldError (fields.py:208-209)."""
    import paper_2106_08817_b200 as mr

    f = mr.ScalarField.from_array(_rng(10).standard_normal((9, 7)))
    out = mr.interpolate(f, mr.SampleGrid.identity(f.geometry))
    assert out.values.tobytes() == f.values.tobytes()
    v = mr.VectorField.from_array(_rng(11).standard_normal((9, 7, 2)))
    assert np.array_equal(mr.interpolate_vec(v, mr.SampleGrid.identity(v.geometry)).values,
                          v.values)
    from paper_2106_08817_b200 import fields as F

    bad = np.moveaxis(_O().identity_coords((4, 4)), 0, -1).copy()
    bad[1, 2, 0] = np.nan
    with pytest.raises(mr.FieldError, match="non-finite"):
        F.bilinear_plan(bad, (4, 4))


def test_dot_and_ssd_device_reductions():
    import paper_2106_08817_b200 as mr

    rng = _rng(12)
    a, b = rng.standard_normal((33, 20)), rng.standard_normal((33, 20))
    fa, fb = mr.ScalarField.from_array(a), mr.ScalarField.from_array(b)
    assert mr.dot(fa, fb) == pytest.approx(float(np.sum(a * b)), rel=1e-13)
    assert mr.ssd(fa, fb) == pytest.approx(0.5 * float(np.sum((a - b) ** 2)), rel=1e-13)
    assert mr.ssd(fa, fa) == 0.0
    # deterministic: same bits twice
    assert mr.dot(fa, fb) == mr.dot(fa, fb)


@pytest.mark.parametrize("scheme", ["semi-lagrangian", "eulerian"])
def test_single_step_operators_match_oracle_and_shoot(scheme):
    """advect_image_* / continuity_* (integrator.py:133-159) against the oracle,
    and one shoot step equals the hand composition bitwise (test_integrator.py:184-194)."""
    import paper_2106_08817_b200 as mr

    O = _O()
    g = load_golden("shoot_E_40x33.npz")
    I0, z0, w = g["source"], g["z0"], g["weights"]
    mu, dt = 0.2, 0.25
    k = mr.GaussianKernel(1.0)
    k.weights = w  # golden taps (same construction)
    fi, fz = mr.ScalarField.from_array(I0), mr.ScalarField.from_array(z0)
    v = mr.velocity_from_momentum(fz, fi, k)
    assert v.tensor.dtype == torch.float64
    vref = O.velocity(z0, O.gradient(I0), w)
    assert rel_l2(np.moveaxis(v.values, -1, 0), vref) < 1e-13
    S = mr.Scheme(scheme)
    if S is mr.Scheme.SEMI_LAGRANGIAN:
        i1 = mr.integrator.advect_image_sl(fi, v, fz, mu, dt)
        z1 = mr.integrator.continuity_sl(fz, v, dt)
    else:
        i1 = mr.integrator.advect_image_euler(fi, v, fz, mu, dt)
        z1 = mr.integrator.continuity_euler(fz, v, dt)
    Iref, zref, _, _ = O.shoot(I0, z0, 1, mu, w, with_phi=False, scheme=scheme)
    # O.shoot uses dt = 1/n_steps = 1: compare a dt = 1 step against it
    if S is mr.Scheme.SEMI_LAGRANGIAN:
        i1b = mr.integrator.advect_image_sl(fi, v, fz, mu, 1.0)
        z1b = mr.integrator.continuity_sl(fz, v, 1.0)
    else:
        i1b = mr.integrator.advect_image_euler(fi, v, fz, mu, 1.0)
        z1b = mr.integrator.continuity_euler(fz, v, 1.0)
    assert rel_l2(i1b.values, Iref[1]) < 1e-12
    assert rel_l2(z1b.values, zref[1]) < 1e-12
    assert i1.values.shape == I0.shape and z1.values.shape == z0.shape
    cfg = mr.ShootingConfig(S, 1, mu, k, dtype=torch.float64)
    traj = mr.shoot(fi, fz, cfg)
    assert np.array_equal(traj.states[1].image.values, i1b.values)
    assert np.array_equal(traj.states[1].momentum.values, z1b.values)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64], ids=["fp32", "fp64"])
def test_path_energy_honours_its_kernel(dtype):
    """integrator.py:280-289: energies from the kernel ARGUMENT, not the shoot's."""
    import paper_2106_08817_b200 as mr

    O = _O()
    g = load_golden("shoot_E_40x33.npz")
    T, mu = int(g["n_steps"]), float(g["mu"])
    k_shoot = mr.GaussianKernel(float(g["sigma"]), int(g["radius"]))
    k_shoot.weights = g["weights"]
    cfg = mr.ShootingConfig(mr.Scheme.SEMI_LAGRANGIAN, T, mu, k_shoot, dtype=dtype)
    traj = mr.shoot(mr.ScalarField.from_array(g["source"]), mr.ScalarField.from_array(g["z0"]),
                    cfg)
    rho = 0.7
    tol = 1e-12 if dtype == torch.float64 else 1e-5
    for k2 in (k_shoot, mr.GaussianKernel(1.25), mr.GaussianKernel(2.0, radius=3)):
        e = mr.path_energy(traj, k2, rho)
        assert len(e) == T + 1
        for t in range(T + 1):
            It, zt = g["I"][t], g["z"][t]
            m = zt * O.gradient(It)
            ref = O.v_norm_sq(m, k2.weights) + rho * float(np.sum(zt * zt))
            assert e[t] == pytest.approx(ref, rel=max(tol, 1e-4 if dtype == torch.float32 else 0))
    # a trajectory without a device copy (states only) gives the same energies
    bare = mr.GeodesicTrajectory(states=traj.states, deformation=traj.deformation)
    assert np.allclose(mr.path_energy(bare, k_shoot, rho), mr.path_energy(traj, k_shoot, rho),
                       rtol=1e-12)
