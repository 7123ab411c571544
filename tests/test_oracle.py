"""Pin the CPU oracle (oracle/morphreg_oracle.py) before trusting it.

2D: against golden vectors produced by running the reference itself
(tests/golden/make_golden.py).  3D (no reference exists): extrusion onto the
2D goldens, dense-transpose checks of every 3D operator, and finite
differences of the 3D gradient.
"""

import numpy as np
import pytest

from conftest import load_golden, rel_l2, scheme_cases, shoot_cases
from oracle import morphreg_oracle as O


# ---- operators vs reference goldens ---------------------------------------------


def test_ops_match_reference_goldens():
    g = load_golden("ops.npz")
    assert np.allclose(O.gradient(g["grad_in"]), g["grad_out"], atol=1e-15)
    assert np.allclose(O.gradient_adjoint(g["gradT_in"]), g["gradT_out"], atol=1e-14)
    assert np.allclose(O.divergence(g["gradT_in"]), g["div_out"], atol=1e-14)
    p = O.Plan(g["bl_coords"], (9, 11))
    assert np.array_equal(O.interp_apply(g["grad_in"], p), g["bl_apply"])
    assert np.allclose(O.interp_adjoint(p, g["bl_gbar"]), g["bl_adjoint"], atol=1e-14)
    assert np.array_equal(np.stack(O.interp_coord_grad(g["grad_in"], p)), g["bl_coord_grad"])
    for n, sigma in [(3, 1.0), (8, 1.0), (16, 2.0), (5, 3.0), (40, 2.5)]:
        key = f"conv_{n}_{sigma}"
        w = O.gaussian_weights(sigma)
        assert np.array_equal(w, g[key + "_w"])
        a = g[key + "_in"]
        assert np.array_equal(O.conv1d_replicate(a, w, 0), g[key + "_ax0"])
        assert np.array_equal(O.conv1d_replicate_adjoint(a, w, 0), g[key + "_adj0"])
        assert np.array_equal(O.smooth(a, w), g[key + "_smooth"])
        assert np.array_equal(O.smooth_adjoint(a, w), g[key + "_smoothT"])


@pytest.mark.parametrize("case", shoot_cases() + scheme_cases())
def test_oracle_shoot_cost_grad_match_reference(case):
    g = load_golden(case)
    w = O.gaussian_weights(float(g["sigma"]), int(g["radius"]))
    assert np.array_equal(w, g["weights"])
    T, mu = int(g["n_steps"]), float(g["mu"])
    scheme = str(g["scheme"])
    I, z, v, phi = O.shoot(g["source"], g["z0"], T, mu, w, scheme=scheme)
    if "I" in g:
        for k in range(T + 1):
            assert np.array_equal(I[k], g["I"][k]), k
            assert np.array_equal(z[k], g["z"][k]), k
            assert np.array_equal(v[k], g["v"][k]), k
    else:
        for k in (0, T):
            assert np.array_equal(I[k], g[f"I{k}"])
            assert np.array_equal(z[k], g[f"z{k}"])
            assert np.array_equal(v[k], g[f"v{k}"])
    assert np.array_equal(phi, g["phi"])
    c = O.cost(g["source"], g["target"], g["z0"], float(g["lam"]), float(g["rho"]), T, mu, w,
               scheme=scheme)
    assert np.allclose(c, g["cost"], rtol=1e-14, atol=0)
    gr = O.grad(g["source"], g["target"], g["z0"], float(g["lam"]), float(g["rho"]), T, mu, w,
                scheme=scheme)
    assert rel_l2(gr, g["grad"]) < 1e-13


def test_oracle_guard_matches_reference():
    g = load_golden("guard.npz")
    w = O.gaussian_weights(float(g["sigma"]))
    with pytest.raises(O.OracleDiverged) as e:
        O.shoot(g["source"], g["z0"], int(g["n_steps"]), float(g["mu"]), w)
    assert e.value.step == int(g["step"])
    assert e.value.what == str(g["what"])


# ---- 3D generalisation --------------------------------------------------------------


@pytest.mark.parametrize("case", ["shoot_A_16sq.npz", "shoot_B_13x21.npz", "shoot_J_48sq_bigdisp.npz"])
def test_oracle_3d_extrusion_reproduces_2d_reference(case):
    """A volume constant along axis 0 must reproduce the 2D reference per slice."""
    g = load_golden(case)
    D = 3
    w = O.gaussian_weights(float(g["sigma"]), int(g["radius"]))
    T, mu, lam, rho = int(g["n_steps"]), float(g["mu"]), float(g["lam"]), float(g["rho"])
    ext = lambda a: np.repeat(a[None], D, axis=0)  # noqa: E731
    I, z, v, phi = O.shoot(ext(g["source"]), ext(g["z0"]), T, mu, w)
    key_I = g["I"][T] if "I" in g else g[f"I{T}"]
    for s in range(D):
        assert rel_l2(I[T][s], key_I) < 1e-13
        assert np.abs(v[0][0]).max() == 0.0  # no motion along the extruded axis
        assert rel_l2(v[0][1][s], (g["v"][0] if "v" in g else g["v0"])[0]) < 1e-13
    gr3 = O.grad(ext(g["source"]), ext(g["target"]), ext(g["z0"]), lam, rho, T, mu, w)
    # d/dz2 H3(E z2) = sum_s dH3/dz0[s] = D dH2/dz2  ->  axis-0 mean equals the 2D gradient
    assert rel_l2(gr3.mean(axis=0), g["grad"]) < 1e-12


def _dense(op, shape):
    n = int(np.prod(shape))
    cols = []
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        cols.append(np.asarray(op(e.reshape(shape))).ravel())
    return np.stack(cols, axis=1)


@pytest.mark.parametrize("shape", [(3, 4, 5), (2, 3, 2)])
def test_oracle_3d_operator_transposes(shape):
    rng = np.random.default_rng(0)
    w = O.gaussian_weights(1.3)
    for ax in range(3):
        A = _dense(lambda a: O.axis_diff(a, ax), shape)
        At = _dense(lambda a: O.axis_diff_adjoint(a, ax), shape)
        assert np.allclose(A.T, At, atol=1e-14)
        K = _dense(lambda a: O.conv1d_replicate(a, w, ax), shape)
        Kt = _dense(lambda a: O.conv1d_replicate_adjoint(a, w, ax), shape)
        assert np.allclose(K.T, Kt, atol=1e-14)
    S = _dense(lambda a: O.smooth(a, w), shape)
    St = _dense(lambda a: O.smooth_adjoint(a, w), shape)
    assert np.allclose(S.T, St, atol=1e-14)
    coords = O.identity_coords(shape) + rng.uniform(-1.5, 1.5, (3,) + shape)
    p = O.Plan(coords, shape)
    B = _dense(lambda a: O.interp_apply(a, p), shape)
    Bt = _dense(lambda a: O.interp_adjoint(p, a), shape)
    assert np.allclose(B.T, Bt, atol=1e-14)


def test_oracle_3d_trilinear_coord_grad_by_finite_differences():
    rng = np.random.default_rng(1)
    shape = (5, 6, 4)
    f = rng.standard_normal(shape)
    coords = O.identity_coords(shape) + rng.uniform(-0.4, 0.4, (3,) + shape)
    p = O.Plan(coords, shape)
    dd = O.interp_coord_grad(f, p)
    eps = 1e-6
    for ax in range(3):
        cp = coords.copy()
        cp[ax] += eps
        cm = coords.copy()
        cm[ax] -= eps
        fd = (O.interp_apply(f, O.Plan(cp, shape)) - O.interp_apply(f, O.Plan(cm, shape))) / (2 * eps)
        mask = p.inside[ax]
        assert np.allclose(dd[ax][mask], fd[mask], atol=1e-7)


def test_oracle_3d_gradient_finite_differences():
    rng = np.random.default_rng(2)
    shape = (6, 7, 6)
    w = O.gaussian_weights(1.0)
    win = np.zeros(shape)
    win[1:-1, 1:-1, 1:-1] = 1.0
    src = np.abs(O.smooth(rng.standard_normal(shape), w)) * win
    tgt = np.abs(O.smooth(rng.standard_normal(shape), w)) * win
    z0 = 0.3 * O.smooth(rng.standard_normal(shape), w) * win
    T, mu, lam, rho = 3, 0.2, 1e-3, 0.5
    g = O.grad(src, tgt, z0, lam, rho, T, mu, w)
    d = rng.standard_normal(shape)
    d /= np.linalg.norm(d)
    eps = 1e-5
    cp = O.cost(src, tgt, z0 + eps * d, lam, rho, T, mu, w)[0]
    cm = O.cost(src, tgt, z0 - eps * d, lam, rho, T, mu, w)[0]
    fd = (cp - cm) / (2 * eps)
    assert float(np.sum(g * d)) == pytest.approx(fd, rel=1e-6)


def test_oracle_mu_zero_equals_reference_lddmm_path():
    """The reference's separate shoot_lddmm routine (integrator.py:222-277) on a config with
    mu = 0.7: the oracle's shoot at mu = 0 reproduces every state bitwise."""
    g = load_golden("lddmm_path.npz")
    I, z, v, phi = O.shoot(g["source"], g["z0"], int(g["n_steps"]), 0.0, g["weights"], with_phi=True)
    assert np.array_equal(np.stack(I), g["I"])
    assert np.array_equal(np.stack(z), g["z"])
    assert np.array_equal(np.stack(v), g["v"])
    assert np.array_equal(phi, g["phi"])
