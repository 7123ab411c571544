"""Generate golden fixtures by running the REFERENCE package (float64 numpy).

Run in the build container only (needs /root/reference, read-only):

    python tests/golden/make_golden.py

Writes tests/golden/*.npz.  The GPU box never reads /root/reference; tests
there use these committed fixtures.  Vector fields are stored channel-first
([d, H, W]) to match the device layout.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, REPO)

import morphreg  # noqa: E402  (the reference)
from morphreg import (  # noqa: E402
    GaussianKernel,
    GridGeometry,
    IntegrationDiverged,
    RegistrationProblem,
    Scheme,
    ScalarField,
    ShootingConfig,
    cost,
    grad,
    shoot,
)
from morphreg import fields as rf  # noqa: E402
from morphreg import kernel as rk  # noqa: E402
from morphreg.kernel import smooth_arr  # noqa: E402

# (name, shape, seed, T, mu, sigma, radius, amp, lam, rho, full_states)
SHOOT_CASES = [
    ("A_16sq", (16, 16), 0, 5, 0.05, 1.0, None, 0.05, 1e-3, 0.5, True),
    ("B_13x21", (13, 21), 1, 3, 0.5, 1.5, None, 0.3, 1e-2, 1.0, True),
    ("C_24sq_lddmm", (24, 24), 2, 6, 0.0, 2.0, None, 0.5, 1e-3, 0.5, True),
    ("D_5x7_bigr", (5, 7), 3, 2, 0.2, 3.0, None, 0.2, 1e-2, 0.3, True),
    ("E_40x33", (40, 33), 4, 4, 0.3, 2.5, None, 1.0, 1e-3, 1.0, True),
    ("F_2x6", (2, 6), 5, 2, 0.1, 1.0, None, 0.5, 1e-2, 0.5, True),
    ("G_64sq_r24", (64, 64), 6, 5, 0.0, 6.0, 24, 3.0, 1e-4, 1.0, False),
    ("H_100x90_r9", (100, 90), 7, 4, 0.5, 3.0, 9, 3.0, 1e-2, 1.0, False),
    ("I_70x150_r32", (70, 150), 8, 3, 0.2, 8.0, 32, 4.0, 1e-3, 1.0, False),
    # large per-step back-trace offsets (out-of-cell gathers, scatter contention)
    ("J_48sq_bigdisp", (48, 48), 9, 4, 0.1, 2.0, None, 250.0, 1e-3, 1.0, True),
    # momentum up to the border: feet leave the domain (clamp + strict inside mask)
    ("K_60x44_border", (60, 44), 10, 3, 0.2, 2.0, None, 40.0, 1e-3, 1.0, True, 0.0),
]


def instance(shape, seed, amp, margin_frac=0.2, sigma=1.0):
    """Smooth nonnegative source/target and smooth momentum (like tests/conftest.py:16-35)."""
    rng = np.random.default_rng(seed)
    kern = GaussianKernel(sigma)
    h, w = shape
    mh, mw = max(1, int(h * margin_frac)), max(1, int(w * margin_frac))
    win = np.zeros(shape)
    win[mh : h - mh, mw : w - mw] = 1.0
    if h <= 2 or w <= 2 or margin_frac == 0.0:
        win[:] = 1.0

    def field(scale=1.0, nonneg=False):
        a = smooth_arr(kern, rng.standard_normal(shape)) * win
        if nonneg:
            a = np.abs(a)
        return scale * a

    return field(nonneg=True), field(nonneg=True), field(scale=amp)


def cf(v):
    """[H, W, 2] -> [2, H, W]."""
    return np.moveaxis(np.asarray(v), -1, 0)


# Eulerian / Hybrid schemes (integrator.py:97-106, objective.py:124-127,148-155):
# (name, scheme, shape, seed, T, mu, sigma, radius, amp, lam, rho, full_states)
SCHEME_CASES = [
    ("eu_A_16sq", "eulerian", (16, 16), 20, 5, 0.05, 1.0, None, 0.05, 1e-3, 0.5, True),
    ("eu_B_13x21", "eulerian", (13, 21), 21, 3, 0.5, 1.5, None, 0.3, 1e-2, 1.0, True),
    ("eu_C_40x36_r12", "eulerian", (40, 36), 22, 4, 0.3, 3.0, 12, 2.0, 1e-3, 1.0, True),
    ("eu_D_72x100_r24", "eulerian", (72, 100), 23, 4, 0.0, 6.0, 24, 3.0, 1e-4, 1.0, False),
    ("hy_A_16sq", "hybrid", (16, 16), 24, 5, 0.05, 1.0, None, 0.05, 1e-3, 0.5, True),
    ("hy_B_24x20", "hybrid", (24, 20), 25, 3, 0.5, 1.5, None, 0.5, 1e-2, 1.0, True),
    ("hy_C_48sq_bigdisp", "hybrid", (48, 48), 26, 4, 0.1, 2.0, None, 40.0, 1e-3, 1.0, True),
    ("hy_D_66x90_r9", "hybrid", (66, 90), 27, 4, 0.3, 3.0, 9, 3.0, 1e-2, 1.0, False),
]


def shoot_case(name, shape, seed, T, mu, sigma, radius, amp, lam, rho, full, margin=0.2,
               scheme=Scheme.SEMI_LAGRANGIAN, prefix="shoot"):
    src, tgt, z0 = instance(shape, seed, amp, margin_frac=margin)
    geom = GridGeometry(*shape)
    kern = GaussianKernel(sigma, radius)
    cfg = ShootingConfig(scheme, T, mu, kern)
    prob = RegistrationProblem(ScalarField(geom, src), ScalarField(geom, tgt), lam, rho, cfg)
    zf = ScalarField(geom, z0)
    traj = shoot(prob.source, zf, cfg)
    rep = cost(prob, zf)
    g = grad(prob, zf).values
    out = dict(
        source=src, target=tgt, z0=z0, n_steps=T, mu=mu, sigma=sigma, radius=kern.radius,
        lam=lam, rho=rho, weights=kern.weights,
        cost=np.array([rep.total, rep.data_term, rep.v_norm, rep.z_norm]), grad=g,
        phi=cf(traj.deformation.coords), scheme=np.array(scheme.value),
    )
    if full:
        out["I"] = np.stack([s.image.values for s in traj.states])
        out["z"] = np.stack([s.momentum.values for s in traj.states])
        out["v"] = np.stack([cf(s.velocity.values) for s in traj.states])
    else:
        for k in (0, T):
            out[f"I{k}"] = traj.states[k].image.values
            out[f"z{k}"] = traj.states[k].momentum.values
            out[f"v{k}"] = cf(traj.states[k].velocity.values)
    np.savez_compressed(os.path.join(HERE, f"{prefix}_{name}.npz"), **out)
    print(name, "cost", rep.total, "max|grad|", np.abs(g).max(),
          "max disp", np.abs(cf(traj.states[0].velocity.values)).max() / T)


def ops_case():
    """Operator-level goldens: stencils, their transposes, bilinear, conv."""
    rng = np.random.default_rng(123)
    out = {}
    f = rng.standard_normal((9, 11))
    out["grad_in"] = f
    out["grad_out"] = cf(rf.gradient_arr(f))
    g = rng.standard_normal((9, 11, 2))
    out["gradT_in"] = cf(g)
    out["gradT_out"] = rf.gradient_adjoint_arr(g)
    out["div_out"] = rf.divergence_arr(g)
    coords = rf.identity_coords((9, 11)) + rng.uniform(-3, 3, (9, 11, 2))
    coords[0, 0] = [-5.0, 20.0]
    coords[1, 1] = [8.0, 10.0]  # exactly on the far corner
    coords[2, 2] = [0.0, 0.0]
    p = rf.bilinear_plan(coords, (9, 11))
    out["bl_coords"] = cf(coords)
    out["bl_apply"] = rf.bilinear_apply(f, p)
    gb = rng.standard_normal((9, 11))
    out["bl_gbar"] = gb
    out["bl_adjoint"] = rf.bilinear_adjoint_values(p, gb, (9, 11))
    dy, dx = rf.bilinear_coord_grad(f, p)
    out["bl_coord_grad"] = np.stack([dy, dx])
    for n, sigma in [(3, 1.0), (8, 1.0), (16, 2.0), (5, 3.0), (40, 2.5)]:
        k = GaussianKernel(sigma)
        a = rng.standard_normal((n, 7))
        out[f"conv_{n}_{sigma}_in"] = a
        out[f"conv_{n}_{sigma}_w"] = k.weights
        out[f"conv_{n}_{sigma}_ax0"] = rk.conv1d_replicate(a, k.weights, 0)
        out[f"conv_{n}_{sigma}_adj0"] = rk.conv1d_replicate_adjoint(a, k.weights, 0)
        out[f"conv_{n}_{sigma}_smooth"] = rk.smooth_arr(k, a)
        out[f"conv_{n}_{sigma}_smoothT"] = rk.smooth_adjoint_arr(k, a)
    np.savez_compressed(os.path.join(HERE, "ops.npz"), **out)


def lddmm_case():
    """The reference's SEPARATE deformation-only path, shoot_lddmm (integrator.py:222-277),
    on a config whose mu is non-zero (it must be ignored), plus shoot() at mu = 0 on the
    same inputs: the reference keeps them bitwise equal (acceptance criterion 2)."""
    from morphreg import shoot_lddmm

    src, _, z0 = instance((40, 33), 4, 1.0)
    geom = GridGeometry(40, 33)
    kern = GaussianKernel(1.5)
    a = shoot_lddmm(ScalarField(geom, src), ScalarField(geom, z0),
                    ShootingConfig(Scheme.SEMI_LAGRANGIAN, 8, 0.7, kern))
    b = shoot(ScalarField(geom, src), ScalarField(geom, z0),
              ShootingConfig(Scheme.SEMI_LAGRANGIAN, 8, 0.0, kern))
    same = all(x.image.values.tobytes() == y.image.values.tobytes() and
               x.momentum.values.tobytes() == y.momentum.values.tobytes()
               for x, y in zip(a.states, b.states))
    np.savez_compressed(os.path.join(HERE, "lddmm_path.npz"), source=src, z0=z0, n_steps=8,
                        sigma=1.5, weights=kern.weights, mu_in_config=0.7,
                        I=np.stack([s.image.values for s in a.states]),
                        z=np.stack([s.momentum.values for s in a.states]),
                        v=np.stack([cf(s.velocity.values) for s in a.states]),
                        phi=cf(a.deformation.coords), reference_paths_bitwise_equal=same)
    print("lddmm path: reference shoot_lddmm == shoot(mu=0) bitwise:", same)


def guard_case():
    """A momentum that diverges: record (step, what) of IntegrationDiverged."""
    src, tgt, z0 = instance((16, 16), 2, 1.0)
    geom = GridGeometry(16, 16)
    cfg = ShootingConfig(Scheme.SEMI_LAGRANGIAN, 4, 50.0, GaussianKernel(1.0))
    z = ScalarField(geom, z0 * 4e5)
    try:
        shoot(ScalarField(geom, src), z, cfg)
        step, what = -1, ""
    except IntegrationDiverged as e:
        step, what = e.step, e.what
    np.savez_compressed(os.path.join(HERE, "guard.npz"), source=src, z0=z0 * 4e5, n_steps=4,
                        mu=50.0, sigma=1.0, step=step, what=what)
    print("guard", step, what)


def config1_case():
    """BASELINE config 1 at full size: inputs from our generator, outputs from the reference."""
    from paper_2106_08817_b200.synthetic import make_config

    c = make_config(1)
    src, tgt, z0 = c.source[0], c.target[0], c.z0[0]
    geom = GridGeometry(*src.shape)
    kern = GaussianKernel(c.sigma, c.radius)
    cfg = ShootingConfig(Scheme.SEMI_LAGRANGIAN, c.n_steps, c.mu, kern)
    prob = RegistrationProblem(ScalarField(geom, src), ScalarField(geom, tgt), c.lam, c.rho, cfg)
    zf = ScalarField(geom, z0)
    traj = shoot(prob.source, zf, cfg)
    rep = cost(prob, zf)
    g = grad(prob, zf).values
    # 20 fixed-step gradient-descent iterations at 1e-2 (the config's schedule)
    z = z0.copy()
    hist = []
    for _ in range(20):
        r = cost(prob, ScalarField(geom, z))
        hist.append([r.total, r.data_term, r.v_norm, r.z_norm])
        z = z - 1e-2 * grad(prob, ScalarField(geom, z)).values
    r = cost(prob, ScalarField(geom, z))
    hist.append([r.total, r.data_term, r.v_norm, r.z_norm])
    np.savez_compressed(
        os.path.join(HERE, "config1.npz"),
        source=src, target=tgt, z0=z0, IT=traj.states[-1].image.values,
        zT=traj.states[-1].momentum.values, v0=cf(traj.states[0].velocity.values),
        cost=np.array([rep.total, rep.data_term, rep.v_norm, rep.z_norm]), grad=g,
        gd_history=np.array(hist), gd_final_z=z,
    )
    print("config1 cost", rep.total, "-> after 20 GD", hist[-1][0])


if __name__ == "__main__":
    print("reference morphreg", morphreg.__version__, "numpy", np.__version__)
    if "--only-lddmm" in sys.argv:
        lddmm_case()
        sys.exit(0)
    ops_case()
    guard_case()
    lddmm_case()
    for case in SHOOT_CASES:
        shoot_case(*case)
    for name, scheme, *rest in SCHEME_CASES:
        shoot_case(name, *rest, scheme=Scheme(scheme), prefix="scheme")
    config1_case()
