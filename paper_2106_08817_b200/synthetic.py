"""Seeded synthetic inputs for the five BASELINE.json configurations.

Input generation only (host, float64, numpy/scipy) -- not part of the shooting
path.  Conventions mirror the reference's ``synthetic.py`` (default_rng seeds,
strict masks ``r < R`` as in synthetic.py:57-61, blur by the replicate-border
Gaussian of kernel.py with radius ceil(4 sigma)).  Every choice the configs
leave open is resolved as in SURVEY.md Appendix C and recorded in
``ConfigData.manifest``.  The benchmark suites of the reference are not used:
these are seeded stand-ins with the configs' shapes, sizes and value ranges.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np
from scipy.ndimage import correlate1d

__all__ = ["ConfigData", "CONFIGS", "make_config", "gaussian_weights", "smooth_np",
           "interp_np", "velocity_np", "calibrate_momentum"]


def gaussian_weights(sigma: float, radius: int | None = None) -> np.ndarray:
    r = int(math.ceil(4 * sigma)) if radius is None else int(radius)
    x = np.arange(-r, r + 1, dtype=np.float64)
    w = np.exp(-0.5 * (x / float(sigma)) ** 2)
    return w / np.sum(w)


def smooth_np(a: np.ndarray, sigma: float, radius: int | None = None) -> np.ndarray:
    """Separable replicate-border Gaussian, last axis first (kernel.py:71-73 order)."""
    w = gaussian_weights(sigma, radius)
    out = np.asarray(a, dtype=np.float64)
    for ax in reversed(range(out.ndim)):
        out = correlate1d(out, w, axis=ax, mode="nearest")
    return out


def _grad_np(f: np.ndarray) -> np.ndarray:
    return np.stack([np.gradient(f, axis=ax) for ax in range(f.ndim)])


def velocity_np(z: np.ndarray, img: np.ndarray, sigma: float, radius: int | None) -> np.ndarray:
    """-K*(z grad I) on the host, used only to calibrate momentum amplitudes."""
    g = _grad_np(img)
    return np.stack([-smooth_np(z * g[c], sigma, radius) for c in range(img.ndim)])


def interp_np(arr: np.ndarray, coords: np.ndarray) -> np.ndarray:
    """Multilinear interpolation with the reference clamp (fields.py:207-240)."""
    shape = arr.shape
    d = arr.ndim
    i0s, fs = [], []
    for ax in range(d):
        n = shape[ax]
        cc = np.clip(coords[ax], 0.0, float(n - 1))
        i0 = np.minimum(np.floor(cc).astype(np.intp), n - 2)
        i0s.append(i0)
        fs.append(cc - i0)
    out = np.zeros(coords.shape[1:])
    for c in range(1 << d):
        w = None
        idx = []
        for ax in range(d):
            bit = (c >> ax) & 1
            wa = fs[ax] if bit else 1.0 - fs[ax]
            w = wa if w is None else w * wa
            idx.append(i0s[ax] + bit)
        out = out + w * arr[tuple(idx)]
    return out


def _identity(shape) -> np.ndarray:
    return np.stack(np.meshgrid(*[np.arange(n, dtype=np.float64) for n in shape], indexing="ij"))


def _random_warp(rng, img: np.ndarray, sigma: float, max_disp: float) -> np.ndarray:
    """J(x) = B(I)(x + u(x)), u a smoothed Gaussian random field scaled to max |u|_2."""
    d = img.ndim
    u = np.stack([smooth_np(rng.standard_normal(img.shape), sigma) for _ in range(d)])
    norm = np.sqrt(np.sum(u * u, axis=0))
    u *= max_disp / max(float(norm.max()), 1e-30)
    return interp_np(img, _identity(img.shape) + u)


def calibrate_momentum(rng, img: np.ndarray, sigma: float, radius: int | None, n_steps: int,
                       offset: float, noise_sigma: float = 2.0) -> np.ndarray:
    """z0 = s (G*xi) |grad I| / max|grad I| with s so that dt * max|v0|_2 == offset."""
    zeta = smooth_np(rng.standard_normal(img.shape), noise_sigma)
    g = _grad_np(img)
    gm = np.sqrt(np.sum(g * g, axis=0))
    z = zeta * gm / max(float(gm.max()), 1e-30)
    v = velocity_np(z, img, sigma, radius)
    vmax = float(np.sqrt(np.sum(v * v, axis=0)).max())
    dt = 1.0 / n_steps
    return z * (offset / max(dt * vmax, 1e-30))


@dataclass
class ConfigData:
    name: str
    source: np.ndarray  # [B, *shape] float64
    target: np.ndarray
    z0: np.ndarray
    n_steps: int
    sigma: float
    radius: int
    mu: float
    lam: float
    rho: float
    manifest: dict = field(default_factory=dict)

    @property
    def batch(self) -> int:
        return self.source.shape[0]

    @property
    def shape(self):
        return tuple(self.source.shape[1:])

    @property
    def voxel_steps(self) -> int:
        return int(np.prod(self.shape)) * self.batch * self.n_steps

    def weights(self) -> np.ndarray:
        return gaussian_weights(self.sigma, self.radius)


CONFIGS = {
    1: dict(name="cfg1_2d_metamorphosis_200", ndim=2, batch=1, shape=(200, 200), n_steps=10,
            sigma=3.0, radius=9, mu=0.5, lam=1e-2, rho=1.0, gd_iters=20, gd_step=1e-2),
    2: dict(name="cfg2_2d_lddmm_64x512", ndim=2, batch=64, shape=(512, 512), n_steps=20,
            sigma=6.0, radius=24, mu=0.0, lam=1e-4, rho=1.0, offset=1.0),
    3: dict(name="cfg3_3d_metamorphosis_160x192x160", ndim=3, batch=1, shape=(160, 192, 160),
            n_steps=20, sigma=4.0, radius=16, mu=0.3, lam=1e-4, rho=1.0, offset=1.0),
    4: dict(name="cfg4_3d_metamorphosis_32x128", ndim=3, batch=32, shape=(128, 128, 128),
            n_steps=15, sigma=3.0, radius=12, mu=0.3, lam=1e-4, rho=1.0, offset=1.0),
    5: dict(name="cfg5_3d_stress_256", ndim=3, batch=1, shape=(256, 256, 256), n_steps=50,
            sigma=8.0, radius=24, mu=0.3, lam=1e-4, rho=1.0, offset=3.0),
}


# --- config 1 ------------------------------------------------------------------


def _config1(seed: int, shape=(200, 200)):
    n0, n1 = shape
    ii, jj = np.meshgrid(np.arange(n0, dtype=np.float64), np.arange(n1, dtype=np.float64),
                         indexing="ij")
    c0, c1 = (n0 - 1) / 2.0, (n1 - 1) / 2.0
    src = (np.hypot(ii - c0, jj - c1) < 40.0).astype(np.float64)
    src = smooth_np(src, 1.5)
    cy, cx = c0 + 8.0, c1 - 5.0
    tgt = (((ii - cy) / 50.0) ** 2 + ((jj - cx) / 32.0) ** 2 < 1.0).astype(np.float64)
    tgt[(np.abs(ii - cy) < 6.0) & (np.abs(jj - cx) < 6.0)] = 0.5
    tgt = smooth_np(tgt, 1.5)
    rng = np.random.default_rng(seed)
    z0 = smooth_np(rng.normal(0.0, 0.01, shape), 2.0)
    return src, tgt, z0


# --- config 2 ------------------------------------------------------------------


def _random_ellipses_2d(rng, shape):
    n0, n1 = shape
    ii, jj = np.meshgrid(np.arange(n0, dtype=np.float64), np.arange(n1, dtype=np.float64),
                         indexing="ij")
    img = np.zeros(shape)
    for _ in range(int(rng.integers(3, 7))):
        a = rng.uniform(20.0, 120.0) / 2.0
        b = rng.uniform(20.0, 120.0) / 2.0
        th = rng.uniform(0.0, math.pi)
        cy = rng.uniform(0.2 * n0, 0.8 * n0)
        cx = rng.uniform(0.2 * n1, 0.8 * n1)
        val = rng.uniform(0.2, 1.0)
        u = (ii - cy) * math.cos(th) + (jj - cx) * math.sin(th)
        w = -(ii - cy) * math.sin(th) + (jj - cx) * math.cos(th)
        img += val * ((u / a) ** 2 + (w / b) ** 2 < 1.0)
    return smooth_np(img, 2.0)


def _config2_pair(seed: int, spec, shape):
    rng = np.random.default_rng(seed)
    src = _random_ellipses_2d(rng, shape)
    tgt = _random_warp(rng, src, 24.0, 10.0)
    z0 = calibrate_momentum(rng, src, spec["sigma"], spec["radius"], spec["n_steps"],
                            spec["offset"])
    return src, tgt, z0


# --- 3D phantoms (configs 3-5) ---------------------------------------------------


def _ellipsoid(shape, center, semi, rot=None):
    grids = np.meshgrid(*[np.arange(n, dtype=np.float64) for n in shape], indexing="ij")
    x = np.stack([g - c for g, c in zip(grids, center)])
    if rot is not None:
        x = np.tensordot(rot, x, axes=1)
    return np.sum((x / np.asarray(semi, dtype=np.float64).reshape(-1, 1, 1, 1)) ** 2, axis=0) < 1.0


def _brain_pair(seed: int, shape, scale: float, lesion_r: float | None, spec):
    rng = np.random.default_rng(seed)
    c = tuple((n - 1) / 2.0 for n in shape)
    outer_s = (70 * scale, 85 * scale, 70 * scale)
    inner_s = (50 * scale, 60 * scale, 50 * scale)
    outer = _ellipsoid(shape, c, outer_s)
    inner = _ellipsoid(shape, c, inner_s)
    img = 0.3 * outer.astype(np.float64)
    img[inner] = 0.7
    img += smooth_np(rng.normal(0.0, 0.02, shape), 3.0 * scale) * outer
    img = smooth_np(img, 1.0)
    tgt = _random_warp(rng, img, 12.0 * scale, 6.0 * scale)
    r = lesion_r if lesion_r is not None else float(rng.uniform(6.0, 16.0))
    room = np.maximum(np.asarray(inner_s) - r - 2.0, 0.0)
    off = rng.uniform(-0.5, 0.5, 3) * room
    sphere = _ellipsoid(shape, tuple(np.asarray(c) + off), (r, r, r))
    tgt[sphere] = 0.9
    z0 = calibrate_momentum(rng, img, spec["sigma"], spec["radius"], spec["n_steps"],
                            spec["offset"])
    return img, tgt, z0, r


def _random_ellipsoids_3d(rng, shape):
    img = np.zeros(shape)
    for _ in range(int(rng.integers(3, 7))):
        semi = rng.uniform(20.0, 120.0, 3) / 2.0
        q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
        center = tuple(rng.uniform(0.2 * n, 0.8 * n) for n in shape)
        img += rng.uniform(0.2, 1.0) * _ellipsoid(shape, center, semi, rot=q)
    return smooth_np(img, 2.0)


def _stress_pair(seed: int, shape, spec):
    rng = np.random.default_rng(seed)
    img = _random_ellipsoids_3d(rng, shape)
    tgt = _random_warp(rng, img, 16.0, 20.0)
    z0 = calibrate_momentum(rng, img, spec["sigma"], spec["radius"], spec["n_steps"],
                            spec["offset"])
    return img, tgt, z0


# --- entry point ------------------------------------------------------------------


def make_config(idx: int, seed: int = 0, batch: int | None = None, pairs=None,
                shape=None, mu: float | None = None) -> ConfigData:
    """Inputs of BASELINE config ``idx`` (1..5).

    ``batch`` truncates a batched config to its first pairs; ``pairs`` selects
    explicit pair indices (per-rank sharding: pair p uses seed ``seed + p``).
    ``shape`` overrides the grid (reduced-size parity cases of the same recipe).
    ``mu`` overrides the metamorphosis weight (e.g. the mu = 0 LDDMM variant of
    config 5, which stays finite at the nominal 3 vox/step offset).
    """
    spec = dict(CONFIGS[idx])
    if mu is not None:
        spec["mu"] = float(mu)
        spec["name"] = spec["name"] + f"_mu{float(mu):g}"
    shp = tuple(shape) if shape is not None else spec["shape"]
    if pairs is None:
        pairs = list(range(batch if batch is not None else spec["batch"]))
    manifest = {"config": idx, "seed": seed, "pairs": list(pairs), "shape": list(shp),
                "ambiguities": "SURVEY.md Appendix C", "offset_nominal": spec.get("offset"),
                "mu": spec["mu"]}
    if idx not in CONFIGS:
        raise ValueError(f"unknown config {idx}")

    def one(p):
        s = seed + p
        if idx == 1:
            return _config1(s, shp) + (None,)
        if idx == 2:
            return _config2_pair(s, spec, shp) + (None,)
        if idx in (3, 4):
            scale = 1.0 if idx == 3 else 128.0 / 192.0
            if shape is not None:
                scale *= shp[1] / spec["shape"][1]
            lr = 14.0 * scale if idx == 3 else None
            return _brain_pair(s, shp, scale, lr, spec)
        return _stress_pair(s, shp, spec) + (None,)

    # pairs are independent and seeded per pair: generate them concurrently
    # (scipy's correlate1d releases the GIL); results do not depend on order
    from concurrent.futures import ThreadPoolExecutor

    workers = max(1, min(len(pairs), os.cpu_count() or 1, 16))
    with ThreadPoolExecutor(workers) as ex:
        out = list(ex.map(one, pairs))
    srcs = [o[0] for o in out]
    tgts = [o[1] for o in out]
    zs = [o[2] for o in out]
    if idx in (3, 4):
        manifest["lesion_radius"] = [o[3] for o in out]
    return ConfigData(
        name=spec["name"], source=np.stack(srcs), target=np.stack(tgts), z0=np.stack(zs),
        n_steps=spec["n_steps"], sigma=spec["sigma"], radius=spec["radius"], mu=spec["mu"],
        lam=spec["lam"], rho=spec["rho"], manifest=manifest,
    )
