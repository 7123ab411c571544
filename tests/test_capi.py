"""CPU-side checks of the boundary: the C-ABI library loads and exports every
symbol include/morphreg_sm100.h declares; host logic needs no GPU."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO, load_golden

HEADER = os.path.join(REPO, "include", "morphreg_sm100.h")
LIB = os.path.join(REPO, "paper_2106_08817_b200", "libmorphreg_sm100.so")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mr_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_expected_entry_points():
    from paper_2106_08817_b200 import _lib

    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        pytest.fail(f"{LIB} not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(LIB)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    lib.mr_version.restype = ctypes.c_int
    assert lib.mr_version() == 1


def test_library_rejects_bad_arguments_without_gpu():
    """Validation happens before any CUDA call, so it runs on the CPU host."""
    from paper_2106_08817_b200 import _lib

    lib = _lib.load_library(require_cuda=False)
    g = _lib.make_grid(1, (1, 5))
    rc = lib.mr_velocity(0, g, _lib.KernelHandle(np.ones(3) / 3).struct, None, None, None, None, None,
                         None)
    assert rc == 1
    assert b"at least 2x2" in lib.mr_last_error()
    g = _lib.make_grid(1, (8, 8))
    k = _lib.MrKernel()
    k.radius = 40
    # 8 scalars per pixel, then the tail: fixed-point accumulators (16 B/px), the
    # per-pair max, the overflow flag and the cost partials (1024 blocks x 4 fp64)
    r = lambda x: (x + 255) // 256 * 256  # noqa: E731
    tail = r(16 * 64) + r(8) + 256 + r(1024 * 4 * 8)
    assert lib.mr_adjoint_workspace_bytes(0, g) == r(8 * 8 * 8 * 4) + tail
    assert lib.mr_adjoint_workspace_bytes(1, g) == r(8 * 8 * 8 * 8) + tail
    assert lib.mr_cost_workspace_bytes(0, g) == 1024 * 4 * 8
    with pytest.raises(Exception):
        _lib.KernelHandle(np.ones(81) / 81)  # radius 40 > MR_MAX_RADIUS


def test_product_path_fails_loudly_without_cuda(monkeypatch):
    import torch

    from paper_2106_08817_b200 import _lib

    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.load_library()


def test_package_never_imports_the_oracle():
    pkg = os.path.join(REPO, "paper_2106_08817_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(root, f)).read()
                for bad in ("import oracle", "from oracle", "morphreg_oracle", "__import__("):
                    assert bad not in src, (f, bad)


def test_config1_generator_reproduces_golden_inputs():
    from paper_2106_08817_b200.synthetic import make_config

    g = load_golden("config1.npz")
    c = make_config(1)
    assert np.allclose(c.source[0], g["source"], rtol=0, atol=1e-15)
    assert np.allclose(c.target[0], g["target"], rtol=0, atol=1e-15)
    assert np.allclose(c.z0[0], g["z0"], rtol=0, atol=1e-17)


def test_guard_bit_order_matches_reference_check_order():
    from paper_2106_08817_b200 import _lib
    from paper_2106_08817_b200.engine import guard_report

    import torch

    g = torch.zeros((2, 5), dtype=torch.int32)
    assert guard_report(g) is None
    g[1, 3] = (1 << 5) | (1 << 2)  # velocity magnitude + momentum non-finite
    g[1, 4] = 1
    assert guard_report(g) == (1, 3, "non-finite momentum")
    assert [w for _, w in _lib.GUARD_BITS][0] == "non-finite image"


def test_operator_entry_points_validate_without_gpu():
    """The array-level operators reject bad arguments before any CUDA call."""
    from paper_2106_08817_b200 import _lib

    lib = _lib.load_library(require_cuda=False)
    g = _lib.make_grid(1, (8, 8))
    assert lib.mr_axis_diff(0, g, 2, None, None, 0, None) == 1  # axis out of range (2D)
    assert b"axis" in lib.mr_last_error()
    assert lib.mr_conv1d(0, g, _lib.KernelHandle(np.ones(3) / 3).struct, 0, None, None, 0,
                         None) == 1
    assert lib.mr_reduce(0, g, 7, None, None, None, None) == 1
    assert lib.mr_scheme_step(0, g, 9, 0.1, 0.0, None, None, None, None, None, None, None,
                              None) == 1
    assert lib.mr_interpolate(0, _lib.make_grid(1, (1, 8)), None, None, None, 1, None,
                              None) == 1


def test_bench_gpus_flag_relaunches_one_rank_per_gpu():
    """`bench.py --gpus N` outside torchrun execs N ranks."""
    import json
    import subprocess
    import sys

    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "4",
                          "--steps", "2", "--print-launch"], capture_output=True, text=True,
                         check=True, env={k: v for k, v in os.environ.items()
                                          if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")})
    cmd = json.loads(out.stdout.strip().splitlines()[-1])["launch"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[cmd.index(os.path.join(REPO, "bench.py")) + 1:][:2] == ["--gpus", "4"]


def test_morphreg_shim_exposes_reference_names():
    """tools/morphreg_shim maps every name the reference's tests import onto the
    facade (fp64 ShootingConfig); importing needs no GPU."""
    import importlib
    import sys

    shim = os.path.join(REPO, "tools", "morphreg_shim")
    sys.path.insert(0, shim)
    try:
        for m in [k for k in sys.modules if k == "morphreg" or k.startswith("morphreg.")]:
            del sys.modules[m]
        mr = importlib.import_module("morphreg")
        import torch

        for name in ("FieldError", "GridGeometry", "ScalarField", "VectorField", "SampleGrid",
                     "gradient", "divergence", "interpolate", "interpolate_vec", "dot", "ssd",
                     "GaussianKernel", "smooth_scalar", "smooth_vector", "v_norm_sq", "Scheme",
                     "ShootingConfig", "GeodesicState", "GeodesicTrajectory",
                     "IntegrationDiverged", "velocity_from_momentum", "shoot", "shoot_lddmm",
                     "path_energy", "RegistrationProblem", "CostReport", "cost", "grad",
                     "OptimizeConfig", "OptimizeResult", "Termination", "optimize",
                     "default_init"):
            assert hasattr(mr, name), name
        fields = importlib.import_module("morphreg.fields")
        for name in ("axis_diff", "axis_diff_adjoint", "bilinear_adjoint_values",
                     "bilinear_apply", "bilinear_plan", "identity_coords", "gradient_arr"):
            assert hasattr(fields, name), name
        kern = importlib.import_module("morphreg.kernel")
        for name in ("conv1d_replicate", "conv1d_replicate_adjoint", "smooth_adjoint_arr",
                     "smooth_arr", "smooth_scalar", "smooth_vector", "v_norm_sq",
                     "v_norm_sq_arr"):
            assert hasattr(kern, name), name
        integ = importlib.import_module("morphreg.integrator")
        for name in ("advect_image_euler", "advect_image_sl", "continuity_euler",
                     "continuity_sl"):
            assert hasattr(integ, name), name
        cfg = mr.ShootingConfig(mr.Scheme.SEMI_LAGRANGIAN, 4, 0.0, mr.GaussianKernel(1.0))
        assert cfg.dtype == torch.float64
    finally:
        sys.path.remove(shim)
        for m in [k for k in sys.modules if k == "morphreg" or k.startswith("morphreg.")]:
            del sys.modules[m]
