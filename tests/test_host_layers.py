"""Host-side layers that need no GPU: PGM parsing and its error messages
(image_io.py:20-81 of the reference), momentum files, shape specs, the CLI's
argument surface and exit codes for bad input, optimize_batch's input checks."""

import json

import numpy as np
import pytest
import torch

from paper_2106_08817_b200 import FieldError, GridGeometry, ScalarField
from paper_2106_08817_b200 import cli, image_io, shapes
from paper_2106_08817_b200.image_io import ImageFormatError


def test_pgm_8_and_16_bit_with_comments(tmp_path):
    p = tmp_path / "a.pgm"
    p.write_bytes(b"P5\n# made by a test\n3 2\n255\n" + bytes([0, 255, 128, 64, 32, 16]))
    f = image_io.read_pgm(p)
    assert f.geometry.shape == (2, 3)
    assert np.allclose(f.values, np.array([[0, 255, 128], [64, 32, 16]]) / 255.0)
    p.write_bytes(b"P5 2 2 65535\n" + ((1000).to_bytes(2, "big") + (65535).to_bytes(2, "big")) * 2)
    assert np.allclose(image_io.read_pgm(p).values, [[1000 / 65535, 1.0]] * 2)


def test_pgm_errors_name_the_offending_byte(tmp_path):
    p = tmp_path / "bad.pgm"
    p.write_bytes(b"P2\n2 2\n255\n" + bytes(4))
    with pytest.raises(ImageFormatError, match="byte 0"):
        image_io.read_pgm(p)
    p.write_bytes(b"P5\n2 x2\n255\n" + bytes(4))
    with pytest.raises(ImageFormatError, match=r"'x2' at byte 5"):
        image_io.read_pgm(p)
    p.write_bytes(b"P5\n4 4\n255\n" + bytes(5))
    with pytest.raises(ImageFormatError, match="expected 16 pixel bytes at byte 11, got 5"):
        image_io.read_pgm(p)
    p.write_bytes(b"P5\n4")
    with pytest.raises(ImageFormatError, match="truncated PGM header"):
        image_io.read_pgm(p)
    p.write_bytes(b"P5\n2 2\n70000\n" + bytes(8))
    with pytest.raises(ImageFormatError, match="invalid PGM dimensions/maxval"):
        image_io.read_pgm(p)


def test_pgm_and_png_round_trip_within_one_level(tmp_path):
    rng = np.random.default_rng(0)
    f = ScalarField.from_array(rng.uniform(0, 1, (9, 7)))
    for name in ("rt.pgm", "rt.png"):
        image_io.write_image(f, tmp_path / name)
        g = image_io.read_image(tmp_path / name)
        assert g.geometry.shape == (9, 7)
        assert np.max(np.abs(f.values - g.values)) <= 0.5 / 255 + 1e-12


def test_momentum_files_and_artifacts(tmp_path):
    z = ScalarField.from_array(np.linspace(-1, 1, 12).reshape(3, 4))
    image_io.save_momentum(z, tmp_path / "z.npy")
    assert np.array_equal(image_io.load_momentum(tmp_path / "z.npy").values, z.values)
    np.save(tmp_path / "bad.npy", np.zeros(5))
    with pytest.raises(ImageFormatError, match="must be 2d"):
        image_io.load_momentum(tmp_path / "bad.npy")
    image_io.write_momentum_heatmap(z.values, tmp_path / "h.png", 1.0)
    from PIL import Image

    rgb = np.asarray(Image.open(tmp_path / "h.png"))
    assert rgb.shape == (3, 4, 3)
    assert tuple(rgb[0, 0]) == (0, 0, 255) and tuple(rgb[-1, -1]) == (255, 0, 0)  # -vmax blue, +vmax red


def test_shape_spec_validation_and_indicator():
    with pytest.raises(FieldError, match="inner < outer"):
        shapes.ShapeSpec(shapes.ShapeKind.ANNULUS, (5, 5), outer=3.0, inner=3.0)
    with pytest.raises(FieldError, match="intensity"):
        shapes.ShapeSpec(shapes.ShapeKind.DISK, (5, 5), outer=3.0, intensity=1.5)
    with pytest.raises(FieldError, match="unknown preset"):
        shapes.preset_pair("nope")
    disk = shapes.render(shapes.ShapeSpec(shapes.ShapeKind.DISK, (10.0, 10.0), outer=4.0, intensity=0.5),
                         GridGeometry(21, 21))  # no blur: pure host rasterisation
    assert disk.values[10, 10] == 0.5 and disk.values[10, 14] == 0.0 and disk.values[10, 13] == 0.5
    ring = shapes.render(shapes.ShapeSpec(shapes.ShapeKind.C_OPENING, (20.0, 20.0), outer=12.0, inner=6.0,
                                          opening_angle=90.0, orientation=0.0), GridGeometry(41, 41))
    assert ring.values[20, 29] == 0.0   # the opening faces +column
    assert ring.values[20, 11] == 1.0 and ring.values[11, 20] == 1.0 and ring.values[29, 20] == 1.0
    assert ring.values[20, 20] == 0.0   # inside the hole


def test_cli_argument_surface_and_input_errors(tmp_path, capsys):
    a = cli.build_parser().parse_args(["register", "--synthetic", "c2disk", "--out", "o"])
    assert (a.steps, a.sigma, a.mu, a.rho, a.lam, a.max_iters, a.size) == (20, 6.0, 0.0, 1.0, 1e-4, 50, 200)
    a = cli.build_parser().parse_args(["compare-schemes", "--synthetic", "disk2c", "--out", "o"])
    assert (a.steps_eulerian, a.steps_sl, a.sigma, a.lam, a.warmup_iters) == (38, 20, 4.0, 3e-5, 20)
    # exit code 1 + one diagnostic line on stderr, nothing on stdout, before any device work
    assert cli.main(["register", "--out", str(tmp_path / "o")]) == 1
    out, err = capsys.readouterr()
    assert out == "" and "error=1 kind=FieldError" in err and "SOURCE and TARGET" in err
    assert cli.main(["shoot", str(tmp_path / "none.npy"), str(tmp_path / "i.pgm"), "--out", "o"]) == 1
    (tmp_path / "m.json").write_text(json.dumps({"command": "shoot", "params": {}}))
    assert cli.main(["register", "--replay", str(tmp_path / "m.json"), "--out", str(tmp_path / "o")]) == 1
    assert "not a register manifest" in capsys.readouterr().err
    assert cli.main(["compare-schemes", "--out", str(tmp_path / "o")]) == 1


def test_optimize_batch_rejects_mismatched_batches():
    import paper_2106_08817_b200 as mr

    cfg = mr.ShootingConfig(mr.Scheme.SEMI_LAGRANGIAN, 2, 0.0, mr.GaussianKernel(1.0))
    with pytest.raises(FieldError, match="batch shapes differ"):
        mr.optimize_batch(torch.zeros(2, 8, 8), torch.zeros(3, 8, 8), torch.zeros(2, 8, 8), cfg,
                          1e-3, 1.0, mr.OptimizeConfig(max_iters=1))
