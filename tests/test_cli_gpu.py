"""The CLI over the device facade (cli.py of the reference): artefacts, exit codes, and
the bitwise manifest replay the reference promises (optimizer.py:5-7)."""

import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(argv, capsys):
    from paper_2106_08817_b200 import cli

    code = cli.main(argv)
    out, err = capsys.readouterr()
    return code, out, err


def test_register_writes_artefacts_and_replays_bitwise(tmp_path, capsys):
    d1, d2 = tmp_path / "run", tmp_path / "again"
    code, out, _ = _run(["register", "--synthetic", "c2disk", "--size", "48", "--steps", "5",
                         "--sigma", "3", "--mu", "0.2", "--max-iters", "3", "--save-frames",
                         "--out", str(d1)], capsys)
    assert code == 0
    summary = json.loads(out)  # exactly one JSON line on stdout
    assert summary["command"] == "register" and summary["frames"] == 6
    assert summary["iterations"] >= 1 and summary["out"] == str(d1)
    for name in ("metrics.csv", "z0.npy", "source.npy", "target.npy", "manifest.json", "grid_t1.png",
                 "frame_000.pgm", "frame_005.pgm", "momentum_003.png"):
        assert (d1 / name).exists(), name
    rows = (d1 / "metrics.csv").read_text().splitlines()
    assert rows[0] == "iteration,total,data_term,v_norm,z_norm,step_size"
    totals = [float(r.split(",")[1]) for r in rows[1:]]
    assert totals == sorted(totals, reverse=True) and len(totals) == summary["iterations"] + 1
    man = json.loads((d1 / "manifest.json").read_text())
    assert man["command"] == "register" and man["params"]["synthetic"] == "c2disk"
    assert man["final"]["total"] == summary["total"]
    # replay: same metrics and momentum, bit for bit
    code, out2, _ = _run(["register", "--replay", str(d1 / "manifest.json"), "--out", str(d2)], capsys)
    assert code == 0
    assert (d2 / "metrics.csv").read_bytes() == (d1 / "metrics.csv").read_bytes()
    assert (d2 / "z0.npy").read_bytes() == (d1 / "z0.npy").read_bytes()
    # shoot from the saved run
    d3 = tmp_path / "shoot"
    code, out3, _ = _run(["shoot", str(d1 / "z0.npy"), str(d1 / "source.npy"), "--steps", "5",
                          "--sigma", "3", "--mu", "0.2", "--out", str(d3)], capsys)
    assert code == 0
    s3 = json.loads(out3)
    energy = (d3 / "energy.csv").read_text().splitlines()
    assert energy[0] == "step,t,energy,max_abs_z" and len(energy) == 7
    assert s3["frames"] == 2 and s3["energy_t0"] == float(energy[1].split(",")[2])


def test_shoot_rejects_mismatched_geometry_and_reports_divergence(tmp_path, capsys):
    np.save(tmp_path / "z.npy", np.zeros((8, 9)))
    np.save(tmp_path / "i.npy", np.zeros((8, 8)))
    code, out, err = _run(["shoot", str(tmp_path / "z.npy"), str(tmp_path / "i.npy"), "--out",
                           str(tmp_path / "o")], capsys)
    assert code == 1 and out == "" and "kind=FieldError" in err
    rng = np.random.default_rng(0)
    np.save(tmp_path / "zbig.npy", 1e7 * rng.standard_normal((16, 16)))
    np.save(tmp_path / "img.npy", rng.random((16, 16)))
    code, out, err = _run(["shoot", str(tmp_path / "zbig.npy"), str(tmp_path / "img.npy"), "--mu", "5",
                           "--steps", "4", "--sigma", "1", "--out", str(tmp_path / "o2")], capsys)
    assert code == 2 and out == "" and "kind=IntegrationDiverged" in err


def test_compare_schemes_from_a_saved_momentum(tmp_path, capsys):
    import paper_2106_08817_b200 as mr

    src, _ = mr.preset_pair("disk2c", 40)
    z = 0.05 * mr.smooth_random_field(src.geometry, 2.0, seed=1).values
    np.save(tmp_path / "z.npy", z)
    np.save(tmp_path / "i.npy", src.values)
    out_dir = tmp_path / "cmp"
    code, out, _ = _run(["compare-schemes", "--z0", str(tmp_path / "z.npy"), "--image",
                         str(tmp_path / "i.npy"), "--sigma", "2", "--steps-eulerian", "12",
                         "--steps-sl", "6", "--out", str(out_dir)], capsys)
    assert code == 0
    verdicts = json.loads(out)["verdicts"]
    assert set(verdicts) == {"eulerian", "semi-lagrangian", "hybrid"}
    assert verdicts["semi-lagrangian"]["status"] == "stable"
    assert json.loads((out_dir / "verdict.json").read_text()) == verdicts
    for name in ("growth_eulerian.csv", "final_hybrid.pgm", "grid_semi-lagrangian.png", "z0.npy"):
        assert (out_dir / name).exists(), name
