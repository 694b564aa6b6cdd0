"""CLI (paper_2509_00774_b200.cli) on CPU: the subcommands that need no GPU, usage errors and
exit codes (the reference's cli.py:336-347 contract: 0 ok, 1 failure, 2 usage). The GPU
subcommands are covered by tests/test_gpu_cli.py."""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from paper_2509_00774_b200 import preset_scenario, scenario_fingerprint
from paper_2509_00774_b200.cli import main
from paper_2509_00774_b200.io import read_scenario

GOLD = Path(__file__).resolve().parent / "golden"


def test_scenario_init_matches_reference_document(tmp_path, capsys):
    """The same flags the reference CLI was run with (tests/golden/make_cli_golden.py) give a
    byte-identical scenario document."""
    from golden.cli_flags import SCENARIO

    out = tmp_path / "scn.json"
    assert main(["scenario-init", *SCENARIO, "--out", str(out)]) == 0
    assert out.read_text() == (GOLD / "cli" / "scn.json").read_text()
    assert "M=60 N=126" in capsys.readouterr().out
    assert main(["scenario-init", "--preset", "paper-v", "--out", str(tmp_path / "p.json")]) == 0
    assert scenario_fingerprint(read_scenario(tmp_path / "p.json")) == scenario_fingerprint(preset_scenario("paper-v"))


def test_scenario_init_default_extent_collapses_single_axes(tmp_path):
    out = tmp_path / "s.json"
    assert main(["scenario-init", "--custom", "--dims", "5,1,3", "--out", str(out)]) == 0
    assert read_scenario(out).voxels.extent == (0.3, 0.0, 0.1)


def test_info(capsys):
    assert main(["info", "--scenario", str(GOLD / "cli" / "scn.json")]) == 0
    lines = capsys.readouterr().out.splitlines()
    assert lines[0] == "channels M=60" and lines[1] == "voxels N=126"
    assert lines[2] == "transmitters=4 receivers=3"
    assert lines[-1].startswith("fingerprint=") and len(lines[-1]) == len("fingerprint=") + 64


def test_psnr(capsys):
    cli = GOLD / "cli"
    assert main(["psnr", "--recon", str(cli / "pgm.nfmv"), "--reference", str(cli / "pgm.nfmv")]) == 0
    assert capsys.readouterr().out.strip() == "psnr_db=inf rmse=0"
    assert main(["psnr", "--recon", str(cli / "spgm.nfmv"), "--reference", str(cli / "meas_truth.nfmv")]) == 0
    out = capsys.readouterr().out
    assert out.startswith("psnr_db=") and "rmse=" in out


def test_exit_codes(tmp_path, capsys):
    cli = GOLD / "cli"
    base = ["reconstruct", "--scenario", str(cli / "scn.json"), "--measurements", str(cli / "meas.nfms"),
            "--out", str(tmp_path / "o.nfmv")]
    assert main(base + ["--method", "spgm"]) == 2  # needs --batch
    assert main(base + ["--method", "pgm", "--batch", "1,1,1"]) == 2
    assert main(["scenario-init", "--out", str(tmp_path / "x.json")]) == 2
    assert main(["scenario-init", "--preset", "paper-v", "--custom", "--out", str(tmp_path / "x.json")]) == 2
    assert main(["info", "--scenario", str(tmp_path / "missing.json")]) == 1
    assert main(["psnr", "--recon", str(cli / "scn.json"), "--reference", str(cli / "pgm.nfmv")]) == 1
    assert main(["scenario-init", "--custom", "--dims", "1,2", "--out", str(tmp_path / "x.json")]) == 2
    assert main(["benchmark", "--scenario", "a", "--measurements", "b", "--compositions", ";", "--seeds", "1",
                 "--out", "c"]) == 2
    assert main([]) == 2
    assert main(["frobnicate"]) == 2
    assert main(["info", "--bogus"]) == 2
    assert main(["info"]) == 2
    assert main(["--help"]) == 0
    err = capsys.readouterr().err
    assert "usage error: --method spgm requires --batch f,tx,rx" in err
    assert "# paper_2509_00774_b200 " in err and "command=reconstruct" in err


def test_reconstruct_rejects_foreign_measurements(tmp_path):
    cli = GOLD / "cli"
    assert main(["reconstruct", "--scenario", str(GOLD / "io" / "small.json"), "--measurements",
                 str(cli / "meas.nfms"), "--method", "pgm", "--out", str(tmp_path / "o.nfmv")]) == 1


def test_phantoms_and_metrics():
    from paper_2509_00774_b200 import Vec3, VoxelGrid
    from paper_2509_00774_b200.metrics import spearman_rank
    from paper_2509_00774_b200.phantoms import make_phantom

    g = VoxelGrid(center=Vec3(0, 0, 0.3), extent=(0.1, 0.1, 0.02), dims=(8, 6, 3))
    bar = make_phantom("bar", g).values.reshape(3, 6, 8)
    assert np.flatnonzero(bar[1, 3]).tolist() == list(range(2, 7)) and np.abs(bar).sum() == 5
    cross = make_phantom("cross", g).values.reshape(3, 6, 8)
    assert np.flatnonzero(cross[1, :, 4]).tolist() == [1, 2, 3, 4] and np.abs(cross).sum() == 8
    pts = make_phantom("points:5", g, rng_seed=4).values
    assert np.count_nonzero(pts) == 5 and np.allclose(np.abs(pts[pts != 0]), 1.0)
    assert np.array_equal(make_phantom("points:5", g, rng_seed=4).values, pts)
    for bad in ("points:0", "points:1000", "sphere"):
        with pytest.raises(ValueError):
            make_phantom(bad, g)
    assert spearman_rank([1, 2, 3, 4], [10, 20, 30, 40]) == pytest.approx(1.0)
    assert spearman_rank([1, 2, 2, 3], [3, 2, 2, 1]) == pytest.approx(-1.0)
    assert spearman_rank([1, 1, 1], [1, 2, 3]) == 0.0
