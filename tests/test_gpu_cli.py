"""The CLI's GPU subcommands (simulate, reconstruct, benchmark) against the outputs the
REFERENCE CLI wrote for the same flags (tests/golden/cli, tests/golden/make_cli_golden.py)."""

from __future__ import annotations

import csv
import json
from pathlib import Path

import numpy as np
import pytest

from conftest import rel_l2
from paper_2509_00774_b200.cli import main
from paper_2509_00774_b200.io import read_measurements, read_scenario, read_volume

pytestmark = pytest.mark.gpu
CLI = Path(__file__).resolve().parent / "golden" / "cli"


def test_simulate_reconstruct_match_reference_cli(tmp_path):
    from golden.cli_flags import RECON

    scn = str(CLI / "scn.json")
    meas = tmp_path / "meas.nfms"
    assert main(["simulate", "--scenario", scn, "--phantom", "points:6", "--noise", "0.001", "--seed", "3",
                 "--out", str(meas)]) == 0
    ref_m = read_measurements(CLI / "meas.nfms", scenario=read_scenario(scn))
    ours = read_measurements(meas, scenario=read_scenario(scn))
    assert rel_l2(ours.values, ref_m.values) <= 1e-10
    assert (tmp_path / "meas_truth.nfmv").read_bytes() == (CLI / "meas_truth.nfmv").read_bytes()
    # reconstruct from the reference's own measurement file
    for method, extra in (("pgm", []), ("spgm", ["--batch", "3,2,2", "--seed", "5"])):
        out = tmp_path / f"{method}.nfmv"
        rep = tmp_path / f"{method}.json"
        assert main(["reconstruct", "--scenario", scn, "--measurements", str(CLI / "meas.nfms"), "--method", method,
                     *extra, *RECON, "--out", str(out), "--report", str(rep), "--slices", str(tmp_path / method)]) == 0
        assert rel_l2(read_volume(out).values, read_volume(CLI / f"{method}.nfmv").values) <= 1e-9
        doc = json.loads(rep.read_text())
        assert doc["iterations"] == 30 and doc["termination"] == "max_iters"
        assert len(list(tmp_path.glob(f"{method}_z*.csv"))) == 3
    ref_rep = json.loads((CLI / "spgm_report.json").read_text())
    ours_rep = json.loads((tmp_path / "spgm.json").read_text())
    assert [r["batch_size"] for r in ours_rep["per_iteration"]] == [r["batch_size"] for r in ref_rep["per_iteration"]]
    assert np.allclose([r["magnitude_change"] for r in ours_rep["per_iteration"]],
                       [r["magnitude_change"] for r in ref_rep["per_iteration"]], rtol=1e-8)


def test_benchmark_sweep_csv(tmp_path, capsys):
    out = tmp_path / "sweep.csv"
    assert main(["benchmark", "--scenario", str(CLI / "scn.json"), "--measurements", str(CLI / "meas.nfms"),
                 "--compositions", "5,4,3;2,2,2", "--seeds", "1,2", "--eta", "2e3", "--alpha", "2e-4",
                 "--max-iters", "20", "--tol", "1e-300", "--out", str(out)]) == 0
    rows = list(csv.reader(out.open()))
    assert rows[0] == ["composition_f", "composition_tx", "composition_rx", "B", "seed", "iterations", "runtime_s",
                       "psnr_db"]
    assert [r[:6] for r in rows[1:]] == [["5", "4", "3", "60", "1", "20"], ["5", "4", "3", "60", "2", "20"],
                                         ["2", "2", "2", "8", "1", "20"], ["2", "2", "2", "8", "2", "20"]]
    assert rows[1][7] == rows[2][7] == "inf"  # the full composition reproduces PGM exactly
    assert "wrote" in capsys.readouterr().out
