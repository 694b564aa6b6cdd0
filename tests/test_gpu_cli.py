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


def _small_case(tmp_path):
    """A small custom scenario and noiseless point-scatterer measurements through the CLI."""
    scn = tmp_path / "s.json"
    assert main(["scenario-init", "--custom", "--tx", "4", "--rx", "4", "--radius", "0.1", "--f-start", "20e9",
                 "--f-stop", "24e9", "--f-count", "4", "--center", "0,0,0.3", "--extent", "0.06,0.06,0",
                 "--dims", "7,7,1", "--out", str(scn)]) == 0
    meas = tmp_path / "m.nfms"
    assert main(["simulate", "--scenario", str(scn), "--phantom", "points:1", "--seed", "4", "--out", str(meas)]) == 0
    return scn, meas


def test_simulate_semantics(tmp_path):
    from paper_2509_00774_b200 import forward_apply

    scn, meas = _small_case(tmp_path)
    truth = read_volume(tmp_path / "m_truth.nfmv")
    s = read_scenario(scn)
    assert rel_l2(read_measurements(meas).values, forward_apply(truth.values, s)) <= 1e-12  # zero noise
    again = tmp_path / "again.nfms"
    assert main(["simulate", "--scenario", str(scn), "--phantom", "points:1", "--seed", "4", "--out", str(again)]) == 0
    assert again.read_bytes() == meas.read_bytes()
    bad = tmp_path / "bad.nfms"
    assert main(["simulate", "--scenario", str(scn), "--phantom", "sphere", "--out", str(bad)]) == 1
    other = tmp_path / "o.json"
    assert main(["scenario-init", "--custom", "--dims", "3,3,1", "--out", str(other)]) == 0
    assert main(["simulate", "--scenario", str(other), "--phantom", f"file:{tmp_path / 'm_truth.nfmv'}",
                 "--out", str(bad)]) == 1


def _eta(scn) -> str:
    from paper_2509_00774_b200 import lipschitz_estimate

    return repr(1.0 / lipschitz_estimate(read_scenario(scn), n_iters=30))


def test_reconstruct_semantics(tmp_path, capsys):
    scn, meas = _small_case(tmp_path)
    truth = read_volume(tmp_path / "m_truth.nfmv").values
    base = ["reconstruct", "--scenario", str(scn), "--measurements", str(meas), "--eta", _eta(scn), "--alpha", "1e-6",
            "--tol", "1e-300", "--max-iters", "60"]
    assert main(base + ["--method", "pgm", "--out", str(tmp_path / "p.nfmv")]) == 0
    rec = read_volume(tmp_path / "p.nfmv").values
    assert int(np.argmax(np.abs(rec))) == int(np.argmax(np.abs(truth)))  # localises the scatterer
    assert main(base + ["--method", "spgm", "--batch", "4,4,4", "--out", str(tmp_path / "q.nfmv")]) == 0
    capsys.readouterr()
    assert main(["psnr", "--recon", str(tmp_path / "q.nfmv"), "--reference", str(tmp_path / "p.nfmv")]) == 0
    assert capsys.readouterr().out.startswith("psnr_db=inf")  # the full composition is PGM
    rep = tmp_path / "r.json"
    assert main(["reconstruct", "--scenario", str(scn), "--measurements", str(meas), "--method", "pgm",
                 "--max-iters", "100000000", "--tol", "1e-300", "--time-budget-s", "0.2", "--out",
                 str(tmp_path / "t.nfmv"), "--report", str(rep)]) == 0
    assert json.loads(rep.read_text())["termination"] == "time_budget"


def test_benchmark_repeat_is_deterministic(tmp_path):
    scn, meas = _small_case(tmp_path)
    cols = []
    for k in range(2):
        out = tmp_path / f"b{k}.csv"
        assert main(["benchmark", "--scenario", str(scn), "--measurements", str(meas), "--compositions", "2,2,2",
                     "--seeds", "1,2", "--max-iters", "15", "--tol", "1e-300", "--eta", _eta(scn), "--alpha", "1e-6",
                     "--out", str(out)]) == 0
        cols.append([r[7] for r in csv.reader(out.open())][1:])
    assert cols[0] == cols[1]
