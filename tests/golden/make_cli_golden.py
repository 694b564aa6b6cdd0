#!/usr/bin/env python3
"""Run the REFERENCE CLI (pkg/src/nfmimo/cli.py) end to end on a small scenario and keep its
files in tests/golden/cli/ for tests/test_gpu_cli.py:

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_cli_golden.py

scenario-init (custom) -> simulate (points:6, noise) -> reconstruct (pgm and spgm) -> benchmark.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

REF = os.environ.get("NFMIMO_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
from nfmimo.cli import main  # noqa: E402

OUT = Path(__file__).resolve().parent / "cli"

sys.path.insert(0, str(Path(__file__).resolve().parent))
from cli_flags import RECON, SCENARIO  # noqa: E402

def run(argv):
    rc = main(argv)
    assert rc == 0, (argv, rc)


def main_():
    OUT.mkdir(parents=True, exist_ok=True)
    o = str(OUT)
    run(["scenario-init", *SCENARIO, "--out", f"{o}/scn.json"])
    run(["simulate", "--scenario", f"{o}/scn.json", "--phantom", "points:6", "--noise", "0.001", "--seed", "3",
         "--out", f"{o}/meas.nfms"])
    run(["reconstruct", "--scenario", f"{o}/scn.json", "--measurements", f"{o}/meas.nfms", "--method", "pgm",
         *RECON, "--out", f"{o}/pgm.nfmv"])
    run(["reconstruct", "--scenario", f"{o}/scn.json", "--measurements", f"{o}/meas.nfms", "--method", "spgm",
         "--batch", "3,2,2", "--seed", "5", *RECON, "--out", f"{o}/spgm.nfmv", "--report", f"{o}/spgm_report.json"])
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main_()
