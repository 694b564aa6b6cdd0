"""Flags of the reference CLI run recorded in tests/golden/cli (no reference import here, so
the tests can use them on the GPU box)."""

SCENARIO = ["--custom", "--tx", "4", "--rx", "3", "--radius", "0.1", "--array-seed", "2", "--f-start", "20e9",
            "--f-stop", "24e9", "--f-count", "5", "--center", "0,0,0.3", "--extent", "0.06,0.06,0.02",
            "--dims", "7,6,3"]
RECON = ["--eta", "2e3", "--alpha", "2e-4", "--tol", "1e-300", "--max-iters", "30"]
