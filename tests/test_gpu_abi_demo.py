"""The C ABI driven from a plain-C host (examples/abi_demo.c, built by __graft_entry__.build()):
forward and adjoint through include/nfgpu.h against the operator entry evaluated in C, in c128
(<= 1e-10) and c64 (<= 1e-5)."""

from __future__ import annotations

import json
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
DEMO = Path(__file__).resolve().parents[1] / "examples" / "abi_demo"


def test_c_host_matches_direct_formula():
    if not DEMO.exists():
        from paper_2509_00774_b200 import _build

        _build.build_abi_demo()
    res = subprocess.run([str(DEMO)], capture_output=True, text=True, timeout=120)
    assert res.returncode == 0, res.stdout + res.stderr
    out = json.loads(res.stdout.strip().splitlines()[-1])
    assert out["c128_rel_l2"] <= 1e-10 and out["c64_rel_l2"] <= 1e-5
