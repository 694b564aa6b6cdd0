#!/usr/bin/env python3
"""c64 precision of the loaded library vs the oracle on Medium/Large/micro spot checks (prints rel L2)."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from oracle import nfmimo_oracle as O
from paper_2509_00774_b200 import configs
from paper_2509_00774_b200.plan import DevicePlan

def rc(rng, n): return rng.standard_normal(n) + 1j * rng.standard_normal(n)
out = {}
for name, scn in (("medium", configs.medium_scenario()), ("large", configs.large_scenario()),
                  ("micro128", configs.micro_scenario("128^3"))):
    geo = O.geom_from_scenario(scn)
    rng = np.random.default_rng(7)
    s = rc(rng, scn.n_voxels).astype(np.complex64).astype(np.complex128)
    idx = np.sort(rng.choice(scn.n_channels, 4096, replace=False))
    plan = DevicePlan(scn, dtype="c64", max_batch=4096)
    plan.prepare(torch.from_numpy(idx.astype(np.int32)).cuda())
    y = plan.forward(plan._as_dev(s, scn.n_voxels, "s")).to(torch.complex128).cpu().numpy()
    rows = rng.choice(idx.size, 12, replace=False)
    ref = O.direct_forward(geo, s, idx[rows], chunk=65536)
    r = rc(rng, idx.size).astype(np.complex64).astype(np.complex128)
    g = plan.adjoint(plan._as_dev(r, idx.size, "r")).to(torch.complex128).cpu().numpy()
    vox = rng.choice(scn.n_voxels, 1024, replace=False)
    gref = O.direct_adjoint(geo, r, idx, voxels=vox)
    out[name] = {"fwd_rel_l2": float(np.linalg.norm(y[rows] - ref) / np.linalg.norm(ref)),
                 "adj_rel_l2": float(np.linalg.norm(g[vox] - gref) / np.linalg.norm(gref))}
    del plan
print(json.dumps(out))
