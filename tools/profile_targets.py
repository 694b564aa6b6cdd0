#!/usr/bin/env python3
"""The launches profiled for profiles/<round>_ncu_summary.json (one each): the Large step's flat forward and
adjoint+prox kernels, the persistent loop on Medium (spgm_loop_kernel, 20 iterations) and on Small
(tiny_loop_kernel, 200 iterations). Run under ncu -k regex:"fwd_kernel|adj_kernel|spgm_loop|tiny_loop"."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_00774_b200 import configs  # noqa: E402
from paper_2509_00774_b200.plan import DevicePlan  # noqa: E402
from paper_2509_00774_b200.solver import SPGMEngine  # noqa: E402

for wl, iters in (("large", 0), ("medium", 20), ("small", 200)):
    w = configs.WORKLOADS[wl]()
    scn = w.scenario
    rng = np.random.default_rng(0)
    y = rng.standard_normal(scn.n_channels) + 1j * rng.standard_normal(scn.n_channels)
    plan = DevicePlan(scn, dtype=w.dtype, device="cuda:0", max_batch=w.batch)
    eng = SPGMEngine(plan, y, eta=1e-3, alpha=1e-7, initial=configs.make_scene(w))
    if iters == 0:
        eng.sample_device(0, 1, w.batch)
        eng.step_staged()
    else:
        eng.run_loop(iters, table=None, seed=0, iter0=1, batch=w.batch, tol=0.0)
        print(wl, eng.loop_result())
    torch.cuda.synchronize()
    del eng, plan
    torch.cuda.empty_cache()
