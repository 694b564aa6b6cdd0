import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2509_00774_b200 import configs
from paper_2509_00774_b200.plan import DevicePlan
from paper_2509_00774_b200.solver import SPGMEngine
w = configs.WORKLOADS[sys.argv[1]]()
scn = w.scenario
rng = np.random.default_rng(0)
y = rng.standard_normal(scn.n_channels) + 1j * rng.standard_normal(scn.n_channels)
plan = DevicePlan(scn, dtype=w.dtype, device="cuda:0", max_batch=w.batch)
eng = SPGMEngine(plan, y, eta=1e-3, alpha=1e-7)
for K in [int(v) for v in sys.argv[2].split(",")]:
    for sampler in ("table", "device"):
        tab = np.stack([np.sort(rng.choice(scn.n_channels, w.batch, replace=False)) for _ in range(K)]) if sampler == "table" else None
        eng.run_loop(K, table=tab, seed=0, iter0=1, batch=w.batch, tol=0.0)
        torch.cuda.synchronize()
        print(K, sampler, eng.loop_result(), flush=True)
