"""Per-iteration time of the theta-step solve at a fixed iteration count
(tol unreachable, max_iter = N: the solve runs exactly N iterations and ends
with the reference's non-convergence error), for latency studies of small
grids. Usage: python tools/k2_iter_time.py <cfg> [N]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2511_20432_b200 as tg  # noqa: E402

cfg = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 200
sim = tg.Simulation(cfg)
nf, nc, n = sim.info["n_free"], sim.info["n_constrained"], sim.info["n_full"]
F = sim.flux_load(5e-3)
g = sim.dirichlet_values(5e-3)
ctx = sim.context()
out = {}
for rep in range(3):
    ctx.set_profiling(True)
    ctx.profile(reset=True)
    try:
        sim.theta_step(np.zeros(nf), g, F, F, g, tol=1e-30, max_iter=N)
    except tg.NumericError:
        pass
    p = ctx.profile()
    out[f"us_per_iter_{rep}"] = 1e3 * p["k2_ms"] / N
print(json.dumps({"cfg": os.path.basename(cfg), "iters": N, **out,
                  "lib": os.path.basename(os.environ.get("TG_LIB_VARIANT", "default"))}))
