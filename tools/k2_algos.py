"""Time the theta-step solve of a config with each Kronecker solver
(TG_K2_ALGO = cg1 | pcg): K2 kernel ms per solve, CG iterations, us/iteration."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2511_20432_b200 as tg  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "configs", "cfg4_large.cfg")
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
for algo in os.environ.get("TG_K2_ALGOS", "cg1,pcg,fdm").split(","):
    os.environ["TG_K2_ALGO"] = "pcg" if algo == "pcg" else "cg1"
    sim = tg.Simulation(cfg, preconditioner="fdm" if algo == "fdm" else "jacobi")
    sim.reset()
    sim.advance(1)
    ctx = sim.context()
    ctx.set_profiling(True)
    ctx.profile(reset=True)
    it, rel = sim.advance(steps)
    p = ctx.profile()
    print(json.dumps({"algo": algo, "solver": sim.info["kronecker"], "iters": it,
                      "k2_ms_per_solve": p["k2_ms"] / max(1, p["k2_launches"]),
                      "us_per_iter": 1e3 * p["k2_ms"] / max(1, it), "rel": rel}), flush=True)
    sim.close()
