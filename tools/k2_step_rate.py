"""Per-CG-iteration K2 time inside real time steps (advance), for tile-shape
studies: python tools/k2_step_rate.py <cfg> [steps]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_20432_b200 as tg  # noqa: E402

cfg = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
sim = tg.Simulation(cfg)
sim.reset()
sim.advance(1)
ctx = sim.context()
ctx.set_profiling(True)
ctx.profile(reset=True)
it, rel = sim.advance(n)
p = ctx.profile()
nf = sim.info["n_free"]
print(json.dumps({"cfg": os.path.basename(cfg), "n_free": nf, "steps": n, "cg_it": it,
                  "k2_ms": p["k2_ms"], "us_per_iter": 1e3 * p["k2_ms"] / max(1, it),
                  "ns_per_dof_iter": 1e6 * p["k2_ms"] / max(1, it) / nf * 1e3,
                  "step_ms": p["step_ms"] / n, "k2_launches": p["k2_launches"]}), flush=True)
