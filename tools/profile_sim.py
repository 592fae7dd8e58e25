"""Drive a few time steps of a config for profiling (ncu -k regex:<kernel>)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2511_20432_b200 as tg  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "configs", "cfg4_large.cfg")
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
sim = tg.Simulation(cfg, preconditioner=os.environ.get("TG_PRECOND", "jacobi"))
sim.reset()
for k in range(steps):
    it, rel = sim.advance(1)
    print(f"step {k + 1}: cg iterations {it} rel {rel:.3e}")
