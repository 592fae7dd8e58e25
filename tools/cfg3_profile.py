"""Drive two config-3 time steps (for ncu -k regex:csr_pcg_kernel)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2511_20432_b200 as tg  # noqa: E402

sim = tg.Simulation(os.path.join(ROOT, "configs", "cfg3_contour_hatch.cfg"))
sim.reset()
for k in range(2):
    it, rel = sim.advance(1)
    print(f"step {k + 1}: cg iterations {it} rel {rel:.3e}")
