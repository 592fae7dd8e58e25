"""Degree-1 cuboid with nx = 34 on the streaming sweep with strip tiles."""
import os, re, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_sim_gpu import box_geometry
import paper_2511_20432_b200 as tg
deg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
xi = 35 - deg - 1 if deg != 2 else 32
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
txt = open(os.path.join(ROOT, "configs", "cfg0_parity.cfg")).read()
head, rest = txt.split("[geometry]", 1)
rest = rest[rest.index("\n\n"):]
rest = re.sub(r"^xi_elements = \d+", f"xi_elements = {34 - deg}", rest, flags=re.M)
p = "/tmp/deg.cfg"
open(p, "w").write(head + box_geometry((deg, deg, deg)) + rest)
s = tg.Simulation(p, t_end=1.5e-4)
print(s.info["nx"], s.info["ny"], s.info["nz"], s.info["kronecker"])
import numpy as np
mode = sys.argv[2] if len(sys.argv) > 2 else "advance"
if mode == "parts":
    F = s.flux_load(5e-5); print("flux ok", flush=True)
    g = s.dirichlet_values(5e-5); print("dirichlet ok", flush=True)
    nf = s.info["n_free"]
    x, it, rel = s.theta_step(np.zeros(nf), g, F, F, g); print("theta ok", it, flush=True)
else:
    s.reset(); print("reset ok", flush=True)
    print(s.advance(3))
