"""Robustness smoke at 4x config 4 (512 x 512 x 64 elements, ~17.4M DOF):
setup, two time steps, and the constant-state property of the theta step."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_20432_b200 as tg  # noqa: E402

txt = open(os.path.join(ROOT, "configs", "cfg4_large.cfg")).read()
txt = txt.replace("xi_elements = 256", "xi_elements = 512").replace("eta_elements = 256",
                                                                  "eta_elements = 512")
path = "/tmp/cfg4x4.cfg"
open(path, "w").write(txt)
t0 = time.perf_counter()
s = tg.Simulation(path)
print("setup_s", round(time.perf_counter() - t0, 2), s.info, flush=True)
s.reset()
t0 = time.perf_counter()
it, rel = s.advance(2)
print("2 steps s", round(time.perf_counter() - t0, 2), "cg", it, "rel", rel, flush=True)
c = 3.5
nf, nc, n = s.info["n_free"], s.info["n_constrained"], s.info["n_full"]
x, _, _ = s.theta_step(np.full(nf, c), np.full(nc, c), np.zeros(n), np.zeros(n), np.full(nc, c))
print("constant state max dev", float(np.abs(x - c).max()), flush=True)
assert np.abs(x - c).max() <= 1e-10 * c
print("ok")
