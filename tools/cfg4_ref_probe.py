"""Config 4 against the unmodified reference on the GPU box host: how long
the reference's setup (prepare_simulation: ~5.3e8-entry CSRs), one threaded
flux load and one serial-PCG theta step take, and how close the device is."""
import os, sys, time, subprocess
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_20432_b200 as tg
from oracle import pyoracle
CFG = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "configs", "cfg4_large.cfg")
nw = lambda a, b: float(np.abs(a - b).max() / np.abs(b).max())
s = tg.Simulation(CFG, solver_tol=1e-12)
s.reset(); s.advance(2)
st = s.state(); dt = s.params["dt"]; t3 = st["time"] + dt
F3 = s.flux_load(t3); g3 = s.dirichlet_values(t3)
x3, it, rel = s.theta_step(st["free"], st["g"], st["F"], F3, g3, tol=1e-12)
print("device step ok", it, rel, flush=True)
R = pyoracle.RefLib()
t0 = time.perf_counter()
rs = R.sim(CFG, threads=os.cpu_count(), solver_tol=1e-12)
print("ref open", round(time.perf_counter() - t0, 1), "s", flush=True)
print(subprocess.run(["free", "-g"], capture_output=True, text=True).stdout, flush=True)
t0 = time.perf_counter(); Fr = rs.flux_load(t3, threads=os.cpu_count()); print("ref flux", round(time.perf_counter() - t0, 1), "s  F rel", nw(F3, Fr), flush=True)
gp = rs.greville_points()
t0 = time.perf_counter()

t0 = time.perf_counter(); xr, itr, relr = rs.theta_step(st["free"], st["g"], st["F"], F3, g3, 1e-12)
print("ref theta", round(time.perf_counter() - t0, 1), "s iters", itr, "vs", it, "x rel", nw(x3, xr), flush=True)
