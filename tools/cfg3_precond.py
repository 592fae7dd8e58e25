"""Config 3 at full size: CG iterations and ms per step, Jacobi against the
scaled separable-approximation preconditioner (preconditioner="fdm")."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2511_20432_b200 as tg
cfg = sys.argv[1] if len(sys.argv) > 1 else "configs/cfg3_contour_hatch.cfg"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
out = {}
for pc in ("jacobi", "fdm"):
    t0 = time.perf_counter()
    s = tg.Simulation(cfg, preconditioner=pc)
    setup = time.perf_counter() - t0
    s.reset()
    s.advance(1)
    ctx = s.context()
    ctx.set_profiling(True); ctx.profile(reset=True)
    t0 = time.perf_counter()
    it, rel = s.advance(steps)
    wall = (time.perf_counter() - t0) * 1e3 / steps
    p = ctx.profile(); ctx.set_profiling(False)
    out[pc] = s.state()["free"]
    print(f"{pc}: setup {setup:.2f} s, {wall:.2f} ms/step, theta solve {p['k2_ms']/steps:.2f} ms, "
          f"{it/steps:.1f} CG it/step", flush=True)
    s.close()
x, y = out["jacobi"], out["fdm"]
print("fdm vs jacobi free coefficients:", np.abs(x - y).max() / np.abs(x).max())
