"""Config-4 (or any config) step timing with the fused K5 path: wall time per
advance() and the profiled K5 contraction / K1 / theta-step shares."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2511_20432_b200 as tg
cfg = sys.argv[1] if len(sys.argv) > 1 else "configs/cfg4_large.cfg"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
t0 = time.perf_counter()
s = tg.Simulation(cfg)
print(f"setup {time.perf_counter() - t0:.2f} s", flush=True)
ctx = s.context()
s.reset()
s.advance(2)
for on in (True, False):
    s.set_sumfact(on)
    s.reset()
    s.advance(2)
    ctx.set_profiling(True)
    ctx.profile(reset=True)
    t0 = time.perf_counter()
    it, _ = s.advance(steps)
    wall = (time.perf_counter() - t0) * 1e3 / steps
    p = ctx.profile()
    ctx.set_profiling(False)
    st = s.sumfact_stats()
    print(f"sumfact={on}: {wall:.2f} ms/step  k5 {p['k5_ms']/steps:.2f}  k1 {p['k1_ms']/steps:.2f}  "
          f"theta {p['theta_step_ms']/steps:.2f} ms/step  cg {it/steps:.1f}  J_flux {st['last_j_flux']} "
          f"J_dir {st['last_j_dirichlet']} flops {st['gemm_flops']:.3e} launches {p['launches']/steps:.1f}",
          flush=True)
s.set_sumfact(True)
t = 3e-5
F = s.flux_load(t); d = s.dirichlet_values(t)
s.set_sumfact(False)
F0 = s.flux_load(t); d0 = s.dirichlet_values(t)
print("K5 vs K1-only: F", np.abs(F - F0).max() / np.abs(F0).max(), "g", np.abs(d - d0).max() / np.abs(d0).max())
