"""Config-4 flux-load call alone (tg_sim_flux_load, K5 + remainder + K3) and the
Dirichlet call alone: device time per call (CUDA events), after warm-up."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_20432_b200 as tg
s = tg.Simulation(sys.argv[1] if len(sys.argv) > 1 else "configs/cfg4_large.cfg")
ctx = s.context()
t = 3e-5
for _ in range(2):
    s.flux_load(t); s.dirichlet_values(t)
for name, fn in (("flux_load", lambda: s.flux_load(t)), ("dirichlet_values", lambda: s.dirichlet_values(t))):
    ctx.set_profiling(True)
    ctx.profile(reset=True)
    n = 5
    for _ in range(n):
        fn()
    p = ctx.profile()
    ctx.set_profiling(False)
    print(f"{name}: K5 contraction {p['k5_ms'] / n:.2f} ms, K1 remainder {p['k1_ms'] / n:.2f} ms per call")
