"""Config 4 with the fast-diagonalization option: theta-step solve time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_20432_b200 as tg
s = tg.Simulation(sys.argv[1] if len(sys.argv) > 1 else "configs/cfg4_large.cfg", preconditioner="fdm")
ctx = s.context()
s.reset()
s.advance(2)
ctx.set_profiling(True); ctx.profile(reset=True)
it, rel = s.advance(5)
p = ctx.profile(); ctx.set_profiling(False)
print(f"fdm solve {p['k2_ms']/5:.3f} ms/step, theta step {p['theta_step_ms']/5:.3f} ms, {it/5:.1f} it, rel {rel:.2e}")
