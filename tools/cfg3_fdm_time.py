"""Config 3 step time with the general preconditioner (and Jacobi), DIA on/off via env."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_20432_b200 as tg
for pc in ("fdm", "jacobi"):
    s = tg.Simulation("configs/cfg3_contour_hatch.cfg", preconditioner=pc)
    s.reset(); s.advance(2)
    ctx = s.context(); ctx.set_profiling(True); ctx.profile(reset=True)
    t0 = time.perf_counter(); it, _ = s.advance(10); w = (time.perf_counter() - t0) * 100
    p = ctx.profile()
    print(pc, f"{w:.3f} ms/step  k2 {p['k2_ms']/10:.3f}  theta_total {p['theta_step_ms']/10:.3f}  it {it/10}", flush=True)
    s.close()
