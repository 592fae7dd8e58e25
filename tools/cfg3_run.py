import time, sys, os
sys.path.insert(0, os.getcwd())
import paper_2511_20432_b200 as tg
os.environ["TG_SETUP_TIMING"] = "1"
t = time.time(); s = tg.Simulation("configs/cfg3_contour_hatch.cfg"); print("setup", time.time() - t, s.info, flush=True)
ctx = s.context()
s.reset()
for k in range(4):
    ctx.set_profiling(True); ctx.profile(reset=True)
    t = time.time(); it, rel = s.advance(1); w = time.time() - t
    p = ctx.profile()
    print(f"step {k+1}: wall {w*1e3:.1f} ms, cg {it}, rel {rel:.2e}, k1 {p['k1_ms']:.2f} ms, solve {p['k2_ms']:.2f} ms, theta {p['theta_step_ms']:.2f} ms", flush=True)
