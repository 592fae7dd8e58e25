"""Config 2: device vs wall time per step, and the kernel split (profiling
counters), Jacobi and fast diagonalization."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_20432_b200 as tg
for pc in ("jacobi", "fdm"):
    s = tg.Simulation("configs/cfg2_raster_layer.cfg", preconditioner=pc)
    ctx = s.context()
    s.reset()
    s.advance(500)
    ctx.set_profiling(True)
    ctx.profile(reset=True)
    t0 = time.perf_counter()
    it, _ = s.advance(200)
    wall = (time.perf_counter() - t0) * 1e3 / 200
    p = ctx.profile()
    ctx.set_profiling(False)
    print(f"{pc}: wall {wall:.3f} ms/step, device {p['step_ms']/200:.3f}, theta {p['theta_step_ms']/200:.3f}, "
          f"k1 {p['k1_ms']/200:.3f}, k5 {p['k5_ms']/200:.3f}, launches {p['launches']/200:.1f}, cg {it/200:.1f}",
          flush=True)
    s.close()
