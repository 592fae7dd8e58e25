"""Config 2 step time with the K5 region machinery on (per-region source
ranges for the pair-wise K1 launch) and off (plain K1 over every point)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_20432_b200 as tg
cfg = sys.argv[1] if len(sys.argv) > 1 else "configs/cfg2_raster_layer.cfg"
s = tg.Simulation(cfg)
ctx = s.context()
for on in (True, False, True):
    s.set_sumfact(on)
    s.reset()
    s.advance(900)
    ctx.set_profiling(True)
    ctx.profile(reset=True)
    t0 = time.perf_counter()
    it, _ = s.advance(200)
    wall = (time.perf_counter() - t0) * 1e3 / 200
    p = ctx.profile()
    ctx.set_profiling(False)
    print(f"sumfact={on}: {wall:.3f} ms/step  k1 {p['k1_ms']/200:.3f}  k5 {p['k5_ms']/200:.3f}  "
          f"k2 {p['k2_ms']/200:.3f}  launches {p['launches']/200:.1f}", flush=True)
