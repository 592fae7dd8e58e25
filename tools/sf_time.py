"""K5 on/off: wall time of config-4 steps (flux + Dirichlet + theta step) and the
per-phase split (TG_STEP_TIMING), GPU box only.

  python tools/sf_time.py [steps]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_20432_b200 as tg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
s = tg.Simulation(os.path.join(ROOT, "configs", "cfg4_large.cfg"))
for on in (True, False, True):
    s.set_sumfact(on)
    s.reset()
    s.advance(1)
    t0 = time.perf_counter()
    s.advance(n)
    dt = (time.perf_counter() - t0) / n
    print(f"sumfact={on}: {dt * 1e3:.2f} ms/step", s.sumfact_stats(), flush=True)
s.close()
