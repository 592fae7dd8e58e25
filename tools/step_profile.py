"""Per-step time split of a config's run_time_loop on the device: wall time
per step vs the CUDA-event times of K1 (all superposition launches) and K2
(solve), over `steps` steps after `skip` untimed ones."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_20432_b200 as tg  # noqa: E402

cfg = sys.argv[1]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 100
sim = tg.Simulation(cfg)
sim.reset()
if skip:
    sim.advance(skip)
ctx = sim.context()
ctx.set_profiling(True)
ctx.profile(reset=True)
t0 = time.perf_counter()
it, _ = sim.advance(steps)
wall = time.perf_counter() - t0
p = ctx.profile()
print(json.dumps({"cfg": os.path.basename(cfg), "wall_ms_per_step": wall * 1e3 / steps,
                  "k1_ms_per_step": p["k1_ms"] / steps, "k2_ms_per_step": p["k2_ms"] / steps,
                  "launches_per_step": p["launches"] / steps, "cg_per_step": it / steps}))
