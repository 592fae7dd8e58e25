"""Config-4 K5 plan after reset + 2 steps: the remainder's pairs per region
((E - J) x points) for the static regions, and the profiled K1 pairs per step."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2511_20432_b200 as tg
s = tg.Simulation(sys.argv[1] if len(sys.argv) > 1 else "configs/cfg4_large.cfg")
s.reset()
s.advance(2)
ctx = s.context()
ctx.set_profiling(True)
ctx.profile(reset=True)
s.advance(1)
p = ctx.profile()
R = s.sumfact_regions()
st = s.state()
t = st["time"]
J, E = s.sumfact_plan(t)
rem = (E - J) * R[:, 7]
print("regions", len(R), "static remainder pairs", rem.sum(), "max per region", rem.max())
print("J min/max", J.min(), J.max(), "E-J min/max", (E - J).min(), (E - J).max())
print("k1 pairs/step", p["k1_pairs"], "k1 ms", p["k1_ms"], "k5 ms", p["k5_ms"], "launches", p["launches"])
order = np.argsort(-rem)[:8]
for r in order:
    print(r, J[r], E[r], R[r, 7], R[r, :6])
