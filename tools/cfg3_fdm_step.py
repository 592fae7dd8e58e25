"""One config-3 step with the general preconditioner (ncu launch-list target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_20432_b200 as tg
cfg = sys.argv[1] if len(sys.argv) > 1 else "configs/cfg3_contour_hatch.cfg"
s = tg.Simulation(cfg, preconditioner="fdm")
s.reset(); s.advance(2)
print(s.advance(1))
