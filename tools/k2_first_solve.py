"""Config-4 reset + one step: the first solve's CG iterations (the ncu target
for the K2 capture)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_20432_b200 as tg
s = tg.Simulation(sys.argv[1] if len(sys.argv) > 1 else "configs/cfg4_large.cfg")
s.reset()
it, rel = s.advance(1)
print("cg iterations", it, "rel", rel)
