"""One config-4 step with the fast-diagonalization preconditioner (ncu target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_20432_b200 as tg
s = tg.Simulation("configs/cfg4_large.cfg", preconditioner="fdm")
s.reset(); s.advance(1)
print(s.advance(1))
