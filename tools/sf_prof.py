"""One config-4 step (reset + advance) for an ncu launch list of the K5 / K1 / K2 kernels."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_20432_b200 as tg  # noqa: E402

s = tg.Simulation(os.path.join(ROOT, "configs", "cfg4_large.cfg"))
s.reset()
s.advance(1)
print(s.sumfact_stats())
s.close()
