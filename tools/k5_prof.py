"""Config-4 reset + one step (the fused K5 path); the ncu target for the
contraction kernel (sf_contract_kernel) and the remainder launch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_20432_b200 as tg
s = tg.Simulation(sys.argv[1] if len(sys.argv) > 1 else "configs/cfg4_large.cfg")
s.reset()
s.advance(1)
print("ok", s.sumfact_stats())
