"""Per-phase timing of the K2 persistent PCG kernel (CTA 0 %globaltimer stamps)."""
import ctypes as C
import os
import sys

os.environ["TG_K2_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2511_20432_b200 as tg  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "configs", "cfg4_large.cfg")
sim = tg.Simulation(cfg)
sim.reset()
sim.advance(1)
L = sim._L
L.tg_sim_debug_trace.argtypes = [C.c_void_p, C.POINTER(C.c_ulonglong), C.c_int]
buf = (C.c_ulonglong * 80)()
sim._check(L.tg_sim_debug_trace(sim._h, buf, 80))
t = np.array(buf[:], dtype=np.float64).reshape(16, 5)
names = ["A' sweep", "reduce pAp", "B stream", "reduce rz/rr", "to next"]
rows = []
for it in range(1, 15):
    if t[it + 1, 0] == 0:
        break
    d = [t[it, 1] - t[it, 0], t[it, 2] - t[it, 1], t[it, 3] - t[it, 2], t[it, 4] - t[it, 3],
         t[it + 1, 0] - t[it, 4]]
    rows.append(d)
rows = np.array(rows) / 1e3
print("phase (us, CTA 0):", {n: round(float(v), 2) for n, v in zip(names, rows.mean(0))})
print("iteration total (us):", round(float(rows.sum(1).mean()), 2))

buf2 = (C.c_ulonglong * 400)()
sim._check(L.tg_sim_debug_trace(sim._h, buf2, 400))
pt = np.array(buf2[80:400], dtype=np.float64).reshape(64, 5)
full = (pt > 0).all(axis=1)
if full.sum() > 2:
    d = np.diff(pt[full], axis=1)
    print("plane sub-steps (SM cycles, CTA 0, %d planes): wait %.0f prep %.0f xpass %.0f "
          "ypass+z+epi %.0f" % (full.sum(), d[:, 0].mean(), d[:, 1].mean(), d[:, 2].mean(),
                                d[:, 3].mean()))
    nz = pt[:, 4] > 0
    idx = np.where(nz)[0]
    per = np.diff(pt[idx, 4]) / np.maximum(1, np.diff(idx))
    print("cycles per plane step: %.0f" % np.median(per))
