"""K1 sweep: pairs/s of the config-1 superposition for each TG_K1_P (or the\ncurrent environment only, with --one)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, os, json, torch
sys.path.insert(0, os.environ["ROOT"])
import paper_2511_20432_b200 as tg
from paper_2511_20432_b200 import workloads as W
ctx = tg.Context(0)
mat = tg.Material(**W.MATERIAL)
src = tg.discretize_scan(tg.ScanPath(W.config1_waypoints(), 0.0, 1e-3), tg.LaserSpec(**W.LASER), mat)[:65536]
t = float(src[-1, 4])
ctx.set_sources(src, mat)
pts = torch.from_numpy(W.config1_points()).cuda()
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
grad = os.environ.get("TG_SWEEP_NOGRAD") is None
for _ in range(2): ctx.superpose(pts, t, grad=grad, stream=s.cuda_stream)
torch.cuda.synchronize()
ctx.set_profiling(True); ctx.profile(reset=True)
for _ in range(3): ctx.superpose(pts, t, grad=grad, stream=s.cuda_stream)
torch.cuda.synchronize()
p = ctx.profile()
ms = p["k1_ms"] / p["k1_launches"]
print(json.dumps({"P": os.environ.get("TG_K1_P"), "P0": os.environ.get("TG_K1_P0"), "grad": grad,
                  "k1_ms": ms, "pairs_per_s": 2**20 * 2**16 / (ms * 1e-3)}))
'''
if "--one" in sys.argv:
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, ROOT=ROOT),
                       capture_output=True, text=True)
    print(r.stdout.strip() or r.stderr[-2000:])
    sys.exit(0)
for P in ("2", "3", "4", "6", "8"):
    env = dict(os.environ, TG_K1_P=P, ROOT=ROOT)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(r.stdout.strip() or r.stderr[-2000:])
