"""Per-iteration K2 time on config-4-like cuboids whose control-point count
per axis is / is not a multiple of the 32-wide tile (tile-waste study).
Usage: python tools/k2_tilewaste.py [N_iters] [elements ...]"""
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N = int(sys.argv[1]) if len(sys.argv) > 1 else 2
els = [int(a) for a in sys.argv[2:]] or [254, 256, 286]
base = open(os.path.join(ROOT, "configs", "cfg4_large.cfg")).read()
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
for e in els:
    txt = re.sub(r"^xi_elements = \d+", f"xi_elements = {e}", base, flags=re.M)
    txt = re.sub(r"^eta_elements = \d+", f"eta_elements = {e}", txt, flags=re.M)
    p = os.path.join(ROOT, "gpurun_out", f"k2tw_{e}.cfg")
    open(p, "w").write(txt)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "k2_step_rate.py"), p, str(N)],
                       capture_output=True, text=True)
    line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-400:]
    try:
        d = json.loads(line)
        nf = (e + 2) ** 2 * 65
        print(json.dumps(d), flush=True)
    except Exception:
        print(e, line, flush=True)
