"""Box probe: host RAM / cores, and the reference's setup + step cost for
configs 2 and 3 at full size (sizes the full-size parity tests)."""
import os, sys, time, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
print(subprocess.run(["free", "-g"], capture_output=True, text=True).stdout)
print("nproc", os.cpu_count())
from oracle import pyoracle
R = pyoracle.RefLib()
for cfg in sys.argv[1:]:
    t0 = time.perf_counter()
    rs = R.sim(cfg, threads=os.cpu_count(), solver_tol=1e-12)
    t1 = time.perf_counter()
    print(cfg, "open", round(t1 - t0, 2), "s", rs.info, flush=True)
    rs.reset()
    t2 = time.perf_counter()
    print(" reset", round(t2 - t1, 2), flush=True)
    for k in range(2):
        t3 = time.perf_counter()
        o = rs.step()
        print(" step", k + 1, round(time.perf_counter() - t3, 2), "s iters", o["iters"], flush=True)
    print(subprocess.run(["free", "-g"], capture_output=True, text=True).stdout, flush=True)
    rs.close()
