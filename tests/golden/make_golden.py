"""Regenerate the committed golden vectors from the UNMODIFIED reference
library (oracle/_ref, built from /root/reference by oracle/Makefile).

    python tests/golden/make_golden.py [k1] [cfg0]

The fixtures let the GPU-side parity tests run on hosts where the reference
sources are not mounted; tests/test_oracle_pins.py re-checks them against the
live reference whenever it is available.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import pyoracle  # noqa: E402
from paper_2511_20432_b200 import workloads as W  # noqa: E402

K1_SAMPLE = 2048


def k1(R):
    kw = dict(**W.MATERIAL, **W.LASER)
    src = R.discretize_scan(W.config1_waypoints(), plane_z=1e-3, **kw)[:W.CONFIG1_SOURCES]
    t = float(src[-1, 4])
    pts = W.config1_points()[:K1_SAMPLE]
    val, grad = R.superpose(src, pts, t, threads=os.cpu_count(), **kw)
    # single dwell source probed around activation (causality, peak, cull)
    dwell = R.discretize_scan([[1e-3, 1e-3]], plane_z=1e-3, **kw)
    g = np.linspace(-2e-4, 2e-4, 9)
    probe = np.array([[1e-3 + a, 1e-3 + b, 1e-3 + c] for a in g for b in g[::2] for c in g[::4]])
    times = np.array([dwell[0, 5] - 1e-9, dwell[0, 5], dwell[0, 5] + 1e-9, dwell[0, 4], 1e-5,
                      1e-4, 1e-3])
    dv = np.zeros((len(times), len(probe)))
    dg = np.zeros((len(times), len(probe), 3))
    for i, tt in enumerate(times):
        dv[i], dg[i] = R.superpose(dwell, probe, tt, **kw)
    np.savez_compressed(os.path.join(HERE, "k1_cfg1.npz"), t=t, n_sources=len(src),
                        sample=K1_SAMPLE, val=val, grad=grad, dwell=dwell, probe=probe,
                        times=times, dwell_val=dv, dwell_grad=dg)
    print("k1_cfg1.npz", val.shape)


if __name__ == "__main__":
    what = sys.argv[1:] or ["k1"]
    pyoracle.build(ref=True)
    R = pyoracle.RefLib()
    if "k1" in what:
        k1(R)


SIM_STEPS = {"cfg0_parity": [1, 2, 3, 5, 10, 25, 50, 75, 100], "qc_small": [1, 2, 5, 12, 24],
             "cfg0_oddx": [1, 2, 10, 40], "cfg3_parity": [1, 2, 5, 10, 20, 40]}


def sim_run(R, name):
    """Per-step F, g, free coefficients and CG iterations of run_time_loop."""
    path = os.path.join(ROOT, "configs", name + ".cfg")
    sim = R.sim(path)
    F0, g0 = sim.reset()
    keep = SIM_STEPS[name]
    out = {"F0": F0, "g0": g0, "steps": np.array(keep)}
    iters = []
    for s in range(1, max(keep) + 1):
        r = sim.step()
        iters.append(r["iters"])
        if s in keep:
            out[f"F{s}"], out[f"g{s}"], out[f"x{s}"] = r["F"], r["g"], r["free"]
    out["iters"] = np.array(iters)
    # one flux load and Dirichlet vector at a mid time, and the operator on a probe vector
    t = 0.37 * max(keep) * sim.params["dt"]
    out["t_mid"] = t
    out["F_mid"] = sim.flux_load(t)
    out["g_mid"] = sim.dirichlet(t)
    rp, ci, v = sim.csr(2)
    x = np.random.default_rng(5).standard_normal(sim.info["n_free"])
    out["Ax_probe"] = x
    out["Ax"] = np.array([np.dot(v[rp[i]:rp[i + 1]], x[ci[rp[i]:rp[i + 1]]])
                          for i in range(len(rp) - 1)])
    np.savez_compressed(os.path.join(HERE, f"sim_{name}.npz"), **out)
    print(f"sim_{name}.npz", sum(iters), "CG iterations")
    sim.close()


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "sim":
    R = pyoracle.RefLib()
    for name in (sys.argv[2:] or SIM_STEPS):
        sim_run(R, name)
