#!/usr/bin/env python3
"""Benchmark of the hot path (BASELINE.json metric: source x point pair
evaluations per second, with the roofline fraction).

Workload (BASELINE.json configs[1], the metric's own configuration): the
point-source superposition microbenchmark — 2^20 seeded evaluation points in a
4x4x1 mm box, 2^16 history sources on a bidirectional raster, T~ and grad T~
evaluated at t_end in fp64. One "step" = one full superpose
over all 2^20 points (6.87e10 pairs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

  * value    — pairs/s over all ranks, inputs resident in HBM, device-timed with
               CUDA events per step (L2 flushed between steps by a 256 MiB write,
               outside the step's events), max over ranks.
  * e2e      — the same metric through the C ABI with host buffers
               (tg_superpose_batch: pinned host points -> device -> host value
               and gradient), wall-clock per synchronous call.
  * roofline — K1 main kernel (k1_partial): 49 algorithmic FP64 flops per pair
                x pairs per launch / mean launch time (CUDA events
               on its stream), against the FP64 DFMA peak measured live on this
               GPU (tg_fp64_peak; MEASURED_PEAKS.json has no fp64 figure).
  * cpu_baseline — the unmodified reference's superpose (oracle/_ref, threaded
               with its own parallel_for over all host cores) on a bounded
               sample of the same workload; the C oracle port if _ref is absent.
  * --impl reference — that CPU path alone, as the reference arm.
Multi-GPU (torchrun): every rank evaluates its own 2^20-point slab against the
replicated sources (weak scaling; no data-path collective — the path shards by
points with no exchange).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def _load_workloads():
    """workloads.py by file path: the seeded inputs without importing the
    product package (the reference arm must not load any of it)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "tg_workloads", os.path.join(ROOT, "paper_2511_20432_b200", "workloads.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


W = _load_workloads()

FLOPS_PER_PAIR = 49.0  # value + gradient, exp counted at libdevice cost
# FP64-pipe instructions per pair actually issued by k1_partial's fast path
# (cuobjdump -sass of k1_partial<7,true>: 9 DFMA + 5 DADD + 3 DMUL; the
# exponential costs 6 of them with its argument where libdevice costs 18, so
# the 49-flop accounting exceeds the DFMA peak — fp64_pipe reports the
# issued-instruction fraction).
PIPE_OPS_PER_PAIR = 17.0
# with every source on one plane (a layer's scan paths; config 1 is one) the
# PLANAR variant takes rz and rz^2 per point: 8 DFMA + 5 DADD + 2 DMUL
PIPE_OPS_PER_PAIR_PLANAR = 15.0
# DRAM bytes (read + write) per launch from one `ncu --set full` capture of each
# dominant kernel (profiles/r02b_*.ncu-rep, profiles/r02_profiles_summary.md)
K1_TRAFFIC_BYTES = 43.56e6 + 81.39e6  # k1_partial<7,1,1>, config 1, one launch (4 source splits)
K2_TRAFFIC_B_PER_DOF_ITER = 72.6      # k2_cg1_kernel<2,2>, config 4 (13.54 + 12.87 GB / 84 sweeps)
K5_TRAFFIC_BYTES = 37.92e6 + 3.89e6   # sf_contract_kernel, config 4 step 1 (flux + Dirichlet)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--points", type=int, default=W.CONFIG1_POINTS)
    ap.add_argument("--sources", type=int, default=W.CONFIG1_SOURCES)
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="target CPU work for the bounded cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ncu", action="store_true", help="profiling run: no clocks/cpu legs")
    ap.add_argument("--theta-steps", type=int, default=3,
                    help="config-4 time steps for the theta-step section (0 = skip)")
    ap.add_argument("--theta-sharded", type=int, default=3,
                    help="config-4 time steps on all ranks with parallel.ShardedTimeLoop "
                         "(strong scaling of the whole step; 0 = skip)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def config1_dict(n_points, n_src, world):
    """The `config` object of both arms (identical by construction)."""
    return {"workload": "config1: 2^20 points x 2^16 raster sources, superpose at t_end",
            "points_per_gpu": n_points, "sources": n_src, "cull_exponent": 60.0,
            "parallelism": f"point slabs x{world}, sources replicated",
            "l2": "flushed between steps (256 MiB write outside the step events)"}


def workload(n_src):
    mat = dict(W.MATERIAL)
    path = dict(waypoints=W.config1_waypoints(), start_time=0.0, plane_z=1e-3)
    return mat, path, n_src


def make_sources(tg, n_src):
    src = tg.discretize_scan(tg.ScanPath(W.config1_waypoints(), 0.0, 1e-3),
                             tg.LaserSpec(**W.LASER), tg.Material(**W.MATERIAL))[:n_src]
    return src, float(src[-1, 4])


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def cpu_baseline(src, t, budget_s, threads=None):
    """Reference superpose on a bounded sample (rank 0, N=1 only)."""
    from oracle import pyoracle
    kw = dict(**W.MATERIAL, **W.LASER)
    threads = threads or os.cpu_count() or 1
    if pyoracle.ref_available():
        impl, kind = pyoracle.RefLib(), "reference"
        call = lambda pts: impl.superpose(src, pts, t, threads=threads, **kw)  # noqa: E731
        cores = threads
    else:
        impl, kind = pyoracle.COracle(), "port"
        call = lambda pts: impl.superpose(src, pts, t, **kw)  # noqa: E731
        cores = 1
    all_pts = W.config1_points()
    # calibrate on a small slice, then size the sample for ~budget_s
    n0 = max(64, min(4096, 8 * cores))
    t0 = time.perf_counter()
    call(all_pts[:n0])
    dt0 = time.perf_counter() - t0
    n = int(min(len(all_pts), max(n0, n0 * budget_s / max(dt0, 1e-6))))
    stride = max(1, len(all_pts) // n)
    pts = np.ascontiguousarray(all_pts[::stride][:n])
    t0 = time.perf_counter()
    call(pts)
    secs = time.perf_counter() - t0
    pairs = float(len(pts)) * len(src)
    return {"value": pairs / secs, "unit": "pairs/s", "cores": cores, "kind": kind,
            "sample": f"{len(pts)} of the 2^20 config-1 points (every {stride}th) x {len(src)} "
                      f"sources, value+grad at t_end, {secs:.2f} s"}


THETA_CFG = os.path.join(ROOT, "configs", "cfg4_large.cfg")
THETA_CPU_CFG = os.path.join(ROOT, "configs", "cfg2_raster_layer.cfg")
CFG3 = os.path.join(ROOT, "configs", "cfg3_contour_hatch.cfg")
HBM_PEAK_FALLBACK = 6555.2


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
    except Exception:
        return HBM_PEAK_FALLBACK, "fallback 6555.2 GB/s (BASELINE.md copy measurement)"


def config3_steps(with_cpu, steps=10):
    """Config 3 (degree-3 rational plate-with-hole part, 128x64x32 elements,
    302,974 free DOF; SURVEY.md Appendix C option A): the assembled-operator
    path. `steps` time steps from the start (contour scan) on the device with
    the reference's Jacobi-PCG and with the scaled separable-approximation
    preconditioner; the reference's own pcg_jacobi timed beside it on the
    identical A_ff for a bounded number of iterations."""
    import paper_2511_20432_b200 as tg
    out = {}
    for pc in ("jacobi", "fdm"):
        t0 = time.perf_counter()
        sim = tg.Simulation(CFG3, preconditioner=pc)
        setup_s = time.perf_counter() - t0
        ctx = sim.context()
        sim.reset()
        sim.advance(1)
        ctx.set_profiling(True)
        ctx.profile(reset=True)
        t0 = time.perf_counter()
        iters, rel = sim.advance(steps)
        wall = time.perf_counter() - t0
        prof = ctx.profile()
        ctx.set_profiling(False)
        res = {"setup_s": setup_s, "steps": steps, "ms_per_step": wall * 1e3 / steps,
               "theta_ms_per_step": prof["k2_ms"] / steps,
               "theta_step_total_ms_per_step": prof["theta_step_ms"] / steps,
               "theta_step_total_ms_per_mdof": prof["theta_step_ms"] / steps
                                               / (sim.info["n_full"] / 1e6),
               "cg_iterations_per_step": iters / steps}
        if pc == "jacobi":
            rp, ci, v = sim.reduced_operator()
            n, nnz = len(rp) - 1, len(v)
            peak, src = hbm_peak()
            us_it = 1e3 * prof["k2_ms"] / max(1, iters)
            # per CG iteration: A_ff once and the vectors p (r), Ap (w, r), x (r, w),
            # r (r, w), D^-1 (r, twice), p (r, w). A_ff is read in the implicit-column
            # layout (csr_make_dia): (2p+1)^3 slots of 8 B per row in 32-row slices,
            # zeros where a boundary row has no such column
            W3 = 7 ** 3
            slots = ((n + 31) // 32) * 32 * W3
            alg_bytes = 8.0 * slots + 8.0 * n * 11
            achieved = alg_bytes / (us_it * 1e-6) / 1e9
            res.update({"us_per_cg_iteration": us_it, "nnz": nnz,
                        "operator": "assembled A_ff with implicit columns (DIA over the free "
                                    "box: 343 offsets per row, 32-row slices), one thread per "
                                    "row, row sums in the reference's CSR order (bit-exact "
                                    "rows, equal to the sliced-ELL copy bit for bit)",
                        "roofline": {"kernel": "csr_pcg_kernel<DevDia>", "bound": "hbm",
                                     "achieved": achieved, "peak": peak, "unit": "GB/s",
                                     "frac": achieved / peak, "peak_source": src,
                                     "bytes_per_iteration": alg_bytes,
                                     "bytes_note": "8 B per stencil slot (343 per row) + 11 "
                                                   "vector streams of 8 B/DOF; the CSR form "
                                                   "would move 12 B per nonzero",
                                     "csr_bytes_per_iteration": 12.0 * nnz + 8.0 * n * 11}})
        else:
            res["preconditioner"] = ("S^-1 A~^-1 S^-1: A~ the separable approximation "
                                     "(mean control-net arc length per axis), inverted by fast "
                                     "diagonalization on DMMA mode products; S = sqrt(diag A / "
                                     "diag A~)")
        out[pc] = res
        sim.close()
    out["workload"] = ("config3: degree-(3,3,3) rational plate-with-hole part (Appendix C "
                       "option A), 128x64x32 elements, 311,885 DOF (302,974 free), contour + "
                       f"hatch path; steps 2..{steps + 1} of the 5000-step run")
    if with_cpu:
        from oracle import pyoracle
        if pyoracle.ref_available():
            sim = tg.Simulation(CFG3)
            rp, ci, v = sim.reduced_operator()
            sim.close()
            n = len(rp) - 1
            R = pyoracle.RefLib()
            b = np.random.default_rng(3).standard_normal(n)
            k = 8
            c0 = time.perf_counter()
            try:
                R.pcg(rp, ci, v, b, np.zeros(n), tol=1e-30, max_iter=k)
            except pyoracle.RefError:
                pass  # the cap: k iterations done
            secs = time.perf_counter() - c0
            ms_it = secs * 1e3 / (k + 1)  # k iterations + the initial residual matvec
            out["cpu_baseline"] = {"ms_per_cg_iteration": ms_it, "kind": "reference",
                                   "cores": 1,
                                   "sample": f"pcg_jacobi (proj/src/sparse.cpp:41-100, serial "
                                             f"as shipped) on the identical A_ff, capped at {k} "
                                             "iterations (time / (k + 1))",
                                   "theta_ms_per_step_estimate":
                                       ms_it * out["jacobi"]["cg_iterations_per_step"]}
    return out


def config2_run(with_cpu):
    """End to end: config 2's whole run_time_loop (2000 θ-steps, 64x64x16
    degree-2 cuboid, one raster layer) on the device, against the reference's
    own step at mid-run, warm-started from the same state (flux load on all
    host cores + Dirichlet values + θ-step with its serial PCG)."""
    import paper_2511_20432_b200 as tg
    sim = tg.Simulation(THETA_CPU_CFG)
    n = sim.info["n_steps"]
    sim.reset()
    sim.advance(5)  # warm-up (module load, first launches)
    sim.reset()
    ctx = sim.context()
    ctx.set_profiling(True)
    ctx.profile(reset=True)
    t0 = time.perf_counter()
    iters, rel = sim.advance(n)
    wall = time.perf_counter() - t0
    prof = ctx.profile()
    ctx.set_profiling(False)
    dofs = sim.info["n_full"]
    out = {"workload": "config2: 64x64x16 degree-2 cuboid (78,408 DOF), one-layer raster "
                       f"({sim.info['n_sources']} sources), {n} theta steps, solver_tol "
                       f"{sim.params['solver_tol']:g}",
           "steps": n, "run_s": wall, "ms_per_step": wall * 1e3 / n,
           "theta_step_total_ms_per_step": prof["theta_step_ms"] / n,
           "theta_step_total_ms_per_mdof": prof["theta_step_ms"] / n / (dofs / 1e6),
           "cg_iterations_per_step": iters / n,
           "solve_ms_per_step": prof["k2_ms"] / n,
           "us_per_cg_iteration": 1e3 * prof["k2_ms"] / max(1, iters),
           "solver": "k2_res_kernel: single-sweep Jacobi-PCG with u, s, w (block + halo), x, p "
                     "and D resident in shared memory, one CTA per 6x6x17 column block, w's "
                     "halo through L2 (csrc/k2_resident.cu)",
           "timing": "wall clock around the "
           "synchronous tg_sim_advance(n) call (device-resident state)"}
    k = n // 2
    if with_cpu:
        from oracle import pyoracle
        if pyoracle.ref_available():
            sim.reset()
            sim.advance(k - 1)
            st = sim.state()  # the step k-1 state both sides continue from
            R = pyoracle.RefLib()
            rs = R.sim(THETA_CPU_CFG)
            dt = rs.params["dt"]
            t0_, t1 = (k - 1) * dt, k * dt
            F0 = rs.flux_load(t0_, threads=os.cpu_count())
            g0 = rs.dirichlet(t0_)
            c0 = time.perf_counter()
            F1 = rs.flux_load(t1, threads=os.cpu_count())
            c1 = time.perf_counter()
            g1 = rs.dirichlet(t1)
            c2 = time.perf_counter()
            _, its, _ = rs.theta_step(st["free"], g0, F0, F1, g1, rs.params["solver_tol"])
            c3 = time.perf_counter()
            rs.close()
            out["cpu_baseline"] = {
                "ms_per_step": (c3 - c0) * 1e3, "kind": "reference", "cores": os.cpu_count(),
                "flux_load_ms": (c1 - c0) * 1e3, "dirichlet_ms": (c2 - c1) * 1e3,
                "theta_step_ms": (c3 - c2) * 1e3,
                "theta_step_ms_per_mdof": (c3 - c2) * 1e3 / (dofs / 1e6),
                "cg_iterations": its,
                "sample": f"the reference's step {k} (t = {t1:g} s), warm-started from the "
                          "device run's step-(k-1) state: assemble_flux_load (threaded over "
                          "all cores), dirichlet_values and theta_step (serial, as shipped)",
                "run_s_estimate": (c3 - c0) * n}
    sim.close()
    return out


def theta_section(steps, warmup, with_cpu):
    """Config 4 (4.39M DOF, 1e5 sources): full run_time_loop steps on the device."""
    import paper_2511_20432_b200 as tg
    t0 = time.perf_counter()
    sim = tg.Simulation(THETA_CFG)
    setup_s = time.perf_counter() - t0
    ctx = sim.context()
    sim.reset()
    if warmup:
        sim.advance(warmup)
    flops0 = sim.sumfact_stats()["gemm_flops"]
    ctx.set_profiling(True)
    ctx.profile(reset=True)
    t0 = time.perf_counter()
    iters, _ = sim.advance(steps)
    wall = time.perf_counter() - t0
    prof = ctx.profile()
    ctx.set_profiling(False)
    sf = sim.sumfact_stats()
    k5_flops = (sf["gemm_flops"] - flops0) / steps
    dmma_peak = ctx.dmma_peak_tflops()
    # the same steps (same step indices, from a reset) with every
    # superposition pair on K1 (K5 off), for the split
    sim.set_sumfact(False)
    sim.reset()
    if warmup:
        sim.advance(warmup)
    ctx.set_profiling(True)
    ctx.profile(reset=True)
    sim.advance(steps)
    prof_k1 = ctx.profile()
    ctx.set_profiling(False)
    sim.set_sumfact(True)
    dofs = sim.info["n_full"]
    solver = {2: "single-sweep Chronopoulos-Gear Jacobi-PCG (one tile sweep + one grid "
                 "reduction per iteration)",
              1: "two-phase Jacobi-PCG (direction sweep + streaming update)",
              0: "assembled CSR Jacobi-PCG"}[sim.info["kronecker"]]
    kernel = {2: "k2_cg1_kernel", 1: "k2_pcg_kernel", 0: "csr_pcg_kernel"}[sim.info["kronecker"]]
    k2_ms = prof["k2_ms"] / steps
    peak, src = hbm_peak()
    achieved = prof["k2_bytes"] / (prof["k2_ms"] * 1e-3) / 1e9 if prof["k2_ms"] else None
    k5_ms = prof["k5_ms"] / steps
    k5_tf = k5_flops / (k5_ms * 1e-3) / 1e12 if k5_ms else None
    out = {
        "workload": "config4: 256x256x64 degree-2 cuboid (4,393,224 DOF), 1e5 sources, "
                    "theta = 0.5, dt = 1e-5, solver_tol 1e-10",
        "steps": steps, "warmup": warmup, "setup_s": setup_s,
        "ms_per_step": prof["step_ms"] / steps,
        "ms_per_step_wall": wall * 1e3 / steps,
        "timing": "ms_per_step: CUDA events on the simulation stream around the "
                  "tg_sim_advance(steps) call (loads + theta steps, no host sync between steps)",
        "theta_ms_per_step": k2_ms,
        "theta_ms_per_step_per_mdof": k2_ms / (dofs / 1e6),
        "theta_step_total_ms_per_step": prof["theta_step_ms"] / steps,
        "theta_step_total_ms_per_mdof": prof["theta_step_ms"] / steps / (dofs / 1e6),
        "theta_step_total_note": "SURVEY.md §8d's 'theta-step time per 1M DOF' is the whole "
                                 "step: expand + theta RHS + solve (theta_step, "
                                 "timestep.cpp:5-24); theta_ms_* are the solve alone",
        "k1_ms_per_step": prof["k1_ms"] / steps,
        "k5": {"note": "fused sum-factorised superposition (csrc/k5_fused.cu): the flux-load and "
                       "Dirichlet sums over the sources no cull reaches in each region, as an "
                       "on-chip exponential generator + DMMA m8n8k4 contraction; the pair-wise "
                       "remainder on K1 (k1_ms_per_step)",
               "kernel": "sf_contract_kernel",
               "contraction_ms_per_step": k5_ms,
               "contraction_flops_per_step": k5_flops,
               "roofline": {"bound": "fp64 tensor (DMMA)", "achieved": k5_tf,
                            "peak": dmma_peak, "unit": "TFLOP/s",
                            "frac": k5_tf / dmma_peak if (k5_tf and dmma_peak) else None,
                            "peak_source": "measured live: tg_dmma_peak (independent DMMA "
                                           "m8n8k4 accumulators) on this GPU",
                            "traffic": K5_TRAFFIC_BYTES,
                            "traffic_source": "ncu --set full, profiles/r02b_k5_contract.ncu-rep "
                                              "(dram read + write per launch)"},
               "min_region_prefix_flux": sf["last_j_flux"],
               "min_region_prefix_dirichlet": sf["last_j_dirichlet"],
               "sources": sim.info["n_sources"],
               "ms_per_step_with_k1_only": prof_k1["step_ms"] / steps},
        "cg_iterations_per_step": iters / steps,
        "solver": solver,
        "roofline": {"kernel": kernel, "bound": "hbm",
                     "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if achieved else None,
                     "traffic": (K2_TRAFFIC_B_PER_DOF_ITER * sim.info["n_free"] * iters / steps
                                 if sim.info["kronecker"] == 2 else None),
                     "traffic_source": "ncu --set full, profiles/r02b_k2_cg1.ncu-rep: "
                                       "72.6 B/DOF/iteration measured, per solve",
                     "peak_source": src,
                     "bytes_per_dof_per_iteration": 104},
    }
    out["cpu_baseline"] = {
        "note": "the reference's own step on config 4 takes ~5 min of host time (138 s setup, "
                "85 s threaded flux load, 66 s serial PCG for one theta step; "
                "profiles/r02_cfg4_ref_theta.md), too long for this bench; the reference's "
                "warm-started step on config 2 is config2_run.cpu_baseline"}
    sim.close()
    try:
        out["fdm_option"] = theta_fdm(steps, warmup)
    except Exception as e:  # reported, not fatal
        out["fdm_option"] = {"error": str(e)}
    try:
        out["config2_run"] = config2_run(with_cpu)
    except Exception as e:  # reported, not fatal
        out["config2_run"] = {"error": str(e)}
    try:
        out["config3_steps"] = config3_steps(with_cpu)
    except Exception as e:  # reported, not fatal
        out["config3_steps"] = {"error": str(e)}
    return out


def theta_sharded_section(steps, rank, world, local):
    """Config-4 time steps on all ranks (strong scaling of the whole step):
    the loads' K5 regions and the θ-step's z-slabs split over the GPUs
    (parallel.ShardedTimeLoop -> tg_sim_shard; one rank: plain advance).
    Device time per step (CUDA events around tg_sim_advance on each rank's
    simulation stream), max over ranks."""
    import torch
    import paper_2511_20432_b200 as tg
    from paper_2511_20432_b200 import parallel
    import torch.distributed as dist
    sim = tg.Simulation(THETA_CFG, device=local)
    loop = parallel.ShardedTimeLoop(sim, parallel.Dist(rank, world, f"cuda:{local}"))
    ctx = sim.context()
    loop.reset()
    loop.step(2)
    ctx.set_profiling(True)
    ctx.profile(reset=True)
    its, _ = loop.step(steps)
    prof = ctx.profile()
    ctx.set_profiling(False)
    ms = prof["step_ms"] / steps  # this rank's; the caller takes the max over ranks
    st = sim.state()
    sim.close()
    return {"workload": f"config4 time steps on {world} GPU(s): K5 regions and theta-step "
                        "z-slabs split over the ranks (NCCL all-reduce of the loads, halo + "
                        "partial-sum exchange per CG iteration)" if world > 1 else
                        "config4 time steps on 1 GPU (no split)",
            "n_gpus": world, "steps": steps, "ms_per_step": float(ms),
            "cg_iterations_per_step": its / steps,
            "state_checksum": float(np.abs(st["free"]).sum()),
            "timing": "CUDA events around tg_sim_advance on each rank's stream, max over ranks",
            "scaling": "strong"}


def theta_fdm(steps, warmup):
    """The opt-in fast-diagonalization preconditioner on the
    same config-4 steps: θ-step solve time and CG iterations."""
    import paper_2511_20432_b200 as tg
    sim = tg.Simulation(THETA_CFG, preconditioner="fdm")
    ctx = sim.context()
    sim.reset()
    if warmup:
        sim.advance(warmup)
    ctx.set_profiling(True)
    ctx.profile(reset=True)
    iters, rel = sim.advance(steps)
    prof = ctx.profile()
    ctx.set_profiling(False)
    dofs = sim.info["n_full"]
    k2_ms = prof["k2_ms"] / steps
    sim.close()
    return {"preconditioner": "fast diagonalization (V diag(1/(a + b(lx+ly+lz))) V^T, "
                              "mode products on the hand-written DMMA GEMM), same PCG stop test",
            "theta_ms_per_step": k2_ms, "theta_ms_per_step_per_mdof": k2_ms / (dofs / 1e6),
            "theta_step_total_ms_per_step": prof["theta_step_ms"] / steps,
            "theta_step_total_ms_per_mdof": prof["theta_step_ms"] / steps / (dofs / 1e6),
            "cg_iterations_per_step": iters / steps, "last_rel_residual": rel}


def run_reference(args):
    """The reference's own CPU implementation of the path: the unmodified
    reference library's superpose (oracle/_ref, its parallel_for over every
    host core), on the same workload. Nothing of the product package is
    imported or loaded here. Each step evaluates a fixed strided sample of
    the 2^20 points against all 2^16 sources (the full set would take ~80 s
    per step on 16 cores); value and ms_per_step are the sample's measured
    rate and time."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import pyoracle
    threads = os.cpu_count() or 1
    kw = dict(**W.MATERIAL, **W.LASER)
    if pyoracle.ref_available():
        impl, kind, cores = pyoracle.RefLib(), "reference", threads
        call = lambda pts: impl.superpose(src, pts, t, threads=threads, **kw)  # noqa: E731
    else:  # the pinned C port (oracle/oracle.c), one thread
        impl, kind, cores = pyoracle.COracle(), "port", 1
        call = lambda pts: impl.superpose(src, pts, t, **kw)  # noqa: E731
    src = impl.discretize_scan(W.config1_waypoints(), start_time=0.0, plane_z=1e-3,
                               **W.LASER, **W.MATERIAL)[:args.sources]
    t = float(src[-1, 4])
    all_pts = W.config1_points(args.points)
    # one step ~ per_step seconds so that the whole --steps/--warmup run ends
    # within a few minutes
    per_step = max(0.5, min(10.0, 100.0 / max(1, args.steps + args.warmup)))
    n0 = max(64, 8 * cores)
    call(all_pts[:n0])  # thread / page warm-up, then calibrate
    c0 = time.perf_counter()
    call(all_pts[:n0])
    dt0 = time.perf_counter() - c0
    n = int(min(len(all_pts), max(n0, n0 * per_step / max(dt0, 1e-6))))
    stride = max(1, len(all_pts) // n)
    sample = np.ascontiguousarray(all_pts[::stride][:n])
    for _ in range(args.warmup):
        call(sample)
    secs = []
    for _ in range(args.steps):
        c0 = time.perf_counter()
        call(sample)
        secs.append(time.perf_counter() - c0)
    pairs = float(len(sample)) * len(src)
    v = pairs * len(secs) / sum(secs)
    desc = (f"{len(sample)} of the 2^20 config-1 points (every {stride}th) x {len(src)} sources "
            f"per step, value+grad at t_end")
    line = {
        "impl": "reference", "metric": "source x point pair evals/s (superpose, value+grad)",
        "value": v, "unit": "pairs/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sum(secs) / len(secs),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, SURVEY.md §8d)",
        "config": config1_dict(W.CONFIG1_POINTS, len(src), args.gpus),
        "sample": {"sample_points": len(sample), "sample_fraction": len(sample) / len(all_pts),
                   "pairs_per_step": pairs,
                   "note": "ms_per_step is the measured time of the sampled step actually run"},
        "cpu_baseline": {"value": v, "unit": "pairs/s", "cores": cores, "kind": kind,
                         "sample": desc},
        "e2e": {"value": v, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import paper_2511_20432_b200 as tg

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
        # a rank stuck in the sharded section's own NCCL calls aborts them and
        # reports an error instead of holding the job (csrc/slab.cu stream_wait)
        os.environ.setdefault("TG_NCCL_TIMEOUT", "90")
    dev = torch.device("cuda", local)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    ctx = tg.Context(local)
    src, t = make_sources(tg, args.sources)
    ctx.set_sources(src, tg.Material(**W.MATERIAL))
    n = args.points
    # weak scaling: each rank owns its own seeded slab of 2^20 points
    pts_np = W.config1_points(n, seed=W.CONFIG1_SEED + rank)
    pts = torch.from_numpy(pts_np).to(dev)
    val = torch.empty(n, dtype=torch.float64, device=dev)
    grad = torch.empty((n, 3), dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.Stream(dev)  # a real stream: events and kernels share it
    torch.cuda.set_stream(stream)
    sp = stream.cuda_stream
    pairs_per_step = float(n) * len(src)

    def step():
        ctx.superpose(pts, t, out=(val, grad), stream=sp)

    fp64_peak = ctx.fp64_peak_tflops() if not args.ncu else None

    for _ in range(args.warmup):
        step()
    barrier()

    ctx.set_profiling(True)
    ctx.profile(reset=True)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    sampler = ClockSampler(local)
    barrier()
    with sampler:
        for i in range(args.steps):
            flush.zero_()  # on `stream`, outside the step's events
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    prof = ctx.profile()
    ctx.set_profiling(False)
    total_ms = float(sum(step_ms))
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    value = world * pairs_per_step * args.steps / (total_ms * 1e-3)

    # e2e through the C ABI with host buffers (pinned), H2D + compute + D2H per step
    pin_pts = torch.from_numpy(pts_np).pin_memory()
    pin_val = torch.empty(n, dtype=torch.float64).pin_memory()
    pin_grad = torch.empty((n, 3), dtype=torch.float64).pin_memory()
    pv, pg = pin_val.numpy(), pin_grad.numpy()
    pp = pin_pts.numpy()
    for _ in range(max(1, args.warmup // 2)):
        ctx.superpose(pp, t, out=(pv, pg))
    barrier()
    e2e_s = 0.0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ctx.superpose(pp, t, out=(pv, pg))
        e2e_s += time.perf_counter() - t0
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    e2e = world * pairs_per_step * args.steps / e2e_s

    sharded = None
    if args.theta_sharded > 0:  # collective: every rank takes part
        try:
            sharded = theta_sharded_section(args.theta_sharded, rank, world, local)
        except Exception as e:
            sharded = {"error": str(e)}
        if world > 1:  # every rank gets here (success or error): one agreement step
            import torch
            import torch.distributed as dist
            t = torch.tensor([sharded.get("ms_per_step", 0.0), 1.0 if "error" in sharded else 0.0],
                             dtype=torch.float64, device=f"cuda:{local}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            if t[1].item() > 0.0 and "error" not in sharded:
                sharded = {"error": "another rank failed in the sharded section"}
            elif "error" not in sharded:
                sharded["ms_per_step"] = float(t[0].item())

    if rank != 0:
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()
        return 0

    k1_mean_ms = prof["k1_ms"] / max(1, prof["k1_launches"])
    pairs_per_launch = prof["k1_pairs"] / max(1, prof["k1_launches"])
    planar = bool(len(src)) and bool(np.all(src[:, 2] == src[0, 2])) and \
        not os.environ.get("TG_K1_NO_PLANAR")
    ops = PIPE_OPS_PER_PAIR_PLANAR if planar else PIPE_OPS_PER_PAIR
    # the roofline: FP64 instructions the kernel must issue per pair x pairs
    # per launch / mean launch time, against the FP64 pipe's DFMA issue rate
    # (peak TFLOP/s / 2 instructions per second); MEASURED_PEAKS.json and the
    # profiling recipe carry no FP64 figure, so the peak is the DFMA-chain
    # microbenchmark run live on this GPU
    pipe_peak = fp64_peak * 1e12 / 2 if fp64_peak else None
    achieved_ops = ops * pairs_per_launch / (k1_mean_ms * 1e-3) if k1_mean_ms else None
    alg = FLOPS_PER_PAIR * pairs_per_launch / (k1_mean_ms * 1e-3) / 1e12 if k1_mean_ms else None
    roof = {"kernel": f"k1_partial<{os.environ.get('TG_K1_P', '7')},true,{str(planar).lower()}>",
            "bound": "fp64",
            "achieved": achieved_ops / 1e12 if achieved_ops else None,
            "peak": pipe_peak / 1e12 if pipe_peak else None,
            "unit": "T FP64 instr/s",
            "frac": (achieved_ops / pipe_peak) if (achieved_ops and pipe_peak) else None,
            "traffic": K1_TRAFFIC_BYTES,
            "traffic_source": "ncu --set full, profiles/r02c_k1_full.ncu-rep (dram "
                              "read+write)",
            "peak_source": "measured live: tg_fp64_peak DFMA-chain microbenchmark on this GPU "
                           "(no FP64 entry in MEASURED_PEAKS.json or the recipe's fallback)",
            "ops_per_pair": ops, "pairs_per_launch": pairs_per_launch,
            "mean_launch_ms": k1_mean_ms,
            "note": "frac = issued FP64-pipe instructions per pair (cuobjdump -sass of the "
                    "kernel: 15 planar / 17 general) x pair rate / the pipe's issue rate. "
                    "flops_49 restates it with SURVEY.md §8d's 49 flops/pair, which counts the "
                    "exponential at its libdevice cost (31 flops) where this kernel spends 6 "
                    "instructions, so that figure exceeds 1 and is not a roofline",
            "flops_49": {"achieved_tflops": alg, "peak_tflops": fp64_peak,
                         "frac": (alg / fp64_peak) if (alg and fp64_peak) else None},
            "k1_share_of_step": prof["k1_ms"] / max(1e-9, float(sum(step_ms)))}
    line = {
        "metric": "source x point pair evals/s (superpose, value+grad)",
        "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, SURVEY.md §8d)",
        "config": config1_dict(n, len(src), world),
        "e2e": {"value": e2e, "unit": "pairs/s", "h2d_bytes_per_step": int(pp.nbytes),
                "d2h_bytes_per_step": int(pv.nbytes + pg.nbytes)},
        "gpu_launches": prof["launches"],
        "roofline": roof,
        "clocks": sampler.summary(),
    }
    if world == 1 and not args.no_cpu_baseline and not args.ncu:
        try:
            line["cpu_baseline"] = cpu_baseline(src, t, args.cpu_seconds)
        except Exception as e:  # reported, not fatal
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    if world == 1 and args.theta_steps > 0:
        try:
            line["theta_step"] = theta_section(args.theta_steps, 1,
                                               not args.no_cpu_baseline and not args.ncu)
        except Exception as e:
            line["theta_step"] = {"error": str(e)}
    if sharded is not None:
        line["theta_step_sharded"] = sharded
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
