"""The reference's remaining known-answer pins for the time-step path
(SURVEY.md §8c), re-run through the GPU path:

* the pipeline fixture's probe history (proj/tests/test_pipeline.cpp:19-64):
  24 steps, T̂ at point A exactly 0 at t = 0, its peak in steps 14..24 and in
  (5, 25) degC — with the reference's bounds — and the whole history against
  the compiled reference's own loop;
* the scalar amplification factor of one θ-step
  (proj/tests/test_timestep.cpp:52-71), on the operator/solver calls;
* the manufactured solution (proj/tests/mms_common.hpp, test_mms.cpp:12-68):
  spatial order >= 2.7 on the 4/8/16 ladder and Crank-Nicolson's factor-4 error
  ratios, with the reference's bounds. The separable loads and the L2
  projection are built here with numpy (1D Gauss rules on scipy B-splines);
  every θ-step and the error quadrature's field evaluation run on the GPU
  (tg_sim_theta_step: K2; tg_sim_field_eval: K4)."""
import os

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.interpolate import BSpline

import paper_2511_20432_b200 as tg
from conftest import ROOT

pytestmark = pytest.mark.gpu


def full_of(info, free, g):
    full = np.zeros((info["nz"], info["ny"], info["nx"]))
    full[1:] = free.reshape(info["nz"] - 1, info["ny"], info["nx"])
    full[0] = g.reshape(info["ny"], info["nx"])
    return full.ravel()


# --- test_pipeline.cpp:40-64 ----------------------------------------------

def test_probe_history_peaks_in_the_reference_window(ref):
    cfg = os.path.join(ROOT, "configs", "qc_single_source_small.cfg")
    A = np.array([[0.5, 0.0, 1.0]])
    sim = tg.Simulation(cfg)
    r = ref.sim(cfg)
    try:
        assert sim.info["n_steps"] == 24
        sim.reset()
        r.reset()
        ours = [sim.probe(A)[0, 5]]
        theirs = [0.0]
        for _ in range(24):
            sim.advance(1)
            ours.append(sim.probe(A)[0, 5])
            st = r.step()
            theirs.append(r.field_at(full_of(r.info, st["free"], st["g"]), A[0])[0])
    finally:
        sim.close()
        r.close()
    ours, theirs = np.array(ours), np.array(theirs)
    assert len(ours) == 25 and ours[0] == 0.0
    peak = int(np.argmax(ours))
    assert 14 <= peak <= 24
    assert 5.0 < ours[peak] < 25.0
    # both loops stop their PCG at 1e-10: the histories agree far inside that
    assert peak == int(np.argmax(theirs))
    assert np.abs(ours - theirs).max() <= 1e-8 * np.abs(theirs).max()


# --- test_timestep.cpp:52-71 ----------------------------------------------

@pytest.mark.parametrize("theta,expect", [(1.0, 0.5), (0.5, 1.0 / 3.0), (0.0, 0.0)])
def test_scalar_amplification_factor(theta, expect):
    lam, dt, u0 = 1.0, 1.0, 1.0
    ctx = tg.Context(0)
    try:
        M = sp.csr_matrix(np.array([[1.0]]))
        K = sp.csr_matrix(np.array([[lam]]))
        A = sp.csr_matrix(M + theta * dt * K)
        B = sp.csr_matrix(M - (1.0 - theta) * dt * K)
        B.eliminate_zeros()
        rhs = ctx.csr_multiply(B, np.array([u0])) if B.nnz else np.zeros(1)
        x, _, _ = ctx.pcg_jacobi(A, rhs, x=np.array([u0]), tol=1e-14, max_iter=100)
    finally:
        ctx.close()
    assert abs(x[0] - expect) <= 1e-12 * max(1.0, abs(expect))


# --- mms_common.hpp / test_mms.cpp ----------------------------------------

EDGE, LAMBDA = 1e-3, 100.0
MAT = dict(conductivity=42.0, density=4420.0, heat_capacity=990.0)  # test_util.hpp ti64()


def cube_cfg(tmp_path, n, dt, t_end):
    h = EDGE / 2
    cps = "\n".join(f"cp = {i * h!r} {j * h!r} {k * h!r} 1"
                    for k in range(3) for j in range(3) for i in range(3))
    txt = f"""[geometry]
degrees = 2 2 2
knots_xi = 0 0 0 1 1 1
knots_eta = 0 0 0 1 1 1
knots_zeta = 0 0 0 1 1 1
grid_dims = 3 3 3
{cps}
[material]
conductivity = {MAT['conductivity']}
density = {MAT['density']}
heat_capacity = {MAT['heat_capacity']}
platform_temperature = 0.0
[laser]
power = 1.0
speed = 1.0
spot_radius = 2e-5
absorptivity = 1.0
dt = 1e-5
[scan]
start_time = 0.0
waypoint = 5e-4 5e-4
[faces]
ximin = lateral
ximax = lateral
etamin = lateral
etamax = lateral
zetamin = bottom
zetamax = top
[mesh]
xi_elements = {n}
eta_elements = {n}
zeta_elements = {n}
[stepping]
theta = 0.5
dt = {dt!r}
t_end = {t_end!r}
solver_tol = 1e-12
max_iter = 4000
"""
    p = tmp_path / f"mms_{n}_{dt:.3e}.cfg"
    p.write_text(txt)
    return str(p)


GX, GW = np.polynomial.legendre.leggauss(8)


def basis_1d(n):
    """Degree-2 open uniform basis on [0, EDGE] with n elements: the values
    at an 8-point Gauss rule per element and the rule (x, w)."""
    kn = np.concatenate([[0.0, 0.0], np.linspace(0.0, 1.0, n + 1), [1.0, 1.0]]) * EDGE
    el = np.linspace(0.0, EDGE, n + 1)
    x = (0.5 * (el[:-1] + el[1:])[:, None] + 0.5 * (EDGE / n) * GX[None, :]).ravel()
    w = np.tile(0.5 * (EDGE / n) * GW, n)
    N = BSpline.design_matrix(x, kn, 2).toarray()  # (points, n + 2)
    return N, x, w


def mms_run(tmp_path, n, dt, t_end):
    k, rc = MAT["conductivity"], MAT["density"] * MAT["heat_capacity"]
    N, x, w = basis_1d(n)
    sx, sy, sz = (np.cos(np.pi * x / (2 * EDGE)), np.cos(np.pi * x / EDGE),
                  np.sin(np.pi * x / (2 * EDGE)))
    fx, fy, fz = (N.T @ (w * s) for s in (sx, sy, sz))
    M1 = N.T @ (w[:, None] * N)
    # F(0): the volumetric source plus k grad(u).n on ximax (the other lateral
    # faces are adiabatic for this mode, the top face too)
    lap = -1.5 * np.pi ** 2 / EDGE ** 2
    F0 = (-rc * LAMBDA - k * lap) * np.einsum("k,j,i->kji", fz, fy, fx)
    F0[:, :, -1] += -k * np.pi / (2 * EDGE) * np.einsum("k,j->kj", fz, fy)
    F0 = F0.ravel()
    # u(0): the L2 projection onto the free DOFs (a Kronecker solve)
    cx, cy = np.linalg.solve(M1, fx), np.linalg.solve(M1, fy)
    cz = np.linalg.solve(M1[1:, 1:], fz[1:])
    free = np.einsum("k,j,i->kji", cz, cy, cx).ravel()

    sim = tg.Simulation(cube_cfg(tmp_path, n, dt, t_end))
    try:
        info = sim.info
        assert info["kronecker"] >= 1 and info["n_free"] == len(free)  # matrix-free K2
        g = np.zeros(info["n_constrained"])
        steps = int(round(t_end / dt))
        Fn = F0
        for s in range(1, steps + 1):
            Fn1 = F0 * np.exp(-LAMBDA * s * dt)
            free, _, _ = sim.theta_step(free, g, Fn, Fn1, g, tol=1e-12, max_iter=4000)
            Fn = Fn1
        # L2 error at t_end with a 5-point rule per element and direction
        gx, gw = np.polynomial.legendre.leggauss(5)
        el = np.linspace(0.0, 1.0, n + 1)
        q = (0.5 * (el[:-1] + el[1:])[:, None] + 0.5 / n * gx[None, :]).ravel()
        qw = np.tile(0.5 * EDGE / n * gw, n)
        Z, Y, X = np.meshgrid(q, q, q, indexing="ij")
        xi = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)
        W3 = np.einsum("k,j,i->kji", qw, qw, qw).ravel()
        xp, f = sim.field_eval(full_of(info, free, g), xi)
    finally:
        sim.close()
    exact = (np.cos(np.pi * xp[:, 0] / (2 * EDGE)) * np.cos(np.pi * xp[:, 1] / EDGE) *
             np.sin(np.pi * xp[:, 2] / (2 * EDGE)) * np.exp(-LAMBDA * t_end))
    return float(np.sqrt(np.sum(W3 * (f[:, 0] - exact) ** 2))), free


def test_mms_spatial_order(tmp_path):
    t_end = 2e-3
    meshes = [4, 8, 16]
    errs = [mms_run(tmp_path, n, t_end / 256.0, t_end)[0] for n in meshes]
    slope = np.polyfit(np.log(1.0 / np.array(meshes)), np.log(errs), 1)[0]
    assert errs[0] > errs[1] > errs[2], errs
    assert slope >= 2.7, (errs, slope)  # p + 0.7 for p = 2 (the reference measures 3.08)


def test_mms_crank_nicolson_order(tmp_path):
    t_end, n = 2e-3, 8
    fine = mms_run(tmp_path, n, t_end / 128.0, t_end)[1]
    errs = [np.linalg.norm(mms_run(tmp_path, n, t_end / d, t_end)[1] - fine) for d in (4, 8, 16)]
    r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
    assert 3.2 <= r1 <= 4.8 and 3.2 <= r2 <= 4.8, errs
    assert np.log2(r1) >= 1.8 and np.log2(r2) >= 1.8


# --- acceptance criteria 5 and 6 (proj/tests/acceptance.cpp:232-294) -------

# the fine level (132 x 24 x 18, t_end = 2.6e-4) run through the compiled
# reference's loop (oracle/_ref, 25 s of host time; the recipe is this test
# with RefSim in place of Simulation): T̂(A, 1.9e-4 s), its peak, the flux ratio
FINE_REF = dict(t_hat=10.306120024655076, peak=10.428042458929205, ratio=0.003494566015296245)
LEVELS = [((16, 10, 9), 1.9e-4), ((23, 13, 11), 1.9e-4), ((32, 16, 14), 1.9e-4),
          ((132, 24, 18), 2.6e-4)]


def level_cfg(tmp_path, el, t_end):
    txt = open(os.path.join(ROOT, "configs", "qc_single_source_small.cfg")).read()
    for old, new in (("\nxi_elements = 16\n", f"\nxi_elements = {el[0]}\n"),
                     ("\neta_elements = 6\n", f"\neta_elements = {el[1]}\n"),
                     ("\nzeta_elements = 6\n", f"\nzeta_elements = {el[2]}\n"),
                     ("\nt_end = 2.4e-4\n", f"\nt_end = {t_end!r}\n")):
        assert old in txt
        txt = txt.replace(old, new)
    p = tmp_path / f"level_{el[0]}.cfg"
    p.write_text(txt)
    return str(p)


def run_level(sim_like, gpu):
    """run_single_source_level: T̂ at A per step, the etamin flux profile's
    integrated |q_net| / |q_tilde| at step 19."""
    A = np.array([[0.5, 0.0, 1.0]])
    out = dict(peak=0.0)
    sim_like.reset()
    for s in range(1, sim_like.info["n_steps"] + 1):
        if gpu:
            sim_like.advance(1)
            v = sim_like.probe(A)[0, 5]
        else:
            st = sim_like.step()
            full = full_of(sim_like.info, st["free"], st["g"])
            v = sim_like.field_at(full, A[0])[0]
        out["peak"] = max(out["peak"], v)
        if s == 19:
            out["t_hat"] = v
            if gpu:
                prof = sim_like.boundary_flux_profile("etamin", 400, theta_axis=(2e-3, 0.0))
                out["ratio"] = tg.integrated_abs_flux(prof)["ratio"]
            else:
                _, met = sim_like.flux_profile(full, 2, 400, s * 1e-5, theta_axis=(2e-3, 0.0))
                out["ratio"] = met[2]
    return out


def test_single_source_ladder_acceptance(tmp_path, ref):
    ours, theirs = [], []
    for k, (el, t_end) in enumerate(LEVELS):
        cfg = level_cfg(tmp_path, el, t_end)
        sim = tg.Simulation(cfg)
        try:
            ours.append(run_level(sim, True))
        finally:
            sim.close()
        if k < 3:
            r = ref.sim(cfg)
            try:
                theirs.append(run_level(r, False))
            finally:
                r.close()
        else:
            theirs.append(FINE_REF)
    for o, t in zip(ours, theirs):
        for key in ("t_hat", "peak", "ratio"):
            assert abs(o[key] - t[key]) <= 1e-7 * abs(t[key]), (key, o, t)
    coarse, mid, work, fine = ours
    rel = lambda a: abs(a - fine["t_hat"]) / abs(fine["t_hat"])  # noqa: E731
    assert rel(work["t_hat"]) <= 0.02 and rel(coarse["t_hat"]) <= 0.10      # criterion 5
    assert 0.01 <= work["ratio"] <= 0.10                                    # criterion 6
    assert coarse["ratio"] > mid["ratio"] > work["ratio"]
    # the values the reference's acceptance run prints (proj/test_output.txt:31-34)
    printed = [(100 * rel(work["t_hat"]), 0.140, 3), (100 * rel(coarse["t_hat"]), 5.177, 3),
               (fine["peak"], 10.428, 3), (100 * coarse["ratio"], 26.03, 2),
               (100 * mid["ratio"], 9.48, 2), (100 * work["ratio"], 4.04, 2)]
    for got, want, digits in printed:
        assert abs(got - want) <= 0.5 * 10.0 ** -digits + 1e-9, (got, want)


# --- acceptance criterion 7 (proj/tests/acceptance.cpp:299-325) ------------

def contour_cfg(tmp_path):
    """The reference's contour-scan case: a quarter arc of radius 1.1 mm about
    (2 mm, 0), one waypoint per degree, 100 um target elements on etamin."""
    phi = np.deg2rad(np.arange(91.0))
    wp = "\n".join(f"waypoint = {x:.16e} {y:.16e}"
                   for x, y in zip(2e-3 - 1.1e-3 * np.cos(phi), 1.1e-3 * np.sin(phi)))
    txt = open(os.path.join(ROOT, "configs", "qc_single_source_small.cfg")).read()
    head, rest = txt.split("[scan]")
    mesh = """[mesh]
target_face = etamin
target_min_size = 100e-6
eta_elements = 16
eta_grading = 1.2
eta_focus = 0
zeta_elements = 18
zeta_grading = 1.2
zeta_focus = 1
boundary_quad_multiplier = 3
elevate_radius = 5e-4

[stepping]
theta = 0.5
dt = 1e-5
t_end = 3.0e-3
"""
    faces = rest[rest.index("[faces]"):rest.index("[mesh]")]
    p = tmp_path / "contour.cfg"
    p.write_text(head + "[scan]\nstart_time = 0.0\n" + wp + "\n\n" + faces + mesh)
    return str(p)


def test_contour_scan_acceptance(tmp_path, ref):
    cfg = contour_cfg(tmp_path)
    sim = tg.Simulation(cfg)
    r = ref.sim(cfg)
    ours, theirs = {}, {}
    try:
        assert sim.info["n_full"] == 6137 and sim.info["n_steps"] == 300
        sim.reset()
        r.reset()
        for s in range(1, 301):
            st = r.step()
            if s in (200, 300):  # step_for_time(2e-3), (3e-3)
                sim.advance(s - (0 if s == 200 else 200))
                prof = sim.boundary_flux_profile("etamin", 400, theta_axis=(2e-3, 0.0))
                ours[s] = tg.integrated_abs_flux(prof)["ratio"]
                full = full_of(r.info, st["free"], st["g"])
                theirs[s] = r.flux_profile(full, 2, 400, s * 1e-5, theta_axis=(2e-3, 0.0))[1][2]
    finally:
        sim.close()
        r.close()
    for s in (200, 300):
        assert abs(ours[s] - theirs[s]) <= 1e-7 * theirs[s], (s, ours, theirs)
    assert ours[300] <= 0.15 and ours[200] > ours[300]
    # proj/test_output.txt:35 prints 11.04 % at 3 ms and 13.35 % at 2 ms
    assert abs(100 * ours[300] - 11.04) <= 0.005 + 1e-9
    assert abs(100 * ours[200] - 13.35) <= 0.005 + 1e-9
