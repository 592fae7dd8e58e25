"""K1 + K3 + K2 parity on the GPU through the C ABI (tg_sim_*), against the
unmodified reference (live when oracle/_ref is present, else the committed
golden vectors of tests/golden/make_golden.py).

Tolerances (BASELINE.json north_star):
  * loads F and Dirichlet values g: normwise max|a-b|/max|b| <= 1e-10, and
    reference zeros reproduced exactly;
  * correction-field coefficients: normwise <= 1e-8 at every compared step,
    both sides run with solver_tol = 1e-12 (configs/*_parity.cfg, qc_small.cfg).
"""
import os

import numpy as np
import pytest

import paper_2511_20432_b200 as tg
from conftest import GOLDEN, ROOT

pytestmark = pytest.mark.gpu
NAMES = ["cfg0_parity", "qc_small", "cfg0_oddx", "cfg3_parity"]


def cfg(name):
    return os.path.join(ROOT, "configs", name + ".cfg")


def golden(name):
    return np.load(os.path.join(GOLDEN, f"sim_{name}.npz"))


def normwise(a, b):
    m = np.abs(b).max()
    return 0.0 if m == 0 else np.abs(a - b).max() / m


@pytest.fixture(scope="module", params=[(n, a) for n in NAMES for a in ("cg1", "pcg")],
                ids=lambda p: f"{p[0]}-{p[1]}")
def sim(request):
    """Each config with both Kronecker solvers: the single-sweep
    Chronopoulos-Gear kernel (default with TMA) and the two-phase PCG kernel
    (TG_K2_ALGO=pcg; the only one without TMA, e.g. cfg0_oddx's odd pitch)."""
    name, algo = request.param
    os.environ["TG_K2_ALGO"] = algo
    try:
        s = tg.Simulation(cfg(name))
    finally:
        os.environ.pop("TG_K2_ALGO")
    if algo == "cg1" and name != "cfg0_oddx" and s.info["kronecker"]:
        assert s.info["kronecker"] == 2
    yield name, s
    s.close()


def test_operator_matches_assembled_reference(sim):
    name, s = sim
    g = golden(name)
    y = s.operator_apply(g["Ax_probe"])
    assert normwise(y, g["Ax"]) <= 1e-13


def test_flux_load_and_dirichlet(sim):
    name, s = sim
    g = golden(name)
    F = s.flux_load(float(g["t_mid"]))
    assert normwise(F, g["F_mid"]) <= 1e-10
    assert np.array_equal(F == 0.0, g["F_mid"] == 0.0)
    d = s.dirichlet_values(float(g["t_mid"]))
    assert normwise(d, g["g_mid"]) <= 1e-10
    F0 = s.flux_load(0.0)  # the first source is already active at t = 0 (tau < 0)
    assert normwise(F0, g["F0"]) <= 1e-10
    assert np.array_equal(F0 == 0.0, g["F0"] == 0.0)
    Fe = s.flux_load(-1.0)  # before every modified time: causal exact zero
    assert not np.any(Fe)


def test_flux_load_live_reference_times(sim, ref):
    """Several instants incl. ones where the fine rule engages (t = 1e-4, 2e-4)."""
    name, s = sim
    r = ref.sim(cfg(name))
    for t in (1e-5, 5e-5, 1e-4, 2e-4, 2.4e-4):
        F = s.flux_load(t)
        Fr = r.flux_load(t)
        assert normwise(F, Fr) <= 1e-10, t
        assert np.array_equal(F == 0.0, Fr == 0.0), t
        d, dr = s.dirichlet_values(t), r.dirichlet(t)
        assert normwise(d, dr) <= 1e-10, t
    # fine rule disabled / always on
    for rad in (0.0, 1.0):
        assert normwise(s.flux_load(1e-4, rad), r.flux_load_radius(1e-4, rad)) <= 1e-10
    r.close()


def test_theta_step_from_reference_inputs(sim):
    name, s = sim
    g = golden(name)
    steps = list(g["steps"])
    for a, b in zip(steps[:-1], steps[1:]):
        if b != a + 1:
            continue
        x, it, rel = s.theta_step(g[f"x{a}"], g[f"g{a}"], g[f"F{a}"], g[f"F{b}"], g[f"g{b}"],
                                  tol=1e-12)
        assert rel <= 1e-12
        assert normwise(x, g[f"x{b}"]) <= 1e-8, (a, b)
        assert abs(it - g["iters"][b - 1]) <= max(3, 0.1 * g["iters"][b - 1])


def test_full_time_loop(sim):
    """run_time_loop on the device: every compared step within tolerance."""
    name, s = sim
    g = golden(name)
    s.reset()
    st = s.state()
    assert st["step"] == 0 and not np.any(st["free"])
    assert normwise(st["F"], g["F0"]) <= 1e-10 and normwise(st["g"], g["g0"]) <= 1e-10
    done = 0
    total_it = 0
    worst = 0.0
    for k in g["steps"]:
        it, rel = s.advance(int(k) - done)
        total_it += it
        done = int(k)
        st = s.state()
        assert st["step"] == k
        assert normwise(st["F"], g[f"F{k}"]) <= 1e-10, k
        assert normwise(st["g"], g[f"g{k}"]) <= 1e-10, k
        err = normwise(st["free"], g[f"x{k}"])
        worst = max(worst, err)
        assert err <= 1e-8, (k, err)
    ref_it = int(g["iters"][:done].sum())
    assert abs(total_it - ref_it) <= 0.05 * ref_it, (total_it, ref_it)


def test_deterministic_reruns(sim):
    name, s = sim
    s.reset()
    s.advance(5)
    a = s.state()
    s.reset()
    s.advance(5)
    b = s.state()
    for k in ("free", "g", "F"):
        assert np.array_equal(a[k], b[k])


def test_step_profile_counters(sim):
    """Profiling brackets the solve (kind 2) inside the whole theta step (kind 3)."""
    name, s = sim
    ctx = s.context()
    s.reset()
    ctx.set_profiling(True)
    ctx.profile(reset=True)
    s.advance(3)
    p = ctx.profile()
    ctx.set_profiling(False)
    assert p["k2_launches"] == 3
    assert 0.0 < p["k2_ms"] <= p["theta_step_ms"]
    assert p["k1_ms"] > 0.0


def test_pcg_error_paths(sim):
    name, s = sim
    g = golden(name)
    # iteration cap -> numeric error with the reference's message (sparse.cpp:98-99)
    with pytest.raises(tg.NumericError, match=r"pcg: no convergence in 1 iterations, "
                                              r"relative residual"):
        s.theta_step(g["x1"], g["g1"], g["F1"], g["F2"], g["g2"], tol=1e-14, max_iter=1)
    # zero right-hand side resets a warm start (sparse.cpp:57-60)
    nf, nc, n = s.info["n_free"], s.info["n_constrained"], s.info["n_full"]
    x, it, rel = s.theta_step(np.ones(nf) * 0.0, np.zeros(nc), np.zeros(n), np.zeros(n),
                              np.zeros(nc))
    assert it == 0 and not np.any(x)


def test_zero_power_gives_platform_temperature(tmp_path):
    # proj/tests/test_pipeline.cpp:66-78: P = 0 -> exactly T_c everywhere
    txt = open(cfg("cfg0_parity")).read().replace("power = 150.0", "power = 0.0")
    p = tmp_path / "zero.cfg"
    p.write_text(txt)
    s = tg.Simulation(str(p), t_end=1e-4)
    s.reset()
    s.advance(s.info["n_steps"])
    st = s.state()
    assert not np.any(st["free"]) and not np.any(st["g"]) and not np.any(st["F"])
    s.close()



@pytest.mark.parametrize("name", ["cfg0_parity", "cfg0_oddx"])
def test_fdm_preconditioner_time_loop(name):
    """The fast-diagonalization preconditioner (opt-in): the
    same run_time_loop within the correction-field tolerance of the
    reference's Jacobi-PCG solution, in 1-2 CG iterations per step, with
    bitwise-deterministic reruns."""
    g = golden(name)
    s = tg.Simulation(cfg(name), preconditioner="fdm")
    assert s.info["kronecker"] == 3
    s.reset()
    done = 0
    for k in g["steps"]:
        it, rel = s.advance(int(k) - done)
        assert it <= 2 * (int(k) - done), (k, it)
        done = int(k)
        st = s.state()
        assert normwise(st["free"], g[f"x{k}"]) <= 1e-8, k
    a = s.state()["free"]
    s.reset()
    s.advance(done)
    assert np.array_equal(s.state()["free"], a)
    with pytest.raises(tg.NumericError, match=r"pcg: no convergence in 1 iterations"):
        s.theta_step(g["x1"], g["g1"], g["F1"], g["F2"], g["g2"], tol=1e-30, max_iter=1)
    s.close()


@pytest.mark.parametrize("name", ["cfg3_parity", "qc_small"])
def test_general_patch_preconditioner_time_loop(name):
    """Non-separable patches (config 3's degree-3 rational part, the reference's
    quarter cylinder) with the scaled separable-approximation preconditioner
    (preconditioner="fdm" on an assembled operator): the run_time_loop within
    the correction-field tolerance of the reference's Jacobi-PCG solution, in
    far fewer CG iterations than Jacobi."""
    g = golden(name)
    s = tg.Simulation(cfg(name), preconditioner="fdm")
    j = tg.Simulation(cfg(name))
    assert s.info["kronecker"] == 0
    s.reset()
    j.reset()
    done = 0
    its = itj = 0
    for k in g["steps"]:
        it, _ = s.advance(int(k) - done)
        it2, _ = j.advance(int(k) - done)
        its += it
        itj += it2
        done = int(k)
        assert normwise(s.state()["free"], g[f"x{k}"]) <= 1e-8, k
    assert its * 2 < itj, (its, itj)
    s.close()
    j.close()



BOTTOMS = {
    "zetamax": dict(zetamin="lateral", zetamax="bottom"),
    "etamin": dict(etamin="bottom", zetamin="lateral"),
    "ximax": dict(ximax="bottom", zetamin="lateral"),
}


@pytest.mark.parametrize("bottom", list(BOTTOMS))
@pytest.mark.parametrize("precond", ["jacobi", "fdm"])
def test_other_bottom_faces_against_live_reference(bottom, precond, ref, tmp_path):
    """The Dirichlet layer on another face (other axis, or the last layer):
    the Kronecker operator on the reduced grid, the expand / RHS kernels and
    both preconditioners, stepped against the unmodified reference."""
    txt = open(cfg("cfg0_parity")).read()
    head, faces = txt.split("[faces]", 1)
    block, rest = faces.split("\n\n", 1)
    roles = dict(line.split(" = ") for line in block.strip().splitlines())
    roles.update(BOTTOMS[bottom])
    faces_txt = "\n".join(f"{k} = {v}" for k, v in roles.items())
    p = tmp_path / f"b_{bottom}.cfg"
    p.write_text(head + "[faces]\n" + faces_txt + "\n\n" + rest)
    s = tg.Simulation(str(p), t_end=2e-4, preconditioner=precond)
    r = ref.sim(str(p), t_end=2e-4)
    # the single-sweep kernel needs TMA (free-grid row pitch a multiple of
    # 16 bytes); otherwise the two-phase kernel with plain loads runs
    assert s.info["kronecker"] in ((3,) if precond == "fdm" else (1, 2))
    s.reset()
    F0, g0 = r.reset()
    st = s.state()
    assert normwise(st["F"], F0) <= 1e-10 and normwise(st["g"], g0) <= 1e-10
    for k in range(1, 21):
        s.advance(1)
        st = s.state()
        o = r.step()
        assert normwise(st["F"], o["F"]) <= 1e-10, (bottom, k)
        assert normwise(st["g"], o["g"]) <= 1e-10, (bottom, k)
        assert normwise(st["free"], o["free"]) <= 1e-8, (bottom, k)
    s.close()
    r.close()


def box_geometry(degrees, size=(2e-3, 1e-3, 0.5e-3)):
    """[geometry] block of an axis-aligned box as a single Bezier patch of the
    given degrees (control points equally spaced: the exact linear map)."""
    lines = ["[geometry]", "degrees = " + " ".join(map(str, degrees))]
    for name, p in zip(("xi", "eta", "zeta"), degrees):
        lines.append(f"knots_{name} = " + " ".join(["0"] * (p + 1) + ["1"] * (p + 1)))
    lines.append("grid_dims = " + " ".join(str(p + 1) for p in degrees))
    px, py, pz = degrees
    for k in range(pz + 1):
        for j in range(py + 1):
            for i in range(px + 1):
                x, y, z = (size[0] * i / px, size[1] * j / py, size[2] * k / pz)
                lines.append(f"cp = {x!r} {y!r} {z!r} 1")
    return "\n".join(lines) + "\n"


@pytest.mark.parametrize("degrees", [(1, 1, 1), (3, 3, 3), (2, 2, 1)],
                         ids=["p1", "p3", "mixed221"])
def test_other_degrees_against_live_reference(degrees, ref, tmp_path):
    """Degree 1 and 3 Kronecker paths, and a mixed-degree cuboid (separable
    but unequal degrees: the assembled-operator path), stepped against the
    unmodified reference."""
    txt = open(cfg("cfg0_parity")).read()
    head, rest = txt.split("[geometry]", 1)
    rest = rest[rest.index("\n\n"):]
    p = tmp_path / "deg.cfg"
    p.write_text(head + box_geometry(degrees) + rest)
    s = tg.Simulation(str(p), t_end=1.5e-4)
    r = ref.sim(str(p), t_end=1.5e-4)
    kron = len(set(degrees)) == 1
    assert (s.info["kronecker"] > 0) == kron
    s.reset()
    F0, g0 = r.reset()
    assert normwise(s.state()["F"], F0) <= 1e-10
    for k in range(1, 16):
        s.advance(1)
        st = s.state()
        o = r.step()
        assert normwise(st["F"], o["F"]) <= 1e-10, (degrees, k)
        assert normwise(st["g"], o["g"]) <= 1e-10, (degrees, k)
        assert normwise(st["free"], o["free"]) <= 1e-8, (degrees, k)
    s.close()
    r.close()


def test_graded_cuboid_against_live_reference(ref, tmp_path):
    """Graded knot vectors in two directions keep the patch separable: the
    Kronecker factors of non-uniform 1D meshes, against the live reference."""
    txt = open(cfg("cfg0_parity")).read()
    txt = txt.replace("zeta_elements = 4", "zeta_elements = 6\nzeta_grading = 1.35\nzeta_focus = 1")
    txt = txt.replace("eta_elements = 8", "eta_elements = 8\neta_grading = 1.2")
    assert "zeta_grading" in txt and "eta_grading" in txt
    p = tmp_path / "graded.cfg"
    p.write_text(txt)
    s = tg.Simulation(str(p), t_end=1.5e-4)
    r = ref.sim(str(p), t_end=1.5e-4)
    assert s.info["kronecker"] == 2
    s.reset()
    r.reset()
    for k in range(1, 16):
        s.advance(1)
        st = s.state()
        o = r.step()
        assert normwise(st["F"], o["F"]) <= 1e-10, k
        assert normwise(st["free"], o["free"]) <= 1e-8, k
    s.close()
    r.close()


@pytest.mark.parametrize("edit", [
    ("theta = 0.5", "theta = 1.0"),
    ("theta = 0.5", "theta = 0.0"),
    ("dt = 1e-5\nt_end", "dt = 1e-5\nsubsteps = 2\nt_end"),
    ("zeta_elements = 4", "zeta_elements = 4\nquad_order = 4"),
], ids=["theta1", "theta0", "substeps2", "quad4"])
def test_stepping_and_quadrature_variants_against_live_reference(edit, ref, tmp_path):
    """Backward Euler, the explicit theta = 0 scheme, solver substeps and an
    explicit quadrature order change the operator and the step sequence: each
    against the unmodified reference."""
    txt = open(cfg("cfg0_parity")).read()
    assert edit[0] in txt
    p = tmp_path / "variant.cfg"
    p.write_text(txt.replace(edit[0], edit[1], 1))
    s = tg.Simulation(str(p), t_end=1.2e-4)
    r = ref.sim(str(p), t_end=1.2e-4)
    assert s.info["n_steps"] == r.info["n_steps"]
    s.reset()
    r.reset()
    for k in range(1, s.info["n_steps"] + 1):
        s.advance(1)
        st = s.state()
        o = r.step()
        assert normwise(st["F"], o["F"]) <= 1e-10, k
        assert normwise(st["free"], o["free"]) <= 1e-8, k
    s.close()
    r.close()
