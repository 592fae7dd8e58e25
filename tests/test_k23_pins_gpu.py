"""The reference's own flux-load and time-step pins re-run through the GPU
path (tg_sim_*), on the reference's test fixture (configs/qc_pins.cfg: the
quarter-cylinder part refined 8 x 4 x 4, Ti64, benchmark laser dwelling at the
single-pulse position — proj/tests/test_util.hpp, test_assembly.cpp,
test_timestep.cpp), with the reference's tolerances. Matrices for the
energy / stability checks come from the reference library (CSR M, K)."""
import os

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2511_20432_b200 as tg
from conftest import ROOT

pytestmark = pytest.mark.gpu
CFG = os.path.join(ROOT, "configs", "qc_pins.cfg")
FACES = (0, 1, 2, 3)  # ximin, ximax, etamin, etamax


def variant(tmp_path, name, **repl):
    txt = open(CFG).read()
    for old, new in repl.items():
        assert old in txt
        txt = txt.replace(old, new)
    p = tmp_path / name
    p.write_text(txt)
    return str(p)


@pytest.fixture(scope="module")
def sim():
    s = tg.Simulation(CFG)
    yield s
    s.close()


@pytest.fixture(scope="module")
def refsim(ref):
    r = ref.sim(CFG)
    yield r
    r.close()


def csr(refsim, which):
    rp, ci, v = refsim.csr(which)
    n = len(rp) - 1
    return sp.csr_matrix((v, ci, rp), shape=(n, n))


def expand(sim, free, g):
    i = sim.info
    full = np.zeros((i["nz"], i["ny"], i["nx"]))
    full[1:] = free.reshape(i["nz"] - 1, i["ny"], i["nx"])
    full[0] = g.reshape(i["ny"], i["nx"])
    return full.ravel()


# --- flux load (test_assembly.cpp:133-233) --------------------------------

def test_causal_zero_before_modified_time(tmp_path):
    s = tg.Simulation(variant(tmp_path, "late.cfg", **{"start_time = 0.0": "start_time = 1e-4"}))
    assert not np.any(s.flux_load(0.0))
    s.close()


def test_interior_source_pushes_heat_back(sim):
    F = sim.flux_load(1.9e-4)
    m = F.max()
    assert m > 0.0 and np.all(F >= -1e-12 * m)


def test_load_sum_matches_independent_quadrature(sim, refsim, coracle):
    t = 1.9e-4
    total = sim.flux_load(t).sum()
    gn, gw = coracle.gauss_rule(10)
    nu, nv = 60, 20
    U = ((np.arange(nu)[:, None] + 0.5 + 0.5 * gn[None, :]) / nu).ravel()
    V = ((np.arange(nv)[:, None] + 0.5 + 0.5 * gn[None, :]) / nv).ravel()
    WU = np.tile(gw, nu)
    WV = np.tile(gw, nv)
    uu, vv = np.meshgrid(U, V, indexing="ij")
    ww = np.outer(WU, WV).ravel()
    uv = np.stack([uu.ravel(), vv.ravel()], axis=1)
    src = sim.sources()
    kw = dict(conductivity=42.0, density=4420.0, heat_capacity=990.0)
    oracle = 0.0
    for f in FACES:
        fp = refsim.face_points(f, uv)
        _, g = coracle.superpose(src, fp[:, :3], t, **kw)
        qn = 42.0 * np.einsum("ij,ij->i", g, fp[:, 3:6])
        oracle += np.sum(-qn * fp[:, 6] * ww) / (4.0 * nu * nv)
    assert total == pytest.approx(oracle, rel=1e-3)
    assert abs(total) > 0.0


def test_elevated_rule_engages_and_converges(sim, tmp_path):
    t = 1.9e-4
    never = sim.flux_load(t, 0.0).sum()  # base rule only
    x3 = sim.flux_load(t).sum()
    s6 = tg.Simulation(variant(tmp_path, "x6.cfg",
                               **{"boundary_quad_multiplier = 3": "boundary_quad_multiplier = 6"}))
    x6 = s6.flux_load(t).sum()
    s6.close()
    assert abs(never - x3) > 0.01 * abs(x3)
    assert x3 == pytest.approx(x6, rel=5e-3)


def test_load_continuous_in_time(sim):
    F0, F1 = sim.flux_load(1.5e-4), sim.flux_load(1.5e-4 + 1e-9)
    assert np.abs(F1 - F0).max() <= 1e-4 * np.abs(F0).max()


def test_repeated_assembly_is_bitwise_identical(sim):
    a, b = sim.flux_load(1.9e-4), sim.flux_load(1.9e-4)
    assert np.array_equal(a, b)


# --- time stepping (test_timestep.cpp) -------------------------------------

@pytest.mark.parametrize("cfgname", ["qc_pins", "cfg0_parity"])
def test_constant_state_preserved(cfgname):
    s = tg.Simulation(os.path.join(ROOT, "configs", cfgname + ".cfg"))
    c = 7.25
    nf, nc, n = s.info["n_free"], s.info["n_constrained"], s.info["n_full"]
    x, g, zero = np.full(nf, c), np.full(nc, c), np.zeros(n)
    for _ in range(5):
        x, _, _ = s.theta_step(x, g, zero, zero, g)
    assert np.all(np.abs(x - c) <= 1e-10 * c)
    s.close()


def test_crank_nicolson_stable_for_huge_steps(tmp_path, ref):
    path = variant(tmp_path, "bigdt.cfg", **{"dt = 1e-5\nt_end": "dt = 1e3\nt_end"})
    s = tg.Simulation(path)
    r = ref.sim(path)
    M = csr(r, 0)
    nf, nc, n = s.info["n_free"], s.info["n_constrained"], s.info["n_full"]
    x = np.random.default_rng(77).uniform(-1.0, 1.0, nf)
    g, zero = np.zeros(nc), np.zeros(n)

    def m_norm(free):
        f = expand(s, free, g)
        return np.sqrt(f @ (M @ f))

    prev = m_norm(x)
    for _ in range(8):
        x, _, _ = s.theta_step(x, g, zero, zero, g, tol=1e-12, max_iter=5000)
        now = m_norm(x)
        assert now <= prev * (1.0 + 1e-10)
        prev = now
    s.close()
    r.close()


def test_discrete_energy_balance(sim, refsim):
    """Free-row residual of the full semi-discrete theta step below 0.5 % of
    the input, every step of the 19-step pulse (test_timestep.cpp:146-199)."""
    M, K = csr(refsim, 0), csr(refsim, 1)
    theta, dt = 0.5, 1e-5
    sim.reset()
    st = sim.state()
    prev, Fn = expand(sim, st["free"], st["g"]), st["F"]
    free_rows = np.ones(sim.info["n_full"], dtype=bool)
    free_rows[: sim.info["nx"] * sim.info["ny"]] = False
    for _ in range(19):
        sim.advance(1)
        st = sim.state()
        now, Fnp1 = expand(sim, st["free"], st["g"]), st["F"]
        f_theta = theta * Fnp1 + (1.0 - theta) * Fn
        res = M @ ((now - prev) / dt) + K @ (theta * now + (1.0 - theta) * prev) - f_theta
        inp = f_theta.sum()
        assert inp > 0.0
        assert abs(res[free_rows].sum()) < 0.005 * inp
        prev, Fn = now, Fnp1
