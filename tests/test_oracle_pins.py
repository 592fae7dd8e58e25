"""Pin the plain-C oracle (oracle/oracle.c) and the committed golden vectors
against the UNMODIFIED reference library and the reference's own known
answers (proj/tests/*.cpp). CPU only."""
import os

import numpy as np
import pytest

from paper_2511_20432_b200 import workloads as W
from conftest import GOLDEN

KW = dict(**W.MATERIAL, **W.LASER)
# proj/tests/test_util.hpp:11-29 fixtures
TI64 = dict(conductivity=42.0, density=4420.0, heat_capacity=990.0)
BENCH_LASER = dict(power=82.5, speed=0.5, spot_radius=20e-6, absorptivity=0.77, dt=1e-5)


def test_gauss_rule_bit_exact(ref, coracle):
    for n in range(1, 13):
        a, b = ref.gauss_rule(n)
        c, d = coracle.gauss_rule(n)
        assert np.array_equal(a, c) and np.array_equal(b, d)


@pytest.mark.parametrize("case", ["cfg1", "dwell", "corner", "line", "late"])
def test_discretize_scan_bit_exact(ref, coracle, case):
    kw = dict(KW)
    if case == "cfg1":
        wp, extra = W.config1_waypoints(), dict(plane_z=1e-3)
    elif case == "dwell":  # test_analytic.cpp:25-38
        wp, extra = [[1e-3, 2e-3]], dict(plane_z=2e-3)
        kw.update(TI64, **BENCH_LASER)
    elif case == "corner":  # test_analytic.cpp:53-60
        wp, extra = [[0, 0], [1e-5, 0], [1e-5, 1e-5]], {}
        kw.update(TI64, **BENCH_LASER)
    elif case == "line":  # test_analytic.cpp:40-51: 201 sources, 5 um apart
        wp, extra = [[0, 0], [1e-3, 0]], {}
        kw.update(TI64, **BENCH_LASER)
    else:
        wp, extra = [[0, 0], [1e-4, 0]], dict(start_time=1e-4)
    a = ref.discretize_scan(wp, **extra, **kw)
    b = coracle.discretize_scan(wp, **extra, **kw)
    assert np.array_equal(a, b)
    if case == "line":
        assert len(a) == 201
        assert np.allclose(np.diff(a[:, 0]), 5e-6, rtol=1e-9)
    if case == "corner":
        assert len(a) == 5


def test_superpose_bit_exact_sample(ref, coracle):
    src = coracle.discretize_scan(W.config1_waypoints(), plane_z=1e-3, **KW)[:W.CONFIG1_SOURCES]
    t = float(src[-1, 4])
    pts = W.config1_points()[::4096]  # 256 points spread over the set
    v1, g1 = ref.superpose(src, pts, t, **KW)
    v2, g2 = coracle.superpose(src, pts, t, **KW)
    assert np.array_equal(v1, v2) and np.array_equal(g1, g2)


def test_k1_golden_matches_live_reference(ref):
    g = np.load(os.path.join(GOLDEN, "k1_cfg1.npz"))
    src = ref.discretize_scan(W.config1_waypoints(), plane_z=1e-3, **KW)[:int(g["n_sources"])]
    pts = W.config1_points()[:256]
    v, gr = ref.superpose(src, pts, float(g["t"]), threads=4, **KW)
    assert np.array_equal(v, g["val"][:256]) and np.array_equal(gr, g["grad"][:256])


def test_k1_golden_matches_c_oracle(coracle):
    g = np.load(os.path.join(GOLDEN, "k1_cfg1.npz"))
    src = coracle.discretize_scan(W.config1_waypoints(), plane_z=1e-3, **KW)[:int(g["n_sources"])]
    pts = W.config1_points()[:64]
    v, gr = coracle.superpose(src, pts, float(g["t"]), **KW)
    assert np.array_equal(v, g["val"][:64]) and np.array_equal(gr, g["grad"][:64])
    for i, tt in enumerate(g["times"]):
        v, gr = coracle.superpose(g["dwell"], g["probe"], float(tt), **KW)
        assert np.array_equal(v, g["dwell_val"][i]) and np.array_equal(gr, g["dwell_grad"][i])


def test_activation_peak_known_answer(coracle):
    # proj/tests/test_analytic.cpp:86-93: peak = E/(rho c (pi r^2/2)^1.5) ~ 9.2e3
    kw = dict(TI64, **BENCH_LASER)
    src = coracle.discretize_scan([[0.0, 0.0]], **kw)
    v, _ = coracle.superpose(src, src[:, :3], float(src[0, 4]), **kw)
    E = 0.77 * 82.5 * 1e-5
    expected = E / (4420.0 * 990.0 * (np.pi * 20e-6 ** 2 / 2.0) ** 1.5)
    assert v[0] == pytest.approx(expected, rel=1e-13)
    assert v[0] == pytest.approx(9.2e3, rel=0.01)
    # causality: exactly zero at and before tau (test_analytic.cpp:79-84)
    v0, g0 = coracle.superpose(src, np.zeros((1, 3)), float(src[0, 5]), **kw)
    assert v0[0] == 0.0 and not np.any(g0)


def test_pcg_known_answers(ref, coracle):
    # proj/tests/test_sparse.cpp:42-48: [[4,1],[1,3]] x = [1,2] -> [1/11, 7/11]
    rp, ci, v = [0, 2, 4], [0, 1, 0, 1], [4.0, 1.0, 1.0, 3.0]
    x, it, rel, rc = coracle.pcg(rp, ci, v, [1.0, 2.0], [0.0, 0.0])
    assert rc == 0 and x == pytest.approx([1 / 11, 7 / 11], rel=1e-10)
    xr, itr, relr = ref.pcg(rp, ci, v, [1.0, 2.0], [0.0, 0.0])
    assert np.array_equal(x, xr) and it == itr
    # iteration cap -> numeric error (test_sparse.cpp:81-85)
    assert coracle.pcg(rp, ci, v, [1.0, 2.0], [0.0, 0.0], tol=1e-14, max_iter=1)[3] == 3
    with pytest.raises(Exception, match="no convergence"):
        ref.pcg(rp, ci, v, [1.0, 2.0], [0.0, 0.0], tol=1e-14, max_iter=1)
    # zero rhs resets a warm start (test_sparse.cpp:101-108)
    x, it, rel, rc = coracle.pcg([0, 1, 2], [0, 1], [2.0, 2.0], [0.0, 0.0], [5.0, -1.0])
    assert rc == 0 and it == 0 and not np.any(x)


def test_pcg_random_spd_matches_reference(ref, coracle):
    rng = np.random.default_rng(33)
    n = 50
    g = rng.standard_normal((n, n))
    a = g.T @ g + n * np.eye(n)
    rp = np.arange(0, n * n + 1, n)
    ci = np.tile(np.arange(n), n)
    b = rng.standard_normal(n)
    x1, it1, r1, rc = coracle.pcg(rp, ci, a.ravel(), b, np.zeros(n), tol=1e-10, max_iter=500)
    x2, it2, r2 = ref.pcg(rp, ci, a.ravel(), b, np.zeros(n), tol=1e-10, max_iter=500)
    assert rc == 0 and it1 == it2 and np.array_equal(x1, x2)
    assert np.linalg.norm(b - a @ x1) / np.linalg.norm(b) <= 1e-9


def test_boundary_load_bit_exact(ref, coracle, configs):
    sim = ref.sim(configs["cfg0"])
    fs = sim.face_sets()
    src = sim.sources()
    for t in (0.0, 3e-5, 5e-4, 1e-3):
        F = sim.flux_load(t)
        Fo = coracle.boundary_load(fs, src, t, fine_radius=5e-4, n_full=sim.info["n_full"], **KW)
        assert np.array_equal(F, Fo)
    sim.close()
