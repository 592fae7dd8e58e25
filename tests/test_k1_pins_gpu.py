"""The reference's own K1 pins (proj/tests/test_analytic.cpp) re-run through
the GPU superposition (tg_superpose_batch): same fixtures (ti64, the
benchmark laser; proj/tests/test_util.hpp), same seeds where the reference
seeds a std::mt19937 (the draws differ, numpy vs libstdc++, so the random
points are different samples of the same distributions), same tolerances."""
import numpy as np
import pytest

import paper_2511_20432_b200 as tg

pytestmark = pytest.mark.gpu

MAT = tg.Material(42.0, 4420.0, 990.0, 0.0)
LASER = tg.LaserSpec(power=82.5, speed=0.5, spot_radius=20e-6, absorptivity=0.77, dt=1e-5)


def sources(wp, start_time=0.0):
    return tg.discretize_scan(tg.ScanPath(wp, start_time, 0.0), LASER, MAT)


@pytest.fixture
def dwell(gpu_ctx):
    """One source: superpose without culling is temp_point_source /
    grad_point_source (analytic.cpp:73-90), the functions these pins test."""
    src = sources([[0.0, 0.0]])
    assert len(src) == 1
    gpu_ctx.set_sources(src, MAT)
    return gpu_ctx, src[0]


NO_CULL = tg.SuperposeOptions(1e30)


def T(ctx, pts, t, opts=NO_CULL):
    v, g = ctx.superpose(np.asarray(pts, dtype=np.float64).reshape(-1, 3), t, opts)
    return v, g


def test_causality_exact_zero(dwell):
    ctx, s = dwell
    tau = s[5]
    v, _ = T(ctx, [[0, 0, 0]], tau)
    assert v[0] == 0.0
    v, _ = T(ctx, [[0, 0, 0]], tau - 1e-9)
    assert v[0] == 0.0
    _, g = T(ctx, [[1e-5, 0, 0]], tau)
    assert np.linalg.norm(g[0]) == 0.0


def test_activation_peak_closed_form(dwell):
    ctx, s = dwell
    v, _ = T(ctx, [s[:3]], s[4])
    r2 = LASER.spot_radius ** 2
    expected = s[3] / (MAT.volumetric_capacity() * (np.pi * r2 / 2.0) ** 1.5)
    assert v[0] == pytest.approx(expected, rel=1e-13)
    assert v[0] == pytest.approx(9.2e3, rel=0.01)


def test_radial_symmetry(dwell):
    ctx, s = dwell
    v, _ = T(ctx, [[3e-5, 4e-5, 0], [0, 0, -5e-5]], 5e-5)
    assert v[0] == pytest.approx(v[1], rel=1e-13)


def test_monotone_decay(dwell):
    ctx, s = dwell
    pts = [s[:3] + [i * 2e-5, 0, 0] for i in range(31)]
    v, _ = T(ctx, pts, 1e-4)
    assert np.all(np.diff(v) < 0)


def test_gradient_matches_finite_differences(dwell):
    ctx, s = dwell
    rng = np.random.default_rng(17)
    h = 1e-8
    for _ in range(50):
        x = rng.uniform(-2e-4, 2e-4, 3)
        t = rng.uniform(1e-5, 3e-4)
        _, g = T(ctx, [x], t)
        for d in range(3):
            xp, xm = x.copy(), x.copy()
            xp[d] += h
            xm[d] -= h
            v, _ = T(ctx, [xp, xm], t)
            fd = (v[0] - v[1]) / (2.0 * h)
            assert abs(fd - g[0, d]) <= 1e-6 * abs(g[0, d]) + 1e-4


def test_gradient_antiparallel(dwell):
    ctx, s = dwell
    x = np.array([1e-4, 5e-5, -2e-5])
    _, g = T(ctx, [x, s[:3]], 1e-4)
    r = x - s[:3]
    assert g[0] @ r < 0.0
    assert np.linalg.norm(np.cross(g[0], r)) <= 1e-12 * np.linalg.norm(g[0]) * np.linalg.norm(r)
    assert np.linalg.norm(g[1]) == 0.0


def test_no_sources_zero_field(gpu_ctx):
    gpu_ctx.set_sources(np.zeros((0, 6)), MAT)
    v, g = T(gpu_ctx, [[0, 0, 0]], 1.0)
    assert v[0] == 0.0 and np.linalg.norm(g[0]) == 0.0


def test_two_sources_sum_linearly(gpu_ctx):
    src = sources([[0.0, 0.0], [1e-5, 0.0]])
    assert len(src) == 3
    src = src[:2]
    x, t = [2e-5, 1e-5, 0], 6e-5
    gpu_ctx.set_sources(src, MAT)
    v, _ = T(gpu_ctx, [x], t, tg.SuperposeOptions())
    direct = 0.0
    for s in src:
        gpu_ctx.set_sources(s[None, :], MAT)
        direct += T(gpu_ctx, [x], t)[0][0]
    assert v[0] == pytest.approx(direct, rel=1e-13)


def test_zero_before_first_modified_time(gpu_ctx):
    src = sources([[0.0, 0.0], [1e-4, 0.0]], start_time=1e-4)
    gpu_ctx.set_sources(src, MAT)
    v, g = T(gpu_ctx, [[0, 0, 0]], 0.0, tg.SuperposeOptions())
    assert v[0] == 0.0 and np.linalg.norm(g[0]) == 0.0


def test_heat_equation_residual(dwell):
    """4th-order FD residual of dT/dt - alpha lap T <= 1e-5 of the rate
    (test_analytic.cpp:192-236), 200 trials, seed 101."""
    ctx, s = dwell
    alpha = MAT.diffusivity()
    rng = np.random.default_rng(101)
    rates, res = [], []
    for _ in range(200):
        age = 1e-6 * (3e-4 / 1e-6) ** rng.uniform()
        t = s[5] + age
        sigma = np.sqrt(4.0 * alpha * age)
        x = s[:3] + (2.0 * rng.uniform(size=3) - 1.0) * (1.5 * sigma)
        ht, hx = 0.004 * age, 0.02 * sigma
        vt = [T(ctx, [x], t + k * ht)[0][0] for k in (-2, -1, 1, 2)]
        dTdt = (vt[0] - 8 * vt[1] + 8 * vt[2] - vt[3]) / (12.0 * ht)
        lap = 0.0
        c = T(ctx, [x], t)[0][0]
        for d in range(3):
            e = np.zeros(3)
            e[d] = 1.0
            v, _ = T(ctx, [x - 2 * hx * e, x - hx * e, x + hx * e, x + 2 * hx * e], t)
            lap += (-v[0] + 16 * v[1] - 30 * c + 16 * v[2] - v[3]) / (12.0 * hx * hx)
        rates.append(abs(dTdt))
        res.append(abs(dTdt - alpha * lap))
    floor = 1e-6 * max(rates)
    for r, q in zip(rates, res):
        assert q <= 1e-5 * max(r, floor)


def test_deposited_energy_by_quadrature(dwell, coracle):
    """rho c * integral of T over a 10-sigma box == E to 1e-3
    (test_analytic.cpp:238-272): 16 panels x 6 Gauss points per axis."""
    ctx, s = dwell
    t = 1.9e-4
    sigma = np.sqrt(4.0 * MAT.diffusivity() * (t - s[5]))
    half = 10.0 * sigma
    gn, gw = coracle.gauss_rule(6)
    nodes, weights = [], []
    for p in range(16):
        a = -half + 2.0 * half * p / 16
        b = -half + 2.0 * half * (p + 1) / 16
        nodes += list(0.5 * (a + b) + 0.5 * (b - a) * gn)
        weights += list(0.5 * (b - a) * gw)
    nodes, weights = np.array(nodes), np.array(weights)
    X, Y, Z = np.meshgrid(nodes, nodes, nodes, indexing="ij")
    W = np.einsum("i,j,k->ijk", weights, weights, weights)
    pts = s[:3] + np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)
    v, _ = T(ctx, pts, t)
    integral = (W.ravel() * v).sum() * MAT.volumetric_capacity()
    assert integral == pytest.approx(s[3], rel=1e-3)
    assert s[3] == pytest.approx(6.35e-4, rel=1e-2)
