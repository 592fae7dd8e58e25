"""K1 parity on the GPU: superpose (proj/src/analytic.cpp:92-109) through the C
ABI against the golden vectors of the unmodified reference and the C oracle.

Tolerances (BASELINE.json north_star): values pointwise relative <= 1e-10
with exact zeros bitwise equal; gradients normwise
max|a-b| / max|b| <= 1e-10."""
import os

import numpy as np
import pytest

import paper_2511_20432_b200 as tg
from paper_2511_20432_b200 import workloads as W
from conftest import GOLDEN

pytestmark = pytest.mark.gpu
KW = dict(**W.MATERIAL, **W.LASER)
MAT = tg.Material(**W.MATERIAL)
TOL = 1e-10


def check_field(v, g, v_ref, g_ref, tol=TOL):
    zero = v_ref == 0.0
    assert np.array_equal(v[zero], v_ref[zero]), "exact zeros (causality/cull) must match"
    nz = ~zero
    if nz.any():
        rel = np.abs(v[nz] - v_ref[nz]) / np.abs(v_ref[nz])
        assert rel.max() <= tol, rel.max()
    if g_ref is not None and np.abs(g_ref).max() > 0:
        err = np.abs(g - g_ref).max() / np.abs(g_ref).max()
        assert err <= tol, err


@pytest.fixture(scope="module")
def cfg1_sources():
    path = tg.ScanPath(W.config1_waypoints(), 0.0, 1e-3)
    src = tg.discretize_scan(path, tg.LaserSpec(**W.LASER), MAT)[:W.CONFIG1_SOURCES]
    return src, float(src[-1, 4])


def test_golden_config1_sample(gpu_ctx, cfg1_sources):
    g = np.load(os.path.join(GOLDEN, "k1_cfg1.npz"))
    src, t = cfg1_sources
    assert t == float(g["t"])
    gpu_ctx.set_sources(src, MAT)
    pts = W.config1_points()[:int(g["sample"])]
    v, gr = gpu_ctx.superpose(pts, t)
    check_field(v, gr, g["val"], g["grad"])


def test_golden_dwell_causality_and_peak(gpu_ctx):
    g = np.load(os.path.join(GOLDEN, "k1_cfg1.npz"))
    gpu_ctx.set_sources(g["dwell"], MAT)
    for i, t in enumerate(g["times"]):
        v, gr = gpu_ctx.superpose(g["probe"], float(t))
        check_field(v, gr, g["dwell_val"][i], g["dwell_grad"][i])
        if t <= g["dwell"][0, 5]:
            assert not np.any(v) and not np.any(gr)


def test_full_size_against_oracle_subset(gpu_ctx, cfg1_sources, coracle):
    """The full 2^20 x 2^16 launch; a strided subset is checked against the C
    oracle and the run is repeated for bitwise determinism."""
    src, t = cfg1_sources
    gpu_ctx.set_sources(src, MAT)
    pts = W.config1_points()
    v, gr = gpu_ctx.superpose(pts, t)
    v2, gr2 = gpu_ctx.superpose(pts, t)
    assert np.array_equal(v, v2) and np.array_equal(gr, gr2)
    sub = np.arange(0, len(pts), len(pts) // 97)[:96]
    vo, go = coracle.superpose(src, pts[sub], t, **KW)
    check_field(v[sub], gr[sub], vo, go)
    assert np.all(v > 0) and np.isfinite(gr).all()


def test_cull_boundary_and_zero_pattern(gpu_ctx, coracle):
    """Points placed so that many pairs sit right at arg ~ cull: the set of
    culled pairs (and so exact zeros) must match the reference exactly."""
    mat = MAT
    src = coracle.discretize_scan([[1e-3, 1e-3], [2e-3, 1e-3]], plane_z=1e-3, **KW)
    t = float(src[-1, 4]) + 2e-5
    alpha = mat.diffusivity()
    rng = np.random.default_rng(7)
    pts = []
    for s in src[::7]:
        spread = 4.0 * alpha * (t - s[5])
        r = np.sqrt(60.0 * spread) * (1 + rng.uniform(-1e-9, 1e-9, 64))
        d = rng.standard_normal((64, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        pts.append(s[:3] + d * r[:, None])
    pts = np.concatenate(pts)
    gpu_ctx.set_sources(src, mat)
    for cull in (60.0, 10.0, 0.0):
        opts = tg.SuperposeOptions(cull)
        v, g = gpu_ctx.superpose(pts, t, opts)
        vo, go = coracle.superpose(src, pts, t, cull=cull, **KW)
        assert np.array_equal(v == 0.0, vo == 0.0)
        check_field(v, g, vo, go)


def test_single_pair_cull_decision_ulp_exact(gpu_ctx, coracle):
    """One source, points whose r.r lands within a few ulp of cull*spread: each
    point's value is non-zero iff its single pair is kept, so the zero pattern
    pins the per-pair decision fl(r.r / spread) > cull (analytic.cpp:103)
    against the reference arithmetic, including the kernel's high-word band."""
    src = coracle.discretize_scan([[1e-3, 1e-3], [1.1e-3, 1e-3]], plane_z=1e-3, **KW)[:1]
    t = float(src[0, 5]) + 3e-5
    alpha = MAT.diffusivity()
    spread = 4.0 * alpha * (t - float(src[0, 5]))
    rng = np.random.default_rng(3)
    gpu_ctx.set_sources(src, MAT)
    for cull in (60.0, 7.5, 1e-3):
        r = np.sqrt(cull * spread) * (1 + rng.integers(-40, 41, 4096) * 2.0**-53)
        d = rng.standard_normal((4096, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        pts = src[0, :3] + d * r[:, None]
        v, g = gpu_ctx.superpose(pts, t, tg.SuperposeOptions(cull))
        vo, go = coracle.superpose(src, pts, t, cull=cull, **KW)
        kept = vo != 0.0
        assert 0 < kept.sum() < len(kept), "sample must straddle the threshold"
        assert np.array_equal(v != 0.0, kept)
        check_field(v, g, vo, go)


def test_cull_invariance_and_no_cull(gpu_ctx, coracle):
    # proj/tests/test_analytic.cpp:178-189
    kw = dict(conductivity=42.0, density=4420.0, heat_capacity=990.0, power=82.5, speed=0.5,
              spot_radius=20e-6, absorptivity=0.77, dt=1e-5)
    mat = tg.Material(42.0, 4420.0, 990.0)
    src = coracle.discretize_scan([[0.0, 0.0], [5e-4, 0.0]], **kw)
    x = np.array([[1e-4, 1e-4, -1e-4]])
    gpu_ctx.set_sources(src, mat)
    a, _ = gpu_ctx.superpose(x, 7e-4)
    b, _ = gpu_ctx.superpose(x, 7e-4, tg.SuperposeOptions(1e30))
    assert a[0] == pytest.approx(b[0], rel=1e-13)
    vo, _ = coracle.superpose(src, x, 7e-4, cull=1e30, **kw)
    assert b[0] == pytest.approx(vo[0], rel=TOL)


def test_edge_cases(gpu_ctx, coracle):
    # no sources -> zero field (test_analytic.cpp:141-145)
    gpu_ctx.set_sources(np.zeros((0, 6)), MAT)
    v, g = gpu_ctx.superpose(np.ones((5, 3)), 1.0)
    assert not np.any(v) and not np.any(g)
    # zero points
    v, g = gpu_ctx.superpose(np.zeros((0, 3)), 1.0)
    assert v.shape == (0,)
    # zero power -> exactly zero (test_pipeline.cpp:66-78)
    zero = dict(KW, power=0.0)
    src = coracle.discretize_scan([[0, 0], [1e-4, 0]], plane_z=0.0, **zero)
    gpu_ctx.set_sources(src, MAT)
    v, g = gpu_ctx.superpose(np.random.default_rng(1).uniform(-1e-4, 1e-4, (100, 3)), 1e-3)
    assert not np.any(v) and not np.any(g)
    # ragged sizes around the tile width
    src = coracle.discretize_scan(W.config1_waypoints()[:3], plane_z=1e-3, **KW)
    gpu_ctx.set_sources(src, MAT)
    for n in (1, 255, 257, 511, 513, 1000):
        pts = W.config1_points(n, seed=n)
        v, g = gpu_ctx.superpose(pts, float(src[-1, 4]))
        vo, go = coracle.superpose(src, pts, float(src[-1, 4]), **KW)
        check_field(v, g, vo, go)


def test_device_path_matches_host_path(gpu_ctx, cfg1_sources):
    import torch
    src, t = cfg1_sources
    gpu_ctx.set_sources(src, MAT)
    pts = W.config1_points(8192, seed=3)
    v, g = gpu_ctx.superpose(pts, t)
    dp = torch.from_numpy(pts).cuda()
    dv, dg = gpu_ctx.superpose(dp, t)
    torch.cuda.synchronize()
    assert np.array_equal(dv.cpu().numpy(), v) and np.array_equal(dg.cpu().numpy(), g)


def test_value_only_launch_matches_value_of_gradient_launch(gpu_ctx, cfg1_sources):
    """Without a gradient output the value-only kernel runs (13 instead of 17
    FP64 ops per pair); the values are the same bits."""
    src, t = cfg1_sources
    gpu_ctx.set_sources(src, MAT)
    pts = W.config1_points()[:50000]
    v, g = gpu_ctx.superpose(pts, t)
    v0, g0 = gpu_ctx.superpose(pts, t, grad=False)
    assert g0 is None and np.array_equal(v0, v)


def test_more_than_2e28_points_in_one_call(gpu_ctx, coracle):
    """Calls beyond one launch's 2^28 points are chunked inside the library;
    points on both sides of the chunk seam match the oracle."""
    import torch
    src = coracle.discretize_scan([[1e-3, 1e-3], [1.02e-3, 1e-3]], plane_z=1e-3, **KW)
    t = float(src[-1, 4])
    gpu_ctx.set_sources(src, MAT)
    n = (1 << 28) + 4096
    g = torch.Generator(device="cuda").manual_seed(5)
    pts = (torch.rand((n, 3), dtype=torch.float64, device="cuda", generator=g) * 4e-4 + 8e-4)
    v, gr = gpu_ctx.superpose(pts, t)
    torch.cuda.synchronize()
    for lo in (0, (1 << 28) - 2048, n - 2048):
        p = pts[lo:lo + 2048].cpu().numpy()
        vo, go = coracle.superpose(src, p, t, **KW)
        check_field(v[lo:lo + 2048].cpu().numpy(), gr[lo:lo + 2048].cpu().numpy(), vo, go)
    del pts, v, gr
    torch.cuda.empty_cache()
