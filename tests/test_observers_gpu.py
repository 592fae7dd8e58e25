"""Observers on the GPU (SURVEY.md §8f "next"): NURBS map_point / field_at
(K4, proj/src/splines.cpp:257-303), total_temperature (postproc.cpp:9-19),
boundary_flux_profile + integrated_abs_flux (:21-95) and export_field
(:101-147) of the device state, against the unmodified reference evaluated on
the same coefficient vector.

Tolerances: geometry x and the field_at value/gradient bit-identical (the K4
kernel rounds every operation in the reference's order); T_tilde-derived
quantities 1e-10 (BASELINE.json north_star)."""
import os

import numpy as np
import pytest

import paper_2511_20432_b200 as tg
from conftest import ROOT

pytestmark = pytest.mark.gpu
KW_CFG = {"cfg0_parity": dict(faces=[0, 1, 2, 3], axis=None),
          "qc_small": dict(faces=[0, 2, 3], axis=(2e-3, 0.0))}


def cfg(name):
    return os.path.join(ROOT, "configs", name + ".cfg")


def full_coeffs(sim):
    """DirichletSystem::expand of the device state (bottom layer zetamin)."""
    st = sim.state()
    i = sim.info
    full = np.zeros((i["nz"], i["ny"], i["nx"]))
    full[1:] = st["free"].reshape(i["nz"] - 1, i["ny"], i["nx"])
    full[0] = st["g"].reshape(i["ny"], i["nx"])
    return full.ravel(), st["time"]


def sample_xi(n, seed):
    rng = np.random.default_rng(seed)
    xi = rng.uniform(0.0, 1.0, (n, 3))
    xi[:8] = [[0, 0, 0], [1, 1, 1], [0, 1, 0.5], [1, 0, 0.25], [0.5, 0.5, 0.5], [0.25, 0.75, 1],
              [1, 0.5, 0], [0.0625, 0.125, 0.75]]  # corners, faces, knot values
    return xi


@pytest.fixture(scope="module", params=list(KW_CFG))
def pair(request, ref):
    s = tg.Simulation(cfg(request.param))
    r = ref.sim(cfg(request.param))
    yield request.param, s, r
    s.close()
    r.close()


def test_field_eval_bitwise(pair):
    name, s, r = pair
    xi = sample_xi(200, 5)
    coeffs = np.random.default_rng(9).standard_normal(s.info["n_full"])
    x, f = s.field_eval(coeffs, xi)
    for k in range(len(xi)):
        assert np.array_equal(x[k], r.map_point(xi[k])), (name, xi[k])
        v, g = r.field_at(coeffs, xi[k])
        assert f[k, 0] == v and np.array_equal(f[k, 1:], g), (name, xi[k])
    xg, fg = s.field_eval(None, xi)
    assert fg is None and np.array_equal(xg, x)


def test_probe_total_temperature(pair, coracle):
    name, s, r = pair
    s.reset()
    s.advance(7)
    full, t = full_coeffs(s)
    xi = sample_xi(64, 6)
    pr = s.probe(xi)
    src = s.sources()
    kw = dict(conductivity=s.params["conductivity"], density=s.params["density"],
              heat_capacity=s.params["heat_capacity"])
    for k in range(len(xi)):
        assert np.array_equal(pr[k, :3], r.map_point(xi[k]))
        v, g = r.field_at(full, xi[k])
        assert pr[k, 5] == v and np.array_equal(pr[k, 9:], g)
        Tref = r.total_temperature(full, xi[k], t)
        assert abs(pr[k, 3] - Tref) <= 1e-10 * abs(Tref), (name, k)
    vo, go = coracle.superpose(src, pr[:, :3], t, cull=s.params["cull"], **kw)
    nz = vo != 0
    assert np.array_equal(pr[:, 4] == 0, vo == 0)
    assert np.all(np.abs(pr[nz, 4] - vo[nz]) <= 1e-10 * np.abs(vo[nz]))
    assert np.abs(pr[:, 6:9] - go).max() <= 1e-10 * max(np.abs(go).max(), 1e-300)
    assert np.array_equal(s.total_temperature(xi), pr[:, 3])


def test_flux_profile_and_metrics(pair):
    name, s, r = pair
    s.reset()
    s.advance(12)
    full, t = full_coeffs(s)
    ax = KW_CFG[name]["axis"]
    for face in KW_CFG[name]["faces"]:
        for edge_v in (1.0, 0.5):
            ours = s.boundary_flux_profile(face, 41, theta_axis=ax, edge_v=edge_v)
            theirs, met = r.flux_profile(full, face, 41, t, theta_axis=ax, edge_v=edge_v)
            assert np.array_equal(ours[:, 0], theirs[:, 0])  # arc length: host, bit-exact
            if ax is None:
                assert np.all(np.isnan(ours[:, 1])) and np.all(np.isnan(theirs[:, 1]))
            else:
                assert np.array_equal(ours[:, 1], theirs[:, 1])
            assert np.array_equal(ours[:, 3], theirs[:, 3])  # q_hat: field_at, bit-exact
            for c in (2, 4):
                m = np.abs(theirs[:, c]).max()
                assert np.abs(ours[:, c] - theirs[:, c]).max() <= 1e-10 * m, (name, face, c)
            mo = tg.integrated_abs_flux(ours)
            assert abs(mo["integral_net"] - met[0]) <= 1e-10 * abs(met[0])
            assert abs(mo["integral_analytic"] - met[1]) <= 1e-10 * abs(met[1])


def test_export_field_matches_reference_writer(pair, tmp_path):
    name, s, r = pair
    s.reset()
    s.advance(3)
    full, t = full_coeffs(s)
    ours, theirs = tmp_path / "ours.vtk", tmp_path / "theirs.vtk"
    s.export_field(str(ours), (5, 4, 3))
    r.export_field(full, (5, 4, 3), t, str(theirs))
    a, b = open(ours).read().splitlines(), open(theirs).read().splitlines()
    assert len(a) == len(b)
    n = 5 * 4 * 3
    # header, points, T_hat block are bit-identical text; T_total / T_tilde within 1e-10
    assert a[:6 + n] == b[:6 + n]
    blocks = {}
    for lines, key in ((a, "a"), (b, "b")):
        i = 6 + n + 1
        for nm in ("T_total", "T_tilde", "T_hat"):
            assert lines[i] == f"SCALARS {nm} double 1"
            blocks[(key, nm)] = np.array([float(v) for v in lines[i + 2:i + 2 + n]])
            i += 2 + n
    assert np.array_equal(blocks[("a", "T_hat")], blocks[("b", "T_hat")])
    for nm in ("T_total", "T_tilde"):
        x, y = blocks[("a", nm)], blocks[("b", nm)]
        assert np.all(np.abs(x - y) <= 1e-10 * np.abs(y))


def test_probe_errors(pair):
    name, s, r = pair
    with pytest.raises(tg.ThermigaError, match="probe parametric coordinates outside the patch"):
        s.probe([[0.5, 0.5, 1.5]])
    assert s.probe(np.zeros((0, 3))).shape == (0, 12)


def test_probe_device_tensor(pair):
    import torch
    name, s, r = pair
    s.reset()
    s.advance(2)
    xi = sample_xi(32, 8)
    host = s.probe(xi)
    dev = s.probe(torch.from_numpy(xi).cuda())
    assert dev.is_cuda and np.array_equal(dev.cpu().numpy(), host)
