"""Config 3 (SURVEY.md §8d, Appendix C option A; §8f item 4) on the CPU side:
the geometry tooling (exact degree elevation, tg_geometry_elevate) checked
through the unmodified reference's own map_point, and the host setup of the
degree-3 rational part against the reference — face sets, Greville points and
the assembled reduced operator bit for bit."""
import os
import re

import numpy as np
import pytest

import paper_2511_20432_b200 as tg
from paper_2511_20432_b200 import workloads as W
from conftest import ROOT

CFG3 = os.path.join(ROOT, "configs", "cfg3_parity.cfg")


def _config_with_geometry(tmp_path, name, geo_text):
    """cfg3_parity.cfg with its geometry file replaced (written next to it)."""
    (tmp_path / f"{name}.geo").write_text(geo_text)
    txt = open(CFG3).read().replace("file = cfg3_plate_hole_p3.geo", f"file = {name}.geo")
    p = tmp_path / f"{name}.cfg"
    p.write_text(txt)
    return str(p)


def _map_points(ref, cfg_path, xi):
    r = ref.sim(cfg_path)
    try:
        return np.array([r.map_point(x) for x in xi]), r.info
    finally:
        r.close()


def test_elevated_part_is_the_same_map(ref, tmp_path):
    """The committed degree-(3,3,3) part and the reference's bundled (2,1,1)
    quarter-cylinder part (z scaled by 0.5) map every parametric point to the
    same place, evaluated by the reference's map_point."""
    src = tmp_path / "src.geo"
    src.write_text("[geometry]\ncase = quarter_cylinder\n")
    tg.elevate_geometry(str(src), str(tmp_path / "scaled.geo"), elevate=(0, 0, 0),
                        scale=(1.0, 1.0, 0.5))
    tg.elevate_geometry(str(src), str(tmp_path / "elev.geo"), elevate=(1, 2, 2),
                        scale=(1.0, 1.0, 0.5))
    assert (tmp_path / "elev.geo").read_text() == open(
        os.path.join(ROOT, "configs", "cfg3_plate_hole_p3.geo")).read()
    a = _config_with_geometry(tmp_path, "a", (tmp_path / "scaled.geo").read_text())
    b = _config_with_geometry(tmp_path, "b", (tmp_path / "elev.geo").read_text())
    xi = np.random.default_rng(31).uniform(0, 1, (200, 3))
    xi[:8] = [[0, 0, 0], [1, 1, 1], [0.5, 0, 1], [0.5, 1, 0], [0.25, 0.5, 0.5], [1, 0, 0],
              [0, 1, 1], [0.5, 0.5, 0.5]]
    xa, ia = _map_points(ref, a, xi)
    xb, ib = _map_points(ref, b, xi)
    assert (ia["px"], ia["py"], ia["pz"]) == (2, 1, 1)
    assert (ib["px"], ib["py"], ib["pz"]) == (3, 3, 3)
    assert np.abs(xa - xb).max() <= 1e-15 * np.abs(xa).max() * 8
    # the part: a quarter of a 4 x 4 x 1 mm plate with a radius-1 mm hole at (2, 0)
    assert np.isclose(xa[:, 2].max(), 1e-3) and np.isclose(xa[:, 2].min(), 0.0)
    r_hole = np.hypot(xb[:, 0] - 2e-3, xb[:, 1])
    assert r_hole.min() >= 1e-3 * (1 - 1e-14)


def test_elevation_of_a_spline_with_simple_interior_knots(ref, tmp_path):
    """A degree-2 B-spline with single interior knots and uneven control
    points: elevation (via Bezier extraction) keeps the map."""
    rng = np.random.default_rng(8)
    lines = ["[geometry]", "degrees = 2 2 1",
             "knots_xi = 0 0 0 0.3 0.7 1 1 1", "knots_eta = 0 0 0 0.5 1 1 1",
             "knots_zeta = 0 0 1 1", "grid_dims = 5 4 2"]
    for k in range(2):
        for j in range(4):
            for i in range(5):
                x = i * 0.5e-3 + rng.uniform(-5e-5, 5e-5)
                y = j * 0.6e-3 + rng.uniform(-5e-5, 5e-5)
                w = 1.0 + 0.2 * rng.uniform()
                lines.append(f"cp = {x!r} {y!r} {k * 1e-3!r} {w!r}")
    src = tmp_path / "spl.geo"
    src.write_text("\n".join(lines) + "\n")
    tg.elevate_geometry(str(src), str(tmp_path / "spl3.geo"), elevate=(1, 1, 2))
    txt = (tmp_path / "spl3.geo").read_text()
    assert "degrees = 3 3 3" in txt
    assert "knots_xi = 0 0 0 0 0.29999999999999999 0.29999999999999999 0.29999999999999999" in txt
    a = _config_with_geometry(tmp_path, "sa", src.read_text())
    b = _config_with_geometry(tmp_path, "sb", txt)
    xi = np.random.default_rng(4).uniform(0, 1, (100, 3))
    xa, _ = _map_points(ref, a, xi)
    xb, _ = _map_points(ref, b, xi)
    assert np.abs(xa - xb).max() <= 1e-14 * np.abs(xa).max()


def test_elevation_errors(tmp_path):
    with pytest.raises(tg.ConfigError, match="cannot open"):
        tg.elevate_geometry(str(tmp_path / "missing.geo"), str(tmp_path / "o.geo"))
    src = tmp_path / "src.geo"
    src.write_text("[geometry]\ncase = quarter_cylinder\n")
    with pytest.raises(tg.ThermigaError, match=">= 0"):
        tg.elevate_geometry(str(src), str(tmp_path / "o.geo"), elevate=(-1, 0, 0))
    with pytest.raises(tg.api.IOError_):
        tg.elevate_geometry(str(src), str(tmp_path / "no" / "such" / "o.geo"))


def test_scan_path_stays_on_the_part():
    wps = np.array(W.contour_hatch_waypoints())
    assert all(W.plate_hole_region_contains(x, y) for x, y in wps)
    seg = np.linalg.norm(np.diff(wps, axis=0), axis=1)
    steps = seg.sum() / (W.LASER["speed"] * W.LASER["dt"])
    assert 3000 < steps < 5000  # the path ends before the 5000-step run does
    # every segment keeps ~0.1 mm from the hole (sampled; arc chords cut in by
    # their sagitta, < 0.5 um with 24 segments)
    for p0, p1 in zip(wps[:-1], wps[1:]):
        for s in np.linspace(0, 1, 9):
            x, y = p0 + s * (p1 - p0)
            assert np.hypot(x - 2e-3, y) >= 1.1e-3 - 1e-6


@pytest.fixture(scope="module")
def pair3(ref):
    s = tg.Simulation(CFG3, host_only=True)
    r = ref.sim(CFG3)
    yield s, r
    s.close()
    r.close()


def test_setup_counts_and_points_bit_exact(pair3):
    s, r = pair3
    for k in ("n_full", "n_free", "n_constrained", "n_steps", "n_sources", "n_face_elems", "nx",
              "ny", "nz", "px", "py", "pz"):
        assert s.info[k] == r.info[k], k
    assert s.info["kronecker"] == 0
    assert np.array_equal(s.sources(), r.sources())
    assert np.array_equal(s.greville_points(), r.greville_points())
    fs, rf = s.face_sets(), r.face_sets()
    tqb = len(rf["wb"])
    assert np.array_equal(fs["xq"][:tqb], rf["xb"]) and np.array_equal(fs["xq"][tqb:], rf["xf"])
    assert np.array_equal(fs["wq"][:tqb], rf["wb"]) and np.array_equal(fs["wq"][tqb:], rf["wf"])
    assert np.array_equal(fs["nq"][:tqb], rf["nb"]) and np.array_equal(fs["nq"][tqb:], rf["nf"])


@pytest.mark.parametrize("name", ["cfg3_parity", "qc_small"])
def test_reduced_operator_bit_exact(ref, name):
    """The assembled reduced operator A_ff (parallel element matrices and a
    row-partitioned scatter in element order) equals the reference's."""
    path = os.path.join(ROOT, "configs", name + ".cfg")
    s = tg.Simulation(path, host_only=True)
    r = ref.sim(path)
    try:
        rp, ci, v = s.reduced_operator()
        rr, rc, rv = r.csr(2)
        assert np.array_equal(rp, rr) and np.array_equal(ci, rc)
        assert np.array_equal(v, rv)
    finally:
        s.close()
        r.close()


def test_reduced_operator_is_refused_for_separable_patches():
    s = tg.Simulation(os.path.join(ROOT, "configs", "cfg0_parity.cfg"), host_only=True)
    with pytest.raises(tg.ThermigaError, match="not assembled"):
        s.reduced_operator()
    s.close()


def test_config3_full_size_files():
    txt = open(os.path.join(ROOT, "configs", "cfg3_contour_hatch.cfg")).read()
    assert re.search(r"xi_elements = 128\s+eta_elements = 64\s+zeta_elements = 32", txt)
    assert "t_end = 0.05" in txt and "file = cfg3_plate_hole_p3.geo" in txt
