"""K2 strip tiles (csrc/k2_kron.cu TileShape / make_tiles_strip): grids whose
x extent leaves a ragged remainder of 1..8 control points past the last full
32-wide tile (config 2: 66 = 2 * 32 + 2, config 4: 258 = 8 * 32 + 2) sweep those
columns with transposed 8 x 32 tiles. The per-point arithmetic is the main
tiles' (same band sums in the same order); only the per-CTA grouping of the
dot products changes. Checked here:
  * against the live reference's time loop (pcg_jacobi, proj/src/sparse.cpp:
    41-100, driven by run_time_loop, proj/src/driver.cpp:126-145) on small
    cuboids with remainders 2, 6 and 8 (normwise <= 1e-8 per step, loads
    <= 1e-10; solver_tol 1e-12 on both sides);
  * against the main-tile-only sweep (TG_K2_NO_STRIP) at config-4 size: the
    same iteration counts and free coefficients within rounding.
The small-grid resident solve (csrc/k2_resident.cu) is checked the same way
against the streaming kernel; the reference-loop parity of small configs
(tests/test_sim_gpu.py) runs through it by default.
"""
import os
import re

import numpy as np
import pytest

import paper_2511_20432_b200 as tg
from conftest import ROOT

pytestmark = pytest.mark.gpu


def normwise(a, b):
    m = np.abs(b).max()
    return 0.0 if m == 0 else float(np.abs(a - b).max() / m)


def cfg_with_xi(tmp_path, xi):
    txt = open(os.path.join(ROOT, "configs", "cfg0_parity.cfg")).read()
    txt, n = re.subn(r"^xi_elements = \d+", f"xi_elements = {xi}", txt, flags=re.M)
    assert n == 1
    p = tmp_path / f"xi{xi}.cfg"
    p.write_text(txt)
    return str(p)


@pytest.mark.parametrize("xi", [32, 36, 38], ids=["rx2", "rx6", "rx8"])
def test_strip_grid_against_live_reference(xi, ref, tmp_path):
    p = cfg_with_xi(tmp_path, xi)
    os.environ["TG_K2_STRIP"] = "1"  # small grids use strips only when forced
    os.environ["TG_K2_NO_RESIDENT"] = "1"  # (and the resident solve would take them)
    try:
        s = tg.Simulation(p, t_end=1.5e-4)
    finally:
        os.environ.pop("TG_K2_STRIP")
        os.environ.pop("TG_K2_NO_RESIDENT")
    r = ref.sim(p, t_end=1.5e-4)
    assert s.info["kronecker"] == 2
    s.reset()
    r.reset()
    for k in range(1, 16):
        s.advance(1)
        st = s.state()
        o = r.step()
        assert normwise(st["F"], o["F"]) <= 1e-10, (xi, k)
        assert normwise(st["g"], o["g"]) <= 1e-10, (xi, k)
        assert normwise(st["free"], o["free"]) <= 1e-8, (xi, k)
    s.close()
    r.close()


@pytest.mark.parametrize("resident", [True, False], ids=["resident", "streaming"])
@pytest.mark.parametrize("deg,xi", [(1, 33), (3, 31)], ids=["p1", "p3"])
def test_even_pitch_other_degrees_against_live_reference(deg, xi, resident, ref, tmp_path):
    """Degree-1 and degree-3 cuboids whose x extent (34) makes the grid
    TMA-addressable: the TMA sweeps are kept to degree 2 (k2_make_map), so
    these take the resident solve or the plain-load kernels; regression test
    for the illegal-instruction fault those bands hit on the TMA path."""
    from test_sim_gpu import box_geometry
    txt = open(os.path.join(ROOT, "configs", "cfg0_parity.cfg")).read()
    head, rest = txt.split("[geometry]", 1)
    rest = rest[rest.index("\n\n"):]
    rest, n = re.subn(r"^xi_elements = \d+", f"xi_elements = {xi}", rest, flags=re.M)
    assert n == 1
    p = tmp_path / f"deg{deg}.cfg"
    p.write_text(head + box_geometry((deg, deg, deg)) + rest)
    if not resident:
        os.environ["TG_K2_NO_RESIDENT"] = "1"
    try:
        s = tg.Simulation(str(p), t_end=1.5e-4)
    finally:
        os.environ.pop("TG_K2_NO_RESIDENT", None)
    r = ref.sim(str(p), t_end=1.5e-4)
    assert s.info["kronecker"] > 0 and s.info["nx"] == 34
    s.reset()
    r.reset()
    for k in range(1, 12):
        s.advance(1)
        st = s.state()
        o = r.step()
        assert normwise(st["F"], o["F"]) <= 1e-10, (deg, k)
        assert normwise(st["free"], o["free"]) <= 1e-8, (deg, k)
    s.close()
    r.close()


def _run(cfg, steps, strip, resident=False):
    """Steps with the streaming single-sweep solve (strip tiles on / off) or,
    resident=True, the shared-memory resident solve (k2_resident.cu)."""
    keys = [] if resident else ["TG_K2_NO_RESIDENT",
                                "TG_K2_STRIP" if strip else "TG_K2_NO_STRIP"]
    for k in keys:
        os.environ[k] = "1"
    try:
        s = tg.Simulation(cfg, solver_tol=1e-12)
    finally:
        for k in keys:
            os.environ.pop(k, None)
    s.reset()
    its = [s.advance(1)[0] for _ in range(steps)]
    x = s.state()["free"]
    s.close()
    return its, x


@pytest.mark.slow
@pytest.mark.parametrize("name", ["cfg2_raster_layer", "cfg4_large"])
def test_strip_matches_main_tiles_full_size(name):
    cfg = os.path.join(ROOT, "configs", name + ".cfg")
    its_s, x_s = _run(cfg, 3, True)
    its_m, x_m = _run(cfg, 3, False)
    assert all(abs(a - b) <= 1 for a, b in zip(its_s, its_m)), (its_s, its_m)
    assert normwise(x_s, x_m) <= 1e-11, normwise(x_s, x_m)
    # the dot products group differently per CTA with strips, so bit-equal
    # states would mean the strip path never ran
    assert not np.array_equal(x_s, x_m)


@pytest.mark.parametrize("name", ["cfg2_raster_layer", "cfg0_single_track"])
def test_resident_solve_matches_streaming(name):
    """The shared-memory resident solve (the default on grids that fit one
    cooperative wave) against the streaming single-sweep kernel: the same
    Krylov iterates up to the per-CTA grouping of the dot products."""
    cfg = os.path.join(ROOT, "configs", name + ".cfg")
    its_r, x_r = _run(cfg, 5, False, resident=True)
    its_m, x_m = _run(cfg, 5, False)
    assert all(abs(a - b) <= 1 for a, b in zip(its_r, its_m)), (its_r, its_m)
    assert normwise(x_r, x_m) <= 1e-11, normwise(x_r, x_m)


@pytest.mark.parametrize("xi,zeta", [(38, 6), (128, 8)], ids=["tb4", "tb12"])
def test_resident_block_shapes_match_streaming(xi, zeta, tmp_path):
    """The resident solve's other block edges (4 x 4 on a 40 x 40 free grid,
    12 x 12 with ragged edge blocks on 130 x 130) against the streaming
    kernel on the same steps."""
    txt = open(os.path.join(ROOT, "configs", "cfg0_parity.cfg")).read()
    txt = re.sub(r"^xi_elements = \d+", f"xi_elements = {xi}", txt, flags=re.M)
    txt = re.sub(r"^eta_elements = \d+", f"eta_elements = {xi}", txt, flags=re.M)
    txt = re.sub(r"^zeta_elements = \d+", f"zeta_elements = {zeta}", txt, flags=re.M)
    p = tmp_path / f"res{xi}.cfg"
    p.write_text(txt)
    its_r, x_r = _run(str(p), 4, False, resident=True)
    its_m, x_m = _run(str(p), 4, False)
    assert all(abs(a - b) <= 1 for a, b in zip(its_r, its_m)), (its_r, its_m)
    assert normwise(x_r, x_m) <= 1e-11, normwise(x_r, x_m)
    assert not np.array_equal(x_r, x_m)  # (the resident path ran: other dot grouping)


@pytest.mark.parametrize("name", ["cfg3_parity", "qc_small"])
def test_dia_operator_bitwise_equals_sell(name):
    """Non-separable patches: A_ff with implicit columns (DevDia, k2_csr.cu)
    against the sliced-ELL copy it is built from. Both sum each row in the
    CSR's column order (the DIA's extra slots hold exact zeros), and the PCG
    dot products do not depend on the format, so whole steps agree bit for
    bit (CsrMatrix::multiply order, proj/src/sparse.cpp:25-31)."""
    cfg = os.path.join(ROOT, "configs", name + ".cfg")
    out = []
    for off in (False, True):
        if off:
            os.environ["TG_K2_NO_DIA"] = "1"
        try:
            s = tg.Simulation(cfg, solver_tol=1e-12)
        finally:
            os.environ.pop("TG_K2_NO_DIA", None)
        assert s.info["kronecker"] == 0
        s.reset()
        its = [s.advance(1)[0] for _ in range(4)]
        out.append((its, s.state()["free"]))
        s.close()
    assert out[0][0] == out[1][0]
    assert np.array_equal(out[0][1], out[1][1])
