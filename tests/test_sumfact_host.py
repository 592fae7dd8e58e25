"""K5's host decisions without a GPU (host-only simulations): which point sets are
tensor grids, how they are cut into regions, and the per-region plan at a time t
— the contraction prefix J and the pair-wise remainder end E — checked against a
numpy restatement of the rule (csrc/k5_fused.cu sf_plan_kernel, restated on the
host by Sim::sf_plan_host): J = the first source with a point of the region's
box (+- delta) it could cull there (r.r > cull * spread * (1 - 1e-9)), 0 when
J x points < the profitability threshold; E = one past the last source not
culled on the whole box. Causally inactive sources are eligible and culled."""
import os

import numpy as np
import pytest

import paper_2511_20432_b200 as tg
from conftest import ROOT
from test_sumfact_gpu import long_history_cfg


def host_sim(path):
    return tg.Simulation(path, host_only=True)


def test_grids_detected_on_cuboids_only():
    s = host_sim(os.path.join(ROOT, "configs", "cfg2_raster_layer.cfg"))
    st = s.sumfact_stats()
    assert st["on"] and st["faces_gridded"] and st["greville_gridded"]
    s.close()
    q = host_sim(os.path.join(ROOT, "configs", "qc_small.cfg"))  # curved quarter cylinder
    st = q.sumfact_stats()
    assert not st["faces_gridded"]
    R = q.sumfact_regions()
    assert (R[:, 7] > 0).all()  # only the (flat, gridded) Greville regions
    q.close()


def test_switch_off():
    s = host_sim(os.path.join(ROOT, "configs", "cfg2_raster_layer.cfg"))
    s.set_sumfact(False)
    assert not s.sumfact_stats()["on"]
    J, E = s.sumfact_plan(0.02)
    assert not J.any() and E.any()  # every pair on K1, still trimmed per region
    s.set_sumfact(True)
    assert s.sumfact_stats()["on"]
    s.close()


def _plan(src, t, alpha, cull, reg, min_pairs):
    dt = t - src[:, 5]
    active = dt > 0.0
    spread = 4.0 * alpha * dt
    p = src[:, :3]
    lo, hi, delta, npts = reg[0:3] - reg[6], reg[3:6] + reg[6], reg[6], reg[7]
    r2max = np.maximum((lo - p) ** 2, (hi - p) ** 2).sum(axis=1)
    ok = ~active | ((r2max * (1.0 + 1e-9) <= cull * spread)
                    & (36.0 * cull * delta * delta <= 1e-24 * spread))
    bad = np.flatnonzero(~ok)
    n_act = int(np.flatnonzero(active)[-1]) + 1 if active.any() else 0
    J = int(bad[0]) if len(bad) and bad[0] < n_act else n_act
    if npts < 0 or (J * npts < min_pairs and J < 16384):
        J = 0
    d = np.maximum(np.maximum(lo - p, p - hi), 0.0)
    culled = ~active | ((d * d).sum(axis=1) * (1.0 - 1e-9) > cull * spread)
    keep = np.flatnonzero(~culled[J:n_act])
    E = J + int(keep[-1]) + 1 if len(keep) else J
    # the contraction's count: + the sources of [J, E) eligible on the box too
    Jc = J + int(ok[J:E].sum()) if J > 0 else J
    return J, E, Jc


def test_regions_cover_the_grids():
    s = host_sim(os.path.join(ROOT, "configs", "cfg2_raster_layer.cfg"))
    R = s.sumfact_regions()
    fs = s.face_sets()
    tqb = s.info["total_qb"]
    n_dir = s.info["n_constrained"]
    # region point counts: every base quadrature point and every Greville
    # point exactly once; every point inside its grid's region boxes
    assert R[:, 7].sum() == tqb + n_dir
    for pts in (fs["xq"][:tqb], s.greville_points()):
        inside = np.zeros(len(pts), dtype=int)
        for r in R:
            lo, hi = r[0:3] - r[6] - 1e-15, r[3:6] + r[6] + 1e-15
            inside += np.all((pts >= lo) & (pts <= hi), axis=1)
        assert inside.min() >= 1
    s.close()


@pytest.mark.parametrize("t", [-1.0, 0.0, 1e-4, 3e-3, 6e-3])
@pytest.mark.parametrize("min_pairs", [0.0, 3e7])
def test_plan_matches_restatement(tmp_path, monkeypatch, t, min_pairs):
    monkeypatch.setenv("TG_SF_MIN_PAIRS", repr(min_pairs))
    s = host_sim(long_history_cfg(tmp_path))
    src = s.sources()
    k, rho, c = (s.params[n] for n in ("conductivity", "density", "heat_capacity"))
    alpha, cull = k / (rho * c), s.params["cull"]
    J, E = s.sumfact_plan(t)
    Jc = s.sumfact_counts(t)
    R = s.sumfact_regions()
    for r in range(len(R)):
        assert (J[r], E[r], Jc[r]) == _plan(src, t, alpha, cull, R[r], min_pairs), (r, t)
    if t == -1.0:  # every source still inactive: nothing to do anywhere
        assert not J.any() and not E.any()
    if t == 0.0 and min_pairs == 0.0:  # the long history: both paths carry sources
        assert J.min() > 0 and (E > J).any()
    if t == 6e-3 and min_pairs == 0.0:  # eligible sources after the prefix join the contraction
        assert (Jc > J).any()
    s.close()
