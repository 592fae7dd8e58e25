"""K5's host decisions without a GPU (host-only simulations): which point sets are
tensor grids, and the source prefix [0, J) that takes the GEMMs at a time t —
checked against a numpy restatement of the rule in csrc/k5_sumfact.cu
(sf_source_eligible: every pair of the source with a point of the face's bounding
box has r.r <= cull * spread * (1 - 1e-9), or the source is causally inactive)."""
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
    assert q.sumfact_prefix(1e-3)[0] == 0
    q.close()


def test_switch_off():
    s = host_sim(os.path.join(ROOT, "configs", "cfg2_raster_layer.cfg"))
    s.set_sumfact(False)
    assert not s.sumfact_stats()["on"] and s.sumfact_prefix(0.02) == (0, 0)
    s.set_sumfact(True)
    assert s.sumfact_stats()["on"]
    s.close()


def _prefix(src, t, alpha, cull, lo, hi):
    dt = t - src[:, 5]
    spread = 4.0 * alpha * dt
    p = src[:, :3]
    r2 = np.maximum((lo - p) ** 2, (hi - p) ** 2).sum(axis=1)
    ok = ~(dt > 0.0) | (r2 * (1.0 + 1e-9) <= cull * spread)
    bad = np.flatnonzero(~ok)
    return int(bad[0]) if len(bad) else len(src)


def _face_boxes(s):
    fs = s.face_sets()
    tqb = s.info["total_qb"]
    nq, xq = fs["nq"], fs["xq"]
    ax = np.abs(nq).argmax(axis=1)
    key = 2 * ax + (nq[np.arange(len(nq)), ax] > 0)
    boxes = {}
    for e in range(s.info["n_face_elems"]):
        b0, b1 = fs["qb_off"][e], fs["qb_off"][e + 1]
        f0, f1 = tqb + fs["qf_off"][e], tqb + fs["qf_off"][e + 1]
        k = int(key[b0])
        pts = np.concatenate([xq[b0:b1], xq[f0:f1]])
        lo, hi = boxes.get(k, (np.full(3, np.inf), np.full(3, -np.inf)))
        boxes[k] = (np.minimum(lo, pts.min(axis=0)), np.maximum(hi, pts.max(axis=0)))
    return boxes


@pytest.mark.parametrize("t", [-1.0, 0.0, 1e-4, 3e-3])
def test_prefix_matches_restatement(tmp_path, monkeypatch, t):
    path = long_history_cfg(tmp_path)
    banded = host_sim(path)  # default: faces cut into bands of element rows
    monkeypatch.setenv("TG_SF_BANDS", "1")  # whole faces: the restatement's boxes
    s = host_sim(path)
    src = s.sources()
    k, rho, c = (s.params[n] for n in ("conductivity", "density", "heat_capacity"))
    alpha, cull = k / (rho * c), s.params["cull"]
    jf = min(_prefix(src, t, alpha, cull, lo, hi) for lo, hi in _face_boxes(s).values())
    g = s.greville_points()
    jd = _prefix(src, t, alpha, cull, g.min(axis=0), g.max(axis=0))
    got = s.sumfact_prefix(t)
    assert got == (jf, jd)
    jb = banded.sumfact_prefix(t)  # smaller boxes: never a shorter prefix
    assert jb[0] >= jf and jb[1] == jd
    banded.close()
    if t == -1.0:  # every source still inactive: all eligible (exact zero columns)
        assert got == (len(src), len(src))
    if t == 0.0:  # the long history: both paths carry sources
        assert 0 < got[0] < len(src) and 0 < got[1] < len(src)
    s.close()
