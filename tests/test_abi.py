"""C-ABI library checks that need no GPU: it builds and loads, exports every
symbol include/thermiga_b200.h declares, the host-side setup reproduces the
reference bit for bit, and compute entry points fail loudly without a B200."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2511_20432_b200 as tg
from paper_2511_20432_b200 import _build
from paper_2511_20432_b200 import workloads as W
from conftest import ROOT


def _declared():
    hdr = open(os.path.join(ROOT, "include", "thermiga_b200.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(tg_[a-z0-9_]+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol():
    lib = tg.lib()
    names = _declared()
    assert len(names) >= 8
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump -lelf {_build.LIB} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out


@pytest.mark.parametrize("case", ["cfg1", "cfg0", "cfg2", "dwell", "corner"])
def test_discretize_scan_matches_reference(ref, case):
    mat = tg.Material(**W.MATERIAL)
    las = tg.LaserSpec(**W.LASER)
    if case == "cfg1":
        path = tg.ScanPath(W.config1_waypoints(), 0.0, 1e-3)
    elif case == "cfg0":
        path = tg.ScanPath([(0.2e-3, 0.5e-3), (1.8e-3, 0.5e-3)], 0.0, 0.5e-3)
    elif case == "cfg2":
        path = tg.ScanPath(W.raster_waypoints(4e-3, 4e-3, 1e-4, 1), 0.0, 1e-3)
    elif case == "dwell":
        path = tg.ScanPath([(1e-3, 2e-3)], 0.0, 2e-3)
    else:
        path = tg.ScanPath([(0, 0), (1e-5, 0), (1e-5, 1e-5)], -0.5, 0.0)
    a = tg.discretize_scan(path, las, mat)
    b = ref.discretize_scan(path.waypoints, start_time=path.start_time, plane_z=path.plane_z,
                            **W.MATERIAL, **W.LASER)
    assert np.array_equal(a, b)
    if case == "cfg2":
        assert len(a) == 19988


def test_discretize_scan_rejects_bad_input():
    mat = tg.Material(**W.MATERIAL)
    with pytest.raises(tg.ThermigaError):
        tg.discretize_scan(tg.ScanPath([]), tg.LaserSpec(**W.LASER), mat)
    bad = dict(W.LASER, absorptivity=1.5)
    with pytest.raises(tg.ThermigaError):
        tg.discretize_scan(tg.ScanPath([(0, 0)]), tg.LaserSpec(**bad), mat)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(tg.CudaError):
        tg.Context(0)
