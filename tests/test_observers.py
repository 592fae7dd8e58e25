"""Observer host logic on CPU: integrated_abs_flux (postproc.cpp:81-95) and the
profile CSV writer (:149-159) against the unmodified reference on a profile
the reference itself computed (boundary_flux_profile of config 0 with a
seeded coefficient vector)."""
import os

import numpy as np
import pytest

import paper_2511_20432_b200 as tg
from conftest import ROOT


@pytest.fixture(scope="module")
def profile(ref):
    r = ref.sim(os.path.join(ROOT, "configs", "cfg0_parity.cfg"))
    full = np.random.default_rng(4).standard_normal(r.info["n_full"]) * 10.0
    rows, met = r.flux_profile(full, 2, 37, 2.5e-4, theta_axis=(1e-3, 0.0), edge_v=1.0)
    yield r, rows, met
    r.close()


def test_integrated_abs_flux_bitwise(profile):
    r, rows, met = profile
    m = tg.integrated_abs_flux(rows)
    assert m["integral_net"] == met[0] and m["integral_analytic"] == met[1]
    assert m["ratio"] == met[2]
    with pytest.raises(ValueError):
        tg.integrated_abs_flux(rows[:1])
    z = rows.copy()
    z[:, 2] = 0.0
    assert tg.integrated_abs_flux(z)["ratio"] is None


def test_profile_csv_byte_identical(profile, tmp_path):
    r, rows, met = profile
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    tg.export_profile_csv(rows, str(a))
    r.export_profile_csv(rows, str(b))
    assert open(a, "rb").read() == open(b, "rb").read()
    nan = rows.copy()
    nan[:, 1] = np.nan
    tg.export_profile_csv(nan, str(a))
    r.export_profile_csv(nan, str(b))
    assert open(a, "rb").read() == open(b, "rb").read()
