"""K6 (csrc/k6_assemble.cu): the general patch's operators assembled on the
device (SURVEY.md §8f "GPU setup path": assemble_matrix / element_quad,
proj/src/assembly.cpp:59-101, 194-228; proj/src/mesh.cpp:65-117).

  * the device-assembled A_ff equals the reference's CSR bit for bit (row
    pointers, columns, values), as the host assembly does (tests/test_cfg3.py);
  * A_fc and B_f (only seen through the θ-step) give time steps bit-identical
    to the host-assembled operators' (TG_HOST_ASSEMBLY=1);
  * config 3 at full size: the device's A_ff equals the host assembly's;
  * the face quadrature sets built on the device (build_face_sets, the
    reference's build_face_element, proj/src/mesh.cpp:158-236) equal the host
    build bit for bit: points, normals, weights, kept N columns, DOFs, centres."""
import os

import numpy as np
import pytest

import paper_2511_20432_b200 as tg
from conftest import ROOT

pytestmark = pytest.mark.gpu


def _sim(path, host, **kw):
    old = os.environ.pop("TG_HOST_ASSEMBLY", None)
    if host:
        os.environ["TG_HOST_ASSEMBLY"] = "1"
    try:
        return tg.Simulation(path, **kw)
    finally:
        os.environ.pop("TG_HOST_ASSEMBLY", None)
        if old is not None:
            os.environ["TG_HOST_ASSEMBLY"] = old


@pytest.mark.parametrize("name", ["cfg3_parity", "qc_small"])
def test_device_operator_bit_exact_against_reference(ref, name):
    path = os.path.join(ROOT, "configs", name + ".cfg")
    s = _sim(path, host=False)
    r = ref.sim(path)
    try:
        assert s.info["kronecker"] == 0
        rp, ci, v = s.reduced_operator()
        rr, rc, rv = r.csr(2)
        assert np.array_equal(rp, rr) and np.array_equal(ci, rc)
        assert np.array_equal(v, rv)
    finally:
        s.close()
        r.close()


@pytest.mark.parametrize("name", ["cfg3_parity", "qc_small"])
def test_device_operators_step_like_host_operators(name):
    path = os.path.join(ROOT, "configs", name + ".cfg")
    d, h = _sim(path, host=False), _sim(path, host=True)
    try:
        d.reset()
        h.reset()
        for _ in range(3):
            d.advance(4)
            h.advance(4)
            sd, sh = d.state(), h.state()
            assert np.array_equal(sd["free"], sh["free"])
            assert np.array_equal(sd["g"], sh["g"]) and np.array_equal(sd["F"], sh["F"])
    finally:
        d.close()
        h.close()


def test_config3_full_size_device_operator_is_the_host_one():
    path = os.path.join(ROOT, "configs", "cfg3_contour_hatch.cfg")
    d = _sim(path, host=False)
    rp, ci, v = d.reduced_operator()
    d.close()
    h = tg.Simulation(path, host_only=True)
    hp, hc, hv = h.reduced_operator()
    h.close()
    assert np.array_equal(rp, hp) and np.array_equal(ci, hc) and np.array_equal(v, hv)


@pytest.mark.parametrize("name", ["cfg0_parity", "qc_small", "cfg3_parity", "cfg2_raster_layer"])
def test_device_face_sets_bit_exact(name):
    path = os.path.join(ROOT, "configs", name + ".cfg")
    d = tg.Simulation(path)  # device face tables
    h = tg.Simulation(path, host_only=True)
    try:
        assert d.info["n_dofs_kept"] == h.info["n_dofs_kept"]
        fd, fh = d.face_sets(), h.face_sets()
        for k in ("qb_off", "qf_off", "centers", "dofs", "xq", "nq", "wq", "Nb", "Nf"):
            assert np.array_equal(fd[k], fh[k]), k
    finally:
        d.close()
        h.close()
