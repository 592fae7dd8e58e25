"""The multi-GPU decomposition's device path on one GPU (csrc/slab.cu,
csrc/k5_fused.cu's region split):
  * the θ-step solve as n z-slabs (k2_slab_kernel per slab, ghost planes and
    partial sums exchanged by device copies, Simulation.set_slabs) against the
    single-GPU persistent solve: same iteration counts, free coefficients
    within rounding (the dot products are summed per slab, then in slab
    order), and the reference's time loop within the parity tolerance;
  * the loads' region split (r % world == rank): every compact flux
    integrand entry and Dirichlet value comes from exactly one rank (the
    others contribute zeros, so the NCCL all-reduce of tg_sim_shard is exact
    and identical on every rank), and the sum equals the unsplit values to
    rounding (the contraction's stream-K partial sums group the sources by
    the CTA split of the rank's own item count);
  * a one-rank NCCL communicator: tg_sim_shard(0, 1) steps bit-equal to
    plain advance().
Tolerances: BASELINE.json north_star (free coefficients <= 1e-8 normwise per
step against the reference)."""
import os

import numpy as np
import pytest

import paper_2511_20432_b200 as tg
from conftest import GOLDEN, ROOT

pytestmark = pytest.mark.gpu
CFG4 = os.path.join(ROOT, "configs", "cfg4_large.cfg")
CFG2 = os.path.join(ROOT, "configs", "cfg2_raster_layer.cfg")


def normwise(a, b):
    m = np.abs(b).max()
    return 0.0 if m == 0 else float(np.abs(a - b).max() / m)


@pytest.fixture(scope="module")
def cfg4():
    s = tg.Simulation(CFG4, solver_tol=1e-12)
    s.reset()
    s.advance(2)
    st = s.state()
    t3 = st["time"] + s.params["dt"]
    inputs = (st["free"], st["g"], st["F"], s.flux_load(t3), s.dirichlet_values(t3))
    yield s, inputs
    s.close()


@pytest.mark.parametrize("n", [2, 3, 8])
def test_slab_solve_matches_single_gpu_config4(cfg4, n):
    s, inp = cfg4
    s.set_slabs(1)
    x1, it1, rel1 = s.theta_step(*inp, tol=1e-12)
    s.set_slabs(n)
    try:
        xn, itn, reln = s.theta_step(*inp, tol=1e-12)
    finally:
        s.set_slabs(1)
    assert abs(itn - it1) <= 1, (itn, it1)
    assert reln <= 1e-12
    assert normwise(xn, x1) <= 1e-11, normwise(xn, x1)


def test_slab_time_loop_against_reference_golden():
    """config 0 (parity size): 2 slabs over the run_time_loop steps of the
    golden reference run (free-grid nz = 5 planes, p = 2)."""
    g = np.load(os.path.join(GOLDEN, "sim_cfg0_parity.npz"))
    s = tg.Simulation(os.path.join(ROOT, "configs", "cfg0_parity.cfg"))
    s.set_slabs(2)
    s.reset()
    done = 0
    for k in g["steps"][:6]:
        s.advance(int(k) - done)
        done = int(k)
        assert normwise(s.state()["free"], g[f"x{k}"]) <= 1e-8, k
    s.close()


def test_slab_config2_steps_match_single():
    a = tg.Simulation(CFG2)
    b = tg.Simulation(CFG2)
    b.set_slabs(4)
    a.reset()
    b.reset()
    a.advance(400)  # mid raster, then 5 steps on both from the same state
    b.advance(400)
    ia, _ = a.advance(5)
    ib, _ = b.advance(5)
    assert abs(ia - ib) <= 5
    assert normwise(b.state()["free"], a.state()["free"]) <= 1e-8
    a.close()
    b.close()


@pytest.mark.parametrize("world", [2, 3])
def test_region_split_partitions_the_loads(cfg4, world):
    s, _ = cfg4
    t = 2.5e-3
    s.set_region_split(0, 1)
    s.flux_load(t)
    gq = s.last_integrand()
    g = s.dirichlet_values(t)
    parts_q, parts_g = [], []
    try:
        for r in range(world):
            s.set_region_split(r, world)
            s.flux_load(t)
            parts_q.append(s.last_integrand())
            parts_g.append(s.dirichlet_values(t))
            s.flux_load(t)  # deterministic per split
            assert np.array_equal(s.last_integrand(), parts_q[-1])
    finally:
        s.set_region_split(0, 1)
    # one contributor per entry: the all-reduce adds zeros only
    assert ((np.stack(parts_q) != 0).sum(axis=0) <= 1).all()
    assert ((np.stack(parts_g) != 0).sum(axis=0) <= 1).all()
    sq, sg = np.sum(parts_q, axis=0), np.sum(parts_g, axis=0)
    assert np.array_equal(sq == 0.0, gq == 0.0)
    assert normwise(sq, gq) <= 1e-13 and normwise(sg, g) <= 1e-13


def test_one_rank_nccl_is_advance():
    uid = tg.api.nccl_unique_id()
    a = tg.Simulation(CFG2)
    b = tg.Simulation(CFG2)
    b.shard(0, 1, uid)
    a.reset()
    b.reset()
    for _ in range(3):
        a.advance(7)
        b.advance(7)
        sa, sb = a.state(), b.state()
        assert np.array_equal(sa["free"], sb["free"]) and np.array_equal(sa["F"], sb["F"])
    a.close()
    b.close()
