"""Multi-rank logic of the multi-GPU step on CPU (gloo; world sizes 2 and 3).

The device path (csrc/slab.cu, sim.cu step_loads) needs GPUs; what these
tests check without them is its decomposition:
  * tg_slab_plan (the product's host function) covers the free grid's planes
    once, with P ghost planes per interior side that are exactly the
    neighbours' own boundary planes;
  * parallel.SlabModel — the slab protocol of k2_slab_kernel in numpy: ghost
    planes of u_0, w^_0 and every w^ exchanged by point-to-point messages,
    own-plane partial sums all-gathered and summed in rank order — gives the
    single-rank solve's iterate count and solution (to rounding) over gloo;
  * the region split of the loads (r % world == rank) covers every region
    once.
The device slabs themselves are compared with the single-GPU solve on a GPU
(tests/test_slab_gpu.py)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2511_20432_b200 as tg
from paper_2511_20432_b200.api import slab_plan
from paper_2511_20432_b200.parallel import Dist, KronOperator, SlabModel, partition
from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(world, fn, tmp, *args):
    port = _free_port()
    mp.spawn(_entry, args=(world, port, fn, str(tmp), args), nprocs=world, join=True)
    return [dict(np.load(os.path.join(tmp, f"out_{r}.npz"))) for r in range(world)]


def _entry(rank, world, port, fn, tmp, args):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = fn(Dist(rank, world, "cpu"), *args)
        np.savez(os.path.join(tmp, f"out_{rank}.npz"), **out)
    finally:
        dist.destroy_process_group()


def test_partition_covers_and_balances():
    for n in (0, 1, 7, 192, 65536):
        for w in (1, 2, 3, 8):
            parts = [partition(n, w, r) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [e - b for b, e in parts]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("nz,p,world", [(65, 2, 8), (65, 2, 2), (17, 2, 3), (5, 2, 2), (9, 3, 3)])
def test_slab_plan(nz, p, world):
    plans = [slab_plan(nz, p, world, r) for r in range(world)]
    own = []
    for r, q in enumerate(plans):
        g0, g1 = q["gz0"] + q["zo0"], q["gz0"] + q["zo1"]
        own.append((g0, g1))
        assert q["zo1"] - q["zo0"] >= p
        assert q["zo0"] == (p if r > 0 else 0)  # ghosts only on interior sides
        assert q["nloc"] - q["zo1"] == (p if r + 1 < world else 0)
        assert q["lo"] == (r - 1 if r > 0 else -1) and q["hi"] == (r + 1 if r + 1 < world else -1)
    assert own[0][0] == 0 and own[-1][1] == nz
    assert all(a[1] == b[0] for a, b in zip(own, own[1:]))
    # a rank's lower ghosts are the lower neighbour's top own planes
    for r in range(1, world):
        assert plans[r]["gz0"] == own[r - 1][1] - p
    with pytest.raises(ValueError):
        slab_plan(nz, p, nz // p + 1, 0)


def _kron_problem():
    """Config 2's free-grid operator (66 x 66 x 17 free planes, degree 2) from
    a host-only Simulation, a seeded right-hand side and warm start."""
    s = tg.Simulation(os.path.join(ROOT, "configs", "cfg2_raster_layer.cfg"), host_only=True)
    p = s.info["px"]
    M = [s.kron_factors(d)[0] for d in range(3)]
    K = [s.kron_factors(d)[1] for d in range(3)]
    M[2], K[2] = M[2][1:], K[2][1:]  # the bottom (constrained) layer is not a free row
    pr = s.params
    a = pr["density"] * pr["heat_capacity"] / pr["dt"]
    b = pr["theta"] * pr["conductivity"]
    shape = (M[2].shape[0], M[1].shape[0], M[0].shape[0])
    s.close()
    rng = np.random.default_rng(7)
    rhs = rng.standard_normal(shape)
    x0 = 1e-3 * rng.standard_normal(shape)
    return KronOperator(M, K, a, b, p), rhs, x0


def _slab_rank(d: Dist):
    op, rhs, x0 = _kron_problem()
    m = SlabModel(op, rhs.shape[0], d)
    x, it, status, rel = m.solve(rhs, x0, 1e-12, 500)
    return {"x": x, "it": it, "status": status, "rel": rel, "z0": m.gz0 + m.zo0}


@pytest.mark.parametrize("world", [2, 3])
def test_slab_protocol_matches_one_rank(tmp_path, world):
    op, rhs, x0 = _kron_problem()
    one = SlabModel(op, rhs.shape[0], Dist(0, 1))
    x1, it1, st1, rel1 = one.solve(rhs, x0, 1e-12, 500)
    assert st1 == 0 and it1 > 10
    # the model is the reference's Jacobi-PCG: the true residual is tol-small
    res = rhs - op.apply(np.pad(x1, ((op.p, op.p), (0, 0), (0, 0))), np.arange(rhs.shape[0]))
    assert np.linalg.norm(res) / np.linalg.norm(rhs) <= 2e-12
    outs = _run(world, _slab_rank, tmp_path)
    x = np.concatenate([o["x"] for o in sorted(outs, key=lambda o: int(o["z0"]))])
    for o in outs:  # every rank took the same decisions
        assert int(o["it"]) == it1 and int(o["status"]) == 0
        assert float(o["rel"]) == float(outs[0]["rel"])
    assert np.abs(x - x1).max() <= 1e-10 * np.abs(x1).max()


@pytest.mark.parametrize("world", [2, 3, 8])
def test_region_split_covers_every_region_once(world):
    s = tg.Simulation(os.path.join(ROOT, "configs", "cfg2_raster_layer.cfg"), host_only=True)
    n = len(s.sumfact_regions())
    s.close()
    owners = [[r for r in range(n) if r % world == rank] for rank in range(world)]
    assert sorted(sum(owners, [])) == list(range(n))
    assert max(map(len, owners)) - min(map(len, owners)) <= 1
