"""Multi-rank logic of paper_2511_20432_b200/parallel.py on CPU (gloo,
world_size 2): element-slab flux load (bit-identical to the reference's serial
scatter) and z-slab Jacobi-PCG with halo exchange (same iterates as one rank).
The compute callbacks are the C oracle (flux) and a numpy Kronecker operator
(K2); the GPU bindings plug the C ABI device calls into the same logic."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_20432_b200.parallel import Dist, SlabPCG, partition, sharded_flux_load
from conftest import ROOT

KW = dict(conductivity=20.0, density=4400.0, heat_capacity=600.0)


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


# --- flux load ------------------------------------------------------------

def _flux_rank(d: Dist, fs_path, t):
    from oracle.pyoracle import COracle
    z = dict(np.load(fs_path))
    src = z.pop("sources")
    n_full = int(z.pop("n_full"))
    fs = z
    o = COracle()
    nd = fs["dofs"].shape[1]

    def local(e0, e1):
        return torch.from_numpy(o.boundary_local(fs, src, t, e0, e1, fine_radius=5e-4, **KW).ravel())

    def gather(loc_all):
        loc = loc_all.numpy().reshape(-1, nd)
        F = np.zeros(n_full)
        for e in range(loc.shape[0]):  # the reference's serial scatter order
            for a in range(nd):
                F[fs["dofs"][e, a]] += loc[e, a]
        return F

    return {"F": sharded_flux_load(local, gather, fs["dofs"].shape[0], nd, d)}


@pytest.mark.parametrize("t", [1e-4, 6e-4])
def test_sharded_flux_load_bit_identical(ref, tmp_path, t):
    sim = ref.sim(os.path.join(ROOT, "configs", "cfg0_parity.cfg"))
    fs = sim.face_sets()
    path = tmp_path / "fs.npz"
    np.savez(path, sources=sim.sources(), n_full=sim.info["n_full"], **fs)
    F_ref = sim.flux_load(t)
    sim.close()
    outs = _run(2, _flux_rank, tmp_path, str(path), t)
    for o in outs:
        assert np.array_equal(o["F"], F_ref)


# --- z-slab PCG -------------------------------------------------------------

def _dense(B):
    n, w = B.shape
    p = w // 2
    A = np.zeros((n, n))
    for i in range(n):
        for d in range(-p, p + 1):
            if 0 <= i + d < n:
                A[i, i + d] = B[i, p + d]
    return A


def _kron_factors():
    import paper_2511_20432_b200 as tg
    s = tg.Simulation(os.path.join(ROOT, "configs", "cfg0_parity.cfg"), host_only=True)
    Ms, Ks = zip(*[s.kron_factors(d) for d in range(3)])
    rc = s.params["density"] * s.params["heat_capacity"]
    a = rc / s.params["dt"]
    b = s.params["theta"] * s.params["conductivity"]
    s.close()
    Mx, My, Mz = (_dense(m) for m in Ms)
    Kx, Ky, Kz = (_dense(k) for k in Ks)
    # free grid: drop the constrained bottom layer (zetamin, k = 0)
    return Mx, Kx, My, Ky, Mz[1:, 1:], Kz[1:, 1:], a, b


def _apply(Mx, Kx, My, Ky, Mz, Kz, a, b, x):
    """Op(a, b) x for x of shape (nz, ny, nx) (first index fastest in memory)."""
    def k3(Z, Y, X):
        return np.einsum("kl,jm,in,lmn->kji", Z, Y, X, x)
    return a * k3(Mz, My, Mx) + b * (k3(Mz, My, Kx) + k3(Mz, Ky, Mx) + k3(Kz, My, Mx))


def _pcg_rank(d: Dist, rhs_path, single=False):
    Mx, Kx, My, Ky, Mz, Kz, a, b = _kron_factors()
    nz, ny, nx = Mz.shape[0], My.shape[0], Mx.shape[0]
    p = 2
    rhs = np.load(rhs_path)["b"].reshape(nz, ny, nx)
    k0, k1 = partition(nz, d.world, d.rank)
    diag = (a * np.einsum("k,j,i->kji", np.diag(Mz), np.diag(My), np.diag(Mx)) +
            b * (np.einsum("k,j,i->kji", np.diag(Mz), np.diag(My), np.diag(Kx)) +
                 np.einsum("k,j,i->kji", np.diag(Mz), np.diag(Ky), np.diag(Mx)) +
                 np.einsum("k,j,i->kji", np.diag(Kz), np.diag(My), np.diag(Mx))))

    def apply_slab(s0, s1, xg):
        g0, g1 = max(0, s0 - p), min(nz, s1 + p)
        x = xg.numpy().reshape(g1 - g0, ny, nx)
        y = _apply(Mx, Kx, My, Ky, Mz[s0:s1, g0:g1], Kz[s0:s1, g0:g1], a, b, x)
        return torch.from_numpy(y.ravel().copy())

    solver = SlabPCG(apply_slab, torch.from_numpy((1.0 / diag[k0:k1]).ravel().copy()), ny * nx,
                     nz, p, d)
    x = torch.zeros((k1 - k0) * ny * nx, dtype=torch.float64)
    it, rel = solver.solve(torch.from_numpy(rhs[k0:k1].ravel().copy()), x, 1e-12, 2000,
                           single_reduction=single)
    return {"x": x.numpy(), "k0": k0, "k1": k1, "it": it, "rel": rel}


@pytest.mark.parametrize("single", [False, True], ids=["two-reductions", "single-reduction"])
def test_slab_pcg_two_ranks_matches_one(tmp_path, single):
    Mx, Kx, My, Ky, Mz, Kz, a, b = _kron_factors()
    nz, ny, nx = Mz.shape[0], My.shape[0], Mx.shape[0]
    rhs = np.random.default_rng(11).standard_normal(nz * ny * nx)
    path = tmp_path / "rhs.npz"
    np.savez(path, b=rhs)
    one = _run(1, _pcg_rank, tmp_path, str(path), False)[0]
    two = _run(2, _pcg_rank, tmp_path, str(path), single)
    x2 = np.concatenate([o["x"] for o in sorted(two, key=lambda o: int(o["k0"]))])
    assert abs(int(two[0]["it"]) - int(one["it"])) <= 1
    assert np.abs(x2 - one["x"]).max() <= 1e-10 * np.abs(one["x"]).max()
    # and the solution solves the assembled system
    A = (a * np.kron(Mz, np.kron(My, Mx)) +
         b * (np.kron(Mz, np.kron(My, Kx)) + np.kron(Mz, np.kron(Ky, Mx)) +
              np.kron(Kz, np.kron(My, Mx))))
    assert np.linalg.norm(A @ x2 - rhs) / np.linalg.norm(rhs) <= 1e-11


def _points_rank(d: Dist, n):
    from paper_2511_20432_b200.parallel import sharded_points
    f = lambda b, e: torch.arange(b, e, dtype=torch.float64) * 0.5 + 1.0  # noqa: E731
    return {"all": sharded_points(f, n, d).numpy(), "own": sharded_points(f, n, d, gather=False).numpy()}


@pytest.mark.parametrize("n", [0, 7, 66564])
def test_sharded_points_two_ranks(tmp_path, n):
    """Point slabs (the Dirichlet values of ShardedTimeLoop) all-gathered in
    rank order reproduce the single evaluation."""
    outs = _run(2, _points_rank, tmp_path, n)
    ref = np.arange(n, dtype=np.float64) * 0.5 + 1.0
    for r, o in enumerate(outs):
        assert np.array_equal(o["all"], ref)
        b, e = partition(n, 2, r)
        assert np.array_equal(o["own"], ref[b:e])
