"""Multi-GPU time stepping: one process per GPU,
torch.distributed for the plumbing, the data path native.

Per step (proj/src/driver.cpp:126-145 on every rank):
  * loads: the K5 regions (face-grid and Greville-grid tiles, the step's fine
    rectangles; csrc/k5_fused.cu) are dealt round-robin to the ranks; each
    rank computes its regions' compact flux integrand and Dirichlet values and
    one NCCL all-reduce per vector sums them (disjoint supports: every entry
    has exactly one nonzero contributor, so the sum is exact and identical on
    every rank), then every rank runs the deterministic K3 local-load / gather;
  * θ-step: the RHS is formed on every rank (cheap, HBM-bound); the Jacobi-PCG
    solve runs on z-slabs of the free grid (csrc/slab.cu): per iteration one
    sweep per rank plus one NCCL group carrying the P ghost planes of w^ to /
    from each neighbour and an all-gather of 4 partial sums (summed in rank
    order, so all ranks take the same alpha, beta and stop decision); after
    the solve every rank broadcasts its own planes of x.
Every rank therefore ends each step with the same state.

This module joins the ranks (ShardedTimeLoop: the NCCL communicator id from
rank 0 to all through torch.distributed, then tg_sim_shard) and holds
SlabModel, a numpy model of the slab protocol — the same slab plan
(tg_slab_plan), ghost planes, own-plane partial sums and scalar recurrences
as k2_slab_kernel — that tests/test_parallel.py runs over gloo on CPU to
check the decomposition logic without GPUs. The device path itself is
checked on one GPU by Simulation.set_slabs (all slabs on one device, halos
by device copies) against the single-GPU solve.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np


def partition(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Balanced contiguous slab [begin, end) of n items for `rank`."""
    return n * rank // world, n * (rank + 1) // world


@dataclass
class Dist:
    """Thin wrapper over torch.distributed (or a single process)."""
    rank: int = 0
    world: int = 1
    device: str = "cpu"

    @staticmethod
    def from_env(device: Optional[str] = None) -> "Dist":
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return Dist(dist.get_rank(), dist.get_world_size(), device or "cpu")
        return Dist(0, 1, device or "cpu")

    def broadcast_bytes(self, data: Optional[bytes]) -> bytes:
        """rank 0's bytes on every rank."""
        if self.world == 1:
            return data
        import torch.distributed as dist
        box = [data if self.rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        return box[0]

    def all_gather_array(self, a: np.ndarray) -> list:
        if self.world == 1:
            return [a]
        import torch.distributed as dist
        out = [None] * self.world
        dist.all_gather_object(out, a)
        return out

    def send_recv(self, send: dict, shapes: dict) -> dict:
        """Point-to-point exchange: send[peer] -> peer, receive shapes[peer]
        from peer (float64 arrays)."""
        import torch
        import torch.distributed as dist
        ops, got = [], {}
        for peer, arr in send.items():
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(arr)), peer))
        for peer, shape in shapes.items():
            got[peer] = torch.empty(shape, dtype=torch.float64)
            ops.append(dist.P2POp(dist.irecv, got[peer], peer))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return {p: t.numpy() for p, t in got.items()}


class ShardedTimeLoop:
    """run_time_loop (proj/src/driver.cpp:105-146) on `dist.world` GPUs, one
    Simulation per rank: the loads' regions and the θ-step's z-slabs split
    over the ranks through one NCCL communicator (tg_sim_shard). With one
    rank nothing is sharded: the steps are Simulation.advance's, bit for bit."""

    def __init__(self, sim, dist: Dist):
        from .api import nccl_unique_id
        self.sim, self.dist = sim, dist
        if dist.world > 1:
            uid = dist.broadcast_bytes(nccl_unique_id() if dist.rank == 0 else None)
            sim.shard(dist.rank, dist.world, uid)

    def reset(self):
        self.sim.reset()

    def step(self, n: int = 1):
        return self.sim.advance(n)


# ---------------------------------------------------------------------------
# numpy model of the slab protocol (CPU tests over gloo)

def _band_apply(band: np.ndarray, v: np.ndarray, axis: int, p: int, rows=None) -> np.ndarray:
    """y = B v along `axis` with B banded, entry [i][p + j - i]; rows selects
    the band rows of the output (a slab's own planes), v spans the rows'
    neighbourhoods (zeros outside)."""
    v = np.moveaxis(v, axis, 0)
    n_out = v.shape[0] if rows is None else len(rows)
    out = np.zeros((n_out,) + v.shape[1:])
    for o in range(n_out):
        i = o if rows is None else rows[o]
        for d in range(2 * p + 1):
            j = i + d - p
            jj = j if rows is None else j - rows[0] + p  # v starts p below rows[0]
            if 0 <= jj < v.shape[0]:
                out[o] += band[i, d] * v[jj]
    return np.moveaxis(out, 0, axis)


class KronOperator:
    """A = a (Mz x My x Mx) + b (Mz x My x Kx + Mz x Ky x Mx + Kz x My x Mx)
    on an (nz, ny, nx) grid from banded 1D factors (k2_kron.cu's operator)."""

    def __init__(self, M, K, a: float, b: float, p: int):
        self.M, self.K, self.a, self.b, self.p = M, K, a, b, p

    def diag(self):
        mx, my, mz = (m[:, self.p] for m in self.M)
        kx, ky, kz = (k[:, self.p] for k in self.K)
        mm = np.einsum("k,j,i->kji", mz, my, mx)
        return self.a * mm + self.b * (np.einsum("k,j,i->kji", mz, my, kx)
                                       + np.einsum("k,j,i->kji", mz, ky, mx)
                                       + np.einsum("k,j,i->kji", kz, my, mx))

    def apply(self, v: np.ndarray, zrows=None) -> np.ndarray:
        """A v on the planes zrows (all when None); v holds zrows +- p planes."""
        (Mx, My, Mz), (Kx, Ky, Kz), p = self.M, self.K, self.p
        ux, kx = _band_apply(Mx, v, 2, p), _band_apply(Kx, v, 2, p)
        w1, w2, w3 = _band_apply(My, ux, 1, p), _band_apply(My, kx, 1, p), _band_apply(Ky, ux, 1, p)
        s1 = self.a * w1 + self.b * (w2 + w3)
        s2 = self.b * w1
        return _band_apply(Mz, s1, 0, p, zrows) + _band_apply(Kz, s2, 0, p, zrows)


class SlabModel:
    """The slab solve of csrc/slab.cu in numpy: this rank's planes (tg_slab_plan)
    with ghost planes, the scaled Chronopoulos-Gear Jacobi-PCG (u = D^-1 r,
    w^ = D^-1 A u, s^ = D^-1 A p) with own-plane partial sums, the ghost planes
    of u_0, w^_0 and every w^ exchanged with the neighbours and the partials
    all-gathered (Dist), scalars advanced from the rank-ordered sums."""

    def __init__(self, op: KronOperator, nz: int, dist: Dist):
        from .api import slab_plan
        self.op, self.d = op, dist
        pl = slab_plan(nz, op.p, dist.world, dist.rank)
        self.gz0, self.nloc, self.zo0, self.zo1 = pl["gz0"], pl["nloc"], pl["zo0"], pl["zo1"]
        self.lo, self.hi = pl["lo"], pl["hi"]
        self.rows = np.arange(self.gz0, self.gz0 + self.nloc)
        self.dg = op.diag()[self.gz0:self.gz0 + self.nloc]

    def _apply(self, v):  # A v on every local plane (ghost rows wrong: exchanged)
        p = self.op.p
        pad = np.zeros((self.nloc + 2 * p,) + v.shape[1:])
        pad[p:p + self.nloc] = v
        return self.op.apply(pad, self.rows)

    def _exchange(self, v, parts):
        p = self.op.p
        send, shapes = {}, {}
        if self.lo >= 0:
            send[self.lo] = v[self.zo0:self.zo0 + p]
            shapes[self.lo] = v[:p].shape
        if self.hi >= 0:
            send[self.hi] = v[self.zo1 - p:self.zo1]
            shapes[self.hi] = v[:p].shape
        got = self.d.send_recv(send, shapes) if self.d.world > 1 else {}
        if self.lo >= 0:
            v[:p] = got[self.lo]
        if self.hi >= 0:
            v[self.zo1:self.zo1 + p] = got[self.hi]
        return sum(self.d.all_gather_array(np.asarray(parts, dtype=np.float64)))

    def solve(self, b_full: np.ndarray, x_full: np.ndarray, tol: float, max_iter: int):
        """(x on this rank's own planes, iterations, status, rel)."""
        sl = slice(self.gz0, self.gz0 + self.nloc)
        own = slice(self.zo0, self.zo1)
        b, x = b_full[sl].copy(), x_full[sl].copy()
        r = b - self._apply(x)
        u = r / self.dg
        tot = self._exchange(u, [np.sum(r[own] ** 2), np.sum(b[own] ** 2),
                                 np.sum((r * u)[own]), 0.0])
        bnorm = np.sqrt(tot[1])
        if bnorm == 0.0:
            return np.zeros_like(x[own]), 0, 0, 0.0
        rel = np.sqrt(tot[0]) / bnorm
        if max_iter <= 0 or rel <= tol:
            return x[own], 0, 3 if max_iter <= 0 else 0, rel
        gamma = tot[2]
        Au = self._apply(u)
        w = Au / self.dg
        tot = self._exchange(w, [np.sum((Au * u)[own]), 0.0, 0.0, 0.0])
        if not tot[0] > 0.0:
            return x[own], 0, 4, rel
        alpha, beta = gamma / tot[0], 0.0
        s = np.zeros_like(u)
        p = np.zeros_like(u)
        it = 0
        while True:
            p = u + beta * p
            x = x + alpha * p
            s = w + beta * s
            u = u - alpha * s
            ru = self.dg * u
            Au = self._apply(u)
            w = Au / self.dg
            tot = self._exchange(w, [np.sum((ru * u)[own]), np.sum((Au * u)[own]),
                                     np.sum((ru * ru)[own]), 0.0])
            it += 1
            if it >= max_iter:
                return x[own], it, 3, rel
            rel = np.sqrt(tot[2]) / bnorm
            if rel <= tol:
                return x[own], it, 0, rel
            g1 = tot[0]
            beta = g1 / gamma
            den = tot[1] - beta * g1 / alpha
            if not den > 0.0:
                return x[own], it, 4, rel
            alpha, gamma = g1 / den, g1


def init_from_env(backend: Optional[str] = None) -> Dist:
    """torchrun-style initialization (MASTER_ADDR/PORT, RANK, WORLD_SIZE)."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 and not dist.is_initialized():
        dist.init_process_group(backend or ("nccl" if torch.cuda.is_available() else "gloo"))
    dev = f"cuda:{int(os.environ.get('LOCAL_RANK', '0'))}" if torch.cuda.is_available() else "cpu"
    return Dist.from_env(dev)
