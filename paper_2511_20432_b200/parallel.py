"""Multi-GPU sharding of the hot path: one process per GPU,
torch.distributed for the plumbing (NCCL on B200s, gloo for the CPU tests).

* K1 superposition shards by points: every rank evaluates a contiguous slab of
  the points against the replicated source history; no exchange is needed
  (bench.py's weak-scaling mode) or one all-gather assembles the field.
* K1 + K3 flux load shards by face elements: each rank computes the local
  loads of its element slab, the slabs are all-gathered and every rank runs
  the deterministic gather in the reference's scatter order
  (proj/src/assembly.cpp:141-144) — bit-identical to one GPU.
* K2 shards the free grid in z-slabs: each CG iteration exchanges p ghost
  planes with the two neighbours (the halo) before the operator apply and
  all-reduces the dot products (SlabPCG below, the reference's
  pcg_jacobi, proj/src/sparse.cpp:41-100, with global dot products).

The compute callbacks are injected so that the partition, exchange and
reduction logic is exercised on CPU (gloo, world_size 2) by
tests/test_parallel.py; the GPU bindings (`gpu_*` helpers) plug in the C ABI
device entry points.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Callable, List, Optional, Tuple

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

    def all_gather_concat(self, part, sizes: List[int]):
        """Concatenate every rank's part (sizes[r] items each, in rank order)."""
        import torch
        import torch.distributed as dist
        t = part if isinstance(part, torch.Tensor) else torch.as_tensor(part)
        if self.world == 1:
            return t
        width = max(sizes)
        pad = torch.zeros(width, dtype=t.dtype, device=t.device)
        pad[: t.numel()] = t.reshape(-1)
        bufs = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(bufs, pad)
        return torch.cat([b[:s] for b, s in zip(bufs, sizes)])

    def all_reduce_sum(self, values):
        """Sum of a small vector over ranks (fixed order per backend)."""
        import torch
        import torch.distributed as dist
        t = torch.as_tensor(np.asarray(values, dtype=np.float64)).to(self.device)
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return t.cpu().numpy()

    def exchange_halo(self, lo_send, hi_send, lo_shape, hi_shape):
        """Send lo_send to rank-1 and hi_send to rank+1; return what they sent
        back (the ghost planes below and above this rank's slab), or None at
        the ends of the rank chain."""
        import torch
        import torch.distributed as dist
        if self.world == 1:
            return None, None
        ops = []
        lo_recv = hi_recv = None
        if self.rank > 0:
            lo_recv = torch.empty(lo_shape, dtype=torch.float64, device=self.device)
            ops.append(dist.P2POp(dist.isend, lo_send.contiguous(), self.rank - 1))
            ops.append(dist.P2POp(dist.irecv, lo_recv, self.rank - 1))
        if self.rank < self.world - 1:
            hi_recv = torch.empty(hi_shape, dtype=torch.float64, device=self.device)
            ops.append(dist.P2POp(dist.isend, hi_send.contiguous(), self.rank + 1))
            ops.append(dist.P2POp(dist.irecv, hi_recv, self.rank + 1))
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        return lo_recv, hi_recv


# ---------------------------------------------------------------------------
# K1 / K3

def sharded_flux_load(local_fn: Callable[[int, int], object], gather_fn: Callable[[object], object],
                      n_elems: int, n_cols: int, dist: Dist):
    """assemble_flux_load over face-element slabs. local_fn(e0, e1) returns the
    local loads of elements [e0, e1) ((e1 - e0) * n_cols values, element-major);
    gather_fn(loc_all) scatters all elements' loads into F in the reference's
    order. Every rank returns the full F."""
    e0, e1 = partition(n_elems, dist.world, dist.rank)
    part = local_fn(e0, e1)
    sizes = [(partition(n_elems, dist.world, r)[1] - partition(n_elems, dist.world, r)[0]) * n_cols
             for r in range(dist.world)]
    return gather_fn(dist.all_gather_concat(part, sizes))


def sharded_points(fn: Callable[[int, int], object], n_points: int, dist: Dist, gather=True):
    """Evaluate fn(begin, end) on this rank's point slab; optionally all-gather."""
    b, e = partition(n_points, dist.world, dist.rank)
    part = fn(b, e)
    if not gather:
        return part
    sizes = [partition(n_points, dist.world, r)[1] - partition(n_points, dist.world, r)[0]
             for r in range(dist.world)]
    return dist.all_gather_concat(part, sizes)


# ---------------------------------------------------------------------------
# K2: z-slab Jacobi-PCG

class SlabPCG:
    """pcg_jacobi (proj/src/sparse.cpp:41-100) on z-slabs of the free grid.

    apply_slab(k0, k1, x_ghosted) -> (A x) on planes [k0, k1), where x_ghosted
    holds planes [max(0, k0 - p), min(nz, k1 + p)) (torch tensor, flat,
    plane-major). inv_diag_owned: 1/diag on this rank's planes."""

    def __init__(self, apply_slab, inv_diag_owned, plane: int, nz: int, p: int, dist: Dist):
        self.apply_slab = apply_slab
        self.dinv = inv_diag_owned
        self.plane, self.nz, self.p, self.dist = plane, nz, p, dist
        self.k0, self.k1 = partition(nz, dist.world, dist.rank)
        if dist.world > 1 and self.k1 - self.k0 < p:
            raise ValueError("z-slabs thinner than the stencil half-width")

    def _ghosted(self, v):
        """v (owned planes) with the neighbours' ghost planes attached."""
        import torch
        p, pl = self.p, self.plane
        k0, k1 = self.k0, self.k1
        lo_n = min(p, k0)                 # ghost planes below
        hi_n = min(p, self.nz - k1)       # ghost planes above
        v2 = v.reshape(k1 - k0, pl)
        lo, hi = self.dist.exchange_halo(v2[:min(p, k1 - k0)], v2[max(0, k1 - k0 - p):],
                                         (lo_n, pl), (hi_n, pl))
        parts = []
        if lo_n:
            parts.append(lo[-lo_n:] if lo is not None else v2.new_zeros((lo_n, pl)))
        parts.append(v2)
        if hi_n:
            parts.append(hi[:hi_n] if hi is not None else v2.new_zeros((hi_n, pl)))
        return torch.cat(parts).reshape(-1)

    def _dot(self, *pairs):
        local = [float((a * b).sum().item()) for a, b in pairs]
        return self.dist.all_reduce_sum(local)

    def solve(self, b, x, tol: float, max_iter: int, single_reduction: bool = False):
        """b, x: owned-plane torch tensors (x = warm start, updated in place).
        Returns (iterations, relative residual); raises like the reference.
        single_reduction: the Chronopoulos-Gear form of the device solver
        (k2_cg1_kernel) — one halo exchange and one 3-scalar allreduce per
        iteration instead of one exchange and two allreduces."""
        if single_reduction:
            return self._solve_cg1(b, x, tol, max_iter)
        bb = self._dot((b, b))[0]
        bnorm = float(np.sqrt(bb))
        if bnorm == 0.0:
            x.zero_()
            return 0, 0.0
        r = b - self.apply_slab(self.k0, self.k1, self._ghosted(x))
        z = self.dinv * r
        rz = self._dot((r, z))[0]
        p = z.clone()
        rel = 0.0
        for it in range(max_iter):
            rr = self._dot((r, r))[0]
            rel = float(np.sqrt(rr)) / bnorm
            if rel <= tol:
                return it, rel
            Ap = self.apply_slab(self.k0, self.k1, self._ghosted(p))
            pAp = self._dot((p, Ap))[0]
            if not pAp > 0.0:
                raise ArithmeticError("pcg: indefinite direction, matrix not SPD")
            alpha = rz / pAp
            x.add_(alpha * p)
            r.sub_(alpha * Ap)
            z = self.dinv * r
            rz_new = self._dot((r, z))[0]
            beta = rz_new / rz
            rz = rz_new
            p = z + beta * p
        raise ArithmeticError(f"pcg: no convergence in {max_iter} iterations, "
                              f"relative residual {rel:.17g}")

    def _solve_cg1(self, b, x, tol, max_iter):
        A = lambda v: self.apply_slab(self.k0, self.k1, self._ghosted(v))  # noqa: E731
        r = b - A(x)
        bb, rr = self._dot((b, b), (r, r))
        bnorm = float(np.sqrt(bb))
        if bnorm == 0.0:  # sparse.cpp:57-60
            x.zero_()
            return 0, 0.0
        rel = float(np.sqrt(rr)) / bnorm
        if max_iter > 0 and rel <= tol:
            return 0, rel
        if max_iter > 0:
            u = self.dinv * r
            w = A(u)
            gamma, delta = self._dot((r, u), (w, u))
            if not delta > 0.0:
                raise ArithmeticError("pcg: indefinite direction, matrix not SPD")
            alpha, beta = gamma / delta, 0.0
            p = u.clone()
            s = w.clone()
            it = 0
            while it < max_iter:
                if it > 0:
                    p = u + beta * p  # p_i = u_i + beta p_{i-1}
                    s = w + beta * s  # s_i = w_i + beta s_{i-1} (= A p_i)
                x.add_(alpha * p)
                r.sub_(alpha * s)
                u = self.dinv * r
                w = A(u)
                g1, d1, rr = self._dot((r, u), (w, u), (r, r))
                it += 1
                if it >= max_iter:
                    break  # the reference leaves after max_iter updates untested
                rel = float(np.sqrt(rr)) / bnorm
                if rel <= tol:
                    return it, rel
                beta = g1 / gamma
                den = d1 - beta * g1 / alpha  # p_{i+1} . A p_{i+1}
                if not den > 0.0:
                    raise ArithmeticError("pcg: indefinite direction, matrix not SPD")
                alpha, gamma = g1 / den, g1
        raise ArithmeticError(f"pcg: no convergence in {max_iter} iterations, "
                              f"relative residual {rel:.17g}")


# ---------------------------------------------------------------------------
# GPU bindings (C ABI device entry points)

def gpu_flux_local(sim, t: float, fine_radius: float = -1.0):
    """local_fn for sharded_flux_load on this rank's GPU."""
    import ctypes as C
    import torch
    L = sim._L
    L.tg_sim_flux_local_device.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_int, C.c_int,
                                           C.c_void_p]
    ndk = sim.info["n_dofs_kept"]

    def local(e0, e1):
        out = torch.empty((e1 - e0) * ndk, dtype=torch.float64, device="cuda")
        sim._check(L.tg_sim_flux_local_device(sim._h, float(t), float(fine_radius), e0, e1,
                                              C.c_void_p(out.data_ptr())))
        return out
    return local


def gpu_flux_gather(sim):
    import ctypes as C
    import torch
    L = sim._L
    L.tg_sim_flux_gather_device.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]

    def gather(loc_all):
        F = torch.empty(sim.info["n_full"], dtype=torch.float64, device="cuda")
        sim._check(L.tg_sim_flux_gather_device(sim._h, C.c_void_p(loc_all.data_ptr()),
                                               C.c_void_p(F.data_ptr())))
        return F
    return gather


def gpu_apply_slab(sim):
    import ctypes as C
    import torch
    L = sim._L
    L.tg_sim_operator_apply_slab_device.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p,
                                                    C.c_void_p]
    plane = sim.info["nx"] * sim.info["ny"]

    def apply(k0, k1, xg):
        y = torch.empty((k1 - k0) * plane, dtype=torch.float64, device="cuda")
        sim._check(L.tg_sim_operator_apply_slab_device(sim._h, k0, k1, C.c_void_p(xg.data_ptr()),
                                                       C.c_void_p(y.data_ptr())))
        return y
    return apply


def gpu_inverse_diagonal(sim):
    """1 / diag(A_ff) of the simulation's operator as a CUDA tensor (the Jacobi
    preconditioner of SlabPCG on this GPU)."""
    import ctypes as C
    import torch
    L = sim._L
    L.tg_sim_inverse_diagonal.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
    out = np.zeros(sim.info["n_free"])
    sim._check(L.tg_sim_inverse_diagonal(sim._h, out.ctypes.data_as(C.POINTER(C.c_double))))
    return torch.from_numpy(out).cuda()


def gpu_dirichlet_range(sim, t: float):
    """fn(c0, c1) -> Dirichlet values of constrained DOFs [c0, c1) at t (CUDA
    tensor) for sharded_points."""
    import ctypes as C
    import torch
    L = sim._L
    L.tg_sim_dirichlet_range_device.argtypes = [C.c_void_p, C.c_double, C.c_int, C.c_int,
                                                C.c_void_p]

    def fn(c0, c1):
        out = torch.empty(max(0, c1 - c0), dtype=torch.float64, device="cuda")
        if c1 > c0:
            sim._check(L.tg_sim_dirichlet_range_device(sim._h, float(t), c0, c1,
                                                       C.c_void_p(out.data_ptr())))
        return out
    return fn


class ShardedTimeLoop:
    """run_time_loop (proj/src/driver.cpp:105-146) on `dist.world` GPUs, one
    Simulation per rank. Per step the superposition work — the flux load over
    face-element slabs and the Dirichlet values over point slabs, >90 % of a
    config-4 step — is split across ranks and all-gathered (two collectives);
    the theta step then runs on every rank from the same loads, so every rank
    holds the same state (bit for bit: all pieces are deterministic and
    shard-independent)."""

    def __init__(self, sim, dist: Dist):
        import ctypes as C
        self.sim, self.dist = sim, dist
        self.L = sim._L
        self.L.tg_sim_advance_with_loads_device.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p,
                                                           C.POINTER(C.c_long),
                                                           C.POINTER(C.c_double)]
        self.dt = sim.params["dt"]
        self.step_index = 0

    def reset(self):
        self.sim.reset()
        self.step_index = 0

    def step(self):
        import ctypes as C
        s, d = self.sim, self.dist
        t1 = (self.step_index + 1) * self.dt  # driver.cpp:127
        F1 = sharded_flux_load(gpu_flux_local(s, t1), gpu_flux_gather(s), s.info["n_face_elems"],
                               s.info["n_dofs_kept"], d)
        g1 = sharded_points(gpu_dirichlet_range(s, t1), s.info["n_constrained"], d)
        it = C.c_long(0)
        rel = C.c_double(0.0)
        s._check(self.L.tg_sim_advance_with_loads_device(s._h, C.c_void_p(F1.data_ptr()),
                                                         C.c_void_p(g1.data_ptr()),
                                                         C.byref(it), C.byref(rel)))
        self.step_index += 1
        return it.value, rel.value


def init_from_env(backend: Optional[str] = None) -> Dist:
    """torchrun-style initialization (MASTER_ADDR/PORT, RANK, WORLD_SIZE)."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 and not dist.is_initialized():
        dist.init_process_group(backend or ("nccl" if torch.cuda.is_available() else "gloo"))
    dev = f"cuda:{int(os.environ.get('LOCAL_RANK', '0'))}" if torch.cuda.is_available() else "cpu"
    return Dist.from_env(dev)
