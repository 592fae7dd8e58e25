"""Python mirror of the reference's hot-path interface over the C ABI.

Names, argument meaning and error behaviour follow proj/include/thermiga/*.hpp:
``discretize_scan`` (analytic.hpp:45-48), ``superpose`` (analytic.hpp:73-75),
``Simulation`` / ``run_time_loop`` (driver.hpp:20-47), ``assemble_flux_load``
(assembly.hpp:37-40), ``dirichlet_values`` (mesh.hpp:121-125), ``theta_step``
(timestep.hpp:26-29).  Every compute call goes through
``_lib/libthermiga_b200.so`` (sm_100a kernels); there is no CPU fallback —
without the library or a B200 the calls raise.

Arrays: numpy arrays are host memory (the C ABI stages them through the
device); torch CUDA tensors are passed as device pointers (no copies).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _build

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class ThermigaError(RuntimeError):
    """Base class; ``code`` is the TG_* status (= reference CLI exit code)."""
    code = 1


class ConfigError(ThermigaError):
    code = 2


class NumericError(ThermigaError):
    code = 3


class IOError_(ThermigaError):
    code = 4


class CudaError(ThermigaError):
    code = 5


_ERRORS = {1: ThermigaError, 2: ConfigError, 3: NumericError, 4: IOError_, 5: CudaError}

TG_OK = 0


class _Material(C.Structure):
    _fields_ = [("conductivity", C.c_double), ("density", C.c_double),
                ("heat_capacity", C.c_double), ("platform_temperature", C.c_double)]


class _Laser(C.Structure):
    _fields_ = [("power", C.c_double), ("speed", C.c_double), ("spot_radius", C.c_double),
                ("absorptivity", C.c_double), ("dt", C.c_double)]


@dataclass
class Material:
    """thermiga::Material (analytic.hpp:10-20)."""
    conductivity: float
    density: float
    heat_capacity: float
    platform_temperature: float = 0.0

    def diffusivity(self) -> float:
        return self.conductivity / (self.density * self.heat_capacity)

    def volumetric_capacity(self) -> float:
        return self.density * self.heat_capacity

    def _c(self):
        return _Material(self.conductivity, self.density, self.heat_capacity,
                         self.platform_temperature)


@dataclass
class LaserSpec:
    """thermiga::LaserSpec (analytic.hpp:22-31)."""
    power: float
    speed: float
    spot_radius: float
    absorptivity: float
    dt: float

    def _c(self):
        return _Laser(self.power, self.speed, self.spot_radius, self.absorptivity, self.dt)


@dataclass
class ScanPath:
    """thermiga::ScanPath (analytic.hpp:42-47)."""
    waypoints: Sequence[Sequence[float]] = field(default_factory=list)
    start_time: float = 0.0
    plane_z: float = 0.0


@dataclass
class SuperposeOptions:
    """thermiga::SuperposeOptions (analytic.hpp:60-66)."""
    cull_exponent: float = 60.0


_LIB = None


def lib(auto_build: bool = True):
    """Load libthermiga_b200.so (building it in-tree with nvcc when missing)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if auto_build and (not os.path.exists(_build.LIB) or os.environ.get("TG_REBUILD")):
        _build.build()
    path = os.environ.get("TG_LIB_VARIANT") or _build.LIB  # tuning builds (tools/k1_variants.py)
    if not os.path.exists(path):
        raise CudaError(f"native library missing: {path}")
    if "TG_NCCL_LIB" not in os.environ:  # the multi-GPU path binds torch's NCCL if present
        import importlib.util
        spec = importlib.util.find_spec("torch")
        if spec and spec.origin:
            cand = os.path.join(os.path.dirname(os.path.dirname(spec.origin)), "nvidia", "nccl",
                                "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["TG_NCCL_LIB"] = cand
    L = C.CDLL(path)
    L.tg_abi_version.restype = C.c_int
    L.tg_ctx_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
    L.tg_ctx_destroy.argtypes = [C.c_void_p]
    L.tg_last_error.restype = C.c_char_p
    L.tg_last_error.argtypes = [C.c_void_p]
    L.tg_set_profiling.argtypes = [C.c_void_p, C.c_int]
    L.tg_profile_read.argtypes = [C.c_void_p, _dp, C.c_int]
    L.tg_fp64_peak.argtypes = [C.c_void_p, _dp]
    L.tg_dmma_peak.argtypes = [C.c_void_p, _dp]
    L.tg_pcg_jacobi.argtypes = [C.c_void_p, C.c_int, _ip, _ip, _dp, _dp, _dp, C.c_double, C.c_int,
                                _ip, _dp]
    L.tg_csr_multiply.argtypes = [C.c_void_p, C.c_int, _ip, _ip, _dp, _dp, _dp]
    L.tg_discretize_scan.argtypes = [_dp, C.c_int, C.c_double, C.c_double,
                                     C.POINTER(_Laser), C.POINTER(_Material), _dp, C.c_int]
    L.tg_set_sources.argtypes = [C.c_void_p, _dp, C.c_int, C.POINTER(_Material)]
    L.tg_superpose_batch.argtypes = [C.c_void_p, _dp, C.c_long, C.c_double, C.c_double, _dp, _dp]
    L.tg_superpose_batch_device.argtypes = [C.c_void_p, C.c_void_p, C.c_long, C.c_double,
                                            C.c_double, C.c_void_p, C.c_void_p, C.c_void_p]
    L.tg_geometry_elevate.argtypes = [C.c_char_p, _ip, _dp, C.c_char_p, C.c_char_p, C.c_int]
    _LIB = L
    return L


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a):
    return None if a is None else a.ctypes.data_as(_dp)


def discretize_scan(path: ScanPath, laser: LaserSpec, mat: Material) -> np.ndarray:
    """Point sources {x, y, z, E, t_activate, tau} (n, 6); analytic.cpp:22-71."""
    L = lib()
    wp = _f64(np.asarray(path.waypoints, dtype=np.float64).reshape(-1, 2))
    las, m = laser._c(), mat._c()
    n = L.tg_discretize_scan(_p(wp), len(wp), path.start_time, path.plane_z, C.byref(las),
                             C.byref(m), None, 0)
    if n < 0:
        raise ThermigaError("discretize_scan: invalid laser, material or empty path")
    out = np.zeros((n, 6))
    L.tg_discretize_scan(_p(wp), len(wp), path.start_time, path.plane_z, C.byref(las),
                         C.byref(m), _p(out), n)
    return out


def elevate_geometry(in_path: str, out_path: str, elevate=(0, 0, 0), scale=None) -> None:
    """Geometry tooling for config 3 (SURVEY.md §8f item 4, Appendix C option A):
    read a geometry file in the reference's format, scale the control
    coordinates per axis, elevate the degree exactly, write a geometry file
    (tg_geometry_elevate)."""
    L = lib()
    t = np.ascontiguousarray(elevate, dtype=np.int32)
    sc = None if scale is None else _f64(scale)
    err = C.create_string_buffer(512)
    rc = L.tg_geometry_elevate(os.fsencode(in_path), t.ctypes.data_as(_ip), _p(sc),
                               os.fsencode(out_path), err, len(err))
    if rc != 0:
        raise _ERRORS.get(rc, ThermigaError)(err.value.decode())


class Context:
    """A device context (one CUDA stream, resident buffers) on one GPU."""

    def __init__(self, device: int = 0):
        L = self._L = lib()
        h = C.c_void_p()
        rc = L.tg_ctx_create(device, C.byref(h))
        self._h = h
        if rc != TG_OK:
            msg = L.tg_last_error(h).decode() if h else "context creation failed"
            if h:
                L.tg_ctx_destroy(h)
            self._h = None
            raise _ERRORS.get(rc, ThermigaError)(msg)
        self.n_sources = 0
        self.material: Optional[Material] = None

    def _check(self, rc):
        if rc != TG_OK:
            raise _ERRORS.get(rc, ThermigaError)(self._L.tg_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            self._L.tg_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- profiling ----------------------------------------------------------
    def set_profiling(self, on: bool = True):
        self._check(self._L.tg_set_profiling(self._h, int(on)))

    def profile(self, reset: bool = False) -> dict:
        out = np.zeros(11)
        self._check(self._L.tg_profile_read(self._h, _p(out), int(reset)))
        return dict(k1_ms=out[0], k1_launches=int(out[1]), k1_pairs=out[2], k2_ms=out[3],
                    k2_launches=int(out[4]), k2_bytes=out[5], launches=int(out[6]),
                    theta_step_ms=out[7], k5_ms=out[8], k5_launches=int(out[9]),
                    step_ms=out[10])

    @staticmethod
    def _csr(A):
        """(row_ptr, col, val) int32/int32/float64 from a scipy sparse matrix,
        a dense array or a (row_ptr, col, val) tuple."""
        if isinstance(A, tuple):
            rp, ci, v = A
        elif hasattr(A, "tocsr"):
            M = A.tocsr()
            M.sort_indices()
            rp, ci, v = M.indptr, M.indices, M.data
        else:
            D = np.asarray(A, dtype=np.float64)
            rp, ci, v = [0], [], []
            for row in D:
                nz = np.nonzero(row)[0]
                ci += nz.tolist()
                v += row[nz].tolist()
                rp.append(len(ci))
        return (np.ascontiguousarray(rp, dtype=np.int32), np.ascontiguousarray(ci, dtype=np.int32),
                _f64(v))

    def pcg_jacobi(self, A, b, x=None, tol: float = 1e-10, max_iter: int = 5000):
        """pcg_jacobi (proj/include/thermiga/sparse.hpp:45-46) on this GPU:
        returns (x, iterations, rel_residual); NumericError with the
        reference's message on the cap or a non-SPD matrix."""
        rp, ci, v = self._csr(A)
        n = len(rp) - 1
        bb = _f64(b)
        xx = np.zeros(n) if x is None else _f64(x).copy()
        it = C.c_int(0)
        rel = C.c_double(0.0)
        ip = C.POINTER(C.c_int)
        self._check(self._L.tg_pcg_jacobi(self._h, n, rp.ctypes.data_as(ip), ci.ctypes.data_as(ip),
                                          _p(v), _p(bb), _p(xx), float(tol), int(max_iter),
                                          C.byref(it), C.byref(rel)))
        return xx, it.value, rel.value

    def csr_multiply(self, A, x):
        """CsrMatrix::multiply (sparse.cpp:25-31) on this GPU."""
        rp, ci, v = self._csr(A)
        n = len(rp) - 1
        xx = _f64(x)
        y = np.zeros(n)
        ip = C.POINTER(C.c_int)
        self._check(self._L.tg_csr_multiply(self._h, n, rp.ctypes.data_as(ip),
                                            ci.ctypes.data_as(ip), _p(v), _p(xx), _p(y)))
        return y

    def fp64_peak_tflops(self) -> float:
        out = C.c_double(0.0)
        self._check(self._L.tg_fp64_peak(self._h, C.byref(out)))
        return out.value

    def dmma_peak_tflops(self) -> float:
        """Measured FP64 tensor-core rate (DMMA m8n8k4, independent accumulators)."""
        out = C.c_double(0.0)
        self._check(self._L.tg_dmma_peak(self._h, C.byref(out)))
        return out.value

    # -- K1 -------------------------------------------------------------------
    def set_sources(self, sources, mat: Material):
        s = _f64(np.asarray(sources).reshape(-1, 6))
        m = mat._c()
        self._check(self._L.tg_set_sources(self._h, _p(s), len(s), C.byref(m)))
        self.n_sources = len(s)
        self.material = mat

    def superpose(self, points, t: float, opts: SuperposeOptions = SuperposeOptions(),
                  grad: bool = True, out=None, stream=None):
        """T~ and grad T~ at every point (superpose, analytic.cpp:92-109).

        numpy input -> numpy (value (n,), grad (n,3)); torch CUDA input -> device
        tensors written in place of ``out`` (or newly allocated)."""
        if hasattr(points, "is_cuda") and points.is_cuda:
            import torch
            n = points.shape[0]
            if out is None:
                val = torch.empty(n, dtype=torch.float64, device=points.device)
                g = torch.empty((n, 3), dtype=torch.float64, device=points.device) if grad else None
            else:
                val, g = out
            st = stream if stream is not None else torch.cuda.current_stream(points.device).cuda_stream
            self._check(self._L.tg_superpose_batch_device(
                self._h, C.c_void_p(points.data_ptr()), n, float(t), float(opts.cull_exponent),
                C.c_void_p(val.data_ptr()), C.c_void_p(g.data_ptr()) if g is not None else None,
                C.c_void_p(st)))
            return val, g
        p = _f64(np.asarray(points).reshape(-1, 3))
        n = len(p)
        if out is None:
            val = np.zeros(n)
            g = np.zeros((n, 3)) if grad else None
        else:
            val, g = out
        self._check(self._L.tg_superpose_batch(self._h, _p(p), n, float(t),
                                               float(opts.cull_exponent), _p(val), _p(g)))
        return val, g


def superpose(sources, mat: Material, x, t: float, opts: SuperposeOptions = SuperposeOptions(),
              ctx: Optional[Context] = None):
    """Reference-shaped convenience: one or many points -> (value, grad)."""
    own = ctx is None
    ctx = ctx or Context()
    try:
        ctx.set_sources(sources, mat)
        pts = np.asarray(x, dtype=np.float64)
        single = pts.ndim == 1
        v, g = ctx.superpose(pts.reshape(-1, 3), t, opts)
        return (v[0], g[0]) if single else (v, g)
    finally:
        if own:
            ctx.close()


class _SimOptions(C.Structure):
    _fields_ = [("t_end", C.c_double), ("solver_tol", C.c_double), ("max_iter", C.c_int),
                ("device", C.c_int), ("host_only", C.c_int), ("preconditioner", C.c_int)]


def _bind_sim(L):
    if getattr(L, "_sim_bound", False):
        return
    L.tg_sim_create.argtypes = [C.c_char_p, C.POINTER(_SimOptions), C.POINTER(C.c_void_p)]
    L.tg_sim_destroy.argtypes = [C.c_void_p]
    L.tg_sim_last_error.restype = C.c_char_p
    L.tg_sim_last_error.argtypes = [C.c_void_p]
    L.tg_sim_context.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
    L.tg_sim_info.argtypes = [C.c_void_p, C.POINTER(C.c_long)]
    L.tg_sim_params.argtypes = [C.c_void_p, _dp]
    L.tg_sim_sources.argtypes = [C.c_void_p, _dp, C.c_int]
    L.tg_sim_face_sets.argtypes = [C.c_void_p, _ip, _ip, _dp, _ip, _dp, _dp, _dp, _dp, _dp]
    L.tg_sim_greville_points.argtypes = [C.c_void_p, _dp]
    L.tg_sim_last_local_loads.argtypes = [C.c_void_p, _dp]
    L.tg_sim_kron_factors.argtypes = [C.c_void_p, C.c_int, _dp, _dp]
    L.tg_sim_reduced_operator.argtypes = [C.c_void_p, _ip, _ip, _ip, _dp]
    L.tg_sim_reduced_operator.restype = C.c_long
    L.tg_sim_flux_load.argtypes = [C.c_void_p, C.c_double, _dp, C.c_double, _dp]
    L.tg_sim_dirichlet_values.argtypes = [C.c_void_p, C.c_double, _dp]
    L.tg_sim_theta_step.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp, C.c_double, C.c_int,
                                    _dp, _ip, _dp]
    L.tg_sim_operator_apply.argtypes = [C.c_void_p, _dp, _dp]
    L.tg_sim_reset.argtypes = [C.c_void_p]
    L.tg_sim_advance.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_long), _dp]
    L.tg_sim_state.argtypes = [C.c_void_p, _ip, _dp, _dp, _dp, _dp]
    L.tg_sim_probe.argtypes = [C.c_void_p, _dp, C.c_long, _dp]
    L.tg_sim_probe_device.argtypes = [C.c_void_p, C.c_void_p, C.c_long, C.c_void_p]
    L.tg_sim_field_eval.argtypes = [C.c_void_p, _dp, _dp, C.c_long, _dp, _dp]
    L.tg_sim_flux_profile.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, _dp, _dp]
    L.tg_sim_set_sumfact.argtypes = [C.c_void_p, C.c_int]
    L.tg_sim_sumfact_stats.argtypes = [C.c_void_p, _dp]
    L.tg_sim_sumfact_regions.argtypes = [C.c_void_p, _dp]
    L.tg_sim_shard.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_char_p]
    L.tg_sim_set_slabs.argtypes = [C.c_void_p, C.c_int]
    L.tg_sim_last_integrand.restype = C.c_long
    L.tg_sim_last_integrand.argtypes = [C.c_void_p, _dp]
    L.tg_sim_set_region_split.argtypes = [C.c_void_p, C.c_int, C.c_int]
    L.tg_sim_sumfact_plan.argtypes = [C.c_void_p, C.c_double, _ip, _ip]
    L.tg_sim_sumfact_last_plan.argtypes = [C.c_void_p, _ip, _ip]
    L.tg_sim_sumfact_counts.argtypes = [C.c_void_p, C.c_double, _ip]
    L.tg_sim_sumfact_last_counts.argtypes = [C.c_void_p, _ip]
    L._sim_bound = True


class _BorrowedContext(Context):
    """The context owned by a Simulation (not destroyed by Python)."""

    def __init__(self, L, h):  # noqa: D401 - no base init: the handle is borrowed
        self._L, self._h = L, h

    def close(self):
        self._h = None


class Simulation:
    """prepare_simulation + run_time_loop of the reference (driver.hpp:20-47) on the GPU.

    The hot-path calls keep the reference's names: ``flux_load`` =
    assemble_flux_load, ``dirichlet_values``, ``theta_step``; ``reset`` /
    ``advance`` / ``state`` run the time loop with the state resident on the device.
    """

    INFO_KEYS = ["n_full", "n_free", "n_constrained", "n_steps", "n_sources", "n_face_elems",
                 "nx", "ny", "nz", "px", "py", "pz", "kronecker", "nq_base", "nq_fine",
                 "n_dofs_kept", "total_qb", "total_qf"]
    PARAM_KEYS = ["dt", "theta", "solver_tol", "elevate_radius", "cull", "conductivity",
                  "density", "heat_capacity", "platform_temperature", "max_iter"]

    PRECONDITIONERS = {"jacobi": 0, "fdm": 1}

    def __init__(self, config_path, t_end=0.0, solver_tol=0.0, max_iter=0, device=0,
                 host_only=False, preconditioner="jacobi"):
        L = self._L = lib()
        _bind_sim(L)
        opt = _SimOptions(t_end, solver_tol, max_iter, device, int(host_only),
                          self.PRECONDITIONERS[preconditioner])
        h = C.c_void_p()
        rc = L.tg_sim_create(str(config_path).encode(), C.byref(opt), C.byref(h))
        self._h = h
        if rc != TG_OK:
            msg = L.tg_sim_last_error(h).decode() if h else "tg_sim_create failed"
            L.tg_sim_destroy(h)
            self._h = None
            raise _ERRORS.get(rc, ThermigaError)(msg)
        info = (C.c_long * 18)()
        self._check(L.tg_sim_info(h, info))
        self.info = {k: int(v) for k, v in zip(self.INFO_KEYS, info)}
        par = np.zeros(10)
        self._check(L.tg_sim_params(h, _p(par)))
        self.params = dict(zip(self.PARAM_KEYS, par.tolist()))

    def _check(self, rc):
        if rc != TG_OK:
            raise _ERRORS.get(rc, ThermigaError)(self._L.tg_sim_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            self._L.tg_sim_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def context(self) -> Context:
        h = C.c_void_p()
        self._check(self._L.tg_sim_context(self._h, C.byref(h)))
        return _BorrowedContext(self._L, h)

    def sources(self):
        out = np.zeros((self.info["n_sources"], 6))
        self._check(self._L.tg_sim_sources(self._h, _p(out), len(out)))
        return out

    def face_sets(self):
        """Face sets as uploaded: qb_off/qf_off per-element offsets, xq/nq/wq all base
        points then all fine points, Nb (total_qb, kept), Nf (total_qf, kept)."""
        i = self.info
        ne, nd, tqb, tqf = i["n_face_elems"], i["n_dofs_kept"], i["total_qb"], i["total_qf"]
        d = dict(qb_off=np.zeros(ne + 1, dtype=np.int32), qf_off=np.zeros(ne + 1, dtype=np.int32),
                 centers=np.zeros((ne, 3)), dofs=np.zeros((ne, nd), dtype=np.int32),
                 xq=np.zeros((tqb + tqf, 3)), nq=np.zeros((tqb + tqf, 3)), wq=np.zeros(tqb + tqf),
                 Nb=np.zeros((tqb, nd)), Nf=np.zeros((tqf, nd)))
        ip = lambda a: a.ctypes.data_as(_ip)  # noqa: E731
        self._check(self._L.tg_sim_face_sets(self._h, ip(d["qb_off"]), ip(d["qf_off"]),
                                             _p(d["centers"]), ip(d["dofs"]), _p(d["xq"]),
                                             _p(d["nq"]), _p(d["wq"]), _p(d["Nb"]), _p(d["Nf"])))
        return d

    def set_sumfact(self, on: bool = True):
        """K5: superposition on the gridded face / Greville point sets as a DGEMM over
        the sources no cull can reach there (default on where the sets are grids);
        off = every pair through K1."""
        self._check(self._L.tg_sim_set_sumfact(self._h, int(on)))

    def sumfact_stats(self) -> dict:
        out = np.zeros(8)
        self._check(self._L.tg_sim_sumfact_stats(self._h, _p(out)))
        return dict(on=bool(out[0]), faces_gridded=bool(out[1]), greville_gridded=bool(out[2]),
                    last_j_flux=int(out[3]), last_j_dirichlet=int(out[4]), gemm_flops=out[5],
                    regions=int(out[6]), item=int(out[7]))

    def shard(self, rank: int, world: int, nccl_id: bytes):
        """Join the NCCL communicator `nccl_id` (nccl_unique_id() on rank 0)
        as rank of world: the loads' regions and the θ-step's z-slabs are then
        split over the ranks (tg_sim_shard)."""
        self._check(self._L.tg_sim_shard(self._h, int(rank), int(world), bytes(nccl_id)))

    def set_slabs(self, n: int):
        """Run the θ-step solve as n z-slabs on this GPU (the multi-GPU
        decomposition's local test bed; n <= 1 turns it off)."""
        self._check(self._L.tg_sim_set_slabs(self._h, int(n)))

    def last_integrand(self):
        """The compact flux integrand of the last flux-load call (one value per
        active face quadrature point, device element order)."""
        n = self._L.tg_sim_last_integrand(self._h, None)
        if n < 0:
            raise _ERRORS.get(-n, ThermigaError)(self._L.tg_sim_last_error(self._h).decode())
        out = np.zeros(n)
        self._L.tg_sim_last_integrand(self._h, _p(out))
        return out

    def set_region_split(self, rank: int, world: int):
        """Compute only the K5 regions r % world == rank (the multi-GPU split)."""
        self._check(self._L.tg_sim_set_region_split(self._h, int(rank), int(world)))

    def sumfact_regions(self):
        """K5 regions (flux tiles, then Greville tiles): (n, 8) = lo[3], hi[3],
        delta, points."""
        out = np.zeros((self.sumfact_stats()["regions"], 8))
        self._check(self._L.tg_sim_sumfact_regions(self._h, _p(out)))
        return out

    def sumfact_plan(self, t: float):
        """The K5 plan at t restated on the host: per region (J, E)."""
        n = self.sumfact_stats()["regions"]
        J = np.zeros(n, dtype=np.int32)
        E = np.zeros(n, dtype=np.int32)
        self._check(self._L.tg_sim_sumfact_plan(self._h, float(t), J.ctypes.data_as(_ip),
                                                E.ctypes.data_as(_ip)))
        return J, E

    def sumfact_last_plan(self):
        """The plan the device computed in the last flux-load / Dirichlet call."""
        n = self.sumfact_stats()["regions"]
        J = np.zeros(n, dtype=np.int32)
        E = np.zeros(n, dtype=np.int32)
        self._check(self._L.tg_sim_sumfact_last_plan(self._h, J.ctypes.data_as(_ip),
                                                     E.ctypes.data_as(_ip)))
        return J, E

    def sumfact_counts(self, t: float = None):
        """Per region the contraction's source count Jc (J + the eligible
        sources of [J, E)): the host restatement at t, or (t None) the last
        device plan."""
        Jc = np.zeros(self.sumfact_stats()["regions"], dtype=np.int32)
        if t is None:
            self._check(self._L.tg_sim_sumfact_last_counts(self._h, Jc.ctypes.data_as(_ip)))
        else:
            self._check(self._L.tg_sim_sumfact_counts(self._h, float(t), Jc.ctypes.data_as(_ip)))
        return Jc

    def last_local_loads(self):
        """Per face element local loads of the last flux_load ((n_face_elems,
        n_dofs_kept), columns as face_sets()['dofs'])."""
        out = np.zeros((self.info["n_face_elems"], self.info["n_dofs_kept"]))
        self._check(self._L.tg_sim_last_local_loads(self._h, _p(out)))
        return out

    def greville_points(self):
        out = np.zeros((self.info["n_constrained"], 3))
        self._check(self._L.tg_sim_greville_points(self._h, _p(out)))
        return out

    def kron_factors(self, d):
        n, p = self.info["nx"] if d == 0 else self.info["ny"] if d == 1 else self.info["nz"], \
            self.info["px"]
        M = np.zeros((n, 2 * p + 1))
        K = np.zeros((n, 2 * p + 1))
        self._check(self._L.tg_sim_kron_factors(self._h, d, _p(M), _p(K)))
        return M, K

    def flux_load(self, t, fine_radius=-1.0, focus=None):
        """assemble_flux_load at t; focus (x, y, z) overrides the fine-rule focus
        (default: the newest source active at t)."""
        F = np.zeros(self.info["n_full"])
        fo = None if focus is None else _f64(focus)
        self._check(self._L.tg_sim_flux_load(self._h, float(t), None if fo is None else _p(fo),
                                             float(fine_radius), _p(F)))
        return F

    def dirichlet_values(self, t):
        g = np.zeros(self.info["n_constrained"])
        self._check(self._L.tg_sim_dirichlet_values(self._h, float(t), _p(g)))
        return g

    def theta_step(self, free_n, g_n, F_n, F_np1, g_np1, tol=None, max_iter=None):
        tol = self.params["solver_tol"] if tol is None else tol
        max_iter = int(self.params["max_iter"]) if max_iter is None else max_iter
        a = [_f64(v) for v in (free_n, g_n, F_n, F_np1, g_np1)]
        out = np.zeros(self.info["n_free"])
        it = C.c_int(0)
        rel = C.c_double(0.0)
        self._check(self._L.tg_sim_theta_step(self._h, *[_p(v) for v in a], float(tol),
                                              int(max_iter), _p(out), C.byref(it), C.byref(rel)))
        return out, it.value, rel.value

    def reduced_operator(self):
        """(row_ptr, col, val) of the assembled reduced operator A_ff
        (non-separable patches; DirichletSystem::reduced_operator)."""
        rows = C.c_int(0)
        nnz = self._L.tg_sim_reduced_operator(self._h, C.byref(rows), None, None, None)
        if nnz < 0:
            raise _ERRORS.get(-nnz, ThermigaError)(self._L.tg_sim_last_error(self._h).decode())
        rp = np.zeros(rows.value + 1, dtype=np.int32)
        ci = np.zeros(nnz, dtype=np.int32)
        v = np.zeros(nnz)
        self._L.tg_sim_reduced_operator(self._h, None, rp.ctypes.data_as(_ip),
                                        ci.ctypes.data_as(_ip), _p(v))
        return rp, ci, v

    def operator_apply(self, x):
        xx = _f64(x)
        y = np.zeros(self.info["n_free"])
        self._check(self._L.tg_sim_operator_apply(self._h, _p(xx), _p(y)))
        return y

    def reset(self):
        self._check(self._L.tg_sim_reset(self._h))

    def advance(self, n_steps=1):
        it = C.c_long(0)
        rel = C.c_double(0.0)
        self._check(self._L.tg_sim_advance(self._h, int(n_steps), C.byref(it), C.byref(rel)))
        return it.value, rel.value

    def state(self):
        step = C.c_int(0)
        t = C.c_double(0.0)
        x = np.zeros(self.info["n_free"])
        g = np.zeros(self.info["n_constrained"])
        F = np.zeros(self.info["n_full"])
        self._check(self._L.tg_sim_state(self._h, C.byref(step), C.byref(t), _p(x), _p(g), _p(F)))
        return dict(step=step.value, time=t.value, free=x, g=g, F=F)

    # -- observers (proj/src/postproc.cpp, driver.cpp:226-254) --
    PROBE_COLUMNS = ["x", "y", "z", "T_total", "T_tilde", "T_hat", "gx_tilde", "gy_tilde",
                     "gz_tilde", "gx_hat", "gy_hat", "gz_hat"]

    def probe(self, xi):
        """The current state (time = step * dt) at parametric points xi (n x 3
        in [0, 1]^3): an (n x 12) array with the columns PROBE_COLUMNS —
        map_point, total_temperature, superpose value/gradient, field_at
        value/gradient (postproc.cpp:9-19, splines.cpp:257-303). A torch CUDA
        tensor input stays on the device (tg_sim_probe_device)."""
        try:
            import torch
            if isinstance(xi, torch.Tensor) and xi.is_cuda:
                x = xi.to(torch.float64).contiguous()
                out = torch.empty((x.numel() // 3, 12), dtype=torch.float64, device=x.device)
                torch.cuda.current_stream().synchronize()
                self._check(self._L.tg_sim_probe_device(self._h, x.data_ptr(), x.numel() // 3,
                                                        out.data_ptr()))
                return out
        except ImportError:
            pass
        x = _f64(np.asarray(xi, dtype=np.float64).reshape(-1, 3))
        out = np.zeros((len(x), 12))
        self._check(self._L.tg_sim_probe(self._h, _p(x), len(x), _p(out)))
        return out

    def total_temperature(self, xi):
        """total_temperature (postproc.cpp:9-19) of the current state: T_c +
        T_tilde + T_hat at each parametric point."""
        return self.probe(xi)[:, 3]

    def field_eval(self, coeffs, xi):
        """map_point and field_at with caller coefficients (n_full, flat
        order): (x (n x 3), f (n x 4: value, physical gradient)); coeffs=None
        evaluates the geometry only."""
        x = _f64(np.asarray(xi, dtype=np.float64).reshape(-1, 3))
        xo = np.zeros((len(x), 3))
        if coeffs is None:
            self._check(self._L.tg_sim_field_eval(self._h, None, _p(x), len(x), _p(xo), None))
            return xo, None
        c = _f64(coeffs)
        fo = np.zeros((len(x), 4))
        self._check(self._L.tg_sim_field_eval(self._h, _p(c), _p(x), len(x), _p(xo), _p(fo)))
        return xo, fo

    FACES = {"ximin": 0, "ximax": 1, "etamin": 2, "etamax": 3, "zetamin": 4, "zetamax": 5}

    def boundary_flux_profile(self, face, n_samples, theta_axis=None, edge_v=1.0):
        """boundary_flux_profile (postproc.cpp:21-79) of the current state:
        (n_samples x 5) array of s, theta, q_tilde, q_hat, q_net (theta NaN
        without theta_axis)."""
        f = self.FACES[face] if isinstance(face, str) else int(face)
        out = np.zeros((int(n_samples), 5))
        ax = None if theta_axis is None else _f64(theta_axis)
        self._check(self._L.tg_sim_flux_profile(self._h, f, int(n_samples), float(edge_v),
                                                _p(ax) if ax is not None else None, _p(out)))
        return out

    def export_field(self, path, grid_dims):
        """export_field (postproc.cpp:101-147) of the current state: legacy
        ASCII VTK structured grid of T_total / T_tilde / T_hat on a parametric
        grid, byte-identical to the reference writer for the same values."""
        nx, ny, nz = (int(d) for d in grid_dims)
        if min(nx, ny, nz) < 2:
            raise ValueError("field grid needs >= 2 per direction")
        k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
        xi = np.stack([i.ravel() / (nx - 1), j.ravel() / (ny - 1), k.ravel() / (nz - 1)], axis=1)
        pr = self.probe(xi)
        t = self.state_time()
        tc = self.params["platform_temperature"]
        n = len(xi)
        g = "%.17g"
        lines = ["# vtk DataFile Version 3.0",
                 f"thermiga temperature field at t={g % t} s", "ASCII",
                 "DATASET STRUCTURED_GRID", f"DIMENSIONS {nx} {ny} {nz}", f"POINTS {n} double"]
        lines += [f"{g % a} {g % b} {g % c}" for a, b, c in pr[:, :3]]
        lines.append(f"POINT_DATA {n}")
        for name, col in (("T_total", None), ("T_tilde", 4), ("T_hat", 5)):
            lines += [f"SCALARS {name} double 1", "LOOKUP_TABLE default"]
            vals = (tc + pr[:, 4] + pr[:, 5]) if col is None else pr[:, col]
            lines += [g % v for v in vals]
        try:
            with open(path, "w") as fh:
                fh.write("\n".join(lines) + "\n")
        except OSError as e:
            raise IOError_(f"cannot open {path}") from e

    def state_time(self):
        step = C.c_int(0)
        t = C.c_double(0.0)
        self._check(self._L.tg_sim_state(self._h, C.byref(step), C.byref(t), None, None, None))
        return t.value


def nccl_unique_id() -> bytes:
    """A new NCCL communicator id (128 bytes) for Simulation.shard."""
    L = lib()
    L.tg_nccl_unique_id.argtypes = [C.c_char_p]
    buf = C.create_string_buffer(128)
    rc = L.tg_nccl_unique_id(buf)
    if rc != TG_OK:
        raise CudaError("NCCL is not available (libnccl.so.2)")
    return buf.raw


def slab_plan(nz: int, p: int, world: int, rank: int) -> dict:
    """The z-slab of one rank (host arithmetic, tg_slab_plan)."""
    L = lib()
    L.tg_slab_plan.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _ip]
    out = np.zeros(6, dtype=np.int32)
    if L.tg_slab_plan(int(nz), int(p), int(world), int(rank), out.ctypes.data_as(_ip)) != TG_OK:
        raise ValueError("slab plan: need nz / world >= p and 0 <= rank < world")
    return dict(zip(("gz0", "nloc", "zo0", "zo1", "lo", "hi"), (int(v) for v in out)))


def integrated_abs_flux(profile):
    """integrated_abs_flux (postproc.cpp:81-95): composite-trapezoid integrals
    of |q_net| and |q_tilde| over arc length; ratio None when the analytic
    integral is zero."""
    p = np.asarray(profile, dtype=np.float64)
    if len(p) < 2:
        raise ValueError("flux metrics need >= 2 samples")
    net = ana = 0.0
    for i in range(1, len(p)):
        ds = p[i, 0] - p[i - 1, 0]
        net += 0.5 * ds * (abs(p[i - 1, 4]) + abs(p[i, 4]))
        ana += 0.5 * ds * (abs(p[i - 1, 2]) + abs(p[i, 2]))
    return {"integral_net": float(net), "integral_analytic": float(ana),
            "ratio": float(net / ana) if ana > 0.0 else None}


def export_profile_csv(profile, path):
    """export_profile_csv (postproc.cpp:149-159)."""
    p = np.asarray(profile, dtype=np.float64)
    if len(p) == 0:
        raise ValueError("refusing to write an empty flux profile")
    g = "%.17g"
    try:
        with open(path, "w") as fh:
            fh.write("s_m,theta_rad,q_tilde_W_m2,q_hat_W_m2,q_net_W_m2\n")
            for r in p:
                fh.write(",".join(g % v for v in r) + "\n")
    except OSError as e:
        raise IOError_(f"cannot open {path}") from e
