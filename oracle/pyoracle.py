"""TEST INFRASTRUCTURE — ctypes access to the checkers under oracle/.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module.  Two checkers:

  * ``RefLib``  — oracle/_ref/libthermiga_ref.so: the UNMODIFIED reference
    library (built from /root/reference/proj/src by oracle/Makefile) behind the
    extern "C" harness oracle/ref_harness.cpp.
  * ``COracle`` — oracle/_build/liboracle.so: the plain-C restatement
    (oracle/oracle.c), pinned against RefLib and the reference's known answers.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libthermiga_ref.so")
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SRC = "/root/reference/proj"

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_lp = C.POINTER(C.c_long)


def _ptr(a, t=_dp):
    return a.ctypes.data_as(t) if a is not None else None


def build(ref: bool | None = None, quiet: bool = True) -> None:
    """Build the C oracle; build the reference too when its sources exist."""
    targets = ["oracle"]
    if ref is None:
        ref = os.path.isdir(os.path.join(REF_SRC, "src"))
    if ref:
        targets.append("ref")
    subprocess.run(["make", "-C", HERE, "-j8", *targets], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class RefError(RuntimeError):
    pass


class RefLib:
    """The reference library, called through oracle/ref_harness.cpp."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.L = C.CDLL(path)
        L.ref_discretize_scan.restype = C.c_int
        L.ref_discretize_scan.argtypes = [_dp, C.c_int] + [C.c_double] * 10 + [_dp, C.c_int, C.c_char_p, C.c_int]
        L.ref_superpose_batch.restype = C.c_double
        L.ref_superpose_batch.argtypes = [_dp, C.c_int, C.c_double, C.c_double, C.c_double, _dp,
                                          C.c_long, C.c_double, C.c_double, _dp, _dp, C.c_int]
        L.ref_point_source.argtypes = [_dp, C.c_double, C.c_double, C.c_double, _dp, C.c_double, _dp]
        L.ref_gauss_rule.argtypes = [C.c_int, _dp, _dp]
        L.ref_sim_open.restype = C.c_void_p
        L.ref_sim_open.argtypes = [C.c_char_p, C.c_int, C.c_double, C.c_double, C.c_char_p, C.c_int]
        L.ref_sim_close.argtypes = [C.c_void_p]
        L.ref_sim_info.argtypes = [C.c_void_p, _lp]
        L.ref_sim_params.argtypes = [C.c_void_p, _dp]
        L.ref_sim_sources.argtypes = [C.c_void_p, _dp]
        L.ref_sim_face_sets.argtypes = [C.c_void_p, _lp, _ip, _ip, _dp, _ip] + [_dp] * 8
        L.ref_sim_greville_points.argtypes = [C.c_void_p, _dp]
        L.ref_sim_knots.argtypes = [C.c_void_p, C.c_int, _dp]
        L.ref_sim_flux_load.argtypes = [C.c_void_p, C.c_double, _dp, C.c_int]
        L.ref_sim_flux_load_radius.argtypes = [C.c_void_p, C.c_double, C.c_double, _dp]
        L.ref_sim_dirichlet.argtypes = [C.c_void_p, C.c_double, _dp]
        L.ref_sim_csr.restype = C.c_long
        L.ref_sim_csr.argtypes = [C.c_void_p, C.c_int, _ip, _ip, _ip, _dp]
        L.ref_sim_reset.argtypes = [C.c_void_p, _dp, _dp, C.c_char_p, C.c_int]
        L.ref_sim_step.argtypes = [C.c_void_p, _dp, _dp, _dp, _ip, _dp, C.c_char_p, C.c_int]
        L.ref_sim_theta_step.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp, C.c_double, C.c_int,
                                         _dp, _ip, _dp, C.c_char_p, C.c_int]
        L.ref_sim_field_at.argtypes = [C.c_void_p, _dp, _dp, _dp]
        L.ref_sim_map_point.argtypes = [C.c_void_p, _dp, _dp]
        L.ref_pcg_csr.argtypes = [C.c_int, _ip, _ip, _dp, _dp, _dp, C.c_double, C.c_int, _ip, _dp,
                                  C.c_char_p, C.c_int]
        L.ref_sim_run.argtypes = [C.c_void_p, C.c_int, _dp, C.c_char_p, C.c_int]
        L.ref_sim_total_temperature.argtypes = [C.c_void_p, _dp, _dp, C.c_double, _dp,
                                                C.c_char_p, C.c_int]
        L.ref_sim_flux_profile.argtypes = [C.c_void_p, _dp, C.c_int, C.c_int, C.c_double, _dp,
                                           C.c_double, _dp, _dp, C.c_char_p, C.c_int]
        L.ref_sim_export_field.argtypes = [C.c_void_p, _dp, _ip, C.c_double, C.c_char_p,
                                           C.c_char_p, C.c_int]
        L.ref_export_profile_csv.argtypes = [_dp, C.c_int, C.c_char_p, C.c_char_p, C.c_int]
        L.ref_sim_face_point.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double, _dp]
        L.ref_sim_face_points.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, _dp]

    # -- analytic ---------------------------------------------------------
    def discretize_scan(self, waypoints, *, start_time=0.0, plane_z=0.0, power, speed,
                        spot_radius, absorptivity, dt, conductivity, density, heat_capacity,
                        **_):
        wp = np.ascontiguousarray(np.asarray(waypoints, dtype=np.float64).reshape(-1, 2))
        err = C.create_string_buffer(512)
        n = self.L.ref_discretize_scan(_ptr(wp), len(wp), start_time, plane_z, power, speed,
                                       spot_radius, absorptivity, dt, conductivity, density,
                                       heat_capacity, None, 0, err, 512)
        if n < 0:
            raise RefError(err.value.decode())
        out = np.zeros((n, 6))
        self.L.ref_discretize_scan(_ptr(wp), len(wp), start_time, plane_z, power, speed,
                                   spot_radius, absorptivity, dt, conductivity, density,
                                   heat_capacity, _ptr(out), n, err, 512)
        return out

    def superpose(self, sources, pts, t, *, conductivity, density, heat_capacity, cull=60.0,
                  threads=1, grad=True, **_):
        s = np.ascontiguousarray(sources, dtype=np.float64)
        p = np.ascontiguousarray(pts, dtype=np.float64)
        n = len(p)
        val = np.zeros(n)
        g = np.zeros((n, 3)) if grad else None
        secs = self.L.ref_superpose_batch(_ptr(s), len(s), conductivity, density, heat_capacity,
                                          _ptr(p), n, t, cull, _ptr(val), _ptr(g), threads)
        self.last_seconds = secs
        return val, g

    def point_source(self, src6, x, t, *, conductivity, density, heat_capacity, **_):
        s = np.ascontiguousarray(src6, dtype=np.float64)
        xx = np.ascontiguousarray(x, dtype=np.float64)
        out = np.zeros(4)
        self.L.ref_point_source(_ptr(s), conductivity, density, heat_capacity, _ptr(xx), t,
                                _ptr(out))
        return out[0], out[1:]

    def gauss_rule(self, n):
        a, b = np.zeros(n), np.zeros(n)
        self.L.ref_gauss_rule(n, _ptr(a), _ptr(b))
        return a, b

    def pcg(self, row_ptr, col, val, b, x0, tol=1e-10, max_iter=5000):
        rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
        ci = np.ascontiguousarray(col, dtype=np.int32)
        v = np.ascontiguousarray(val, dtype=np.float64)
        bb = np.ascontiguousarray(b, dtype=np.float64)
        x = np.array(x0, dtype=np.float64)
        it = C.c_int(0)
        rel = C.c_double(0)
        err = C.create_string_buffer(512)
        rc = self.L.ref_pcg_csr(len(bb), _ptr(rp, _ip), _ptr(ci, _ip), _ptr(v), _ptr(bb), _ptr(x),
                                tol, max_iter, C.byref(it), C.byref(rel), err, 512)
        if rc != 0:
            raise RefError(err.value.decode())
        return x, it.value, rel.value

    def sim(self, cfg_path, threads=1, t_end=0.0, solver_tol=0.0):
        return RefSim(self, cfg_path, threads, t_end, solver_tol)


class RefSim:
    """prepare_simulation + stepwise run_time_loop of the reference."""

    INFO_KEYS = ["n_full", "n_free", "n_constrained", "n_steps", "n_sources", "n_face_elems",
                 "nx", "ny", "nz", "px", "py", "pz", "n_elements", "threads"]
    PARAM_KEYS = ["dt", "theta", "solver_tol", "elevate_radius", "cull", "conductivity",
                  "density", "heat_capacity", "platform_temperature"]

    def __init__(self, lib: RefLib, cfg_path, threads, t_end, solver_tol):
        self.lib, self.L = lib, lib.L
        err = C.create_string_buffer(1024)
        self.h = self.L.ref_sim_open(str(cfg_path).encode(), threads, t_end, solver_tol, err, 1024)
        if not self.h:
            raise RefError(err.value.decode())
        info = np.zeros(32, dtype=np.int64)
        n = self.L.ref_sim_info(self.h, _ptr(info, _lp))
        self.info = {k: int(v) for k, v in zip(self.INFO_KEYS, info[:n])}
        par = np.zeros(16)
        self.L.ref_sim_params(self.h, _ptr(par))
        self.params = {k: float(v) for k, v in zip(self.PARAM_KEYS, par)}

    def close(self):
        if self.h:
            self.L.ref_sim_close(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sources(self):
        out = np.zeros((self.info["n_sources"], 6))
        self.L.ref_sim_sources(self.h, _ptr(out))
        return out

    def knots(self, d):
        n = self.L.ref_sim_knots(self.h, d, None)
        out = np.zeros(n)
        self.L.ref_sim_knots(self.h, d, _ptr(out))
        return out

    def face_sets(self):
        """Flattened face sets: per-element rule sizes nqb/nqf, qps in
        (face, element, q) order (xb: (total_base, 3), Nb: (total_base, nd), ...)."""
        cnt = np.zeros(4, dtype=np.int64)
        self.L.ref_sim_face_sets(self.h, _ptr(cnt, _lp), None, None, None, None, *([None] * 8))
        ne, tqb, tqf, nd = (int(c) for c in cnt)
        d = dict(nqb=np.zeros(ne, dtype=np.int32), nqf=np.zeros(ne, dtype=np.int32),
                 centers=np.zeros((ne, 3)), dofs=np.zeros((ne, nd), dtype=np.int32),
                 xb=np.zeros((tqb, 3)), nb=np.zeros((tqb, 3)), wb=np.zeros(tqb),
                 Nb=np.zeros((tqb, nd)), xf=np.zeros((tqf, 3)), nf=np.zeros((tqf, 3)),
                 wf=np.zeros(tqf), Nf=np.zeros((tqf, nd)))
        self.L.ref_sim_face_sets(self.h, _ptr(cnt, _lp), _ptr(d["nqb"], _ip), _ptr(d["nqf"], _ip),
                                 _ptr(d["centers"]), _ptr(d["dofs"], _ip),
                                 _ptr(d["xb"]), _ptr(d["nb"]), _ptr(d["wb"]), _ptr(d["Nb"]),
                                 _ptr(d["xf"]), _ptr(d["nf"]), _ptr(d["wf"]), _ptr(d["Nf"]))
        return d

    def greville_points(self):
        out = np.zeros((self.info["n_constrained"], 3))
        self.L.ref_sim_greville_points(self.h, _ptr(out))
        return out

    def flux_load(self, t, threads=1):
        F = np.zeros(self.info["n_full"])
        self.L.ref_sim_flux_load(self.h, t, _ptr(F), threads)
        return F

    def flux_load_radius(self, t, radius):
        F = np.zeros(self.info["n_full"])
        self.L.ref_sim_flux_load_radius(self.h, t, radius, _ptr(F))
        return F

    def dirichlet(self, t):
        g = np.zeros(self.info["n_constrained"])
        self.L.ref_sim_dirichlet(self.h, t, _ptr(g))
        return g

    def csr(self, which):
        rows = C.c_int(0)
        nnz = self.L.ref_sim_csr(self.h, which, C.byref(rows), None, None, None)
        rp = np.zeros(rows.value + 1, dtype=np.int32)
        ci = np.zeros(nnz, dtype=np.int32)
        v = np.zeros(nnz)
        self.L.ref_sim_csr(self.h, which, C.byref(rows), _ptr(rp, _ip), _ptr(ci, _ip), _ptr(v))
        return rp, ci, v

    def reset(self):
        F0 = np.zeros(self.info["n_full"])
        g0 = np.zeros(self.info["n_constrained"])
        err = C.create_string_buffer(1024)
        if self.L.ref_sim_reset(self.h, _ptr(F0), _ptr(g0), err, 1024):
            raise RefError(err.value.decode())
        return F0, g0

    def step(self):
        F = np.zeros(self.info["n_full"])
        g = np.zeros(self.info["n_constrained"])
        x = np.zeros(self.info["n_free"])
        it = C.c_int(0)
        rel = C.c_double(0)
        err = C.create_string_buffer(1024)
        if self.L.ref_sim_step(self.h, _ptr(F), _ptr(g), _ptr(x), C.byref(it), C.byref(rel), err,
                               1024):
            raise RefError(err.value.decode())
        return dict(F=F, g=g, free=x, iters=it.value, rel=rel.value)

    def theta_step(self, free_n, g_n, F_n, F_np1, g_np1, tol, max_iter=5000):
        out = np.zeros(self.info["n_free"])
        it = C.c_int(0)
        rel = C.c_double(0)
        err = C.create_string_buffer(1024)
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (free_n, g_n, F_n, F_np1, g_np1)]
        if self.L.ref_sim_theta_step(self.h, *[_ptr(a) for a in arrs], tol, max_iter, _ptr(out),
                                     C.byref(it), C.byref(rel), err, 1024):
            raise RefError(err.value.decode())
        return out, it.value, rel.value

    def field_at(self, full, xi):
        out = np.zeros(4)
        f = np.ascontiguousarray(full, dtype=np.float64)
        x = np.ascontiguousarray(xi, dtype=np.float64)
        self.L.ref_sim_field_at(self.h, _ptr(f), _ptr(x), _ptr(out))
        return out[0], out[1:]

    def face_point(self, face, u, v):
        """face_point: (x (3), normal (3), area scale)."""
        out = np.zeros(7)
        self.L.ref_sim_face_point(self.h, int(face), u, v, _ptr(out))
        return out[:3], out[3:6], out[6]

    def face_points(self, face, uv):
        """face_point at many (u, v): (n x 7) = x, normal, area scale."""
        p = np.ascontiguousarray(uv, dtype=np.float64).reshape(-1, 2)
        out = np.zeros((len(p), 7))
        self.L.ref_sim_face_points(self.h, int(face), len(p), _ptr(p), _ptr(out))
        return out

    def map_point(self, xi):
        out = np.zeros(3)
        x = np.ascontiguousarray(xi, dtype=np.float64)
        self.L.ref_sim_map_point(self.h, _ptr(x), _ptr(out))
        return out

    def total_temperature(self, full, xi, t):
        """total_temperature (postproc.cpp:9-19) with caller coefficients."""
        out = np.zeros(1)
        err = C.create_string_buffer(1024)
        f = np.ascontiguousarray(full, dtype=np.float64)
        x = np.ascontiguousarray(xi, dtype=np.float64)
        if self.L.ref_sim_total_temperature(self.h, _ptr(f), _ptr(x), t, _ptr(out), err, 1024):
            raise RefError(err.value.decode())
        return float(out[0])

    def flux_profile(self, full, face, n, t, theta_axis=None, edge_v=1.0):
        """boundary_flux_profile + integrated_abs_flux: (rows (n x 5), metrics[3])."""
        out = np.zeros((n, 5))
        met = np.zeros(3)
        err = C.create_string_buffer(1024)
        f = np.ascontiguousarray(full, dtype=np.float64)
        ax = None if theta_axis is None else np.ascontiguousarray(theta_axis, dtype=np.float64)
        if self.L.ref_sim_flux_profile(self.h, _ptr(f), int(face), int(n), t,
                                       _ptr(ax) if ax is not None else None, edge_v, _ptr(out),
                                       _ptr(met), err, 1024):
            raise RefError(err.value.decode())
        return out, met

    def export_field(self, full, dims, t, path):
        err = C.create_string_buffer(1024)
        f = np.ascontiguousarray(full, dtype=np.float64)
        d = np.ascontiguousarray(dims, dtype=np.int32)
        if self.L.ref_sim_export_field(self.h, _ptr(f), _ptr(d, _ip), t, str(path).encode(), err,
                                       1024):
            raise RefError(err.value.decode())

    def export_profile_csv(self, rows, path):
        err = C.create_string_buffer(1024)
        r = np.ascontiguousarray(rows, dtype=np.float64)
        if self.L.ref_export_profile_csv(_ptr(r), len(r), str(path).encode(), err, 1024):
            raise RefError(err.value.decode())

    def run(self, n_steps=0):
        t = np.zeros(8)
        err = C.create_string_buffer(1024)
        if self.L.ref_sim_run(self.h, n_steps, _ptr(t), err, 1024):
            raise RefError(err.value.decode())
        return dict(time_assembly=t[0], time_loads=t[1], time_solve=t[2], cg_iterations=int(t[3]),
                    n_steps=int(t[4]), wall=t[5])


class COracle:
    """The plain-C restatement (oracle/oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.L = C.CDLL(path)
        L.or_discretize_scan.restype = C.c_int
        L.or_discretize_scan.argtypes = [_dp, C.c_int] + [C.c_double] * 10 + [_dp, C.c_int]
        L.or_superpose_batch.argtypes = [_dp, C.c_int, C.c_double, C.c_double, C.c_double, _dp,
                                         C.c_long, C.c_double, C.c_double, _dp, _dp]
        L.or_gauss_rule.argtypes = [C.c_int, _dp, _dp]
        L.or_csr_spmv.argtypes = [C.c_int, _ip, _ip, _dp, _dp, _dp]
        L.or_pcg_jacobi.restype = C.c_int
        L.or_pcg_jacobi.argtypes = [C.c_int, _ip, _ip, _dp, _dp, _dp, C.c_double, C.c_int, _ip, _dp]
        L.or_boundary_load.argtypes = [C.c_int, C.c_int, _ip, _ip, _ip, _dp, _dp, _dp, _dp, _dp,
                                       _dp, _dp, _dp, _dp, C.c_int, _dp, C.c_int, C.c_double,
                                       C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                       _dp]

    def discretize_scan(self, waypoints, *, start_time=0.0, plane_z=0.0, power, speed,
                        spot_radius, absorptivity, dt, conductivity, density, heat_capacity, **_):
        wp = np.ascontiguousarray(np.asarray(waypoints, dtype=np.float64).reshape(-1, 2))
        n = self.L.or_discretize_scan(_ptr(wp), len(wp), start_time, plane_z, power, speed,
                                      spot_radius, absorptivity, dt, conductivity, density,
                                      heat_capacity, None, 0)
        if n < 0:
            raise ValueError("invalid scan")
        out = np.zeros((n, 6))
        self.L.or_discretize_scan(_ptr(wp), len(wp), start_time, plane_z, power, speed,
                                  spot_radius, absorptivity, dt, conductivity, density,
                                  heat_capacity, _ptr(out), n)
        return out

    def superpose(self, sources, pts, t, *, conductivity, density, heat_capacity, cull=60.0,
                  grad=True, **_):
        s = np.ascontiguousarray(sources, dtype=np.float64)
        p = np.ascontiguousarray(pts, dtype=np.float64)
        n = len(p)
        val = np.zeros(n)
        g = np.zeros((n, 3)) if grad else None
        self.L.or_superpose_batch(_ptr(s), len(s), conductivity, density, heat_capacity, _ptr(p),
                                  n, t, cull, _ptr(val), _ptr(g))
        return val, g

    def gauss_rule(self, n):
        a, b = np.zeros(n), np.zeros(n)
        self.L.or_gauss_rule(n, _ptr(a), _ptr(b))
        return a, b

    def spmv(self, row_ptr, col, val, x):
        rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
        ci = np.ascontiguousarray(col, dtype=np.int32)
        v = np.ascontiguousarray(val, dtype=np.float64)
        xx = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(len(rp) - 1)
        self.L.or_csr_spmv(len(y), _ptr(rp, _ip), _ptr(ci, _ip), _ptr(v), _ptr(xx), _ptr(y))
        return y

    def pcg(self, row_ptr, col, val, b, x0, tol=1e-10, max_iter=5000):
        rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
        ci = np.ascontiguousarray(col, dtype=np.int32)
        v = np.ascontiguousarray(val, dtype=np.float64)
        bb = np.ascontiguousarray(b, dtype=np.float64)
        x = np.array(x0, dtype=np.float64)
        it = C.c_int(0)
        rel = C.c_double(0)
        rc = self.L.or_pcg_jacobi(len(bb), _ptr(rp, _ip), _ptr(ci, _ip), _ptr(v), _ptr(bb),
                                  _ptr(x), tol, max_iter, C.byref(it), C.byref(rel))
        return x, it.value, rel.value, rc

    def boundary_local(self, fs, sources, t, e0, e1, *, fine_radius, conductivity, density,
                       heat_capacity, cull=60.0, **_):
        """Local loads of face elements [e0, e1) ((e1 - e0), n_dofs) — no scatter."""
        L = self.L
        if not getattr(L, "_local_bound", False):
            L.or_boundary_local.argtypes = [C.c_int, C.c_int, _ip, _ip] + [_dp] * 9 + [
                C.c_int, _dp] + [C.c_double] * 6 + [C.c_int, C.c_int, _dp]
            L._local_bound = True
        ne, nd = fs["dofs"].shape
        arr = {k: np.ascontiguousarray(v) for k, v in fs.items()}
        s = np.ascontiguousarray(sources, dtype=np.float64)
        loc = np.zeros((max(0, e1 - e0), nd))
        L.or_boundary_local(ne, nd, _ptr(arr["nqb"], _ip), _ptr(arr["nqf"], _ip),
                            _ptr(arr["centers"]), _ptr(arr["xb"]), _ptr(arr["nb"]),
                            _ptr(arr["wb"]), _ptr(arr["Nb"]), _ptr(arr["xf"]), _ptr(arr["nf"]),
                            _ptr(arr["wf"]), _ptr(arr["Nf"]), len(s), _ptr(s), t, fine_radius,
                            cull, conductivity, density, heat_capacity, e0, e1, _ptr(loc))
        return loc

    def boundary_load(self, fs, sources, t, *, fine_radius, n_full, conductivity, density,
                      heat_capacity, cull=60.0, **_):
        """assemble_flux_load restated (face sets as exported by RefSim.face_sets)."""
        ne, nd = fs["dofs"].shape
        arr = {k: np.ascontiguousarray(v) for k, v in fs.items()}
        s = np.ascontiguousarray(sources, dtype=np.float64)
        F = np.zeros(n_full)
        self.L.or_boundary_load(ne, nd, _ptr(arr["nqb"], _ip), _ptr(arr["nqf"], _ip),
                                _ptr(arr["dofs"], _ip), _ptr(arr["centers"]),
                                _ptr(arr["xb"]), _ptr(arr["nb"]), _ptr(arr["wb"]), _ptr(arr["Nb"]),
                                _ptr(arr["xf"]), _ptr(arr["nf"]), _ptr(arr["wf"]), _ptr(arr["Nf"]),
                                len(s), _ptr(s), n_full, t, fine_radius, cull,
                                conductivity, density, heat_capacity, _ptr(F))
        return F
