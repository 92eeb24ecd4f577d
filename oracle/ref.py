"""ORACLE TEST INFRASTRUCTURE ONLY -- ctypes binding of oracle/_ref/libcdg_ref.so.

The library is the UNMODIFIED reference (``/root/reference/proj/core/src``)
compiled in place against the in-repo Eigen/doctest API shims plus the
``extern "C"`` façade ``oracle/ref_capi.cpp``. Only tests/, the graft smoke
check and bench.py's CPU-baseline leg may import this module; the product
package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_ref" / "libcdg_ref.so"
# the same sources built with BASELINE.md §3's flags (-O3 -march=native): the
# CPU baseline / reference arm of bench.py; the bitwise-pinned build above is
# the checker everywhere else
PERF_LIB_PATH = HERE / "_ref" / "perf" / "libcdg_ref_perf.so"


def use_perf_build() -> bool:
    """Bind to the -O3 -march=native build (before the first call). True when
    it exists and this CPU has the AVX-512 it was compiled for."""
    global LIB_PATH
    if _lib is not None or not PERF_LIB_PATH.exists():
        return False
    try:
        flags = Path("/proc/cpuinfo").read_text()
    except OSError:
        return False
    if "avx512f" not in flags or "amx_tile" not in flags:
        return False
    LIB_PATH = PERF_LIB_PATH
    return True


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class RunCfg(C.Structure):
    """Mirrors ``ref_run_cfg`` (oracle/ref_capi.cpp) and ``cdg_gpu_run_config``."""
    _fields_ = [("riemann", C.c_int), ("gamma", C.c_double), ("visc_enabled", C.c_int),
                ("eps0", C.c_double), ("kappa", C.c_double), ("s0_offset", C.c_double),
                ("indicator_component", C.c_int), ("jacobian_weighted", C.c_int),
                ("cfl", C.c_double)]


def make_cfg(riemann="llf", gamma=1.4, viscosity=None, cfl=0.5) -> RunCfg:
    v = dict(enabled=False, eps0=0.3, kappa=4.0, s0_offset=0.0, indicator_component=0,
             jacobian_weighted=False)
    v.update(viscosity or {})
    return RunCfg(1 if riemann == "hllc" else 0, gamma, int(v["enabled"]), v["eps0"], v["kappa"],
                  v["s0_offset"], v["indicator_component"], int(v["jacobian_weighted"]), cfl)


def available() -> bool:
    return LIB_PATH.exists()


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise FileNotFoundError(f"{LIB_PATH} not built (make -C oracle ref)")
        L = C.CDLL(str(LIB_PATH))
        L.ref_mesh_cube.restype = C.c_void_p
        L.ref_mesh_cube.argtypes = [C.c_int, C.c_double]
        L.ref_mesh_single_tet.restype = C.c_void_p
        L.ref_mesh_two_tets.restype = C.c_void_p
        L.ref_mesh_sphere_shell.restype = C.c_void_p
        L.ref_mesh_sphere_shell.argtypes = [C.c_double, C.c_double, C.c_int, C.c_int]
        L.ref_mesh_free.argtypes = [C.c_void_p]
        L.ref_mesh_from_arrays.restype = C.c_void_p
        L.ref_mesh_from_arrays.argtypes = [C.c_int, _dp, C.c_int, _ip, C.c_int, _ip, _ip, _ip, C.c_char_p, C.c_char_p,
                                           C.c_size_t]
        L.ref_mesh_set_curved.argtypes = [C.c_void_p, C.c_int, C.c_int, _ip, _dp, C.c_char_p, C.c_size_t]
        L.ref_mesh_sphere_curved.restype = C.c_void_p
        L.ref_mesh_sphere_curved.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_size_t]
        L.ref_level_nodes.argtypes = [C.c_void_p, _dp, _ip]
        L.ref_mesh_sizes.argtypes = [C.c_void_p, _ip]
        L.ref_mesh_export.argtypes = [C.c_void_p, _dp, _ip, _ip, _ip, _ip, _ip]
        L.ref_level_create.restype = C.c_void_p
        L.ref_level_create.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.c_char_p, C.c_size_t]
        L.ref_level_free.argtypes = [C.c_void_p]
        L.ref_level_make_periodic.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_double, C.c_char_p,
                                              C.c_size_t]
        L.ref_level_sizes.argtypes = [C.c_void_p, _ip]
        L.ref_level_geometry.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp, _dp, _ip, _ip, _ip, _ip]
        L.ref_level_operators.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, _dp]
        L.ref_random_admissible_store.argtypes = [C.c_void_p, C.c_uint, _dp]
        L.ref_compute_rhs.argtypes = [C.c_void_p, C.POINTER(RunCfg), _dp, _dp, _dp, C.c_char_p, C.c_size_t]
        L.ref_interpolate_to_faces.argtypes = [C.c_void_p, _dp, _dp]
        L.ref_rk_steps.argtypes = [C.c_void_p, C.POINTER(RunCfg), _dp, C.c_double, C.c_int, _dp, _dp,
                                   C.c_char_p, C.c_size_t]
        L.ref_rk_steps_timed.argtypes = [C.c_void_p, C.POINTER(RunCfg), _dp, C.c_double, C.c_int, _dp, _dp, _dp,
                                         C.c_char_p, C.c_size_t]
        L.ref_last_viscosity.argtypes = [C.c_void_p, _dp, _dp]
        L.ref_compute_timestep.argtypes = [C.c_void_p, C.POINTER(RunCfg), _dp, _dp, _dp, C.c_char_p,
                                           C.c_size_t]
        L.ref_refelem_sizes.argtypes = [C.c_int, C.c_int, C.c_int, _ip]
        L.ref_refelem_tables.argtypes = [C.c_int, C.c_int, C.c_int] + [_dp] * 12
        L.ref_num_threads.argtypes = [C.c_int]
        L.ref_run_steady.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(RunCfg), _ip, C.c_int,
                                     C.POINTER(C.c_long), C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                     C.c_int, C.c_double, _dp, _dp, C.c_int, _ip, _ip, _ip, _dp, C.c_long,
                                     C.c_char_p, C.c_size_t]
        _lib = L
    return _lib


def _p(a):
    if a is None:
        return None
    return a.ctypes.data_as(_dp if a.dtype == np.float64 else _ip)


class RefError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(msg)
        self.status = status


def num_threads(n=0) -> int:
    return lib().ref_num_threads(n)


def refelem_tables(p, cub_override=0, face_override=0) -> dict:
    L = lib()
    sz = np.zeros(4, np.int32)
    if L.ref_refelem_sizes(p, cub_override, face_override, _p(sz)) != 0:
        raise RefError(2, f"bad degree {p}")
    n_p, ncub, ng = int(sz[0]), int(sz[1]), int(sz[2])
    out = dict(colloc_nodes=np.zeros((n_p, 3)), cub_nodes=np.zeros((ncub, 3)), cub_weights=np.zeros(ncub),
               face_nodes=np.zeros((4 * ng, 3)), face_weights=np.zeros(ng),
               vandermonde=np.zeros((n_p, n_p)), vandermonde_inv=np.zeros((n_p, n_p)),
               interp_cub=np.zeros((ncub, n_p)), interp_face=np.zeros((4 * ng, n_p)),
               deriv_r=np.zeros((ncub, n_p)), deriv_s=np.zeros((ncub, n_p)), deriv_t=np.zeros((ncub, n_p)))
    L.ref_refelem_tables(p, cub_override, face_override, *[_p(out[k]) for k in out])
    return out


class Mesh:
    def __init__(self, kind="cube", n=2, scale=1.0, sphere=(1.0, 8.0, 2, 5), arrays=None):
        """arrays (kind "arrays"): dict(vertices, tets, bf_elem, bf_face, bf_tag, tags) -- any
        mesh through the reference's build_connectivity (cases.py generators)."""
        L = lib()
        if kind == "arrays":
            a = arrays
            v = np.ascontiguousarray(a["vertices"], np.float64)
            t = np.ascontiguousarray(a["tets"], np.int32)
            be, bfc, bt = (np.ascontiguousarray(a[k], np.int32) for k in ("bf_elem", "bf_face", "bf_tag"))
            err = C.create_string_buffer(512)
            self.h = L.ref_mesh_from_arrays(len(v), _p(v), len(t), _p(t), len(be), _p(be), _p(bfc), _p(bt),
                                            ",".join(a["tags"]).encode(), err, 512)
            if not self.h:
                raise RefError(3, err.value.decode())
        elif kind == "cube":
            self.h = L.ref_mesh_cube(n, scale)
        elif kind == "single_tet":
            self.h = L.ref_mesh_single_tet()
        elif kind == "two_tets":
            self.h = L.ref_mesh_two_tets()
        elif kind == "sphere":
            self.h = L.ref_mesh_sphere_shell(*sphere)
        elif kind == "sphere_curved":
            # sphere=(subdiv, layers, p_curve, p_fem)
            err = C.create_string_buffer(512)
            self.h = L.ref_mesh_sphere_curved(*sphere, err, 512)
            if not self.h:
                raise RefError(3, err.value.decode())
        else:
            raise ValueError(kind)
        sz = np.zeros(3, np.int32)
        L.ref_mesh_sizes(self.h, _p(sz))
        self.n_vertices, self.n_elements = int(sz[0]), int(sz[1])

    def set_curved(self, degree: int, ids, nodes):
        """CurvedMesh of `degree` with elements ids curved to nodes [n][N_p][3]."""
        ids = np.ascontiguousarray(ids, np.int32)
        x = np.ascontiguousarray(nodes, np.float64)
        err = C.create_string_buffer(512)
        if lib().ref_mesh_set_curved(self.h, degree, len(ids), _p(ids), _p(x), err, 512):
            raise RefError(1, err.value.decode())

    def export(self) -> dict:
        nv, ne = self.n_vertices, self.n_elements
        out = dict(vertices=np.zeros((nv, 3)), tets=np.zeros((ne, 4), np.int32),
                   neighbor=np.zeros((ne, 4), np.int32), neighbor_face=np.zeros((ne, 4), np.int32),
                   perm=np.zeros((ne, 4), np.int32), bnd_tag=np.zeros((ne, 4), np.int32))
        lib().ref_mesh_export(self.h, *[_p(out[k]) for k in out])
        return out

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_mesh_free(self.h)
            self.h = None


def run_steady(mesh, cfg: RunCfg, freestream, p_schedule, fixed=(), final_tol=1e-9, inter_tol=1e-4,
               max_iters=20000, check_interval=1000, residual="inf", dt_override=0.0, bc_wall=0, bc_far=1,
               u_cap=None):
    """The reference's run_steady (solver.cpp:594-676) on `mesh` (Mesh handle).
    Returns (rows [n][5] = level, iteration, dt, residual, wall_s; converged;
    final_degree; solution raw store)."""
    ps = np.ascontiguousarray(p_schedule, np.int32)
    fx = (C.c_long * max(1, len(fixed)))(*fixed)
    rows = np.zeros((4096, 5))
    n = np.zeros(1, np.int32)
    conv = np.zeros(1, np.int32)
    fdeg = np.zeros(1, np.int32)
    ex = mesh.export()
    K = len(ex["tets"])
    pmax = int(max(p_schedule))
    cap = u_cap or K * 5 * 176 * (pmax + 1)
    u = np.zeros(cap)
    fs = np.ascontiguousarray(freestream, np.float64)
    err = C.create_string_buffer(512)
    st = lib().ref_run_steady(mesh.h, bc_wall, bc_far, C.byref(cfg), _p(ps), len(ps), fx, len(fixed), final_tol,
                              inter_tol, max_iters, check_interval, 1 if residual == "l2" else 0, dt_override,
                              _p(fs), _p(rows), rows.shape[0], _p(n), _p(conv), _p(fdeg), _p(u), cap, err, 512)
    if st:
        raise RefError(st, err.value.decode())
    return rows[: int(n[0])], bool(conv[0]), int(fdeg[0]), u


class Level:
    """A reference DgLevel + RhsWorkspace on a reference mesh."""

    def __init__(self, mesh: Mesh, p: int, bc_wall=0, bc_far=1, padded=True, curved_quadrature=True):
        L = lib()
        err = C.create_string_buffer(512)
        self.mesh = mesh
        self.h = L.ref_level_create(mesh.h, p, bc_wall, bc_far, int(padded), int(curved_quadrature), err, 512)
        if not self.h:
            raise RefError(3, err.value.decode())
        sz = np.zeros(7, np.int32)
        L.ref_level_sizes(self.h, _p(sz))
        (self.K, self.n_basis, self.n_cub, self.n_face_quad, self.block, self.trace_block,
         self.degree) = (int(x) for x in sz)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_level_free(self.h)
            self.h = None

    @property
    def store_size(self):
        return self.K * 5 * self.block

    def geometry(self) -> dict:
        K, ncub, nf, ng = self.K, self.n_cub, 4 * self.n_face_quad, self.n_face_quad
        g = dict(cub_dr=np.zeros((K, ncub, 9)), cub_jac=np.zeros((K, ncub)), face_normal=np.zeros((K, nf, 3)),
                 face_sjac=np.zeros((K, nf)), face_phys=np.zeros((K, nf, 3)), h=np.zeros(K),
                 neighbor=np.zeros((K, 4), np.int32), neighbor_face=np.zeros((K, 4), np.int32),
                 bc=np.zeros((K, 4), np.int32), node_map=np.zeros((K, 4, ng), np.int32))
        lib().ref_level_geometry(self.h, *[_p(g[k]) for k in g])
        return g

    def nodes(self):
        x = np.zeros((self.K, self.n_basis, 3))
        cv = np.zeros(self.K, np.int32)
        lib().ref_level_nodes(self.h, _p(x), _p(cv))
        return x, cv.astype(bool)

    def operators(self, e: int) -> dict:
        np_, ncub, nf = self.n_basis, self.n_cub, 4 * self.n_face_quad
        o = dict(S=np.zeros((3, np_, ncub)), face_mass=np.zeros((np_, nf)), mass=np.zeros((np_, np_)),
                 mass_chol=np.zeros((np_, np_)))
        lib().ref_level_operators(self.h, e, *[_p(o[k]) for k in o])
        return o

    def random_admissible_store(self, seed=42) -> np.ndarray:
        u = np.zeros(self.store_size)
        lib().ref_random_admissible_store(self.h, seed, _p(u))
        return u

    def compute_rhs(self, u, cfg: RunCfg, freestream) -> np.ndarray:
        u = np.ascontiguousarray(u, np.float64)
        fs = np.ascontiguousarray(freestream, np.float64)
        rhs = np.zeros(self.store_size)
        err = C.create_string_buffer(512)
        st = lib().ref_compute_rhs(self.h, C.byref(cfg), _p(fs), _p(u), _p(rhs), err, 512)
        if st:
            raise RefError(st, err.value.decode())
        return rhs

    def interpolate_to_faces(self, u) -> np.ndarray:
        u = np.ascontiguousarray(u, np.float64)
        t = np.zeros(self.K * 5 * self.trace_block)
        lib().ref_interpolate_to_faces(self.h, _p(u), _p(t))
        return t

    def rk_steps(self, u, res, cfg: RunCfg, freestream, dt, nsteps=1):
        u = np.array(u, np.float64, copy=True)
        res = np.array(res, np.float64, copy=True)
        fs = np.ascontiguousarray(freestream, np.float64)
        err = C.create_string_buffer(512)
        st = lib().ref_rk_steps(self.h, C.byref(cfg), _p(fs), dt, nsteps, _p(u), _p(res), err, 512)
        if st:
            raise RefError(st, err.value.decode())
        return u, res

    def make_periodic(self, period):
        """Link the cube level's boundary faces to their translates (ref_periodic.cpp)."""
        err = C.create_string_buffer(512)
        if lib().ref_level_make_periodic(self.h, *[float(x) for x in period], err, 512):
            raise RefError(1, err.value.decode())

    def rk_steps_timed(self, u, res, cfg: RunCfg, freestream, dt, nsteps=1):
        """nsteps x rk_step with only the step loop timed (store copies outside);
        returns (u, res, seconds per step)."""
        u = np.array(u, np.float64, copy=True)
        res = np.array(res, np.float64, copy=True)
        fs = np.ascontiguousarray(freestream, np.float64)
        secs = np.zeros(nsteps)
        err = C.create_string_buffer(512)
        st = lib().ref_rk_steps_timed(self.h, C.byref(cfg), _p(fs), dt, nsteps, _p(u), _p(res), _p(secs), err, 512)
        if st:
            raise RefError(st, err.value.decode())
        return u, res, secs

    def last_viscosity(self, with_q=True):
        eps = np.zeros(self.K)
        q = np.zeros(3 * self.store_size) if with_q else None
        st = lib().ref_last_viscosity(self.h, _p(eps), _p(q))
        if with_q and st != 0:
            q = None
        return eps, (q.reshape(3, -1) if q is not None else None)

    def compute_timestep(self, u, cfg: RunCfg, eps=None) -> float:
        u = np.ascontiguousarray(u, np.float64)
        dt = np.zeros(1)
        err = C.create_string_buffer(512)
        st = lib().ref_compute_timestep(self.h, C.byref(cfg), _p(u), _p(eps), _p(dt), err, 512)
        if st:
            raise RefError(st, err.value.decode())
        return float(dt[0])
