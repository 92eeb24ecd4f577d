"""ctypes binding of the C ABI (include/cdg_gpu.h) + a host-side mirror of the
reference solver interface (solver.hpp:83-116) for tests, bench and drivers.

The shared library ``libcdg_gpu.so`` is built in-tree by ``build.py`` (nvcc,
sm_100a). There is no CPU fallback: if the library is missing, or no CUDA
device is visible, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import refelem as R
from .level import LevelArrays
from .mesh import Mesh

LIB_PATH = Path(__file__).resolve().parent / "libcdg_gpu.so"

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)

# rk.hpp:13-30 (Carpenter-Kennedy 5-stage, 4th-order low-storage RK)
LSRK_A = np.array([0.0, -567301805773.0 / 1357537059087.0, -2404267990393.0 / 2016746695238.0,
                   -3550918686646.0 / 2091501179385.0, -1275806237668.0 / 842570457699.0])
LSRK_B = np.array([1432997174477.0 / 9575080441755.0, 5161836677717.0 / 13612068292357.0,
                   1720146321549.0 / 2090206949498.0, 3134564353537.0 / 4481467310338.0,
                   2277821191437.0 / 14882151754819.0])


class NumericsError(RuntimeError):
    """cdg::NumericsError (types.hpp:46-49)."""


class ConfigError(RuntimeError):
    """cdg::ConfigError (types.hpp:34-37)."""


class CudaError(RuntimeError):
    pass


class RunConfig(C.Structure):
    """cdg_gpu_run_config == RunConfig fields read by the hot path."""
    _fields_ = [("riemann", C.c_int), ("gamma", C.c_double), ("visc_enabled", C.c_int),
                ("eps0", C.c_double), ("kappa", C.c_double), ("s0_offset", C.c_double),
                ("indicator_component", C.c_int), ("jacobian_weighted", C.c_int),
                ("cfl", C.c_double)]


def run_config(riemann="llf", gamma=1.4, viscosity=None, cfl=0.5) -> RunConfig:
    if riemann not in ("llf", "hllc"):
        raise ConfigError(f"unknown Riemann solver '{riemann}' (llf|hllc)")
    v = dict(enabled=False, eps0=0.3, kappa=4.0, s0_offset=0.0, indicator_component=0,
             jacobian_weighted=False)
    v.update(viscosity or {})
    return RunConfig(1 if riemann == "hllc" else 0, gamma, int(v["enabled"]), v["eps0"], v["kappa"],
                     v["s0_offset"], v["indicator_component"], int(v["jacobian_weighted"]), cfl)


class SteadyParams(C.Structure):
    """cdg_gpu_steady_params: the RunConfig fields run_steady reads per level."""
    _fields_ = [("max_iterations", C.c_long), ("fixed_iterations", C.c_long), ("check_interval", C.c_int),
                ("residual_kind", C.c_int), ("tolerance", C.c_double), ("dt_override", C.c_double),
                ("degree", C.c_int)]


class MeshDesc(C.Structure):
    """cdg_gpu_mesh_desc: the caller's Mesh for cdg_gpu_level_create_from_mesh."""
    _fields_ = [("n_vertices", C.c_int), ("vertices", _dp), ("n_elements", C.c_int), ("n_halo", C.c_int),
                ("tets", _ip), ("neighbor", _ip), ("neighbor_face", _ip), ("face_perm", _ip), ("bc", _ip),
                ("face_nodes", _dp)]


class LevelDesc(C.Structure):
    _fields_ = [("degree", C.c_int), ("n_basis", C.c_int), ("n_cub", C.c_int), ("n_face_quad", C.c_int),
                ("n_elements", C.c_int), ("n_halo", C.c_int), ("padded", C.c_int),
                ("interp_cub", _dp), ("interp_face", _dp), ("deriv_r", _dp), ("deriv_s", _dp),
                ("deriv_t", _dp), ("cub_weights", _dp), ("face_weights", _dp), ("vandermonde_inv", _dp),
                ("metric", _dp), ("jac", _dp), ("face_normal", _dp), ("face_sjac", _dp), ("h", _dp),
                ("neighbor", _ip), ("neighbor_face", _ip), ("bc", _ip), ("node_map", _ip),
                ("face_code", _ip), ("code_node_map", _ip), ("n_codes", C.c_int),
                ("freestream", C.c_double * 5),
                ("n_curved", C.c_int), ("curved_ids", _ip), ("curved_jwr", _dp), ("curved_face", _dp),
                ("curved_minv", _dp), ("modal_cub", _dp), ("curved_jac", _dp)]


_lib = None


def use_library(path) -> None:
    """Load a different build of the C ABI (tuning experiments: build.build_variant).
    Must be called before the first call into the library."""
    global LIB_PATH
    if _lib is not None:
        raise RuntimeError("library already loaded")
    LIB_PATH = Path(path).resolve()


def lib():
    """Load libcdg_gpu.so (fails loudly: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is not built; run `python __graft_entry__.py build` "
                              "(the GPU path has no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        vp = C.c_void_p
        L.cdg_gpu_level_create.argtypes = [C.POINTER(LevelDesc), C.c_int, C.POINTER(vp), C.c_char_p, C.c_size_t]
        L.cdg_gpu_level_destroy.argtypes = [vp]
        L.cdg_gpu_level_sizes.argtypes = [vp, _ip]
        L.cdg_gpu_set_state.argtypes = [vp, _dp, _dp]
        L.cdg_gpu_get_state.argtypes = [vp, _dp, _dp]
        L.cdg_gpu_set_state_device.argtypes = [vp, C.c_void_p, C.c_void_p]
        L.cdg_gpu_device_buffers.argtypes = [vp, C.POINTER(_dp), C.POINTER(_dp), C.POINTER(_dp)]
        L.cdg_gpu_interpolate_to_faces.argtypes = [vp, _dp]
        L.cdg_gpu_compute_rhs.argtypes = [vp, C.POINTER(RunConfig), _dp, C.c_char_p, C.c_size_t]
        L.cdg_gpu_rk_steps.argtypes = [vp, C.POINTER(RunConfig), C.c_int, C.c_double, _dp, _dp, C.c_char_p,
                                       C.c_size_t]
        L.cdg_gpu_viscosity.argtypes = [vp, _dp]
        L.cdg_gpu_aux_gradient.argtypes = [vp, C.c_int, _dp]
        L.cdg_gpu_timestep.argtypes = [vp, C.POINTER(RunConfig), C.c_int, _dp, C.c_char_p, C.c_size_t]
        L.cdg_gpu_snapshot.argtypes = [vp]
        L.cdg_gpu_residual.argtypes = [vp, C.c_int, C.c_double, _dp]
        L.cdg_gpu_halo_setup.argtypes = [vp, C.c_int, _ip, C.c_int, _ip, C.c_void_p, C.c_void_p]
        L.cdg_gpu_halo_pack.argtypes = [vp]
        L.cdg_gpu_halo_unpack.argtypes = [vp]
        L.cdg_gpu_rk_stage_phase.argtypes = [vp, C.POINTER(RunConfig), C.c_int, C.c_int, C.c_double, _dp, _dp,
                                             C.c_char_p, C.c_size_t]
        L.cdg_gpu_stream.argtypes = [vp]
        L.cdg_gpu_stream.restype = vp
        L.cdg_gpu_launch_count.argtypes = [vp]
        L.cdg_gpu_launch_count.restype = C.c_longlong
        L.cdg_gpu_set_profiling.argtypes = [vp, C.c_int]
        L.cdg_gpu_set_max_ctas.argtypes = [vp, C.c_int]
        L.cdg_gpu_set_kernel_path.argtypes = [vp, C.c_int]
        L.cdg_gpu_last_profile.argtypes = [vp, _dp]
        L.cdg_gpu_version.restype = C.c_char_p
        L.cdg_gpu_measure_fp64_peak.argtypes = [C.c_int, _dp]
        L.cdg_gpu_fill_freestream.argtypes = [vp]
        L.cdg_gpu_fused_traces.argtypes = [vp]
        L.cdg_gpu_p_refine_embed.argtypes = [vp, vp, _dp]
        L.cdg_gpu_run_level.argtypes = [vp, C.POINTER(RunConfig), C.POINTER(SteadyParams), _dp, C.c_int, _ip, _ip,
                                        C.c_char_p, C.c_size_t]
        L.cdg_gpu_level_create_from_mesh.argtypes = [C.POINTER(LevelDesc), C.POINTER(MeshDesc), C.c_int,
                                                     C.POINTER(vp), C.c_char_p, C.c_size_t]
        L.cdg_gpu_rhs_kernel.argtypes = [vp]
        L.cdg_gpu_rhs_kernel.restype = C.c_char_p
        L.cdg_gpu_curved_kernel.argtypes = [vp]
        L.cdg_gpu_curved_kernel.restype = C.c_char_p
        L.cdg_gpu_hllc_fallbacks.argtypes = [vp, C.POINTER(C.c_longlong)]
        L.cdg_gpu_halo_define.argtypes = [vp, C.c_int, _ip, _ip, _ip, _ip, _ip]
        L.cdg_gpu_comm_unique_id.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t]
        L.cdg_gpu_comm_create_nccl.argtypes = [vp, C.c_char_p, C.c_int, C.c_int, C.POINTER(vp), C.c_char_p,
                                               C.c_size_t]
        L.cdg_gpu_comm_create_local.argtypes = [C.c_int, C.POINTER(vp), C.POINTER(vp), C.c_char_p, C.c_size_t]
        L.cdg_gpu_comm_destroy.argtypes = [vp]
        L.cdg_gpu_comm_rk_steps.argtypes = [vp, C.POINTER(RunConfig), C.c_int, C.c_double, _dp, _dp, C.c_char_p,
                                            C.c_size_t]
        L.cdg_gpu_comm_timestep.argtypes = [vp, C.POINTER(RunConfig), C.c_int, _dp, C.c_char_p, C.c_size_t]
        L.cdg_gpu_comm_snapshot.argtypes = [vp]
        L.cdg_gpu_comm_residual.argtypes = [vp, C.c_int, C.c_double, _dp]
        L.cdg_gpu_comm_fill_freestream.argtypes = [vp]
        L.cdg_gpu_comm_run_level.argtypes = [vp, C.POINTER(RunConfig), C.POINTER(SteadyParams), C.c_void_p,
                                             C.c_void_p, _dp, C.c_int, _ip, _ip, C.c_char_p, C.c_size_t]
        L.cdg_gpu_comm_exchange_count.argtypes = [vp]
        _lib = L
    return _lib


def _p(a):
    if a is None:
        return None
    return a.ctypes.data_as(_dp if a.dtype == np.float64 else _ip)


def _raise(status: int, msg: str):
    if status == 0:
        return
    if status == 3:
        raise NumericsError(msg)
    if status == 2:
        raise ConfigError(msg)
    if status == 4:
        raise CudaError(msg)
    raise RuntimeError(msg)


class GpuLevel:
    """One polynomial level resident on a GPU: the drop-in for
    DgLevel + RhsWorkspace + the solver kernels (solver.hpp:52-116)."""

    def __init__(self, mesh: Mesh, p: int, bc=0, freestream=None, curved_quadrature: bool = False,
                 padded: bool = True, device: int = 0, re: R.ReferenceElement | None = None,
                 curved: tuple | None = None):
        """curved = (element ids, physical collocation nodes [Kc, N_p, 3]) of the
        isoparametric elements (CurvedMesh); a mesh with curved elements uses the
        raised quadrature for every element (solver.cpp:551-557)."""
        if curved is not None and len(curved[0]):
            curved_quadrature = True
        self.re = re or R.level_reference_element(p, curved_quadrature)
        self.arrays = a = LevelArrays(mesh, self.re, bc=bc, freestream=freestream, padded=padded,
                                      curved=curved)
        re = self.re
        d = LevelDesc()
        d.degree, d.n_basis, d.n_cub, d.n_face_quad = re.degree, re.n_basis, re.n_cub, re.n_face_quad
        d.n_elements, d.n_halo, d.padded = a.K, a.n_halo, int(padded)
        t = a.tables
        d.interp_cub, d.interp_face = _p(t["interp_cub"]), _p(t["interp_face"])
        d.deriv_r, d.deriv_s, d.deriv_t = _p(t["deriv_r"]), _p(t["deriv_s"]), _p(t["deriv_t"])
        d.cub_weights, d.face_weights, d.vandermonde_inv = (_p(t["cub_weights"]), _p(t["face_weights"]),
                                                             _p(t["vandermonde_inv"]))
        d.metric, d.jac, d.face_normal, d.face_sjac, d.h = (_p(a.metric), _p(a.jac), _p(a.face_normal),
                                                            _p(a.face_sjac), _p(a.h))
        d.neighbor, d.neighbor_face, d.bc = _p(a.neighbor), _p(a.neighbor_face), _p(a.bc)
        d.node_map = None
        d.face_code, d.code_node_map, d.n_codes = _p(a.face_code), _p(a.code_node_map), a.code_node_map.shape[0]
        for c in range(5):
            d.freestream[c] = a.freestream[c]
        if a.curved_ids is not None:
            d.n_curved = len(a.curved_ids)
            d.curved_ids, d.curved_jwr = _p(a.curved_ids), _p(a.curved_jwr)
            d.curved_face, d.curved_minv = _p(a.curved_face), _p(a.curved_minv)
            d.curved_jac = _p(a.curved_jac)
        d.modal_cub = _p(t["modal_cub"])
        self._desc = d
        h = C.c_void_p()
        err = C.create_string_buffer(1024)
        st = lib().cdg_gpu_level_create(C.byref(d), device, C.byref(h), err, 1024)
        _raise(st, err.value.decode())
        self.h = h
        sz = np.zeros(8, np.int32)
        lib().cdg_gpu_level_sizes(self.h, _p(sz))
        self.K, self.n_basis, self.n_cub, self.n_face_quad = (int(x) for x in sz[:4])
        self.block, self.trace_block, self.device_block, self.n_halo = (int(x) for x in sz[4:])
        self.degree = p

    @classmethod
    def from_mesh(cls, mesh: Mesh, p: int, bc: int = 0, freestream=None, padded: bool = True, device: int = 0):
        """Straight-sided level built INSIDE the library from the mesh
        (cdg_gpu_level_create_from_mesh: affine geometry + perm-based pairing in
        C++, the scalable setup a C++ caller gets without a DgLevel)."""
        from .mesh import PERMS
        self = cls.__new__(cls)
        self.re = re = R.level_reference_element(p, False)
        K = mesh.n_owned
        t = {k: np.ascontiguousarray(getattr(re, k)) for k in
             ("interp_cub", "interp_face", "deriv_r", "deriv_s", "deriv_t", "cub_weights", "face_weights",
              "vandermonde_inv")}
        t["modal_cub"] = np.ascontiguousarray(R.modal_basis_eval(re.degree, re.cub_nodes))
        d = LevelDesc()
        d.degree, d.n_basis, d.n_cub, d.n_face_quad = re.degree, re.n_basis, re.n_cub, re.n_face_quad
        d.padded = int(padded)
        d.interp_cub, d.interp_face = _p(t["interp_cub"]), _p(t["interp_face"])
        d.deriv_r, d.deriv_s, d.deriv_t = _p(t["deriv_r"]), _p(t["deriv_s"]), _p(t["deriv_t"])
        d.cub_weights, d.face_weights, d.vandermonde_inv = (_p(t["cub_weights"]), _p(t["face_weights"]),
                                                             _p(t["vandermonde_inv"]))
        d.modal_cub = _p(t["modal_cub"])
        fs = np.zeros(5) if freestream is None else np.asarray(freestream, float)
        for c in range(5):
            d.freestream[c] = fs[c]
        nb = np.ascontiguousarray(mesh.neighbor[:K], np.int32)
        perm = np.asarray(PERMS, np.int32)[np.maximum(mesh.perm_code[:K], 0)]
        arrs = dict(vertices=np.ascontiguousarray(mesh.vertices, np.float64),
                    tets=np.ascontiguousarray(mesh.tets, np.int32), neighbor=nb,
                    neighbor_face=np.ascontiguousarray(np.maximum(mesh.neighbor_face[:K], 0), np.int32),
                    face_perm=np.ascontiguousarray(perm, np.int32),
                    bc=np.ascontiguousarray(np.where(nb < 0, int(bc), 0), np.int32),
                    face_nodes=np.ascontiguousarray(re.face_nodes[: re.n_face_quad], np.float64))
        md = MeshDesc()
        md.n_vertices, md.n_elements, md.n_halo = mesh.vertices.shape[0], K, mesh.n_halo
        for k, a in arrs.items():
            setattr(md, k, _p(a))
        h = C.c_void_p()
        err = C.create_string_buffer(1024)
        _raise(lib().cdg_gpu_level_create_from_mesh(C.byref(d), C.byref(md), device, C.byref(h), err, 1024),
               err.value.decode())
        self.h, self._keep = h, (t, arrs, d, md)
        self.arrays = None
        sz = np.zeros(8, np.int32)
        lib().cdg_gpu_level_sizes(self.h, _p(sz))
        self.K, self.n_basis, self.n_cub, self.n_face_quad = (int(x) for x in sz[:4])
        self.block, self.trace_block, self.device_block, self.n_halo = (int(x) for x in sz[4:])
        self.degree = p
        return self

    # -- lifecycle --------------------------------------------------------------
    def close(self):
        if getattr(self, "h", None):
            lib().cdg_gpu_level_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def store_size(self) -> int:
        return self.K * 5 * self.block

    def make_store(self) -> np.ndarray:
        """DgLevel::make_store (solver.cpp:181-183): zero padded store."""
        return np.zeros(self.store_size)

    # -- state ------------------------------------------------------------------
    def set_state(self, u: np.ndarray, res: np.ndarray | None = None):
        u = np.ascontiguousarray(u, np.float64)
        res = None if res is None else np.ascontiguousarray(res, np.float64)
        _raise(lib().cdg_gpu_set_state(self.h, _p(u), _p(res)), "set_state failed")

    def set_state_device(self, u_ptr: int, res_ptr: int | None = None):
        """Copy the state from device memory (e.g. a torch CUDA tensor's data_ptr())."""
        _raise(lib().cdg_gpu_set_state_device(self.h, u_ptr, res_ptr), "set_state_device failed")

    def get_state(self):
        u = np.zeros(self.store_size)
        res = np.zeros(self.store_size)
        _raise(lib().cdg_gpu_get_state(self.h, _p(u), _p(res)), "get_state failed")
        return u, res

    def device_buffers(self):
        u, r, t = _dp(), _dp(), _dp()
        lib().cdg_gpu_device_buffers(self.h, C.byref(u), C.byref(r), C.byref(t))
        return (C.cast(u, C.c_void_p).value, C.cast(r, C.c_void_p).value, C.cast(t, C.c_void_p).value)

    # -- kernels ----------------------------------------------------------------
    def interpolate_to_faces(self) -> np.ndarray:
        out = np.zeros(self.K * 5 * self.trace_block)
        _raise(lib().cdg_gpu_interpolate_to_faces(self.h, _p(out)), "interpolate_to_faces failed")
        return out

    def compute_rhs(self, cfg: RunConfig, u: np.ndarray | None = None) -> np.ndarray:
        if u is not None:
            self.set_state(u)
        out = np.zeros(self.store_size)
        err = C.create_string_buffer(1024)
        _raise(lib().cdg_gpu_compute_rhs(self.h, C.byref(cfg), _p(out), err, 1024), err.value.decode())
        return out

    def rk_steps(self, cfg: RunConfig, dt: float, nsteps: int = 1, a=LSRK_A, b=LSRK_B):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        err = C.create_string_buffer(1024)
        _raise(lib().cdg_gpu_rk_steps(self.h, C.byref(cfg), nsteps, dt, _p(a), _p(b), err, 1024),
               err.value.decode())

    def rk_step(self, u, res, cfg: RunConfig, dt: float, nsteps: int = 1):
        """rk_step adapter semantics (solver.cpp:469-492): upload, step, download."""
        self.set_state(u, res)
        self.rk_steps(cfg, dt, nsteps)
        return self.get_state()

    def viscosity(self) -> np.ndarray:
        eps = np.zeros(self.K)
        _raise(lib().cdg_gpu_viscosity(self.h, _p(eps)), "viscosity failed")
        return eps

    def aux_gradient(self, m: int) -> np.ndarray:
        q = np.zeros(self.store_size)
        _raise(lib().cdg_gpu_aux_gradient(self.h, m, _p(q)), "aux_gradient: no viscous RHS evaluated")
        return q

    def compute_timestep(self, cfg: RunConfig, use_viscosity: bool = False) -> float:
        dt = np.zeros(1)
        err = C.create_string_buffer(1024)
        _raise(lib().cdg_gpu_timestep(self.h, C.byref(cfg), int(use_viscosity), _p(dt), err, 1024),
               err.value.decode())
        return float(dt[0])

    def snapshot(self):
        _raise(lib().cdg_gpu_snapshot(self.h), "snapshot failed")

    def residual(self, dt: float, kind: str = "inf") -> float:
        out = np.zeros(1)
        _raise(lib().cdg_gpu_residual(self.h, 1 if kind == "l2" else 0, dt, _p(out)), "residual failed")
        return float(out[0])

    def rhs_kernel(self) -> str:
        """The affine RHS + update kernel this level runs (k_rhs_wa / k_rhs_row / ...)."""
        return lib().cdg_gpu_rhs_kernel(self.h).decode()

    def curved_kernel(self) -> str:
        """The curved-element RHS + update kernel ('' without curved elements)."""
        return lib().cdg_gpu_curved_kernel(self.h).decode()

    def hllc_fallbacks(self) -> int:
        """HLLC -> LLF fallbacks since creation (RhsWorkspace::hllc_fallbacks, solver.cpp:52,436)."""
        n = C.c_longlong(0)
        _raise(lib().cdg_gpu_hllc_fallbacks(self.h, C.byref(n)), "hllc_fallbacks failed")
        return int(n.value)

    def fused_traces(self) -> bool:
        return bool(lib().cdg_gpu_fused_traces(self.h))

    def launch_count(self) -> int:
        return int(lib().cdg_gpu_launch_count(self.h))

    def set_max_ctas(self, n: int):
        """Cap persistent-kernel grids at n CTAs (0: default); results are grid-independent."""
        _raise(lib().cdg_gpu_set_max_ctas(self.h, int(n)), "set_max_ctas failed")

    def set_kernel_path(self, path: str):
        """'default' (per-order compiled choice), 'generic' (CTA kernels
        everywhere) or 'traced' (default without the neighbour-state kernel:
        every stage through stored traces, bitwise equal to the split paths)."""
        code = {"default": 0, "generic": 1, "traced": 2}[path]
        _raise(lib().cdg_gpu_set_kernel_path(self.h, code), "set_kernel_path failed")

    def set_profiling(self, on: bool):
        lib().cdg_gpu_set_profiling(self.h, int(on))

    def last_profile(self):
        out = np.zeros(3)
        lib().cdg_gpu_last_profile(self.h, _p(out))
        return out

    # -- multi-GPU halo ---------------------------------------------------------
    def halo_setup(self, send_elem_face: np.ndarray, recv_elem_face: np.ndarray, send_ptr: int, recv_ptr: int):
        """Register halo rows and the caller-owned device buffers (torch tensors)."""
        s = np.ascontiguousarray(send_elem_face, np.int32)
        r = np.ascontiguousarray(recv_elem_face, np.int32)
        _raise(lib().cdg_gpu_halo_setup(self.h, len(s), _p(s), len(r), _p(r), send_ptr, recv_ptr),
               "halo_setup failed")

    def halo_define(self, peers):
        """Register this shard's halo rows peer by peer (partition.HaloPeer list);
        the library owns the transfer buffers (multi-rank driver, GpuComm)."""
        ranks = np.array([pe.rank for pe in peers], np.int32)
        sc = np.array([len(pe.send_elem_face) for pe in peers], np.int32)
        rc = np.array([len(pe.recv_elem_face) for pe in peers], np.int32)
        s = np.ascontiguousarray(np.concatenate([pe.send_elem_face for pe in peers] or [np.zeros(0)]), np.int32)
        r = np.ascontiguousarray(np.concatenate([pe.recv_elem_face for pe in peers] or [np.zeros(0)]), np.int32)
        _raise(lib().cdg_gpu_halo_define(self.h, len(peers), _p(ranks), _p(sc), _p(rc), _p(s), _p(r)),
               "halo_define failed")

    def stage_phase(self, cfg: RunConfig, stage: int, phase: int, dt: float, a=LSRK_A, b=LSRK_B):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        err = C.create_string_buffer(1024)
        _raise(lib().cdg_gpu_rk_stage_phase(self.h, C.byref(cfg), stage, phase, dt, _p(a), _p(b), err, 1024),
               err.value.decode())

    def stream(self) -> int:
        return int(lib().cdg_gpu_stream(self.h) or 0)

    # -- device-resident run_steady (solver.cpp:594-676) -------------------------
    def fill_freestream(self):
        _raise(lib().cdg_gpu_fill_freestream(self.h), "fill_freestream failed")

    def p_refine_embed(self, src: "GpuLevel"):
        """self.u = p_refine_embed(src.u) (solver.cpp:528-549)."""
        e = embed_matrix(src.re, self.re)
        _raise(lib().cdg_gpu_p_refine_embed(self.h, src.h, _p(e)), "p_refine_embed failed")

    def run_level(self, cfg: RunConfig, params: SteadyParams, max_rows: int = 100000):
        rows = np.zeros((max_rows, 3))
        n = np.zeros(1, np.int32)
        conv = np.zeros(1, np.int32)
        err = C.create_string_buffer(1024)
        st = lib().cdg_gpu_run_level(self.h, C.byref(cfg), C.byref(params), _p(rows), max_rows, _p(n), _p(conv),
                                     err, 1024)
        _raise(st, err.value.decode())
        return rows[: min(int(n[0]), max_rows)], bool(conv[0])


def _torch_nccl_first():
    """The library resolves libnccl.so.2 at run time (dlopen): load torch (and
    the NCCL it is built against) first, so that one NCCL serves both -- the
    soname would otherwise bind torch to whichever NCCL was loaded first."""
    import torch  # noqa: F401


class GpuComm:
    """Multi-rank driver over shards (GpuLevel with ghost elements + halo_define):
    rk_steps / timestep / residual / run_level over every rank (cdg_gpu_comm_*).

    GpuComm.local(levels): one process drives every shard (one GPU or several,
    peer copies over NVLink); GpuComm.nccl(level, uid, rank, nranks): one
    process per GPU, NCCL inside the library (uid from unique_id() on rank 0,
    broadcast by the caller)."""

    def __init__(self, h, levels):
        self.h = h
        self.levels = levels  # keep the shards alive

    @staticmethod
    def unique_id() -> bytes:
        _torch_nccl_first()
        buf = C.create_string_buffer(128)
        err = C.create_string_buffer(1024)
        _raise(lib().cdg_gpu_comm_unique_id(buf, err, 1024), err.value.decode())
        return buf.raw

    @classmethod
    def local(cls, levels):
        arr = (C.c_void_p * len(levels))(*[lv.h.value for lv in levels])
        h = C.c_void_p()
        err = C.create_string_buffer(1024)
        _raise(lib().cdg_gpu_comm_create_local(len(levels), arr, C.byref(h), err, 1024), err.value.decode())
        return cls(h, list(levels))

    @classmethod
    def nccl(cls, level, uid: bytes, rank: int, nranks: int):
        _torch_nccl_first()
        h = C.c_void_p()
        err = C.create_string_buffer(1024)
        _raise(lib().cdg_gpu_comm_create_nccl(level.h, uid, rank, nranks, C.byref(h), err, 1024),
               err.value.decode())
        return cls(h, [level])

    def close(self):
        if getattr(self, "h", None):
            lib().cdg_gpu_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def rk_steps(self, cfg: RunConfig, dt: float, nsteps: int = 1, a=LSRK_A, b=LSRK_B):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        err = C.create_string_buffer(1024)
        _raise(lib().cdg_gpu_comm_rk_steps(self.h, C.byref(cfg), nsteps, dt, _p(a), _p(b), err, 1024),
               err.value.decode())

    def compute_timestep(self, cfg: RunConfig, use_viscosity: bool = False) -> float:
        dt = np.zeros(1)
        err = C.create_string_buffer(1024)
        _raise(lib().cdg_gpu_comm_timestep(self.h, C.byref(cfg), int(use_viscosity), _p(dt), err, 1024),
               err.value.decode())
        return float(dt[0])

    def snapshot(self):
        _raise(lib().cdg_gpu_comm_snapshot(self.h), "snapshot failed")

    def residual(self, dt: float, kind: str = "inf") -> float:
        out = np.zeros(1)
        _raise(lib().cdg_gpu_comm_residual(self.h, 1 if kind == "l2" else 0, dt, _p(out)), "residual failed")
        return float(out[0])

    def fill_freestream(self):
        _raise(lib().cdg_gpu_comm_fill_freestream(self.h), "fill_freestream failed")

    def run_level(self, cfg: RunConfig, params: SteadyParams, max_rows: int = 100000):
        rows = np.zeros((max_rows, 3))
        n = np.zeros(1, np.int32)
        conv = np.zeros(1, np.int32)
        err = C.create_string_buffer(1024)
        st = lib().cdg_gpu_comm_run_level(self.h, C.byref(cfg), C.byref(params), None, None, _p(rows), max_rows,
                                          _p(n), _p(conv), err, 1024)
        _raise(st, err.value.decode())
        return rows[: min(int(n[0]), max_rows)], bool(conv[0])

    def exchange_count(self) -> int:
        return int(lib().cdg_gpu_comm_exchange_count(self.h))


def embed_matrix(re_from: R.ReferenceElement, re_to: R.ReferenceElement) -> np.ndarray:
    """p_refine_embed's matrix V_to[:, :np_from] V_from^-1 (solver.cpp:536-537)."""
    if re_to.degree < re_from.degree:
        raise ConfigError("p_refine_embed: target degree must not decrease")
    return np.ascontiguousarray(re_to.vandermonde[:, : re_from.n_basis] @ re_from.vandermonde_inv)


def run_steady(make_level, p_schedule, cfg: RunConfig, final_tolerance=1e-9, intermediate_tolerance=1e-4,
               max_iterations=20000, fixed_iterations=(), check_interval=1000, residual="inf", dt_override=0.0,
               on_row=None):
    """run_steady (solver.cpp:594-676) with every level device-resident.

    make_level(p) -> GpuLevel builds the level of degree p (host setup, as the
    reference's DgLevel). Returns (rows [(level, iteration, dt, residual,
    wall_seconds)], converged, final_degree, final level)."""
    import time
    if not p_schedule:
        raise ConfigError("run_steady: empty p-schedule")
    if any(b <= a for a, b in zip(p_schedule, p_schedule[1:])):
        raise ConfigError("run_steady: p-schedule must be strictly increasing")
    t0 = time.perf_counter()
    rows, converged, prev = [], False, None
    for li, p in enumerate(p_schedule):
        lv = make_level(p)
        if prev is None:
            lv.fill_freestream()
        else:
            lv.p_refine_embed(prev)
            prev.close()
        last = li + 1 == len(p_schedule)
        fixed = fixed_iterations[li] if li < len(fixed_iterations) else -1
        sp = SteadyParams(max_iterations, fixed, check_interval, 1 if residual == "l2" else 0,
                          final_tolerance if last else intermediate_tolerance, dt_override, p)
        lrows, conv = lv.run_level(cfg, sp)
        wall = time.perf_counter() - t0
        for it, dt, r in lrows:
            row = (p, int(it), float(dt), float(r), wall)
            rows.append(row)
            if on_row:
                on_row(row)
        if last:
            converged = conv
            if fixed > 0 and rows:
                converged = rows[-1][3] < final_tolerance
        prev = lv
    return rows, converged, p_schedule[-1], prev


def measure_fp64_peak(device: int = 0):
    """(DMMA m16n8k4, DFMA, DMMA m16n8k8, DMMA m16n8k16) TFLOP/s measured on the device."""
    out = np.zeros(4)
    _raise(lib().cdg_gpu_measure_fp64_peak(device, _p(out)), "fp64 peak measurement failed")
    return tuple(float(x) for x in out)


def freestream_store(level: GpuLevel, u_inf) -> np.ndarray:
    """freestream_store (solver.cpp:559-568)."""
    u = np.zeros((level.K, 5, level.block))
    u[:, :, : level.n_basis] = np.asarray(u_inf, float)[None, :, None]
    return u.reshape(-1)


def random_admissible_store(level: GpuLevel, seed: int = 42) -> np.ndarray:
    """The bench.cpp:22-40 recipe (+/-0.05 jitter around rho=1, v=(0.3,0,0),
    p=1) with numpy's generator (same distribution, different stream)."""
    rng = np.random.default_rng(seed)
    K, npb = level.K, level.n_basis
    j = rng.uniform(-0.05, 0.05, size=(K, npb, 6))
    rho = 1.0 + j[..., 0]
    vx, vy, vz = 0.3 + j[..., 1], j[..., 2], j[..., 3]
    p = 1.0 + j[..., 4]
    u = np.zeros((K, 5, level.block))
    u[:, 0, :npb] = rho
    u[:, 1, :npb] = rho * vx
    u[:, 2, :npb] = rho * vy
    u[:, 3, :npb] = rho * vz
    u[:, 4, :npb] = p / 0.4 + 0.5 * rho * (vx * vx + vy * vy + vz * vz)
    return u.reshape(-1)


def make_state(rho, v, p, gamma=1.4):
    v = np.asarray(v, float)
    return np.array([rho, rho * v[0], rho * v[1], rho * v[2], p / (gamma - 1.0) + 0.5 * rho * v.dot(v)])
