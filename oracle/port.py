"""ORACLE TEST INFRASTRUCTURE ONLY -- ctypes binding of the plain-C
restatement ``oracle/cdg_oracle.c`` (built to oracle/_ref/libcdg_oracle.so).

This is the checker the GPU parity tests compare against; it is validated
against the real reference (oracle/_ref/libcdg_ref.so) in
tests/test_oracle_port.py (golden vectors dumped from oracle/_ref). The product never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_ref" / "libcdg_oracle.so"
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class Desc(C.Structure):
    _fields_ = [("p", C.c_int), ("np", C.c_int), ("ncub", C.c_int), ("ng", C.c_int), ("K", C.c_int),
                ("padded", C.c_int)] + [(k, _dp) for k in (
                    "icub", "ig", "dr", "ds", "dt", "fdr", "fds", "fdt", "cub_w", "face_w", "vinv",
                    "elem_nodes", "pair_scale")] + [
                ("neighbor", _ip), ("neighbor_face", _ip), ("bc", _ip), ("freestream", C.c_double * 5),
                ("period", C.c_double * 3)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            env = dict(os.environ)
            env.pop("CC", None)
            env.pop("CXX", None)
            subprocess.run(["make", "-s", "-C", str(HERE), "port"], check=True, env=env)
        L = C.CDLL(str(LIB_PATH))
        vp = C.c_void_p
        L.cdgo_level_create.argtypes = [C.POINTER(Desc), C.POINTER(vp), C.c_char_p, C.c_size_t]
        L.cdgo_level_destroy.argtypes = [vp]
        L.cdgo_level_sizes.argtypes = [vp, _ip]
        L.cdgo_level_export.argtypes = [vp, _dp, _ip]
        L.cdgo_interpolate_to_faces.argtypes = [vp, _dp, _dp]
        L.cdgo_compute_rhs.argtypes = [vp, vp, _dp, _dp, C.c_char_p, C.c_size_t]
        L.cdgo_rk_steps.argtypes = [vp, vp, C.c_double, C.c_int, _dp, _dp, _dp, _dp, C.c_char_p, C.c_size_t]
        L.cdgo_compute_timestep.argtypes = [vp, vp, _dp, _dp, _dp, C.c_char_p, C.c_size_t]
        L.cdgo_last_viscosity.argtypes = [vp, _dp, _dp]
        _lib = L
    return _lib


def _p(a):
    if a is None:
        return None
    return a.ctypes.data_as(_dp if a.dtype == np.float64 else _ip)


class OracleError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(msg)
        self.status = status


def straight_nodes(vertices, tets, colloc):
    """CurvedMesh::straight_nodes (curved_mesh.cpp:5-18): barycentric affine map."""
    v = vertices[tets]                                       # [K,4,3]
    r, s, t = colloc[:, 0], colloc[:, 1], colloc[:, 2]
    l2, l3, l4 = (1.0 + r) / 2.0, (1.0 + s) / 2.0, (1.0 + t) / 2.0
    l1 = 1.0 - l2 - l3 - l4
    return (l1[None, :, None] * v[:, None, 0] + l2[None, :, None] * v[:, None, 1]
            + l3[None, :, None] * v[:, None, 2] + l4[None, :, None] * v[:, None, 3])


class OracleLevel:
    def __init__(self, mesh, re, bc=0, freestream=None, padded=True, elem_nodes=None):
        from paper_1208_4772_b200.level import BC_KINDS  # noqa: host tables only
        K = mesh.n_owned
        self.K, self.re = K, re
        nodes = straight_nodes(mesh.vertices, mesh.tets[:K], re.colloc_nodes) if elem_nodes is None else elem_nodes
        self._keep = dict(
            icub=np.ascontiguousarray(re.interp_cub), ig=np.ascontiguousarray(re.interp_face),
            dr=np.ascontiguousarray(re.deriv_r), ds=np.ascontiguousarray(re.deriv_s),
            dt=np.ascontiguousarray(re.deriv_t), fdr=np.ascontiguousarray(re.face_deriv_r),
            fds=np.ascontiguousarray(re.face_deriv_s), fdt=np.ascontiguousarray(re.face_deriv_t),
            cub_w=np.ascontiguousarray(re.cub_weights), face_w=np.ascontiguousarray(re.face_weights),
            vinv=np.ascontiguousarray(re.vandermonde_inv), elem_nodes=np.ascontiguousarray(nodes),
        )
        v = mesh.vertices[mesh.tets[:K]]
        vol = np.einsum("ij,ij->i", np.cross(v[:, 1] - v[:, 0], v[:, 2] - v[:, 0]), v[:, 3] - v[:, 0]) / 6.0
        self._keep["pair_scale"] = np.cbrt(np.abs(vol))
        nb = np.ascontiguousarray(mesh.neighbor[:K], np.int32)
        if isinstance(bc, (int, np.integer)):
            kinds = np.full((K, 4), int(bc), np.int32)
        else:
            kinds = np.zeros((K, 4), np.int32)
            for tag_id, tag in enumerate(mesh.tags):
                val = bc[tag]
                kinds[mesh.boundary_tag[:K] == tag_id] = BC_KINDS[val] if isinstance(val, str) else val
        self._ints = dict(neighbor=nb, neighbor_face=np.ascontiguousarray(mesh.neighbor_face[:K], np.int32),
                          bc=np.ascontiguousarray(np.where(nb < 0, kinds, 0), np.int32))
        d = Desc()
        d.p, d.np, d.ncub, d.ng, d.K, d.padded = re.degree, re.n_basis, re.n_cub, re.n_face_quad, K, int(padded)
        for k, a in self._keep.items():
            setattr(d, k, _p(a))
        for k, a in self._ints.items():
            setattr(d, k, _p(a))
        fs = np.zeros(5) if freestream is None else np.asarray(freestream, float)
        for c in range(5):
            d.freestream[c] = fs[c]
        for a, L in enumerate(getattr(mesh, "period", None) or (0.0, 0.0, 0.0)):
            d.period[a] = L
        self._desc = d
        h = C.c_void_p()
        err = C.create_string_buffer(512)
        st = lib().cdgo_level_create(C.byref(d), C.byref(h), err, 512)
        if st:
            raise OracleError(st, err.value.decode())
        self.h = h
        sz = np.zeros(3, np.int32)
        lib().cdgo_level_sizes(self.h, _p(sz))
        self.block, self.trace_block = int(sz[1]), int(sz[2])

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.cdgo_level_destroy(self.h)
            self.h = None

    @property
    def store_size(self):
        return self.K * 5 * self.block

    def export(self):
        h = np.zeros(self.K)
        nm = np.zeros((self.K, 4, self.re.n_face_quad), np.int32)
        lib().cdgo_level_export(self.h, _p(h), _p(nm))
        return h, nm

    def interpolate_to_faces(self, u):
        u = np.ascontiguousarray(u, np.float64)
        t = np.zeros(self.K * 5 * self.trace_block)
        lib().cdgo_interpolate_to_faces(self.h, _p(u), _p(t))
        return t

    def compute_rhs(self, u, cfg):
        u = np.ascontiguousarray(u, np.float64)
        rhs = np.zeros(self.store_size)
        err = C.create_string_buffer(512)
        st = lib().cdgo_compute_rhs(self.h, C.addressof(cfg), _p(u), _p(rhs), err, 512)
        if st:
            raise OracleError(st, err.value.decode())
        return rhs

    def rk_steps(self, u, res, cfg, dt, nsteps=1, a=None, b=None):
        from paper_1208_4772_b200.gpu import LSRK_A, LSRK_B
        a = np.ascontiguousarray(LSRK_A if a is None else a, np.float64)
        b = np.ascontiguousarray(LSRK_B if b is None else b, np.float64)
        u = np.array(u, np.float64, copy=True)
        res = np.array(res, np.float64, copy=True)
        err = C.create_string_buffer(512)
        st = lib().cdgo_rk_steps(self.h, C.addressof(cfg), dt, nsteps, _p(a), _p(b), _p(u), _p(res), err, 512)
        if st:
            raise OracleError(st, err.value.decode())
        return u, res

    def compute_timestep(self, u, cfg, eps=None):
        u = np.ascontiguousarray(u, np.float64)
        dt = np.zeros(1)
        err = C.create_string_buffer(512)
        st = lib().cdgo_compute_timestep(self.h, C.addressof(cfg), _p(u), _p(eps), _p(dt), err, 512)
        if st:
            raise OracleError(st, err.value.decode())
        return float(dt[0])

    def last_viscosity(self, with_q=True):
        eps = np.zeros(self.K)
        q = np.zeros(3 * self.store_size) if with_q else None
        st = lib().cdgo_last_viscosity(self.h, _p(eps), _p(q))
        return eps, (q.reshape(3, -1) if (with_q and st == 0) else None)
