"""Level setup for the GPU path: affine geometry, face coupling, node maps.

Host-side restatement of the parts of ``DgLevel`` (solver.cpp:97-179) the
kernels need, in compact per-element form (SURVEY.md §7 "Memory layout at
scale": 26 doubles per affine element instead of ~125 KB of per-element
operator matrices):

* ``affine_geometry`` -- compute_mapping (operators.cpp:32-121) for a straight
  tet: dx/dr = (v1-v0, v2-v0, v3-v0)/2, J = det, dr_m/dx_i = inverse, face
  normal/sjac from the face-chart tangents (operators.cpp:98-118),
  h = 6V/A (operators.hpp:37).
* ``perm_node_maps`` -- the face-node pairing. The reference pairs nodes by
  nearest physical point (solver.cpp:144-172); on conforming faces with the
  symmetric face rules (quadrature.hpp:33-36) that pairing is the barycentric
  permutation induced by FaceLink.perm (mesh.hpp:23-27), so one table per
  vertex permutation replaces the per-face node_map (verified against the
  reference's node_map in tests/test_mesh_level.py and tests/test_gpu_curved.py).
"""
from __future__ import annotations

import numpy as np

from .mesh import PERMS, Mesh
from .refelem import FACE_VERTS, TET_VERTS, ReferenceElement, modal_basis_eval, pad16, tri_quadrature

BC_KINDS = {"slip_wall": 0, "wall": 0, "farfield": 1, "symmetry": 2}


def affine_geometry(vertices: np.ndarray, tets: np.ndarray, re: ReferenceElement):
    v = vertices[tets]                                   # [K,4,3]
    fwd = np.stack([(v[:, 1] - v[:, 0]) * 0.5, (v[:, 2] - v[:, 0]) * 0.5, (v[:, 3] - v[:, 0]) * 0.5],
                   axis=2)                               # f[i][m] = dx_i/dr_m
    jac = np.linalg.det(fwd)
    if np.any(jac <= 1e-14):
        e = int(np.argmax(jac <= 1e-14))
        raise ArithmeticError(f"inverted element {e}: mapping Jacobian {jac[e]} at quadrature node 0")
    inv = np.linalg.inv(fwd)                             # inv[m][i] = dr_m/dx_i
    metric = inv.reshape(-1, 9)
    normals = np.empty((tets.shape[0], 4, 3))
    sjac = np.empty((tets.shape[0], 4))
    for f, (a, b, c) in enumerate(FACE_VERTS):
        ra = 0.5 * (TET_VERTS[b] - TET_VERTS[a])
        rb = 0.5 * (TET_VERTS[c] - TET_VERTS[a])
        xa = fwd @ ra
        xb = fwd @ rb
        nraw = np.cross(xa, xb)
        s = np.linalg.norm(nraw, axis=1)
        sjac[:, f] = s
        normals[:, f] = nraw / s[:, None]
    volume = jac * re.cub_weights.sum()
    area = (sjac * re.face_weights.sum()).sum(axis=1)
    return metric, jac, normals, sjac, 6.0 * volume / area


def curved_geometry(nodes: np.ndarray, re: ReferenceElement):
    """compute_mapping + build_operators (operators.cpp:32-167) for curved
    elements from their physical collocation nodes [Kc, N_p, 3]:
    per-cubature-node J*W*dr_m/dx_d [Kc, N_cub, 9], per-face-node
    (n, sjac*w) [Kc, 4N_g, 4], M_e^-1 [Kc, N_p, N_p] and h = 6V/A [Kc]."""
    X = np.asarray(nodes, float)
    ng = re.n_face_quad
    K = X.shape[0]
    # Every per-element quantity is computed by the same batched (stacked)
    # routine whatever the batch: an element's geometry does not depend on
    # which or how many elements are built with it (a shard's curved elements
    # get bit-identical tables to the whole mesh's; tests/test_gpu_comm.py).

    def fwd_at(dr, ds, dt):  # F[i][m] = dx_i/dr_m at the n points, [Kc, n] each
        dx = [np.matmul(d, X) for d in (dr, ds, dt)]  # stacked [Kc, n, 3] per m
        return [[np.ascontiguousarray(dx[m][..., i]) for m in range(3)] for i in range(3)]

    F = fwd_at(re.deriv_r, re.deriv_s, re.deriv_t)
    # 3x3 determinant and inverse by cofactors, inv[m][i] = dr_m/dx_i
    inv = [[None] * 3 for _ in range(3)]
    inv[0][0] = F[1][1] * F[2][2] - F[1][2] * F[2][1]
    inv[1][0] = F[1][2] * F[2][0] - F[1][0] * F[2][2]
    inv[2][0] = F[1][0] * F[2][1] - F[1][1] * F[2][0]
    jac = F[0][0] * inv[0][0] + F[0][1] * inv[1][0] + F[0][2] * inv[2][0]
    if np.any(jac <= 1e-14):
        k, q = np.argwhere(jac <= 1e-14)[0]
        raise ArithmeticError(f"inverted curved element (list index {k}): mapping Jacobian {jac[k, q]} "
                              f"at quadrature node {q}")
    inv[0][1] = F[0][2] * F[2][1] - F[0][1] * F[2][2]
    inv[1][1] = F[0][0] * F[2][2] - F[0][2] * F[2][0]
    inv[2][1] = F[0][1] * F[2][0] - F[0][0] * F[2][1]
    inv[0][2] = F[0][1] * F[1][2] - F[0][2] * F[1][1]
    inv[1][2] = F[0][2] * F[1][0] - F[0][0] * F[1][2]
    inv[2][2] = F[0][0] * F[1][1] - F[0][1] * F[1][0]
    jw = jac * re.cub_weights[None, :]
    # J W dr_m/dx_i = W x cofactor (the 1/J of the inverse cancels)
    jwr = np.stack([inv[m][i] * re.cub_weights[None, :] for m in range(3) for i in range(3)], axis=2)
    FF = fwd_at(re.face_deriv_r, re.face_deriv_s, re.face_deriv_t)  # [i][m] -> [Kc, 4 N_g]
    face = np.empty((K, 4 * ng, 4))
    area = np.zeros(K)
    for fi, (a, b, c) in enumerate(FACE_VERTS):
        ra = 0.5 * (TET_VERTS[b] - TET_VERTS[a])
        rb = 0.5 * (TET_VERTS[c] - TET_VERTS[a])
        sl = slice(fi * ng, (fi + 1) * ng)
        xa = [sum(FF[i][m][:, sl] * ra[m] for m in range(3)) for i in range(3)]
        xb = [sum(FF[i][m][:, sl] * rb[m] for m in range(3)) for i in range(3)]
        n0 = xa[1] * xb[2] - xa[2] * xb[1]
        n1 = xa[2] * xb[0] - xa[0] * xb[2]
        n2 = xa[0] * xb[1] - xa[1] * xb[0]
        s = np.sqrt(n0 * n0 + n1 * n1 + n2 * n2)
        face[:, sl, 0], face[:, sl, 1], face[:, sl, 2] = n0 / s, n1 / s, n2 / s
        face[:, sl, 3] = s * re.face_weights[None, :]
        area += (s * re.face_weights[None, :]).sum(axis=1)
    # M_e = I_cub^T diag(J W) I_cub, stacked per element (chunks bound the temporary)
    npb = re.n_basis
    minv = np.empty((K, npb, npb))
    it = re.interp_cub.T[None]
    for c0 in range(0, K, 8192):
        sl = slice(c0, min(K, c0 + 8192))
        minv[sl] = np.linalg.inv(np.matmul(it * jw[sl, None, :], re.interp_cub))
    h = 6.0 * jw.sum(axis=1) / area
    return np.ascontiguousarray(jwr), np.ascontiguousarray(face), np.ascontiguousarray(minv), h, \
        np.ascontiguousarray(jac)


def perm_node_maps(re: ReferenceElement) -> np.ndarray:
    """[6][N_g] node maps, one per face-vertex permutation (PERMS order)."""
    ng = re.n_face_quad
    # barycentric coordinates of the 2D rule on (A, B, C): (1-u-v, u, v)
    a, b = _face_rule_ab(re)
    u, w = (a + 1.0) / 2.0, (b + 1.0) / 2.0
    lam = np.stack([1.0 - u - w, u, w], axis=1)          # [ng,3]
    maps = np.empty((len(PERMS), ng), np.int32)
    for code, p in enumerate(PERMS):
        theirs = np.empty_like(lam)
        for i in range(3):
            theirs[:, p[i]] = lam[:, i]
        d = np.linalg.norm(theirs[:, None, :] - lam[None, :, :], axis=2)
        maps[code] = np.argmin(d, axis=1)
        if np.max(np.min(d, axis=1)) > 1e-10:
            raise ArithmeticError("face rule is not invariant under the vertex permutation")
    return maps


def _face_rule_ab(re: ReferenceElement):
    # recover (a, b) of face 0's chart from the embedded nodes: x = A + u(B-A) + v(C-A)
    A, B, C = (TET_VERTS[i] for i in FACE_VERTS[0])
    x = re.face_nodes[: re.n_face_quad]
    m = np.stack([B - A, C - A], axis=1)
    uv, *_ = np.linalg.lstsq(m, (x - A).T, rcond=None)
    return 2.0 * uv[0] - 1.0, 2.0 * uv[1] - 1.0


class LevelArrays:
    """All host arrays behind one cdg_gpu_level_desc (kept alive by the owner)."""

    def __init__(self, mesh: Mesh, re: ReferenceElement, bc: dict | int = 0, freestream=None,
                 padded: bool = True, curved: tuple | None = None):
        """curved = (ids [Kc], nodes [Kc, N_p, 3]) for isoparametric elements."""
        K = mesh.n_owned
        self.re = re
        self.K = K
        self.n_halo = mesh.n_halo
        self.padded = padded
        self.block = pad16(re.n_basis) if padded else re.n_basis
        self.trace_block = pad16(4 * re.n_face_quad) if padded else 4 * re.n_face_quad
        metric, jac, normals, sjac, h = affine_geometry(mesh.vertices, mesh.tets[:K], re)
        self.metric = np.ascontiguousarray(metric)
        self.jac = np.ascontiguousarray(jac)
        self.face_normal = np.ascontiguousarray(normals)
        self.face_sjac = np.ascontiguousarray(sjac)
        self.h = np.ascontiguousarray(h)
        self.neighbor = np.ascontiguousarray(mesh.neighbor[:K], np.int32)
        self.neighbor_face = np.ascontiguousarray(np.maximum(mesh.neighbor_face[:K], 0), np.int32)
        self.face_code = np.ascontiguousarray(np.maximum(mesh.perm_code[:K], 0), np.int32)
        self.code_node_map = np.ascontiguousarray(perm_node_maps(re))
        if isinstance(bc, (int, np.integer)):
            kinds = np.full(K * 4, int(bc), np.int32).reshape(K, 4)
        else:
            kinds = np.zeros((K, 4), np.int32)
            for tag_id, tag in enumerate(mesh.tags):
                sel = mesh.boundary_tag[:K] == tag_id
                if tag not in bc:
                    if sel.any():  # validate_boundary_tags (cli_ops.cpp:80-91)
                        raise ValueError(f"boundary tag '{tag}' has no boundary condition")
                    continue
                kinds[sel] = BC_KINDS[bc[tag]] if isinstance(bc[tag], str) else bc[tag]
        self.bc = np.ascontiguousarray(np.where(self.neighbor < 0, kinds, 0), np.int32)
        self.freestream = np.zeros(5) if freestream is None else np.asarray(freestream, float)
        self.curved_ids = None
        if curved is not None and len(curved[0]):
            ids = np.ascontiguousarray(curved[0], np.int32)
            self.curved_ids = ids
            self.curved_jwr, self.curved_face, self.curved_minv, hc, self.curved_jac = curved_geometry(curved[1], re)
            self.h[ids] = hc
        self.tables = {k: np.ascontiguousarray(getattr(re, k)) for k in
                       ("interp_cub", "interp_face", "deriv_r", "deriv_s", "deriv_t", "cub_weights",
                        "face_weights", "vandermonde_inv")}
        # modal basis at the cubature nodes (refelem.hpp:21), J-weighted indicator
        self.tables["modal_cub"] = np.ascontiguousarray(modal_basis_eval(re.degree, re.cub_nodes))
