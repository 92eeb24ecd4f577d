"""Tetrahedral meshes and face connectivity (host setup, numpy).

Scalable replacement for the reference's mesh generators and
``build_connectivity`` on the synthetic workloads: the
reference keeps per-face ``std::map`` lookups and ~140 KB of per-element
operator tables, which cannot reach the 4M-element configuration; here
everything is vectorised and O(K log K).

* ``cube_mesh`` -- ``make_cube_mesh`` (meshgen.cpp:41-88): (n+1)^3 lattice,
  vertex id (k(n+1)+j)(n+1)+i, 6 Kuhn tets per cell around the main
  diagonal, element order (k, j, i, tet), orientation fixed by swapping
  vertices 0/1. ``cube_mesh(n, k_range=...)`` builds one z-slab of cells
  (multi-GPU partition) with its halo.
* ``single_tet`` / ``two_tets`` -- meshgen.cpp:90-110.
* ``connectivity`` -- build_connectivity (mesh.cpp:26-84): faces matched by
  sorted vertex triple; FaceLink.perm = position of my face vertex i in the
  neighbour's face (mesh.hpp:23-27).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .refelem import FACE_VERTS

# meshgen.cpp:14-15
KUHN_TETS = np.array([[0, 1, 3, 7], [0, 3, 2, 7], [0, 2, 6, 7], [0, 6, 4, 7], [0, 4, 5, 7], [0, 5, 1, 7]])
FACE_VERTS_ARR = np.array(FACE_VERTS)
PERMS = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]
PERM_INDEX = {p: i for i, p in enumerate(PERMS)}


@dataclass
class Mesh:
    vertices: np.ndarray            # [nv,3]
    tets: np.ndarray                # [K,4] int64 (owned elements first)
    neighbor: np.ndarray = None     # [K,4] int32, -1 boundary
    neighbor_face: np.ndarray = None
    perm_code: np.ndarray = None    # [K,4] index into PERMS (-1 boundary)
    boundary_tag: np.ndarray = None  # [K,4] int8: -1 interior, 0 "wall"
    n_owned: int = 0                # K (rows that get a RHS)
    n_halo: int = 0                 # ghost elements appended after the owned ones
    global_ids: np.ndarray = None   # [K+halo] global element ids
    tags: list = field(default_factory=lambda: ["wall"])
    period: tuple | None = None     # box lengths of a periodic mesh (faces wrap around)

    @property
    def n_elements(self) -> int:
        return self.n_owned


def signed_volumes(vertices, tets):
    """Mesh::signed_volume (mesh.cpp:23-26), vectorised."""
    v = vertices[tets]
    return np.einsum("ij,ij->i", np.cross(v[:, 1] - v[:, 0], v[:, 2] - v[:, 0]), v[:, 3] - v[:, 0]) / 6.0


def _orient(vertices, tets):
    neg = signed_volumes(vertices, tets) < 0.0
    tets[neg, 0], tets[neg, 1] = tets[neg, 1].copy(), tets[neg, 0].copy()
    return tets


def _cube_cells(n, k0, k1):
    """Element vertex ids for cells k in [k0,k1) in reference order."""
    kk, jj, ii = np.meshgrid(np.arange(k0, k1), np.arange(n), np.arange(n), indexing="ij")
    kk, jj, ii = kk.ravel(), jj.ravel(), ii.ravel()
    corners = np.empty((kk.size, 8), np.int64)
    for b in range(8):
        corners[:, b] = ((kk + ((b >> 2) & 1)) * (n + 1) + (jj + ((b >> 1) & 1))) * (n + 1) + (ii + (b & 1))
    return corners[:, KUHN_TETS].reshape(-1, 4)


def connectivity(tets: np.ndarray, n_owned: int | None = None):
    """Face matching by sorted vertex triples (mesh.cpp:26-84).

    Returns neighbor, neighbor_face, perm_code for every element row of
    ``tets``; faces seen once are boundary faces (-1)."""
    K = tets.shape[0]
    fv = tets[:, FACE_VERTS_ARR]                      # [K,4,3]
    key = np.sort(fv, axis=2).reshape(-1, 3)
    order = np.lexsort((key[:, 2], key[:, 1], key[:, 0]))
    ks = key[order]
    same = np.all(ks[1:] == ks[:-1], axis=1)
    if np.any(same[1:] & same[:-1]):
        raise ValueError("nonconforming mesh: face shared by >2 tets")
    a = order[:-1][same]
    b = order[1:][same]
    neighbor = np.full(K * 4, -1, np.int64)
    nface = np.full(K * 4, -1, np.int64)
    neighbor[a], nface[a] = b // 4, b % 4
    neighbor[b], nface[b] = a // 4, a % 4
    perm = np.full(K * 4, -1, np.int64)
    fvf = fv.reshape(-1, 3)
    for x, y in ((a, b), (b, a)):
        ida, idb = fvf[x], fvf[y]
        # perm[i] = j with idb[j] == ida[i]
        p = np.argmax(ida[:, :, None] == idb[:, None, :], axis=2)
        perm[x] = _perm_codes(p)
    return (neighbor.reshape(K, 4).astype(np.int32), nface.reshape(K, 4).astype(np.int32),
            perm.reshape(K, 4).astype(np.int32))


def _perm_codes(p):
    code = p[:, 0] * 9 + p[:, 1] * 3 + p[:, 2]
    lut = np.full(27, -1, np.int64)
    for i, q in enumerate(PERMS):
        lut[q[0] * 9 + q[1] * 3 + q[2]] = i
    out = lut[code]
    if np.any(out < 0):
        raise ValueError("degenerate face permutation")
    return out


def cube_mesh(n: int, scale: float = 1.0, k_range: tuple[int, int] | None = None,
              periodic: bool = False) -> Mesh:
    """make_cube_mesh(n, "wall") (meshgen.cpp:41-88), optionally one z-slab.

    ``periodic=True``: the same elements with every boundary face linked to its
    translate on the opposite side of the box (no boundary faces; BASELINE
    config 1's periodic domain). The Kuhn split is translation invariant, so
    opposite boundary faces are congruent triangles and the face links (and
    their vertex permutations) come from matching vertex ids modulo n.

    With ``k_range=(k0,k1)`` the mesh holds the owned elements of cells
    k0..k1-1 followed by the ghost elements of the neighbouring cell layers
    that share a face with them (their global ids in ``global_ids``)."""
    verts = None
    if k_range is None:
        k0, k1 = 0, n
    else:
        k0, k1 = k_range
    g0, g1 = max(k0 - 1, 0), min(k1 + 1, n)
    tets_all = _cube_cells(n, g0, g1)
    # vertex coordinates from ids (lattice), scaled
    vid = np.arange((n + 1) ** 3, dtype=np.int64) if (n + 1) ** 3 <= 3_000_000 else None
    if vid is None:
        # only the vertices that are referenced
        used, inv = np.unique(tets_all, return_inverse=True)
        tets_all = inv.reshape(-1, 4)
        vid = used
    i = vid % (n + 1)
    j = (vid // (n + 1)) % (n + 1)
    k = vid // ((n + 1) ** 2)
    verts = np.stack([i / n, j / n, k / n], axis=1) * scale
    tets_all = _orient(verts, tets_all)
    if periodic:
        if k_range is not None or n < 3:
            raise ValueError("periodic cube meshes: whole mesh, n >= 3")
        vi = vid[tets_all]
        canon = (vi % (n + 1)) % n + n * (((vi // (n + 1)) % (n + 1)) % n + n * ((vi // (n + 1) ** 2) % n))
        nb, nf, pc = connectivity(canon)
        assert np.all(nb >= 0)
        K = tets_all.shape[0]
        return Mesh(vertices=verts, tets=tets_all, neighbor=nb, neighbor_face=nf, perm_code=pc,
                    boundary_tag=np.full((K, 4), -1, np.int8), n_owned=K, n_halo=0,
                    global_ids=np.arange(K, dtype=np.int64), tags=[], period=(scale, scale, scale))
    per_layer = 6 * n * n
    first = (k0 - g0) * per_layer
    owned = slice(first, first + (k1 - k0) * per_layer)
    gid_all = np.arange(g0 * per_layer, g1 * per_layer, dtype=np.int64)
    nb, nf, pc = connectivity(tets_all)
    own_idx = np.arange(owned.start, owned.stop)
    nb_o = nb[own_idx]
    # ghosts: non-owned elements referenced by owned faces
    is_ghost_ref = (nb_o >= 0) & ((nb_o < owned.start) | (nb_o >= owned.stop))
    ghosts = np.unique(nb_o[is_ghost_ref])
    remap = np.full(tets_all.shape[0], -1, np.int64)
    remap[own_idx] = np.arange(own_idx.size)
    remap[ghosts] = own_idx.size + np.arange(ghosts.size)
    neighbor = np.where(nb_o >= 0, remap[np.maximum(nb_o, 0)], -1).astype(np.int32)
    tets = np.concatenate([tets_all[own_idx], tets_all[ghosts]])
    bt = np.where(nb_o < 0, 0, -1).astype(np.int8)
    return Mesh(vertices=verts, tets=tets, neighbor=neighbor, neighbor_face=nf[own_idx],
                perm_code=pc[own_idx], boundary_tag=bt, n_owned=own_idx.size, n_halo=ghosts.size,
                global_ids=np.concatenate([gid_all[own_idx], gid_all[ghosts]]))


def _small_mesh(verts, tets) -> Mesh:
    verts = np.asarray(verts, float)
    tets = _orient(verts, np.asarray(tets, np.int64))
    nb, nf, pc = connectivity(tets)
    return Mesh(vertices=verts, tets=tets, neighbor=nb, neighbor_face=nf, perm_code=pc,
                boundary_tag=np.where(nb < 0, 0, -1).astype(np.int8), n_owned=tets.shape[0],
                global_ids=np.arange(tets.shape[0]))


def single_tet() -> Mesh:
    """make_single_tet (meshgen.cpp:90-98)."""
    return _small_mesh([[-1, -1, -1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1]], [[0, 1, 2, 3]])


def two_tets() -> Mesh:
    """make_two_tets (meshgen.cpp:100-110)."""
    return _small_mesh([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 1, 1]], [[0, 1, 2, 3], [1, 2, 3, 4]])


def from_arrays(vertices, tets, neighbor, neighbor_face, perm_code, boundary_tag) -> Mesh:
    """Wrap externally built connectivity (e.g. exported from the reference)."""
    K = tets.shape[0]
    return Mesh(vertices=np.asarray(vertices, float), tets=np.asarray(tets, np.int64),
                neighbor=np.asarray(neighbor, np.int32), neighbor_face=np.asarray(neighbor_face, np.int32),
                perm_code=np.asarray(perm_code, np.int32), boundary_tag=np.asarray(boundary_tag, np.int8),
                n_owned=K, global_ids=np.arange(K))


def slab_ranges(n: int, nranks: int):
    """Contiguous z-slabs of cells (the reference's element order is k-outer,
    meshgen.cpp:53-66, so slabs are contiguous element ranges)."""
    bounds = [round(r * n / nranks) for r in range(nranks + 1)]
    return [(bounds[r], bounds[r + 1]) for r in range(nranks)]


def warped_nodes(mesh: Mesh, re, amp: float = 0.02, ids=None) -> np.ndarray:
    """Physical collocation nodes [len(ids), N_p, 3] of the owned elements `ids`
    (default: all) under the smooth global map x -> x + amp sin(2 pi y) sin(2 pi z)
    e_x + (cyclic): continuous across faces, so the face pairing is unchanged.
    The synthetic curved (isoparametric) workload of the bench and of the
    partitioned curved tests (every element it lists is a CurvedMesh element,
    curved_mesh.hpp:14-51)."""
    ids = np.arange(mesh.n_owned) if ids is None else np.asarray(ids)
    lam = (re.colloc_nodes + 1.0) / 2.0
    bary = np.concatenate([1.0 - lam.sum(axis=1, keepdims=True), lam], axis=1)  # [N_p, 4]
    X = np.einsum("jv,kvd->kjd", bary, mesh.vertices[mesh.tets[ids]])
    x, y, z = X[..., 0].copy(), X[..., 1].copy(), X[..., 2].copy()
    t = 2.0 * np.pi
    X[..., 0] = x + amp * np.sin(t * y) * np.sin(t * z)
    X[..., 1] = y + amp * np.sin(t * z) * np.sin(t * x)
    X[..., 2] = z + amp * np.sin(t * x) * np.sin(t * y)
    return X
