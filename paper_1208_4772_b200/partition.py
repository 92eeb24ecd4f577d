"""Partitions (cube-mesh slabs; any mesh by recursive coordinate bisection)
and the per-stage halo lists.

Multi-GPU layout: rank r owns the contiguous element range of
z-cell-layers [k0, k1) (the reference's element order is k-outer,
meshgen.cpp:53-66). Ghost elements are the face neighbours owned by the
adjacent ranks; every RK stage each rank sends the 5*N_g face-trace values of
each shared face and receives the neighbour's side (NCCL send/recv over
NVLink). Both sides enumerate the shared faces in one canonical order -- sorted
by (global element id, local face) of the lower-ranked side -- so send row i of
one rank is receive row i of the other without exchanging index lists.
Per-element arithmetic does not depend on the partition, so N-rank results are
bitwise identical to the 1-rank run (tests/test_partition.py,
tests/test_gpu_partition.py).

General meshes: ``rcb_owner`` splits the elements of any
mesh by recursive coordinate bisection of their centroids (balanced element
counts, deterministic), ``mesh_part`` cuts rank r's owned elements plus their
face-neighbour ghosts out of the global mesh, and the halo lists follow the
same canonical order, so the exchange and the bitwise 1-vs-R property are
unchanged (the owned elements of a rank are no longer one contiguous range).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .mesh import Mesh, cube_mesh, slab_ranges


@dataclass
class HaloPeer:
    rank: int
    send_elem_face: np.ndarray  # [n] int32: local owned element*4 + face
    recv_elem_face: np.ndarray  # [n] int32: local ghost element*4 + face


@dataclass
class RankPart:
    rank: int
    nranks: int
    mesh: Mesh
    elem_range: tuple[int, int] | None   # global element ids [lo, hi) (slabs), else None
    peers: list[HaloPeer]
    owned: np.ndarray | None = None      # global ids of the owned elements (general partitions)


def owner_of(gids: np.ndarray, n: int, nranks: int) -> np.ndarray:
    per_layer = 6 * n * n
    bounds = np.array([lo for lo, _ in slab_ranges(n, nranks)] + [n]) * per_layer
    return np.searchsorted(bounds, gids, side="right") - 1


def _halo_peers(m: Mesh, rank: int, owner_of_gid) -> list[HaloPeer]:
    """Send/receive lists per peer rank in the canonical shared-face order:
    sorted by (global element id, local face) of the lower-ranked side."""
    K = m.n_owned
    e_idx, f_idx = np.nonzero(m.neighbor >= K)
    ghost = m.neighbor[e_idx, f_idx].astype(np.int64)
    nface = m.neighbor_face[e_idx, f_idx].astype(np.int64)
    gid_e = m.global_ids[e_idx]
    gid_g = m.global_ids[ghost]
    owner = owner_of_gid(gid_g)
    peers = []
    for s in sorted(set(owner.tolist())):
        sel = owner == s
        if rank < s:
            key = gid_e[sel] * 4 + f_idx[sel]
        else:
            key = gid_g[sel] * 4 + nface[sel]
        order = np.argsort(key, kind="stable")
        send = (e_idx[sel][order] * 4 + f_idx[sel][order]).astype(np.int32)
        recv = (ghost[sel][order] * 4 + nface[sel][order]).astype(np.int32)
        peers.append(HaloPeer(int(s), send, recv))
    return peers


def rank_part(n: int, nranks: int, rank: int, scale: float = 1.0) -> RankPart:
    """Rank r's z-slab of make_cube_mesh(n), built directly (no global mesh)."""
    k0, k1 = slab_ranges(n, nranks)[rank]
    m = cube_mesh(n, scale=scale, k_range=(k0, k1))
    peers = _halo_peers(m, rank, lambda gids: owner_of(gids, n, nranks))
    per_layer = 6 * n * n
    return RankPart(rank, nranks, m, (k0 * per_layer, k1 * per_layer), peers)


def rcb_owner(mesh: Mesh, nranks: int) -> np.ndarray:
    """Owner rank of every element: recursive coordinate bisection of the
    element centroids, each cut along the widest extent of its subset and
    placed so that the two sides get element counts proportional to their
    rank counts (ties broken by element id: deterministic)."""
    K = mesh.n_owned
    cen = mesh.vertices[mesh.tets[:K]].mean(axis=1)
    owner = np.zeros(K, np.int32)

    def split(ids, r0, nr):
        if nr == 1:
            owner[ids] = r0
            return
        nl = nr // 2
        c = cen[ids]
        ax = int(np.argmax(c.max(axis=0) - c.min(axis=0)))
        order = ids[np.lexsort((ids, c[:, ax]))]
        cut = (len(ids) * nl) // nr
        split(order[:cut], r0, nl)
        split(order[cut:], r0 + nl, nr - nl)

    split(np.arange(K), 0, nranks)
    return owner


def submesh(g: Mesh, owned: np.ndarray) -> Mesh:
    """The owned elements (global ids, kept in global order) followed by the
    ghost elements their faces reference, with local neighbour indices."""
    K = g.n_owned
    own = np.sort(np.asarray(owned, np.int64))
    is_own = np.zeros(K, bool)
    is_own[own] = True
    nb = g.neighbor[own].astype(np.int64)
    ghosts = np.unique(nb[(nb >= 0) & ~is_own[np.maximum(nb, 0)]])
    remap = np.full(K, -1, np.int64)
    remap[own] = np.arange(own.size)
    remap[ghosts] = own.size + np.arange(ghosts.size)
    neighbor = np.where(nb >= 0, remap[np.maximum(nb, 0)], -1).astype(np.int32)
    return Mesh(vertices=g.vertices, tets=np.concatenate([g.tets[own], g.tets[ghosts]]), neighbor=neighbor,
                neighbor_face=g.neighbor_face[own], perm_code=g.perm_code[own], boundary_tag=g.boundary_tag[own],
                n_owned=own.size, n_halo=ghosts.size, global_ids=np.concatenate([own, ghosts]), tags=g.tags)


def mesh_part(g: Mesh, owner: np.ndarray, rank: int) -> RankPart:
    """Rank r's part of any mesh under an owner map (e.g. rcb_owner)."""
    owned = np.nonzero(owner == rank)[0]
    m = submesh(g, owned)
    peers = _halo_peers(m, rank, lambda gids: owner[gids])
    return RankPart(rank, int(owner.max()) + 1, m, None, peers, owned=owned)
