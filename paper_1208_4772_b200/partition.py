"""Slab partition of the cube mesh and the per-stage halo lists.

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
    elem_range: tuple[int, int]   # global element ids [lo, hi)
    peers: list[HaloPeer]


def owner_of(gids: np.ndarray, n: int, nranks: int) -> np.ndarray:
    per_layer = 6 * n * n
    bounds = np.array([lo for lo, _ in slab_ranges(n, nranks)] + [n]) * per_layer
    return np.searchsorted(bounds, gids, side="right") - 1


def rank_part(n: int, nranks: int, rank: int, scale: float = 1.0) -> RankPart:
    k0, k1 = slab_ranges(n, nranks)[rank]
    m = cube_mesh(n, scale=scale, k_range=(k0, k1))
    K = m.n_owned
    e_idx, f_idx = np.nonzero(m.neighbor >= K)
    ghost = m.neighbor[e_idx, f_idx].astype(np.int64)
    nface = m.neighbor_face[e_idx, f_idx].astype(np.int64)
    gid_e = m.global_ids[e_idx]
    gid_g = m.global_ids[ghost]
    owner = owner_of(gid_g, n, nranks)
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
    per_layer = 6 * n * n
    return RankPart(rank, nranks, m, (k0 * per_layer, k1 * per_layer), peers)
