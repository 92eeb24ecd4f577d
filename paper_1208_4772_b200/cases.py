"""Input cases of BASELINE.json's configs that the reference does not ship
(SURVEY.md §8 row f3): the periodic isentropic vortex (config 1).

The reference solves steady problems with wall / farfield / symmetry
boundaries only (BcKind, euler.hpp:65); config 1 names "2D isentropic vortex
on a periodic square". Its 3D-tet form here: ``periodic_cube`` (cube_mesh with
every boundary face linked to its translate, mesh.cube_mesh(periodic=True))
and a z-invariant vortex advected diagonally through the x-y period. The
same RK-stage kernels run it unchanged (periodicity lives in the face
coupling only); the exact solution is the initial vortex translated by
u_inf t, which gives an accuracy check on top of the oracle parity
(tests/test_gpu_vortex.py).
"""
from __future__ import annotations

import numpy as np

from .mesh import Mesh, cube_mesh


def periodic_cube(n: int, length: float = 10.0) -> Mesh:
    """make_cube_mesh(n) scaled to [0, length]^3, periodic in x, y and z."""
    return cube_mesh(n, scale=length, periodic=True)


def element_nodes(mesh: Mesh, re) -> np.ndarray:
    """Physical collocation nodes of the owned straight elements [K, N_p, 3]
    (CurvedMesh::straight_nodes, curved_mesh.cpp:5-18)."""
    v = mesh.vertices[mesh.tets[: mesh.n_owned]]
    r = re.colloc_nodes
    l2, l3, l4 = (1.0 + r[:, 0]) / 2.0, (1.0 + r[:, 1]) / 2.0, (1.0 + r[:, 2]) / 2.0
    l1 = 1.0 - l2 - l3 - l4
    return (l1[None, :, None] * v[:, None, 0] + l2[None, :, None] * v[:, None, 1]
            + l3[None, :, None] * v[:, None, 2] + l4[None, :, None] * v[:, None, 3])


def isentropic_vortex(X: np.ndarray, t: float = 0.0, length: float = 10.0, beta: float = 5.0,
                      u_inf=(1.0, 1.0), center=(5.0, 5.0), gamma: float = 1.4) -> np.ndarray:
    """Conserved state [..., 5] of the (z-invariant) isentropic vortex at time t:
    free stream rho = p = 1, velocity (u_inf, 0), perturbation
    du = -beta/(2 pi) e^{(1-r^2)/2} (y - yc), dv = beta/(2 pi) e^{(1-r^2)/2} (x - xc),
    T = 1 - (gamma-1) beta^2 / (8 gamma pi^2) e^{1-r^2}, rho = T^{1/(gamma-1)},
    p = rho^gamma; the centre moves with u_inf (periodic images: minimum image)."""
    X = np.asarray(X, float)
    xc = np.array(center, float) + np.array(u_inf, float) * t
    dx = X[..., 0] - xc[0]
    dy = X[..., 1] - xc[1]
    dx -= length * np.round(dx / length)
    dy -= length * np.round(dy / length)
    r2 = dx * dx + dy * dy
    f = np.exp(0.5 * (1.0 - r2))
    u = u_inf[0] - beta / (2 * np.pi) * f * dy
    v = u_inf[1] + beta / (2 * np.pi) * f * dx
    T = 1.0 - (gamma - 1.0) * beta * beta / (8.0 * gamma * np.pi * np.pi) * f * f
    rho = T ** (1.0 / (gamma - 1.0))
    p = rho ** gamma
    out = np.empty(X.shape[:-1] + (5,))
    out[..., 0] = rho
    out[..., 1] = rho * u
    out[..., 2] = rho * v
    out[..., 3] = 0.0
    out[..., 4] = p / (gamma - 1.0) + 0.5 * rho * (u * u + v * v)
    return out


def vortex_store(mesh: Mesh, re, block: int, t: float = 0.0, **kw) -> np.ndarray:
    """SolutionStore raw() layout [K*5*block] of the vortex at the collocation nodes."""
    X = element_nodes(mesh, re)
    s = isentropic_vortex(X, t, **kw)                  # [K, N_p, 5]
    u = np.zeros((mesh.n_owned, 5, block))
    u[:, :, : re.n_basis] = np.transpose(s, (0, 2, 1))
    return u.reshape(-1)
