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


# ---------------------------------------------------------------------------
# Configs 2 and 3: O-grids around a cylinder and a NACA0012 section, every
# element curved (isoparametric) by the exact smooth map of the grid
# ---------------------------------------------------------------------------
def ogrid_mesh(n_xi: int, n_eta: int, n_z: int, mapping, tags=("wall", "farfield", "symmetry")):
    """Structured O-grid in parameter space (xi periodic in [0, 1), eta in
    [0, 1] from the body to the far field, zeta in [0, 1] across the span),
    each cell split into the 6 Kuhn tets of make_cube_mesh (meshgen.cpp:41-88),
    physical vertices X = mapping(xi, eta, zeta) (arrays). Returns (Mesh,
    params [K, 4, 3]): the (unwrapped) parameters of each tet's vertices, from
    which ``ogrid_nodes`` places the curved collocation nodes.
    Boundary faces: eta = 0 -> tags[0] (body), eta = 1 -> tags[1] (far field),
    zeta = 0 / 1 -> tags[2] (symmetry planes: a 2D flow in a 3D slab)."""
    from .mesh import KUHN_TETS, Mesh, _orient, connectivity
    ni, nj, nk = n_xi, n_eta + 1, n_z + 1
    vid = lambda i, j, k: ((k * nj + j) * ni + (i % ni))  # noqa: E731  (xi wraps)
    kk, jj, ii = np.meshgrid(np.arange(n_z), np.arange(n_eta), np.arange(n_xi), indexing="ij")
    kk, jj, ii = kk.ravel(), jj.ravel(), ii.ravel()
    corners = np.empty((kk.size, 8), np.int64)
    cpar = np.empty((kk.size, 8, 3))
    for b in range(8):
        di, dj, dk = b & 1, (b >> 1) & 1, (b >> 2) & 1
        corners[:, b] = vid(ii + di, jj + dj, kk + dk)
        cpar[:, b] = np.stack([(ii + di) / n_xi, (jj + dj) / n_eta, (kk + dk) / n_z], axis=1)
    tets = corners[:, KUHN_TETS].reshape(-1, 4)
    par = cpar[:, KUHN_TETS].reshape(-1, 4, 3)
    gi, gj, gk = np.meshgrid(np.arange(ni), np.arange(nj), np.arange(nk), indexing="ij")
    order = np.argsort(((gk * nj + gj) * ni + gi).ravel())
    P = np.stack([gi.ravel() / n_xi, gj.ravel() / n_eta, gk.ravel() / n_z], axis=1)[order]
    verts = np.stack(mapping(P[:, 0], P[:, 1], P[:, 2]), axis=1)
    t0 = tets.copy()
    tets = _orient(verts, tets)
    swapped = tets[:, 0] != t0[:, 0]
    par[swapped, 0], par[swapped, 1] = par[swapped, 1].copy(), par[swapped, 0].copy()
    nb, nf, pc = connectivity(tets)
    K = tets.shape[0]
    # boundary tag of each unmatched face from its vertices' parameters
    from .mesh import FACE_VERTS_ARR
    fpar = par[:, FACE_VERTS_ARR]  # [K, 4, 3 verts, 3]
    bt = np.full((K, 4), -1, np.int8)
    bnd = nb < 0
    eta, zeta = fpar[..., 1], fpar[..., 2]
    bt[bnd & np.all(eta < 1e-12, axis=2)] = 0
    bt[bnd & np.all(eta > 1 - 1e-12, axis=2)] = 1
    bt[bnd & (np.all(zeta < 1e-12, axis=2) | np.all(zeta > 1 - 1e-12, axis=2))] = 2
    if np.any(bnd & (bt < 0)):
        raise ValueError("ogrid_mesh: unclassified boundary face")
    m = Mesh(vertices=verts, tets=tets, neighbor=nb, neighbor_face=nf, perm_code=pc, boundary_tag=bt, n_owned=K,
             n_halo=0, global_ids=np.arange(K, dtype=np.int64), tags=list(tags))
    return m, par


def ogrid_nodes(params: np.ndarray, re, mapping) -> np.ndarray:
    """Curved collocation nodes [K, N_p, 3]: the grid map applied to the
    barycentric interpolation of each tet's vertex parameters (an exact
    isoparametric description of the body, continuous across faces)."""
    r = re.colloc_nodes
    lam = np.stack([1.0 - (3.0 + r.sum(axis=1)) / 2.0, (1.0 + r[:, 0]) / 2.0, (1.0 + r[:, 1]) / 2.0,
                    (1.0 + r[:, 2]) / 2.0], axis=1)  # [N_p, 4]
    q = np.einsum("jv,kvd->kjd", lam, params)
    return np.stack(mapping(q[..., 0], q[..., 1], q[..., 2]), axis=-1)


def cylinder_map(r0=0.5, r1=10.0, height=1.0):
    """BASELINE config 3: circular cylinder of radius r0, far field at r1
    (geometric radial spacing), span `height`."""
    def f(xi, eta, zeta):
        r = r0 * (r1 / r0) ** eta
        th = 2.0 * np.pi * xi
        return r * np.cos(th), r * np.sin(th), height * zeta
    return f


def naca0012_map(r_far=8.0, height=0.25, beta=3.0, t=0.12):
    """BASELINE config 2: NACA0012 section (closed trailing edge,
    y_t = 5t(0.2969 sqrt(x) - 0.1260x - 0.3516x^2 + 0.2843x^3 - 0.1036x^4)),
    xi = 0 at the trailing edge over the upper surface to the leading edge
    (xi = 1/2) and back along the lower surface (cosine clustering at both
    edges); linear blend to a far-field circle of radius r_far about the
    mid-chord, exponential clustering of eta at the wall."""
    def f(xi, eta, zeta):
        x = 0.5 * (1.0 + np.cos(2.0 * np.pi * xi))
        yt = 5.0 * t * (0.2969 * np.sqrt(np.maximum(x, 0.0)) - 0.1260 * x - 0.3516 * x ** 2 + 0.2843 * x ** 3
                        - 0.1036 * x ** 4)
        y = np.where(np.mod(xi, 1.0) <= 0.5, yt, -yt)
        th = 2.0 * np.pi * xi
        cx, cy = 0.5 + r_far * np.cos(th), r_far * np.sin(th)
        s = np.expm1(beta * eta) / np.expm1(beta)
        return x + s * (cx - x), y + s * (cy - y), height * zeta
    return f


def freestream(mach: float, alpha_deg: float = 0.0, rho: float = 1.0, p: float = 1.0, gamma: float = 1.4):
    """FreestreamConfig::state (config.cpp:12-24): flow in the x-y plane."""
    c = np.sqrt(gamma * p / rho)
    a = np.radians(alpha_deg)
    v = mach * c * np.array([np.cos(a), np.sin(a), 0.0])
    return np.array([rho, rho * v[0], rho * v[1], rho * v[2], p / (gamma - 1.0) + 0.5 * rho * v.dot(v)])


def reference_arrays(mesh) -> dict:
    """The mesh as the oracle façade's ref_mesh_from_arrays wants it."""
    e, f = np.nonzero(mesh.neighbor < 0)
    return dict(vertices=mesh.vertices, tets=mesh.tets, bf_elem=e, bf_face=f,
                bf_tag=mesh.boundary_tag[e, f].astype(np.int32), tags=mesh.tags)
