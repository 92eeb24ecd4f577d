"""Reference-tetrahedron tables for the RKDG hot path (host setup, numpy).

This is the host-side table builder that feeds ``cdg_gpu_level_create``: the
degree-p nodal/modal basis, cubature, face quadrature and the interpolation /
differentiation operators. It restates the reference's algorithms so that the
GPU path consumes the same tables the reference's ``DgLevel`` would
(parity is pinned against the reference's own table dump in
tests/test_refelem_tables.py and tests/golden/refelem_p*.npz):

* orthonormal Jacobi recurrence / Gauss-Jacobi (Golub-Welsch) / GLL nodes
  -- ``proj/core/src/jacobi.cpp:15-100``
* Grundmann-Moller tet/tri rules, Dunavant orbits with refitted weights
  -- ``proj/core/src/quadrature.cpp:44-244``
* collapsed-coordinate Dubiner basis + gradients, warp & blend nodes,
  face embedding, ``ReferenceElement`` tables
  -- ``proj/core/src/refelem.cpp:15-358``
* curved quadrature strengths -- ``proj/core/include/cdg/refelem.hpp:118-119``

All arrays are float64, row-major, rows = evaluation points.
"""
from __future__ import annotations

import functools
import math
from dataclasses import dataclass

import numpy as np

TET_VERTS = np.array([[-1.0, -1.0, -1.0], [1.0, -1.0, -1.0], [-1.0, 1.0, -1.0], [-1.0, -1.0, 1.0]])
TRI_VERTS = np.array([[-1.0, -1.0], [1.0, -1.0], [-1.0, 1.0]])
# refelem.cpp:291-299: faces t=-1, s=-1, r+s+t=-1, r=-1 ordered outward.
FACE_VERTS = ((0, 2, 1), (0, 1, 3), (1, 2, 3), (0, 3, 2))


def basis_count(p: int) -> int:
    """refelem.hpp:14."""
    return (p + 1) * (p + 2) * (p + 3) // 6


def curved_volume_strength(p: int) -> int:
    """refelem.hpp:118."""
    return max(2 * p + 1, 3 * p - 3)


def curved_face_strength(p: int) -> int:
    """refelem.hpp:119."""
    return max(2 * p, 3 * p - 2)


def pad16(n: int) -> int:
    """padded.hpp:12."""
    return 16 * ((n + 15) // 16)


# ---------------------------------------------------------------------------
# jacobi.cpp
# ---------------------------------------------------------------------------

def jacobi_p(x, alpha: float, beta: float, n: int):
    """Orthonormal Jacobi polynomial (jacobi.cpp:15-44), vectorised over x."""
    x = np.asarray(x, dtype=np.float64)
    ab = alpha + beta
    gamma0 = math.exp((ab + 1.0) * math.log(2.0) + math.lgamma(alpha + 1.0)
                      + math.lgamma(beta + 1.0) - math.lgamma(ab + 1.0)) / (ab + 1.0)
    p_prev = np.full_like(x, 1.0 / math.sqrt(gamma0))
    if n == 0:
        return p_prev
    gamma1 = (alpha + 1.0) * (beta + 1.0) / (ab + 3.0) * gamma0
    p_cur = ((ab + 2.0) * x / 2.0 + (alpha - beta) / 2.0) / math.sqrt(gamma1)
    if n == 1:
        return p_cur
    a_old = 2.0 / (2.0 + ab) * math.sqrt((alpha + 1.0) * (beta + 1.0) / (ab + 3.0))
    for i in range(1, n):
        h1 = 2.0 * i + ab
        a_new = 2.0 / (h1 + 2.0) * math.sqrt((i + 1.0) * (i + 1.0 + ab) * (i + 1.0 + alpha)
                                             * (i + 1.0 + beta) / ((h1 + 1.0) * (h1 + 3.0)))
        b_new = -(alpha * alpha - beta * beta) / (h1 * (h1 + 2.0))
        p_next = (-a_old * p_prev + (x - b_new) * p_cur) / a_new
        p_prev, p_cur, a_old = p_cur, p_next, a_new
    return p_cur


def grad_jacobi_p(x, alpha: float, beta: float, n: int):
    """jacobi.cpp:46-49."""
    x = np.asarray(x, dtype=np.float64)
    if n == 0:
        return np.zeros_like(x)
    return math.sqrt(n * (n + alpha + beta + 1.0)) * jacobi_p(x, alpha + 1.0, beta + 1.0, n - 1)


def gauss_jacobi(n: int, alpha: float, beta: float):
    """Golub-Welsch Gauss-Jacobi rule (jacobi.cpp:51-89)."""
    if n < 1:
        raise ValueError("gauss_jacobi: n must be >= 1")
    ab = alpha + beta
    mu0 = math.exp((ab + 1.0) * math.log(2.0) + math.lgamma(alpha + 1.0)
                   + math.lgamma(beta + 1.0) - math.lgamma(ab + 2.0))
    if n == 1:
        return np.array([-(alpha - beta) / (ab + 2.0)]), np.array([mu0])
    j = np.zeros((n, n))
    for i in range(n):
        h1 = 2.0 * i + ab
        j[i, i] = (beta - alpha) / (ab + 2.0) if i == 0 else -(alpha * alpha - beta * beta) / (h1 * (h1 + 2.0))
        if i < n - 1:
            off = 2.0 / (h1 + 2.0) * math.sqrt((i + 1.0) * (i + 1.0 + ab) * (i + 1.0 + alpha)
                                               * (i + 1.0 + beta) / ((h1 + 1.0) * (h1 + 3.0)))
            j[i, i + 1] = j[i + 1, i] = off
    evals, evecs = np.linalg.eigh(j)
    return evals, mu0 * evecs[0, :] ** 2


def gauss_lobatto(n: int) -> np.ndarray:
    """GLL nodes, n+1 points (jacobi.cpp:91-100)."""
    x = np.empty(n + 1)
    x[0], x[-1] = -1.0, 1.0
    if n >= 2:
        x[1:-1] = gauss_jacobi(n - 1, 1.0, 1.0)[0]
    return x


# ---------------------------------------------------------------------------
# quadrature.cpp
# ---------------------------------------------------------------------------

def _compositions(total: int, length: int):
    """enumerate_compositions order (quadrature.cpp:26-39)."""
    if length == 1:
        yield (total,)
        return
    for v in range(total + 1):
        for rest in _compositions(total - v, length - 1):
            yield (v,) + rest


def _grundmann_moller(s: int, d: int):
    """Barycentric points + weights on the unit d-simplex (quadrature.cpp:44-63)."""
    bary, weights = [], []
    deg = 2 * s + 1
    for i in range(s + 1):
        denom = d + deg - 2.0 * i
        w = (1.0 if i % 2 == 0 else -1.0) * 2.0 ** (-2.0 * s) * denom ** deg / (
            math.factorial(i) * math.factorial(d + deg - i))
        for k in _compositions(s - i, d + 1):
            bary.append([(2.0 * kj + 1.0) / denom for kj in k])
            weights.append(w)
    return np.array(bary), np.array(weights)


def tet_cubature(strength: int):
    """Grundmann-Moller tet rule of at least `strength` (quadrature.cpp:149-169).

    Returns (nodes[n,3], weights[n]) on the reference tet (volume 4/3)."""
    s = max(0, strength // 2)
    bary, w = _grundmann_moller(s, 3)
    nodes = bary @ TET_VERTS
    return nodes, w * (4.0 / 3.0) * 6.0


def _tri_monomial_integral(p: int, q: int) -> float:
    """quadrature.cpp:68-78."""
    total = 0.0
    for i in range(p + 1):
        for j in range(q + 1):
            sign = 1.0 if ((p - i) + (q - j)) % 2 == 0 else -1.0
            total += (sign * math.comb(p, i) * math.comb(q, j) * 2.0 ** (i + j)
                      * math.factorial(i) * math.factorial(j) / math.factorial(i + j + 2))
    return 4.0 * total


_TRI_ORBITS = {
    # quadrature.cpp:110-145 (Dunavant orbit positions; weights refitted)
    0: [(1, 0.0, 0.0)], 1: [(1, 0.0, 0.0)],
    2: [(3, 2.0 / 3.0, 1.0 / 6.0)],
    3: [(3, 0.108103018168070, 0.445948490915965), (3, 0.816847572980459, 0.091576213509771)],
    5: [(1, 0.0, 0.0), (3, 0.059715871789770, 0.470142064105115),
        (3, 0.797426985353087, 0.101286507323456)],
    6: [(3, 0.501426509658179, 0.249286745170910), (3, 0.873821971016996, 0.063089014491502),
        (6, 0.053145049844816, 0.310352451033785)],
    7: [(1, 0.0, 0.0), (3, 0.081414823414554, 0.459292588292723),
        (3, 0.658861384496480, 0.170569307751760), (3, 0.898905543365938, 0.050547228317031),
        (6, 0.008394777409958, 0.263112829634638)],
}
_TRI_ORBITS[4] = _TRI_ORBITS[3]
_TRI_ORBITS[8] = _TRI_ORBITS[7]


def _orbit_points(kind: int, a: float, b: float):
    """quadrature.cpp:85-105."""
    if kind == 1:
        return [(1.0 / 3.0, 1.0 / 3.0, 1.0 / 3.0)]
    if kind == 3:
        c = 1.0 - 2.0 * b
        return [(c, b, b), (b, c, b), (b, b, c)]
    c = 1.0 - a - b
    return [(a, b, c), (a, c, b), (b, a, c), (b, c, a), (c, a, b), (c, b, a)]


def tri_quadrature(strength: int):
    """Symmetric triangle rule on {-1<=a,b; a+b<=0}, weights sum 2
    (quadrature.cpp:171-244). Returns (a[n], b[n], w[n])."""
    if strength not in _TRI_ORBITS:
        s = max(0, strength // 2)
        bary, w = _grundmann_moller(s, 2)
        ab = bary @ TRI_VERTS
        return ab[:, 0].copy(), ab[:, 1].copy(), w * 2.0 * 2.0
    orbits = _TRI_ORBITS[strength]
    orbit_ab = [np.array(_orbit_points(*o)) @ TRI_VERTS for o in orbits]
    monomials = [(p, total - p) for total in range(strength + 1) for p in range(total + 1)]
    amat = np.array([[np.sum(ab[:, 0] ** p * ab[:, 1] ** q) for ab in orbit_ab] for p, q in monomials])
    rhs = np.array([_tri_monomial_integral(p, q) for p, q in monomials])
    w, *_ = np.linalg.lstsq(amat, rhs, rcond=None)
    if np.max(np.abs(amat @ w - rhs)) > 1e-12:
        raise ArithmeticError(f"tri_quadrature: tabulated rule fails moment equations, strength {strength}")
    pts = np.concatenate(orbit_ab)
    weights = np.concatenate([np.full(len(ab), w[o]) for o, ab in enumerate(orbit_ab)])
    return pts[:, 0].copy(), pts[:, 1].copy(), weights


# ---------------------------------------------------------------------------
# refelem.cpp
# ---------------------------------------------------------------------------

def _rst_to_abc(pts):
    """refelem.cpp:17-22."""
    r, s, t = pts[:, 0], pts[:, 1], pts[:, 2]
    st = s + t
    a = np.where(np.abs(st) > 1e-14, 2.0 * (1.0 + r) / np.where(np.abs(st) > 1e-14, -st, 1.0) - 1.0, -1.0)
    omt = 1.0 - t
    b = np.where(np.abs(omt) > 1e-14, 2.0 * (1.0 + s) / np.where(np.abs(omt) > 1e-14, omt, 1.0) - 1.0, -1.0)
    return a, b, t.copy()


def modal_index_order(p: int):
    """Degree-graded (i,j,k) ordering (refelem.cpp:26-33)."""
    return [(i, j, total - i - j) for total in range(p + 1) for i in range(total + 1)
            for j in range(total - i + 1)]


def modal_basis_eval(p: int, pts, tol: float = 1e-12) -> np.ndarray:
    """Orthonormal Dubiner basis at points (refelem.cpp:35-41,148-160)."""
    pts = np.asarray(pts, dtype=np.float64).reshape(-1, 3)
    bad = ((pts[:, 0] < -1 - tol) | (pts[:, 1] < -1 - tol) | (pts[:, 2] < -1 - tol)
           | (pts.sum(axis=1) > -1 + tol))
    if np.any(bad):
        raise ValueError("point outside reference tetrahedron")
    a, b, c = _rst_to_abc(pts)
    cols = []
    for i, j, k in modal_index_order(p):
        h1 = jacobi_p(a, 0.0, 0.0, i)
        h2 = jacobi_p(b, 2.0 * i + 1.0, 0.0, j)
        h3 = jacobi_p(c, 2.0 * (i + j) + 2.0, 0.0, k)
        cols.append(2.0 * math.sqrt(2.0) * h1 * h2 * (1.0 - b) ** i * h3 * (1.0 - c) ** (i + j))
    return np.stack(cols, axis=1)


def modal_basis_grad(p: int, pts):
    """Gradients of the modal basis (refelem.cpp:44-74,162-179)."""
    pts = np.asarray(pts, dtype=np.float64).reshape(-1, 3)
    a, b, c = _rst_to_abc(pts)
    vr, vs, vt = [], [], []
    for i, j, k in modal_index_order(p):
        fa, dfa = jacobi_p(a, 0.0, 0.0, i), grad_jacobi_p(a, 0.0, 0.0, i)
        gb, dgb = jacobi_p(b, 2.0 * i + 1.0, 0.0, j), grad_jacobi_p(b, 2.0 * i + 1.0, 0.0, j)
        hc = jacobi_p(c, 2.0 * (i + j) + 2.0, 0.0, k)
        dhc = grad_jacobi_p(c, 2.0 * (i + j) + 2.0, 0.0, k)
        r_ = dfa * gb * hc
        if i > 0:
            r_ = r_ * (0.5 * (1.0 - b)) ** (i - 1)
        if i + j > 0:
            r_ = r_ * (0.5 * (1.0 - c)) ** (i + j - 1)
        s_ = 0.5 * (1.0 + a) * r_
        tmp = dgb * (0.5 * (1.0 - b)) ** i
        if i > 0:
            tmp = tmp + (-0.5 * i) * gb * (0.5 * (1.0 - b)) ** (i - 1)
        if i + j > 0:
            tmp = tmp * (0.5 * (1.0 - c)) ** (i + j - 1)
        tmp = fa * tmp * hc
        s_ = s_ + tmp
        t_ = 0.5 * (1.0 + a) * r_ + 0.5 * (1.0 + b) * tmp
        tmp2 = dhc * (0.5 * (1.0 - c)) ** (i + j)
        if i + j > 0:
            tmp2 = tmp2 - 0.5 * (i + j) * hc * (0.5 * (1.0 - c)) ** (i + j - 1)
        tmp2 = fa * gb * tmp2 * (0.5 * (1.0 - b)) ** i
        t_ = t_ + tmp2
        scale = 2.0 ** (2.0 * i + j + 1.5)
        vr.append(r_ * scale)
        vs.append(s_ * scale)
        vt.append(t_ * scale)
    return np.stack(vr, 1), np.stack(vs, 1), np.stack(vt, 1)


def _eval_warp(p: int, xnodes, xout):
    """refelem.cpp:89-110."""
    xeq = np.array([-1.0 + 2.0 * (p - i) / p for i in range(p + 1)])
    warp = np.zeros_like(xout)
    for i in range(p + 1):
        d = np.full_like(xout, xnodes[i] - xeq[i])
        for j in range(1, p):
            if i != j:
                d = d * (xout - xeq[j]) / (xeq[i] - xeq[j])
        if i != 0:
            d = -d / (xeq[i] - xeq[0])
        if i != p:
            d = d / (xeq[i] - xeq[p])
        warp = warp + d
    return warp


def _eval_shift(p: int, pval: float, l1, l2, l3):
    """refelem.cpp:113-144."""
    gauss_x = -gauss_lobatto(p)
    warp1 = 4.0 * _eval_warp(p, gauss_x, l3 - l2)
    warp2 = 4.0 * _eval_warp(p, gauss_x, l1 - l3)
    warp3 = 4.0 * _eval_warp(p, gauss_x, l2 - l1)
    c1, s1 = math.cos(2.0 * math.pi / 3.0), math.sin(2.0 * math.pi / 3.0)
    c2, s2 = math.cos(4.0 * math.pi / 3.0), math.sin(4.0 * math.pi / 3.0)
    b1 = l2 * l3 * warp1 * (1.0 + (pval * l1) ** 2)
    b2 = l1 * l3 * warp2 * (1.0 + (pval * l2) ** 2)
    b3 = l1 * l2 * warp3 * (1.0 + (pval * l3) ** 2)
    return 1.0 * b1 + c1 * b2 + c2 * b3, 0.0 * b1 + s1 * b2 + s2 * b3


_ALPHA_STORE = (0.0, 0.0, 0.0, 0.1002, 1.1332, 1.5608, 1.3413, 1.2577, 1.1603, 1.10153,
                0.6080, 0.4523, 0.8856, 0.8717, 0.9655)


def build_colloc_nodes(p: int) -> np.ndarray:
    """Warburton warp & blend nodes on the reference tet (refelem.cpp:181-283)."""
    if p < 1 or p > 9:
        raise ValueError(f"build_colloc_nodes: supported degrees are 1..9, got {p}")
    alpha = _ALPHA_STORE[p - 1]
    tol = 1e-10
    r, s, t = [], [], []
    for n in range(p + 1):
        for m in range(p - n + 1):
            for q in range(p - n - m + 1):
                r.append(-1.0 + 2.0 * q / p)
                s.append(-1.0 + 2.0 * m / p)
                t.append(-1.0 + 2.0 * n / p)
    r, s, t = np.array(r), np.array(s), np.array(t)
    l1 = (1.0 + t) / 2.0
    l2 = (1.0 + s) / 2.0
    l3 = -(1.0 + r + s + t) / 2.0
    l4 = (1.0 + r) / 2.0
    v1 = np.array([-1.0, -1.0 / math.sqrt(3.0), -1.0 / math.sqrt(6.0)])
    v2 = np.array([1.0, -1.0 / math.sqrt(3.0), -1.0 / math.sqrt(6.0)])
    v3 = np.array([0.0, 2.0 / math.sqrt(3.0), -1.0 / math.sqrt(6.0)])
    v4 = np.array([0.0, 0.0, 3.0 / math.sqrt(6.0)])
    t1 = [v2 - v1, v2 - v1, v3 - v2, v3 - v1]
    t2 = [v3 - (v1 + v2) * 0.5, v4 - (v1 + v2) * 0.5, v4 - (v2 + v3) * 0.5, v4 - (v1 + v3) * 0.5]
    t1 = [x / np.linalg.norm(x) for x in t1]
    t2 = [x / np.linalg.norm(x) for x in t2]
    xyz = l3[:, None] * v1 + l4[:, None] * v2 + l2[:, None] * v3 + l1[:, None] * v4
    shift = np.zeros_like(xyz)
    lam = {1: l1, 2: l2, 3: l3, 4: l4}
    order = ((1, 2, 3, 4), (2, 1, 3, 4), (3, 1, 4, 2), (4, 1, 3, 2))
    for face in range(4):
        la, lb, lc, ld = (lam[k] for k in order[face])
        w1, w2 = _eval_shift(p, alpha, lb, lc, ld)
        blend = lb * lc * ld
        denom = (lb + 0.5 * la) * (lc + 0.5 * la) * (ld + 0.5 * la)
        blend = np.where(denom > tol, (1.0 + (alpha * la) ** 2) * blend / np.where(denom > tol, denom, 1.0), blend)
        shift = shift + (blend * w1)[:, None] * t1[face] + (blend * w2)[:, None] * t2[face]
        on_face = la < tol
        interior = (lb > tol).astype(int) + (lc > tol).astype(int) + (ld > tol).astype(int)
        sel = on_face & (interior < 3)
        shift[sel] = (w1[:, None] * t1[face] + w2[:, None] * t2[face])[sel]
    xyz = xyz + shift
    a = np.stack([0.5 * (v2 - v1), 0.5 * (v3 - v1), 0.5 * (v4 - v1)], axis=1)
    rst = (np.linalg.inv(a) @ (xyz - v1).T).T
    return rst - 1.0


@dataclass(frozen=True)
class ReferenceElement:
    """All degree-dependent tables (refelem.hpp:51-112)."""
    degree: int
    n_basis: int
    n_cub: int
    n_face_quad: int
    colloc_nodes: np.ndarray   # [np,3]
    cub_nodes: np.ndarray      # [ncub,3]
    cub_weights: np.ndarray    # [ncub]
    face_nodes: np.ndarray     # [4ng,3] face-major
    face_weights: np.ndarray   # [ng]  (2D rule, sums to 2)
    vandermonde: np.ndarray    # [np,np]
    vandermonde_inv: np.ndarray
    interp_cub: np.ndarray     # [ncub,np]
    interp_face: np.ndarray    # [4ng,np]
    deriv_r: np.ndarray        # [ncub,np]
    deriv_s: np.ndarray
    deriv_t: np.ndarray
    face_deriv_r: np.ndarray   # [4ng,np]
    face_deriv_s: np.ndarray
    face_deriv_t: np.ndarray


@functools.lru_cache(maxsize=None)
def get_reference_element(p: int, cub_override: int = 0, face_override: int = 0) -> ReferenceElement:
    """refelem.cpp:301-358 / 401-413 (cached per (p, strengths))."""
    if p < 1 or p > 9:
        raise ValueError(f"ReferenceElement: supported degrees are 1..9, got {p}")
    colloc = build_colloc_nodes(p)
    cub_nodes, cub_w = tet_cubature(cub_override if cub_override > 0 else 2 * p + 1)
    fa, fb, fw = tri_quadrature(face_override if face_override > 0 else 2 * p)
    ng = len(fa)
    face_nodes = []
    for f in range(4):
        a, b, c = (TET_VERTS[v] for v in FACE_VERTS[f])
        u, v = (fa + 1.0) / 2.0, (fb + 1.0) / 2.0
        face_nodes.append(a + u[:, None] * (b - a) + v[:, None] * (c - a))
    face_nodes = np.concatenate(face_nodes)
    vand = modal_basis_eval(p, colloc)
    vinv = np.linalg.inv(vand)
    vr, vs, vt = modal_basis_grad(p, cub_nodes)
    fvr, fvs, fvt = modal_basis_grad(p, face_nodes)
    return ReferenceElement(
        degree=p, n_basis=basis_count(p), n_cub=len(cub_w), n_face_quad=ng,
        colloc_nodes=colloc, cub_nodes=cub_nodes, cub_weights=cub_w, face_nodes=face_nodes,
        face_weights=fw, vandermonde=vand, vandermonde_inv=vinv,
        interp_cub=modal_basis_eval(p, cub_nodes) @ vinv,
        interp_face=modal_basis_eval(p, face_nodes) @ vinv,
        deriv_r=vr @ vinv, deriv_s=vs @ vinv, deriv_t=vt @ vinv,
        face_deriv_r=fvr @ vinv, face_deriv_s=fvs @ vinv, face_deriv_t=fvt @ vinv)


def level_reference_element(p: int, curved: bool) -> ReferenceElement:
    """solver.cpp:551-557: curved meshes raise the strengths for all elements."""
    if curved:
        return get_reference_element(p, curved_volume_strength(p), curved_face_strength(p))
    return get_reference_element(p)
