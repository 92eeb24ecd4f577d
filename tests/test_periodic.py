"""BASELINE config 1's periodic box on the CPU: the periodic cube mesh, its
face-node pairing, and the two oracles on it (the reference's own kernels
with the periodic coupling of oracle/ref_periodic.cpp, and the C
restatement with minimum-image pairing) against each other. The reference
has no periodic boundary (euler.hpp:65); its compute_rhs / rk_step read the
face graph only through DgLevel::coupling (solver.cpp:228,292,418)."""
import numpy as np
import pytest

from paper_1208_4772_b200 import cases, mesh as M, refelem as R
from paper_1208_4772_b200.level import LevelArrays


def test_periodic_cube_links_translates():
    n, L = 4, 10.0
    m = cases.periodic_cube(n, L)
    K = m.n_owned
    assert K == 6 * n ** 3 and np.all(m.neighbor >= 0) and m.period == (L, L, L)
    e = np.repeat(np.arange(K), 4)
    f = np.tile(np.arange(4), K)
    nb, nf = m.neighbor.ravel(), m.neighbor_face.ravel()
    assert np.array_equal(m.neighbor[nb, nf], e) and np.array_equal(m.neighbor_face[nb, nf], f)
    fv = M.FACE_VERTS_ARR
    c_mine = m.vertices[m.tets[e[:, None], fv[f]]].mean(axis=1)
    c_nb = m.vertices[m.tets[nb[:, None], fv[nf]]].mean(axis=1)
    d = c_mine - c_nb
    d -= L * np.round(d / L)
    assert np.max(np.abs(d)) < 1e-12  # the linked face is the same face or its translate
    wrapped = np.any(np.abs(c_mine - c_nb) > L / 2, axis=1)
    assert wrapped.sum() == 6 * 2 * n * n  # every boundary triangle of the box wraps


@pytest.mark.parametrize("p", [1, 3, 4])
def test_periodic_node_maps_match_minimum_image_pairing(p):
    """The GPU's per-permutation node maps == nearest-point pairing by minimum
    image (the C restatement's pairing, solver.cpp:144-172 + translation)."""
    from oracle import port
    m = cases.periodic_cube(3)
    re = R.get_reference_element(p)
    a = LevelArrays(m, re)
    ol = port.OracleLevel(m, re)
    _, nm = ol.export()
    assert np.array_equal(a.code_node_map[a.face_code], nm)


@pytest.mark.parametrize("p,riemann", [(2, "llf"), (3, "hllc")])
def test_reference_and_restatement_agree_on_periodic_vortex(refmod, p, riemann):
    from oracle import port
    from paper_1208_4772_b200 import gpu
    ref = refmod
    n, L = 3, 10.0
    m = cases.periodic_cube(n, L)
    re = R.get_reference_element(p)
    rl = ref.Level(ref.Mesh("cube", n, scale=L), p, bc_wall=0, bc_far=1)
    rl.make_periodic((L, L, L))
    g = rl.geometry()
    assert np.all(g["neighbor"] >= 0)
    ol = port.OracleLevel(m, re)
    _, nm = ol.export()
    assert np.array_equal(g["node_map"], nm) and np.array_equal(g["neighbor"], m.neighbor)
    u = cases.vortex_store(m, re, ol.block)
    cfg_r, cfg_o = ref.make_cfg(riemann), gpu.run_config(riemann)
    fs = np.array([1.0, 1.0, 1.0, 0.0, 2.5 + 1.0])
    rhs_r = rl.compute_rhs(u, cfg_r, fs)
    rhs_o = ol.compute_rhs(u, cfg_o)
    assert np.max(np.abs(rhs_r - rhs_o)) / np.max(np.abs(rhs_r)) < 1e-12
    dt = 0.3 * ol.compute_timestep(u, cfg_o)
    ur, _ = rl.rk_steps(u, np.zeros_like(u), cfg_r, fs, dt, 2)
    uo, _ = ol.rk_steps(u, np.zeros_like(u), cfg_o, dt, 2)
    assert np.max(np.abs(ur - uo)) / np.max(np.abs(ur)) < 1e-13
