"""Host mesh/level setup vs the reference's DgLevel (golden fixtures)."""
from pathlib import Path

import numpy as np
import pytest

from paper_1208_4772_b200 import level as L, mesh as M, refelem as R

G = Path(__file__).resolve().parent / "golden"


@pytest.mark.parametrize("n,p", [(2, 3), (2, 4), (3, 2)])
def test_level_matches_reference(n, p):
    gold = np.load(G / "level_geometry.npz")
    key = f"n{n}_p{p}"
    m = M.cube_mesh(n)
    assert np.array_equal(m.tets, gold[key + "_tets"])
    assert np.array_equal(m.neighbor, gold[key + "_neighbor"])
    la = L.LevelArrays(m, R.get_reference_element(p), bc=0)
    nm = la.code_node_map[la.face_code]
    mask = la.neighbor >= 0
    assert np.array_equal(nm[mask], gold[key + "_node_map"][mask])
    assert np.max(np.abs(la.h - gold[key + "_h"]) / gold[key + "_h"]) < 1e-12
    assert np.max(np.abs(la.metric - gold[key + "_metric0"])) < 1e-12 * np.max(np.abs(la.metric))
    assert np.max(np.abs(la.jac - gold[key + "_jac0"]) / gold[key + "_jac0"]) < 1e-12


def test_cube_counts_and_orientation():
    m = M.cube_mesh(5)
    assert m.n_owned == 6 * 125
    assert np.all(M.signed_volumes(m.vertices, m.tets) > 0)
    # every interior link is symmetric
    K = m.n_owned
    e, f = np.nonzero(m.neighbor >= 0)
    nb, nf = m.neighbor[e, f], m.neighbor_face[e, f]
    assert np.array_equal(m.neighbor[nb, nf], e)
    assert np.array_equal(m.neighbor_face[nb, nf], f)
    # boundary faces: 2 per cell face on the cube surface
    assert np.sum(m.neighbor < 0) == 6 * 2 * 25


def test_perm_node_maps_are_permutations_for_dunavant_rules():
    # p <= 4 uses the Dunavant orbits (distinct points); p >= 5 face rules are
    # Grundmann-Moller with coincident points, where the reference's
    # nearest-point pairing (solver.cpp:155-171) keeps the first match
    for p in (1, 2, 3, 4):
        re = R.get_reference_element(p)
        maps = L.perm_node_maps(re)
        assert maps.shape == (6, re.n_face_quad)
        for row in maps:
            assert sorted(row.tolist()) == list(range(re.n_face_quad))


@pytest.mark.parametrize("p", [5, 6, 7, 8])
def test_node_maps_high_p_match_live_reference(refmod, p):
    ref = refmod
    rm = ref.Mesh("cube", 1)
    g = ref.Level(rm, p).geometry()
    la = L.LevelArrays(M.cube_mesh(1), R.get_reference_element(p), bc=0)
    nm = la.code_node_map[la.face_code]
    mask = la.neighbor >= 0
    assert np.array_equal(nm[mask], g["node_map"][mask])
