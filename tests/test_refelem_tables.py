"""Host table builder (paper_1208_4772_b200/refelem.py) vs the reference's own
tables (golden fixtures dumped from oracle/_ref, refelem.cpp:301-358)."""
from pathlib import Path

import numpy as np
import pytest

from paper_1208_4772_b200 import refelem as R

G = Path(__file__).resolve().parent / "golden"


def _cases():
    for p in range(1, 9):
        yield p, False
        if R.curved_volume_strength(p) != 2 * p + 1 or R.curved_face_strength(p) != 2 * p:
            yield p, True


@pytest.mark.parametrize("p,curved", list(_cases()))
def test_tables_match_reference(p, curved):
    f = G / f"refelem_p{p}{'_curved' if curved else ''}.npz"
    gold = np.load(f)
    re = R.level_reference_element(p, curved)
    for key in gold.files:
        base = key.split("__")[0]
        mine = np.asarray(getattr(re, base))
        if key.endswith("__rowsum"):
            mine = mine.sum(axis=1)
        elif key.endswith("__colsum"):
            mine = mine.sum(axis=0)
        elif key.endswith("__rows"):
            mine = mine[gold[base + "__rowidx"]]
        elif key.endswith("__rowidx"):
            continue
        ref = gold[key]
        assert mine.shape == ref.shape, key
        scale = max(1.0, np.max(np.abs(ref)))
        assert np.max(np.abs(mine - ref)) / scale < 5e-13, (key, np.max(np.abs(mine - ref)) / scale)


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_counts_and_exactness(p):
    """C01/C02 style properties: counts, weights sum, derivative exactness."""
    re = R.get_reference_element(p)
    assert re.n_basis == R.basis_count(p)
    assert abs(re.cub_weights.sum() - 4.0 / 3.0) < 1e-13
    assert abs(re.face_weights.sum() - 2.0) < 1e-13
    x = re.colloc_nodes
    f = x[:, 0] ** p + x[:, 1] * x[:, 2]
    dfr = p * re.cub_nodes[:, 0] ** (p - 1)
    assert np.max(np.abs(re.deriv_r @ f - dfr)) < 1e-11
    if p == 4:
        assert (re.n_basis, re.n_cub, re.n_face_quad) == (35, 70, 16)
