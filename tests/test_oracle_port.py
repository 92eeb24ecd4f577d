"""The C restatement (oracle/cdg_oracle.c) pinned against the reference's
golden vectors (tests/golden/*.npz, dumped from oracle/_ref) and the
reference's own property tests (test_solver.cpp)."""
from pathlib import Path

import numpy as np
import pytest

from oracle import port
from paper_1208_4772_b200 import gpu, mesh as M, refelem as R

G = Path(__file__).resolve().parent / "golden"
FS = gpu.make_state(1.0, [0.4, 0.05, -0.1], 1.0)


def rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


@pytest.mark.parametrize("p,riem,bc", [(p, r, b) for p in (1, 2, 3, 4) for r, b in (("llf", 0), ("hllc", 1))])
def test_port_matches_reference_golden(p, riem, bc):
    gold = np.load(G / "rhs_cube2.npz")
    key = f"p{p}_{riem}_bc{bc}"
    m = M.cube_mesh(2, scale=4.0)
    ol = port.OracleLevel(m, R.get_reference_element(p), bc=bc, freestream=gold["freestream"])
    cfg = gpu.run_config(riem)
    u = gold[f"p{p}_u"]
    assert rel(ol.compute_rhs(u, cfg), gold[key + "_rhs"]) < 1e-11
    dt = float(gold[key + "_dt"][0])
    assert 0.25 * ol.compute_timestep(u, cfg) == pytest.approx(dt, rel=1e-12)
    u2, _ = ol.rk_steps(u, np.zeros_like(u), cfg, dt, 2)
    assert rel(u2, gold[key + "_u2"]) < 1e-12


def test_port_viscous_matches_reference_golden():
    gold = np.load(G / "viscous_cube3_p2.npz")
    m = M.cube_mesh(3)
    ol = port.OracleLevel(m, R.get_reference_element(2), bc=1, freestream=gold["freestream"])
    cfg = gpu.run_config("llf", viscosity=dict(enabled=True, eps0=0.04, kappa=4.0, s0_offset=-100.0))
    rhs = ol.compute_rhs(gold["forced_u"], cfg)
    eps, q = ol.last_viscosity()
    assert np.allclose(eps, gold["forced_eps"], rtol=1e-13, atol=0)
    assert rel(q, gold["forced_q"]) < 1e-11
    assert rel(rhs, gold["forced_rhs"]) < 1e-11
    cfg2 = gpu.run_config("hllc", viscosity=dict(enabled=True, eps0=0.3, kappa=4.0, s0_offset=0.0))
    rhs2 = ol.compute_rhs(gold["ramp_u"], cfg2)
    eps2, _ = ol.last_viscosity(with_q=False)
    assert np.max(np.abs(eps2 - gold["ramp_eps"])) < 1e-12
    assert rel(rhs2, gold["ramp_rhs"]) < 1e-11


def test_port_freestream_and_conservation():
    """test_solver.cpp:115-183 properties on the restatement."""
    m = M.cube_mesh(2, scale=4.0)
    cfg = gpu.run_config("llf")
    for p, tol in ((1, 1e-12), (2, 1e-12), (3, 1e-12), (4, 2e-11)):
        ol = port.OracleLevel(m, R.get_reference_element(p), bc=1, freestream=FS)
        u = np.zeros(ol.store_size).reshape(ol.K, 5, ol.block)
        u[:, :, : R.basis_count(p)] = FS[None, :, None]
        assert np.max(np.abs(ol.compute_rhs(u.reshape(-1), cfg))) < tol


def test_port_inadmissible_message():
    m = M.cube_mesh(1)
    ol = port.OracleLevel(m, R.get_reference_element(2), bc=1, freestream=FS)
    u = np.zeros(ol.store_size).reshape(ol.K, 5, ol.block)
    u[:, :, :10] = FS[None, :, None]
    u[3, 0, :10] = -1.0
    with pytest.raises(port.OracleError) as ei:
        ol.compute_rhs(u.reshape(-1), gpu.run_config("llf"))
    assert "inadmissible" in str(ei.value) and "node" in str(ei.value)
