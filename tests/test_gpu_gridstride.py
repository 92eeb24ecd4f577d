"""GPU parity in the benchmark's own regime: persistent (grid-stride) kernels
that walk MANY tiles per CTA.

The production launch at BASELINE config 5 (4.09M tets, 255,552 16-element
tiles on 592 resident CTAs) runs ~432 tiles per CTA through the grid-stride
loop of k_rhs_row (cross-tile smem restaging, the fused-trace double buffer).
A small mesh at the default grid gives each CTA one tile, so these tests
(1) run a mesh with more tiles than resident CTAs (make_cube_mesh(14): 16,464
tets = 1,029 tiles) against the reference's own rk_step (oracle/_ref), and
(2) cap the grid with cdg_gpu_set_max_ctas so every kernel family walks
hundreds of tiles per CTA, which must reproduce the default grid BIT FOR BIT
(per-element arithmetic does not depend on the grid) and the oracle.

Tolerances (north_star): conserved variables within 1e-12 normwise-relative
L_inf after the first RK step, drift over the steps below 1e-11.
Reference: solver.cpp:469-492 (rk_step), euler.cpp:59-138 (LLF, HLLC)."""
import numpy as np
import pytest

from oracle import port
from paper_1208_4772_b200 import mesh as M
from paper_1208_4772_b200 import refelem as R

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


def _fs(gpu):
    return gpu.make_state(1.0, [0.4, 0.05, -0.1], 1.0)


def _ref_cube(ref, n):
    """The reference's make_cube_mesh(n) (all faces tagged "wall") as a GPU mesh
    with the same element order and face pairing."""
    rm = ref.Mesh("cube", n)
    ex = rm.export()
    lut = {q[0] + 3 * q[1] + 9 * q[2]: i for i, q in enumerate(M.PERMS)}
    perm = ex["perm"]
    code = np.where(perm >= 0, np.vectorize(lambda x: lut.get(int(x), 0))(perm), -1)
    mesh = M.from_arrays(ex["vertices"], ex["tets"], ex["neighbor"], ex["neighbor_face"], code,
                         np.where(ex["neighbor"] >= 0, -1, ex["bnd_tag"]))
    mesh.tags = ["wall", "farfield"]
    return rm, mesh


_CUBE14 = {}


def _cube14(ref):
    if not _CUBE14:
        rm, mesh = _ref_cube(ref, 14)
        rl = ref.Level(rm, 4, bc_wall=0, bc_far=1)
        _CUBE14.update(rm=rm, mesh=mesh, rl=rl)
    return _CUBE14["rm"], _CUBE14["mesh"], _CUBE14["rl"]


@pytest.mark.parametrize("riemann", ["llf", "hllc"])
def test_p4_cube14_rk_steps_match_reference_default_and_capped_grid(gpu_lib, refmod, riemann):
    """BASELINE config 5's kernel (P=4, slip walls, fused traces) on 1,029 tiles:
    3 RK steps against the reference's own rk_step, at the default grid (592
    CTAs: the grid-stride loop runs) and capped at 7 CTAs (147 tiles per CTA)."""
    gpu, ref = gpu_lib, refmod
    rm, mesh, rl = _cube14(ref)
    assert rl.K == 16464 and (rl.K + 15) // 16 == 1029
    fs = _fs(gpu)
    lv = gpu.GpuLevel(mesh, 4, bc={"wall": 0, "farfield": 1}, freestream=fs, re=R.get_reference_element(4))
    assert lv.fused_traces()
    cfg_r = ref.make_cfg(riemann)
    u0 = rl.random_admissible_store(42)     # bench.cpp:22-40 recipe (mt19937(42))
    dt = 0.5 * rl.compute_timestep(u0, cfg_r)
    lv.set_state(u0)
    assert lv.compute_timestep(gpu.run_config(riemann)) == pytest.approx(dt / 0.5, rel=1e-13)
    u_ref, res_ref = u0.copy(), np.zeros_like(u0)
    states = {}
    for cap in (0, 7):
        lv.set_max_ctas(cap)
        lv.set_state(u0)
        states[cap] = []
        for _ in range(3):
            lv.rk_steps(gpu.run_config(riemann), dt, 1)
            states[cap].append(lv.get_state())
    lv.close()
    for step in range(3):
        u_ref, res_ref = rl.rk_steps(u_ref, res_ref, cfg_r, fs, dt, 1)
        for cap in (0, 7):
            u, res = states[cap][step]
            e = rel(u, u_ref)
            assert e < (1e-12 if step == 0 else 1e-11), (cap, step, e)
            assert rel(res, res_ref) < 1e-10, (cap, step, rel(res, res_ref))
        # the grid does not change any element's arithmetic
        assert np.array_equal(states[0][step][0], states[7][step][0])
        assert np.array_equal(states[0][step][1], states[7][step][1])


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("riemann", ["llf", "hllc"])
@pytest.mark.parametrize("path", ["default", "generic", "traced"])
def test_capped_grid_is_bitwise_default_grid_and_matches_oracle(gpu_lib, p, riemann, path):
    """Every kernel family (neighbour-state p=1, warp-tile p=1 on the traced
    path, row-per-warp / warp-autonomous p=2..5 with fused traces at p<=4, CTA
    kernel p>=6 and the generic path everywhere) with 2 CTAs in
    the grid: RHS and 3 RK steps bitwise equal to the default grid, and the
    RK steps within the north_star tolerance of the oracle."""
    gpu = gpu_lib
    n = 6 if p <= 3 else (4 if p <= 5 else 3)
    m = M.cube_mesh(n, scale=2.0)
    fs = _fs(gpu)
    re = R.get_reference_element(p)
    lv = gpu.GpuLevel(m, p, bc=0, freestream=fs, re=re)
    lv.set_kernel_path(path)
    cfg = gpu.run_config(riemann)
    u0 = gpu.random_admissible_store(lv, seed=50 + p)
    lv.set_state(u0)
    dt = (0.25 if p <= 6 else 0.1) * lv.compute_timestep(cfg)
    out = {}
    for cap in (0, 2):
        lv.set_max_ctas(cap)
        rhs = lv.compute_rhs(cfg, u0)
        lv.set_state(u0)
        lv.rk_steps(cfg, dt, 3)
        out[cap] = (rhs,) + lv.get_state()
    lv.close()
    tiles = (m.n_owned + 15) // 16
    assert tiles >= 8, tiles  # >= 4 tiles per CTA at the cap
    for a, b in zip(out[0], out[2]):
        assert np.array_equal(a, b)
    ol = port.OracleLevel(m, re, bc=0, freestream=fs)
    u_ref, _ = ol.rk_steps(u0, np.zeros_like(u0), cfg, dt, 3)
    assert rel(out[0][1], u_ref) < 1e-11, rel(out[0][1], u_ref)


@pytest.mark.parametrize("p", [5, 6, 7, 8])
@pytest.mark.parametrize("riemann", ["llf", "hllc"])
def test_rk_steps_high_order_match_oracle(gpu_lib, p, riemann):
    """rk_steps at p = 5..8 (row kernel p=5, CTA kernel p>=6) step by step
    against the oracle: first step 1e-12, drift 1e-11."""
    gpu = gpu_lib
    m = M.cube_mesh(2, scale=2.0)
    fs = _fs(gpu)
    re = R.get_reference_element(p)
    lv = gpu.GpuLevel(m, p, bc=0, freestream=fs, re=re)
    ol = port.OracleLevel(m, re, bc=0, freestream=fs)
    cfg = gpu.run_config(riemann)
    u0 = gpu.random_admissible_store(lv, seed=70 + p)
    lv.set_state(u0)
    dt = 0.1 * lv.compute_timestep(cfg)
    u_ref, res = u0.copy(), np.zeros_like(u0)
    worst = 0.0
    for step in range(5):
        lv.rk_steps(cfg, dt, 1)
        u_ref, res = ol.rk_steps(u_ref, res, cfg, dt, 1)
        e = rel(lv.get_state()[0], u_ref)
        worst = max(worst, e)
        if step == 0:
            assert e < 1e-12, e
    assert worst < 1e-11, worst


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
def test_traces_match_oracle_all_orders(gpu_lib, p):
    gpu = gpu_lib
    m = M.cube_mesh(2)
    fs = _fs(gpu)
    re = R.get_reference_element(p)
    lv = gpu.GpuLevel(m, p, bc=1, freestream=fs, re=re)
    ol = port.OracleLevel(m, re, bc=1, freestream=fs)
    u = gpu.random_admissible_store(lv, seed=3 + p)
    lv.set_state(u)
    t_gpu = lv.interpolate_to_faces()
    assert rel(t_gpu, ol.interpolate_to_faces(u)) < 1e-13
    tb = t_gpu.reshape(lv.K, 5, lv.trace_block)
    assert np.all(tb[:, :, 4 * lv.n_face_quad:] == 0.0)


@pytest.mark.parametrize("visc", [dict(enabled=True, eps0=0.04, kappa=4.0, s0_offset=-100.0),
                                  dict(enabled=True, eps0=0.3, kappa=4.0, s0_offset=0.0)])
def test_viscous_capped_grid_is_bitwise_default_grid(gpu_lib, visc):
    """The artificial-viscosity stage (sensor, aux gradient, q traces, viscous
    RHS; gated inside one CUDA graph per step) with 3 CTAs per kernel."""
    gpu = gpu_lib
    m = M.cube_mesh(5, scale=2.0)
    fs = _fs(gpu)
    lv = gpu.GpuLevel(m, 3, bc=1, freestream=fs, re=R.get_reference_element(3))
    cfg = gpu.run_config("hllc", viscosity=visc)
    u0 = gpu.random_admissible_store(lv, seed=21)
    lv.set_state(u0)
    dt = 0.1 * lv.compute_timestep(cfg)
    out = {}
    for cap in (0, 3):
        lv.set_max_ctas(cap)
        lv.set_state(u0)
        lv.rk_steps(cfg, dt, 2)
        out[cap] = lv.get_state()[0]
    assert np.array_equal(out[0], out[3])
    ol = port.OracleLevel(m, R.get_reference_element(3), bc=1, freestream=fs)
    u_ref, _ = ol.rk_steps(u0, np.zeros_like(u0), cfg, dt, 2)
    assert rel(out[0], u_ref) < 1e-12


@pytest.mark.parametrize("frac", [1.0, 0.4])
@pytest.mark.parametrize("riemann", ["llf", "hllc"])
def test_curved_capped_grid_is_bitwise_default_grid(gpu_lib, frac, riemann):
    """k_rhs_rowc (curved elements) + the affine row kernel on the mixed tiles,
    6,000 tets on 3 CTAs per kernel vs the default grid."""
    gpu = gpu_lib
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_curved", "scripts/bench_curved.py")
    bcm = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bcm)
    mesh = M.cube_mesh(10)
    re = R.level_reference_element(4, True)
    X = bcm.curved_nodes(mesh, re, 0.02)
    ids = np.arange(int(round(frac * mesh.n_owned)))
    fs = _fs(gpu)
    lv = gpu.GpuLevel(mesh, 4, bc=0, freestream=fs, curved=(ids, X[ids]))
    cfg = gpu.run_config(riemann)
    u0 = gpu.random_admissible_store(lv, seed=9)
    lv.set_state(u0)
    dt = 0.3 * lv.compute_timestep(cfg)
    out = {}
    for cap in (0, 3):
        lv.set_max_ctas(cap)
        lv.set_state(u0)
        lv.rk_steps(cfg, dt, 3)
        out[cap] = lv.get_state()
    assert np.array_equal(out[0][0], out[3][0]) and np.array_equal(out[0][1], out[3][1])
