"""Device-resident run_steady (solver.cpp:594-676) through the
C ABI (cdg_gpu_fill_freestream / cdg_gpu_p_refine_embed / cdg_gpu_run_level):
the reference's own run_steady tests (test_solver.cpp:481-567) on the GPU,
plus the convergence log and final state against the reference's run_steady
(oracle/_ref) on a non-trivial slip-wall run."""
import numpy as np
import pytest

from paper_1208_4772_b200 import mesh as M
from paper_1208_4772_b200 import refelem as R

pytestmark = pytest.mark.gpu

FS = None


def _fs(gpu):
    return gpu.make_state(1.0, [0.4, 0.05, -0.1], 1.0)


def _cube(ref, n):
    """The reference's make_cube_mesh(n, "wall") as a GPU mesh (same element order)."""
    rm = ref.Mesh("cube", n)
    ex = rm.export()
    lut = {q[0] + 3 * q[1] + 9 * q[2]: i for i, q in enumerate(M.PERMS)}
    perm = ex["perm"]
    code = np.where(perm >= 0, np.vectorize(lambda x: lut.get(int(x), 0))(perm), -1)
    mesh = M.from_arrays(ex["vertices"], ex["tets"], ex["neighbor"], ex["neighbor_face"], code,
                         np.where(ex["neighbor"] >= 0, -1, ex["bnd_tag"]))
    mesh.tags = ["wall", "farfield"]
    return rm, mesh


def _maker(gpu, mesh, fs, bc):
    return lambda p: gpu.GpuLevel(mesh, p, bc=bc, freestream=fs, re=R.get_reference_element(p))


def rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


def test_run_steady_matches_reference_log_and_state(gpu_lib, refmod):
    gpu, ref = gpu_lib, refmod
    fs = _fs(gpu)
    rm, mesh = _cube(ref, 2)
    rows_r, conv_r, deg_r, u_r = ref.run_steady(rm, ref.make_cfg("llf"), fs, [1, 2], fixed=(12, 12),
                                                 check_interval=5, bc_wall=0)
    rows, conv, deg, lv = gpu.run_steady(_maker(gpu, mesh, fs, {"wall": 0, "farfield": 1}), [1, 2],
                                         gpu.run_config("llf"), fixed_iterations=(12, 12), check_interval=5)
    assert deg == deg_r == 2 and conv == conv_r
    rows = np.array(rows)
    assert np.array_equal(rows[:, :2], rows_r[:, :2])          # (level, iteration) of every check
    assert rel(rows[:, 2], rows_r[:, 2]) < 1e-12                # dt
    assert rel(rows[:, 3], rows_r[:, 3]) < 1e-10                # residual
    u = lv.get_state()[0]
    assert rel(u, u_r[: u.size]) < 1e-11


def test_run_steady_l2_residual_matches_reference(gpu_lib, refmod):
    gpu, ref = gpu_lib, refmod
    fs = _fs(gpu)
    rm, mesh = _cube(ref, 2)
    rows_r, _, _, _ = ref.run_steady(rm, ref.make_cfg("hllc"), fs, [2], fixed=(8,), check_interval=4,
                                     residual="l2", bc_wall=0)
    rows, _, _, _ = gpu.run_steady(_maker(gpu, mesh, fs, {"wall": 0, "farfield": 1}), [2], gpu.run_config("hllc"),
                                   fixed_iterations=(8,), check_interval=4, residual="l2")
    rows = np.array(rows)
    assert np.array_equal(rows[:, :2], rows_r[:, :2])
    assert rel(rows[:, 3], rows_r[:, 3]) < 1e-10


def test_run_steady_freestream_converges_one_check_per_level(gpu_lib, refmod):
    """test_solver.cpp:481-515."""
    gpu, ref = gpu_lib, refmod
    fs = _fs(gpu)
    _, mesh = _cube(ref, 2)
    make = _maker(gpu, mesh, fs, {"wall": 1})
    rows, conv, deg, _ = gpu.run_steady(make, [1, 2, 3], gpu.run_config("llf"), final_tolerance=1e-9,
                                        intermediate_tolerance=1e-9, max_iterations=50, check_interval=10)
    assert conv and deg == 3
    assert [r[0] for r in rows] == [1, 2, 3]
    assert rows[0][2] > rows[1][2] > rows[2][2]
    assert all(r[1] == 10 and r[3] < 1e-9 for r in rows)
    single, _, _, _ = gpu.run_steady(make, [3], gpu.run_config("llf"), max_iterations=50, check_interval=10)
    assert len(single) == 1
    with pytest.raises(gpu.ConfigError):
        gpu.run_steady(make, [2, 2], gpu.run_config("llf"))


def test_run_steady_fixed_iterations(gpu_lib, refmod):
    """test_solver.cpp:517-538."""
    gpu, ref = gpu_lib, refmod
    fs = _fs(gpu)
    _, mesh = _cube(ref, 1)
    rows, _, _, _ = gpu.run_steady(_maker(gpu, mesh, fs, {"wall": 1}), [1, 2], gpu.run_config("llf"),
                                   check_interval=10, fixed_iterations=(20, 30), max_iterations=100)
    assert max(r[1] for r in rows if r[0] == 1) == 20
    assert max(r[1] for r in rows if r[0] == 2) == 30


def test_run_steady_divergence_detector(gpu_lib, refmod):
    """test_solver.cpp:540-554: dt 8x above the stability limit aborts."""
    gpu, ref = gpu_lib, refmod
    fs = _fs(gpu)
    _, mesh = _cube(ref, 1)
    make = _maker(gpu, mesh, fs, {"wall": 1})
    probe = make(2)
    probe.fill_freestream()
    dt = 8.0 * probe.compute_timestep(gpu.run_config("llf"))
    with pytest.raises(gpu.NumericsError):
        gpu.run_steady(make, [2], gpu.run_config("llf"), check_interval=25, max_iterations=4000,
                       final_tolerance=1e-14, dt_override=dt)


def test_run_steady_hllc_converges_on_freestream(gpu_lib, refmod):
    """test_solver.cpp:556-567."""
    gpu, ref = gpu_lib, refmod
    fs = _fs(gpu)
    _, mesh = _cube(ref, 1)
    _, conv, _, _ = gpu.run_steady(_maker(gpu, mesh, fs, {"wall": 1}), [2], gpu.run_config("hllc"),
                                   check_interval=5, final_tolerance=1e-9, max_iterations=20)
    assert conv
