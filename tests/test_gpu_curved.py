"""Curved (isoparametric) elements on the GPU vs the reference itself: the
acceptance sphere-shell fixture curved through the reference's own
elasticity pipeline (acceptance_main.cpp:82-120), mixed affine + curved
level with the raised quadrature (solver.cpp:551-557). Needs oracle/_ref."""
import numpy as np
import pytest

from paper_1208_4772_b200 import mesh as M

pytestmark = pytest.mark.gpu

_CACHE = {}


def sphere_case(ref, p):
    key = p
    if key not in _CACHE:
        rm = ref.Mesh("sphere_curved", sphere=(2, 5, p, p))
        rl = ref.Level(rm, p, bc_wall=0, bc_far=1)
        ex = rm.export()
        nodes, curved = rl.nodes()
        perm = ex["perm"]
        # reference FaceLink.perm packed p0+3p1+9p2 -> PERMS index
        lut = {q[0] + 3 * q[1] + 9 * q[2]: i for i, q in enumerate(M.PERMS)}
        code = np.where(perm >= 0, np.vectorize(lambda x: lut.get(int(x), 0))(perm), -1)
        mesh = M.from_arrays(ex["vertices"], ex["tets"], ex["neighbor"], ex["neighbor_face"], code,
                             np.where(ex["neighbor"] >= 0, -1, ex["bnd_tag"]))
        mesh.tags = ["sphere", "farfield"]
        ids = np.nonzero(curved)[0]
        _CACHE[key] = (rm, rl, mesh, ids, nodes)
    return _CACHE[key]


def rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


FS = None


def _fs(gpu):
    # sphere_m038.json-like freestream: M=0.38, rho=p=1, alpha=0
    c = np.sqrt(1.4)
    return gpu.make_state(1.0, [0.38 * c, 0.0, 0.0], 1.0)


# p=6 passes too (2.7 min of reference-side curving on the host; run with
# CDG_SLOW=1) -- the BASELINE "cylinder P=1..6" sweep on the curved sphere
@pytest.mark.parametrize("kernel", ["row", "cta"])
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5] + ([6] if __import__("os").environ.get("CDG_SLOW") else []))
def test_curved_sphere_rhs_and_steps_match_reference(gpu_lib, refmod, p, kernel):
    """kernel: the row-per-warp curved kernel (k_rhs_rowc, default for p <= 5)
    or the CTA kernels (k_rhs_curved + k_rhs: the generic path, default for
    p >= 6)."""
    gpu, ref = gpu_lib, refmod
    rm, rl, mesh, ids, nodes = sphere_case(ref, p)
    assert len(ids) > 0 and rl.n_cub > 0
    fs = _fs(gpu)
    lv = gpu.GpuLevel(mesh, p, bc={"sphere": 0, "farfield": 1}, freestream=fs, curved=(ids, nodes[ids]))
    lv.set_kernel_path("generic" if kernel == "cta" else "default")
    assert (lv.n_cub, lv.n_face_quad) == (rl.n_cub, rl.n_face_quad)
    # node pairing identical to the reference's nearest-point pairing
    g = rl.geometry()
    a = lv.arrays
    nm = a.code_node_map[a.face_code]
    mask = a.neighbor >= 0
    assert np.array_equal(nm[mask], g["node_map"][mask])
    for riem in ("llf", "hllc"):
        cfg = gpu.run_config(riem)
        u = rl.random_admissible_store(5)
        r_ref = rl.compute_rhs(u, ref.make_cfg(riem), fs)
        r_gpu = lv.compute_rhs(cfg, u)
        assert rel(r_gpu, r_ref) < 1e-10, (riem, rel(r_gpu, r_ref))
    dt = 0.2 * rl.compute_timestep(u, ref.make_cfg("llf"))
    lv.set_state(u)
    assert 0.2 * lv.compute_timestep(gpu.run_config("llf")) == pytest.approx(dt, rel=1e-10)
    lv.rk_steps(gpu.run_config("llf"), dt, 2)
    u_ref, _ = rl.rk_steps(u, np.zeros_like(u), ref.make_cfg("llf"), fs, dt, 2)
    assert rel(lv.get_state()[0], u_ref) < 1e-12


@pytest.mark.parametrize("p", [2, 3, 4])
def test_curved_sphere_freestream_preservation(gpu_lib, refmod, p):
    """Acceptance C03 (acceptance_main.cpp:264-298): ||RHS||_inf < 1e-8."""
    gpu, ref = gpu_lib, refmod
    rm, rl, mesh, ids, nodes = sphere_case(ref, p)
    fs = _fs(gpu)
    lv = gpu.GpuLevel(mesh, p, bc={"sphere": 0, "farfield": 1}, freestream=fs, curved=(ids, nodes[ids]))
    # farfield everywhere (as C03) -- freestream ghost on the sphere too
    lv2 = gpu.GpuLevel(mesh, p, bc={"sphere": 1, "farfield": 1}, freestream=fs, curved=(ids, nodes[ids]))
    r = lv2.compute_rhs(gpu.run_config("llf"), gpu.freestream_store(lv2, fs))
    assert np.max(np.abs(r)) < 1e-8, np.max(np.abs(r))


# ---- artificial viscosity on curved elements (the NACA-type configuration:
# curved wall elements + Persson-Peraire AV; BASELINE config 2 kernel proxy) --
VISC_FORCED = dict(enabled=True, eps0=0.04, kappa=4.0, s0_offset=-100.0)
VISC_RAMP = dict(enabled=True, eps0=0.3, kappa=4.0, s0_offset=0.0)


@pytest.mark.parametrize("kernel", ["row", "cta"])
@pytest.mark.parametrize("p", [2, 3, 4])
@pytest.mark.parametrize("visc,riem", [(VISC_FORCED, "llf"), (VISC_RAMP, "hllc")])
def test_curved_sphere_viscous_matches_reference(gpu_lib, refmod, p, visc, riem, kernel):
    gpu, ref = gpu_lib, refmod
    rm, rl, mesh, ids, nodes = sphere_case(ref, p)
    fs = _fs(gpu)
    lv = gpu.GpuLevel(mesh, p, bc={"sphere": 0, "farfield": 1}, freestream=fs, curved=(ids, nodes[ids]))
    lv.set_kernel_path("generic" if kernel == "cta" else "default")
    u = rl.random_admissible_store(11)
    r_ref = rl.compute_rhs(u, ref.make_cfg(riem, viscosity=visc), fs)
    eps_ref, q_ref = rl.last_viscosity()
    r_gpu = lv.compute_rhs(gpu.run_config(riem, viscosity=visc), u)
    eps = lv.viscosity()
    assert np.allclose(eps, eps_ref, rtol=1e-12, atol=1e-15)
    assert (eps > 0).any()
    q = np.stack([lv.aux_gradient(m) for m in range(3)])
    assert rel(q, q_ref) < 1e-10, rel(q, q_ref)
    assert rel(r_gpu, r_ref) < 1e-10, rel(r_gpu, r_ref)
    # two RK steps (sensor + aux gradient + viscous RHS in every stage)
    cfg_r = ref.make_cfg(riem, viscosity=visc)
    dt = 0.1 * rl.compute_timestep(u, ref.make_cfg(riem), eps_ref)
    lv.set_state(u)
    lv.rk_steps(gpu.run_config(riem, viscosity=visc), dt, 2)
    u_ref, _ = rl.rk_steps(u, np.zeros_like(u), cfg_r, fs, dt, 2)
    assert rel(lv.get_state()[0], u_ref) < 1e-12


@pytest.mark.parametrize("p", [2, 3])
def test_curved_sphere_jacobian_weighted_indicator(gpu_lib, refmod, p):
    """The physical-space (J-weighted) smoothness indicator (viscosity.cpp:28-45,
    ViscosityModel::jacobian_weighted) with per-node Jacobians on the curved
    elements, against the reference."""
    gpu, ref = gpu_lib, refmod
    rm, rl, mesh, ids, nodes = sphere_case(ref, p)
    fs = _fs(gpu)
    lv = gpu.GpuLevel(mesh, p, bc={"sphere": 0, "farfield": 1}, freestream=fs, curved=(ids, nodes[ids]))
    visc = dict(VISC_RAMP, jacobian_weighted=True, s0_offset=1.0)
    u = rl.random_admissible_store(13)
    r_ref = rl.compute_rhs(u, ref.make_cfg("llf", viscosity=visc), fs)
    eps_ref, _ = rl.last_viscosity(with_q=False)
    r_gpu = lv.compute_rhs(gpu.run_config("llf", viscosity=visc), u)
    eps = lv.viscosity()
    assert (eps_ref > 0).any()
    assert np.allclose(eps, eps_ref, rtol=1e-10, atol=1e-14)
    assert rel(r_gpu, r_ref) < 1e-10


# ---- the curved kernels at GPU-filling sizes: make_cube_mesh(n) with the
# collocation nodes moved by a smooth global map (scripts/bench_curved.py) ---
def _mapped_cube(gpu, R, n, p, amp, frac=1.0, kernel="row"):
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_curved", "scripts/bench_curved.py")
    bcm = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bcm)
    mesh = M.cube_mesh(n)
    re = R.level_reference_element(p, True)
    X = bcm.curved_nodes(mesh, re, amp)
    ids = np.arange(int(round(frac * mesh.n_owned)))
    fs = gpu.make_state(1.0, [0.4, 0.05, -0.1], 1.0)
    lv = gpu.GpuLevel(mesh, p, bc=0, freestream=fs, curved=(ids, X[ids]))
    lv.set_kernel_path("generic" if kernel == "cta" else "default")
    return lv, mesh, fs


def _smooth_state(lv, seed):
    rng = np.random.default_rng(seed)
    K, npb = lv.K, lv.n_basis
    u = np.zeros((K, 5, lv.block))
    j = lambda: (rng.random((K, npb)) - 0.5) * 0.1
    rho, vx, vy, vz, pr = 1.0 + j(), 0.3 + j(), j(), j(), 1.0 + j()
    u[:, 0, :npb], u[:, 1, :npb], u[:, 2, :npb], u[:, 3, :npb] = rho, rho * vx, rho * vy, rho * vz
    u[:, 4, :npb] = pr / 0.4 + 0.5 * rho * (vx * vx + vy * vy + vz * vz)
    return u.reshape(-1)


@pytest.mark.parametrize("p", [2, 3, 4, 5])
def test_curved_path_on_straight_elements_equals_affine_path(gpu_lib, p):
    """With the map switched off (amp 0) every element goes through the curved
    kernels (per-node metrics, per-face-node normals, per-element M_e^-1) and
    must reproduce the affine kernels (constant metrics, M^-1 folded into the
    shared operators) on the same straight mesh and quadrature."""
    gpu = gpu_lib
    from paper_1208_4772_b200 import refelem as R
    lvc, mesh, fs = _mapped_cube(gpu, R, 5, p, 0.0)
    lva = gpu.GpuLevel(mesh, p, bc=0, freestream=fs, curved_quadrature=True)
    u = _smooth_state(lva, 3)
    for riem in ("llf", "hllc"):
        cfg = gpu.run_config(riem)
        ra, rc = lva.compute_rhs(cfg, u), lvc.compute_rhs(cfg, u)
        assert rel(rc, ra) < 1e-11, (riem, rel(rc, ra))
    lva.close()
    lvc.close()


@pytest.mark.parametrize("frac", [1.0, 0.3])
def test_curved_row_kernel_matches_cta_kernel_mapped_cube(gpu_lib, frac):
    """k_rhs_rowc vs k_rhs_curved on 6,000 curved (or 30% curved + affine)
    elements, RHS and three RK steps (the affine kernels skip the all-curved
    tiles, the mixed tiles keep their affine rows)."""
    gpu = gpu_lib
    from paper_1208_4772_b200 import refelem as R
    out = {}
    for kernel in ("row", "cta"):
        lv, mesh, fs = _mapped_cube(gpu, R, 10, 4, 0.02, frac, kernel)
        u = _smooth_state(lv, 5)
        cfg = gpu.run_config("llf")
        r = lv.compute_rhs(cfg, u)
        lv.set_state(u)
        dt = 0.3 * lv.compute_timestep(cfg)
        lv.rk_steps(cfg, dt, 3)
        out[kernel] = (r, lv.get_state()[0])
        lv.close()
    assert rel(out["row"][0], out["cta"][0]) < 1e-11
    assert rel(out["row"][1], out["cta"][1]) < 1e-12
