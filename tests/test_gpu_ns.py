"""The neighbour-state kernel (cdg_ns.cuh; the default p=1 path on
single-shard straight meshes): no stored traces -- own and neighbour face
states interpolated from the nodal states -- and a ping-pong state buffer.

It sums the face interpolation in another order than the DMMA trace kernel,
so it agrees with the stored-trace path ("traced", the reference's
interpolate_to_faces + node-map gather, solver.cpp:200-208, 415-457) to
rounding, and with the reference's rk_step (oracle) within the north_star
tolerance. The buffer swap must be invisible to every other entry point:
switching paths mid-run, viscous steps, the device driver loop and the
state accessors all see the current state.

Tolerances: 1e-13 normwise-relative per step against the traced path
(rounding of two 4-term sums per face node), 1e-11 against the oracle after
3 steps (test_gpu_gridstride.py)."""
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


def _drop_last(m, k):
    """cube mesh without its last k elements (their faces become walls): an
    element count that is not a multiple of the 16-element tile and a tail
    tile with an odd number of elements (half-valid metric piece)."""
    K = m.n_owned - k
    nb = m.neighbor[:K].copy()
    nf = m.neighbor_face[:K].copy()
    code = m.perm_code[:K].copy()
    tag = m.boundary_tag[:K].copy()
    gone = nb >= K
    nb[gone], nf[gone], code[gone], tag[gone] = -1, -1, -1, 0
    return M.from_arrays(m.vertices, m.tets[:K], nb, nf, code, tag)


def _levels(gpu, m, p, bc, fs):
    re = R.get_reference_element(p)
    a = gpu.GpuLevel(m, p, bc=bc, freestream=fs, re=re)
    b = gpu.GpuLevel(m, p, bc=bc, freestream=fs, re=re)
    b.set_kernel_path("traced")
    return re, a, b


@pytest.mark.parametrize("riemann", ["llf", "hllc"])
@pytest.mark.parametrize("bc", [0, 1, 2])
@pytest.mark.parametrize("drop", [0, 3])
def test_ns_matches_traced_path_and_oracle(gpu_lib, riemann, bc, drop):
    gpu = gpu_lib
    m = M.cube_mesh(5, scale=2.0)
    if drop:
        m = _drop_last(m, drop)
    fs = _fs(gpu)
    re, a, b = _levels(gpu, m, 1, bc, fs)
    assert a.K % 16 != 0 and (not drop or (a.K % 16) % 2 == 1)
    cfg = gpu.run_config(riemann)
    u0 = gpu.random_admissible_store(a, seed=11 + bc)
    a.set_state(u0)
    b.set_state(u0)
    dt = 0.3 * a.compute_timestep(cfg)
    for step in range(5):
        a.rk_steps(cfg, dt, 1)
        b.rk_steps(cfg, dt, 1)
        ua, ra = a.get_state()
        ub, rb = b.get_state()
        assert rel(ua, ub) < 1e-13 and rel(ra, rb) < 1e-12, (step, rel(ua, ub), rel(ra, rb))
        pad = ua.reshape(a.K, 5, a.block)[:, :, a.n_basis:]
        assert np.all(pad == 0.0)
    a.set_state(u0)
    a.rk_steps(cfg, dt, 3)
    ol = port.OracleLevel(m, re, bc=bc, freestream=fs)
    u_ref, _ = ol.rk_steps(u0, np.zeros_like(u0), cfg, dt, 3)
    assert rel(a.get_state()[0], u_ref) < 1e-11, rel(a.get_state()[0], u_ref)
    a.close()
    b.close()


def test_ns_buffer_swap_is_invisible(gpu_lib):
    """odd / even step counts (the state changes buffer every step), a switch
    to the stored-trace path and back, a viscous step, the device driver loop
    and set_state in between: the same states as a level that never used the
    neighbour-state kernel."""
    gpu = gpu_lib
    m = M.cube_mesh(5, scale=2.0)
    fs = _fs(gpu)
    _, a, b = _levels(gpu, m, 1, 1, fs)
    cfg = gpu.run_config("hllc")
    visc = gpu.run_config("hllc", viscosity=dict(enabled=True, eps0=0.02, kappa=4.0, s0_offset=-100.0))
    u0 = gpu.random_admissible_store(a, seed=3)
    a.set_state(u0)
    b.set_state(u0)
    dt = 0.2 * b.compute_timestep(cfg)

    def both(fn):
        fn(a)
        fn(b)
        assert rel(a.get_state()[0], b.get_state()[0]) < 1e-12

    both(lambda L: L.rk_steps(cfg, dt, 3))          # a: state now in the second buffer
    a.set_kernel_path("traced")
    both(lambda L: L.rk_steps(cfg, dt, 2))          # stored traces from the swapped state
    a.set_kernel_path("default")
    both(lambda L: L.rk_steps(cfg, dt, 1))
    both(lambda L: L.rk_steps(visc, 0.5 * dt, 1))   # viscous stages (CTA kernels) on it
    both(lambda L: L.rk_steps(cfg, dt, 2))
    assert a.compute_timestep(cfg) == pytest.approx(b.compute_timestep(cfg), rel=1e-13)
    u1 = gpu.random_admissible_store(a, seed=4)
    both(lambda L: L.set_state(u1))
    both(lambda L: L.rk_steps(cfg, dt, 1))
    sp = gpu.SteadyParams(12, -1, 4, 0, 1e-30, 0.0, 1)
    rows_a, _ = a.run_level(cfg, sp)
    rows_b, _ = b.run_level(cfg, sp)
    # rows (iteration, dt, residual): same checks, time steps and residuals to rounding
    assert len(rows_a) == len(rows_b) == 3 and np.array_equal(rows_a[:, 0], rows_b[:, 0])
    assert np.allclose(rows_a[:, 1], rows_b[:, 1], rtol=1e-12, atol=0)
    assert np.allclose(rows_a[:, 2], rows_b[:, 2], rtol=1e-8, atol=0)
    assert rel(a.get_state()[0], b.get_state()[0]) < 1e-11
    a.close()
    b.close()
