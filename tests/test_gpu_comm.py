"""The library's multi-rank driver (cdg_gpu_comm_*, csrc/cdg_comm.cuh) on ONE
GPU: R shards driven in-process (peer copies between the shards' buffers,
the same stage sequence the NCCL transport runs), inviscid, viscous (the
reference's barrier-separated sensor -> aux gradient -> RHS phases with the
sqrt(eps) and q-trace exchanges and the all-rank viscous gate,
solver.cpp:239-321,438-453) and curved shards (the curved tiles split into
interior / halo as well). Per-element arithmetic does not depend on the
partition, so R-shard states must be BITWISE equal to the single-level run;
the global dt (MIN) and inf-residual (MAX) too; the l2 residual to rounding."""
import numpy as np
import pytest

from paper_1208_4772_b200 import mesh as M, partition as P

pytestmark = pytest.mark.gpu

FORCED = dict(enabled=True, eps0=0.01, kappa=4.0, s0_offset=-100.0)   # eps = eps0 everywhere
RAMP = dict(enabled=True, eps0=0.02, kappa=4.0, s0_offset=2.0)        # mixed eps (ramp + zero)


def _levels(gpu, g, p, parts, owned, fs, u0, curved_frac, bc=1):
    levels = []
    for pt, own in zip(parts, owned):
        curved = None
        if curved_frac:
            re = gpu.R.level_reference_element(p, True)
            ids = np.nonzero(own < int(curved_frac * g.n_owned))[0]
            curved = (ids, M.warped_nodes(pt.mesh, re, ids=ids))
        L = gpu.GpuLevel(pt.mesh, p, bc=bc, freestream=fs, curved=curved)
        L.set_state(np.ascontiguousarray(u0[own]).reshape(-1))
        L.halo_define(pt.peers)
        levels.append(L)
    return levels


def _single(gpu, g, p, fs, curved_frac, bc=1):
    curved = None
    if curved_frac:
        re = gpu.R.level_reference_element(p, True)
        ids = np.arange(int(curved_frac * g.n_owned))
        curved = (ids, M.warped_nodes(g, re, ids=ids))
    return gpu.GpuLevel(g, p, bc=bc, freestream=fs, curved=curved)


def _parts(g, n, R, kind):
    if kind == "slab":
        parts = [P.rank_part(n, R, r) for r in range(R)]
    else:
        owner = P.rcb_owner(g, R)
        parts = [P.mesh_part(g, owner, r) for r in range(R)]
    owned = [np.arange(*pt.elem_range) if pt.owned is None else pt.owned for pt in parts]
    return parts, owned


@pytest.mark.parametrize("R,p,kind,riemann,visc,curved", [
    (2, 4, "slab", "llf", None, 0.0), (3, 4, "rcb", "hllc", None, 0.0), (4, 3, "rcb", "llf", None, 0.0),
    (2, 2, "slab", "llf", FORCED, 0.0), (3, 3, "rcb", "hllc", FORCED, 0.0), (3, 2, "rcb", "llf", RAMP, 0.0),
    (3, 4, "rcb", "llf", None, 1.0), (2, 3, "rcb", "hllc", None, 0.4), (3, 3, "rcb", "llf", FORCED, 0.4),
    (2, 4, "slab", "llf", FORCED, 1.0)])
def test_comm_rk_steps_bitwise_equal(gpu_lib, R, p, kind, riemann, visc, curved):
    gpu = gpu_lib
    n = 4
    fs = gpu.make_state(1.0, [0.3, 0.1, 0.0], 1.0)
    cfg = gpu.run_config(riemann, viscosity=visc)
    g = M.cube_mesh(n)
    lv = _single(gpu, g, p, fs, curved)
    u0 = gpu.random_admissible_store(lv, seed=23)
    lv.set_state(u0)
    dt = 0.1 * lv.compute_timestep(gpu.run_config(riemann))
    lv.rk_steps(cfg, dt, 3)
    u_ref = lv.get_state()[0].reshape(lv.K, 5, lv.block)
    u0 = u0.reshape(lv.K, 5, lv.block)
    parts, owned = _parts(g, n, R, kind)
    levels = _levels(gpu, g, p, parts, owned, fs, u0, curved)
    comm = gpu.GpuComm.local(levels)
    comm.rk_steps(cfg, dt, 3)
    out = np.empty_like(u_ref)
    for L, own in zip(levels, owned):
        out[own] = L.get_state()[0].reshape(L.K, 5, L.block)
    assert np.array_equal(out, u_ref), f"max diff {np.max(np.abs(out - u_ref)):.3e}"
    assert comm.exchange_count() == 3 * 5 * (2 if visc else 1)
    if visc:
        for L, own in zip(levels, owned):
            assert np.array_equal(L.viscosity(), lv.viscosity()[own])
    comm.close()


def test_comm_reductions_and_run_level(gpu_lib):
    """global dt (MIN), residual (inf: MAX, bitwise; l2: SUM, to rounding) and a
    run_steady level through cdg_gpu_comm_run_level == the single level's."""
    gpu = gpu_lib
    n, p, R = 4, 2, 3
    fs = gpu.make_state(1.0, [0.3, 0.1, 0.0], 1.0)
    cfg = gpu.run_config("llf", cfl=0.3)
    g = M.cube_mesh(n)
    lv = _single(gpu, g, p, fs, 0.0)
    u0 = gpu.random_admissible_store(lv, seed=5).reshape(lv.K, 5, lv.block)
    lv.set_state(u0.reshape(-1))
    parts, owned = _parts(g, n, R, "rcb")
    levels = _levels(gpu, g, p, parts, owned, fs, u0, 0.0)
    comm = gpu.GpuComm.local(levels)
    assert comm.compute_timestep(cfg) == lv.compute_timestep(cfg)
    dt = lv.compute_timestep(cfg)
    lv.snapshot()
    comm.snapshot()
    lv.rk_steps(cfg, dt, 1)
    comm.rk_steps(cfg, dt, 1)
    assert comm.residual(dt, "inf") == lv.residual(dt, "inf")
    assert comm.residual(dt, "l2") == pytest.approx(lv.residual(dt, "l2"), rel=1e-13)
    sp = gpu.SteadyParams(40, -1, 10, 0, 1e-30, 0.0, p)
    rows_1, _ = lv.run_level(cfg, sp)
    rows_r, _ = comm.run_level(cfg, sp)
    assert np.array_equal(rows_1, rows_r)
    out = np.empty((lv.K, 5, lv.block))
    for L, own in zip(levels, owned):
        out[own] = L.get_state()[0].reshape(L.K, 5, L.block)
    assert np.array_equal(out, lv.get_state()[0].reshape(lv.K, 5, lv.block))
    comm.close()


def test_comm_numerics_error_reaches_caller(gpu_lib):
    """An inadmissible state on one shard aborts the multi-rank step with the
    reference's NumericsError (solver.cpp:54-69)."""
    gpu = gpu_lib
    n, p, R = 3, 2, 2
    fs = gpu.make_state(1.0, [0.3, 0.1, 0.0], 1.0)
    g = M.cube_mesh(n)
    lv = _single(gpu, g, p, fs, 0.0)
    u0 = gpu.random_admissible_store(lv, seed=5).reshape(lv.K, 5, lv.block)
    u0[7, 0, :] = -1.0
    parts, owned = _parts(g, n, R, "slab")
    levels = _levels(gpu, g, p, parts, owned, fs, u0, 0.0)
    comm = gpu.GpuComm.local(levels)
    with pytest.raises(gpu.NumericsError, match="inadmissible"):
        comm.rk_steps(gpu.run_config("llf"), 1e-3, 1)
    comm.close()


def test_comm_nccl_single_rank_matches_level(gpu_lib):
    """The NCCL transport's plumbing on a one-GPU box: libnccl.so.2 resolved
    at run time, unique id, a 1-rank communicator over a whole-mesh shard
    (no peers), the all-reduces of the viscous gate, dt, residual and the
    error flag. Bitwise equal to the level's own rk_steps / run_level."""
    gpu = gpu_lib
    fs = gpu.make_state(1.0, [0.3, 0.1, 0.0], 1.0)
    g = M.cube_mesh(4)
    a = gpu.GpuLevel(g, 3, bc=1, freestream=fs)
    b = gpu.GpuLevel(g, 3, bc=1, freestream=fs)
    u0 = gpu.random_admissible_store(a, seed=9)
    b.halo_define([])
    comm = gpu.GpuComm.nccl(b, gpu.GpuComm.unique_id(), 0, 1)
    for visc in (None, FORCED):
        cfg = gpu.run_config("hllc", viscosity=visc)
        for lv in (a, b):
            lv.set_state(u0)
        dt = 0.1 * a.compute_timestep(gpu.run_config("hllc"))
        assert comm.compute_timestep(gpu.run_config("hllc")) == a.compute_timestep(gpu.run_config("hllc"))
        a.rk_steps(cfg, dt, 2)
        comm.rk_steps(cfg, dt, 2)
        assert np.array_equal(a.get_state()[0], b.get_state()[0])
    sp = gpu.SteadyParams(20, -1, 10, 1, 1e-30, 0.0, 3)
    cfg = gpu.run_config("llf", cfl=0.3)
    rows_a, _ = a.run_level(cfg, sp)
    rows_b, _ = comm.run_level(cfg, sp)
    assert np.allclose(rows_a, rows_b, rtol=1e-13, atol=0)  # l2 residual: the same partial sums
    comm.close()
