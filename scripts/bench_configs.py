"""Throughput of the BASELINE.json configs other than the headline (which is
bench.py): the GPU path (device-resident cdg_gpu_rk_steps) against the
reference's own rk_step (oracle/_ref, all host threads) on the SAME level and
state. Writes one JSON object per config to stdout.

  C1  isentropic vortex on the periodic box periodic_cube(11) = 7,986 affine
      tets, P=3, LLF (cases.py; the reference's kernels on the same periodic
      coupling, oracle/ref_periodic.cpp)
  C2  NACA0012 O-grid (cases.naca0012_map), every element curved, P=4,
      M=0.8, alpha=1.25 deg, HLLC, Persson-Peraire AV (ramp)
  C3  cylinder O-grid (cases.cylinder_map), every element curved, M=0.3,
      P=1..6, LLF
  plus GPU-only lines of C2 / C3 at a GPU-filling size.

usage: python scripts/bench_configs.py [--quick]
"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import ref  # noqa: E402
from paper_1208_4772_b200 import gpu, mesh as M  # noqa: E402

QUICK = "--quick" in sys.argv


def smooth_state(rl):
    """test_solver.cpp:44-59: rho = 1 + 0.1 sin(2x) cos(y), v = (0.3+0.05z,
    0.02x, -0.04y), p = 1 + 0.08 cos(x+y+z), gamma = 1.4, at the level's nodes."""
    nodes, _ = rl.nodes()
    x, y, z = nodes[..., 0], nodes[..., 1], nodes[..., 2]
    rho = 1.0 + 0.1 * np.sin(2 * x) * np.cos(y)
    vx, vy, vz = 0.3 + 0.05 * z, 0.02 * x, -0.04 * y
    p = 1.0 + 0.08 * np.cos(x + y + z)
    u = np.zeros((rl.K, 5, rl.block))
    npb = nodes.shape[1]
    u[:, 0, :npb] = rho
    u[:, 1, :npb] = rho * vx
    u[:, 2, :npb] = rho * vy
    u[:, 3, :npb] = rho * vz
    u[:, 4, :npb] = p / 0.4 + 0.5 * rho * (vx * vx + vy * vy + vz * vz)
    return u.reshape(-1)


def gpu_mesh(rm, tags):
    ex = rm.export()
    lut = {q[0] + 3 * q[1] + 9 * q[2]: i for i, q in enumerate(M.PERMS)}
    perm = ex["perm"]
    code = np.where(perm >= 0, np.vectorize(lambda v: lut.get(int(v), 0))(perm), -1)
    mesh = M.from_arrays(ex["vertices"], ex["tets"], ex["neighbor"], ex["neighbor_face"], code,
                         np.where(ex["neighbor"] >= 0, -1, ex["bnd_tag"]))
    mesh.tags = tags
    return mesh


def time_gpu(lv, cfg, u, dt, steps):
    lv.set_state(u)
    lv.rk_steps(cfg, dt, 2)  # warm-up (graph capture)
    lv.set_state(u)
    t0 = time.perf_counter()
    lv.rk_steps(cfg, dt, steps)
    return (time.perf_counter() - t0) / steps


def time_cpu(rl, cfg, fs, u, dt, steps):
    res = np.zeros_like(u)
    rl.rk_steps(u, res, cfg, fs, dt, 1)
    t0 = time.perf_counter()
    rl.rk_steps(u, res, cfg, fs, dt, steps)
    return (time.perf_counter() - t0) / steps


def run(name, rm, rl, lv, cfg_g, cfg_r, fs, u, p, gpu_steps, cpu_steps, note):
    dt = 0.25 * rl.compute_timestep(u, cfg_r)
    u_g = None
    tg = time_gpu(lv, cfg_g, u, dt, gpu_steps)
    tc = time_cpu(rl, cfg_r, fs, u, dt, cpu_steps)
    # parity of the timed trajectory's first step
    lv.set_state(u)
    lv.rk_steps(cfg_g, dt, 1)
    u_g = lv.get_state()[0]
    u_r, _ = rl.rk_steps(u, np.zeros_like(u), cfg_r, fs, dt, 1)
    err = float(np.max(np.abs(u_g - u_r)) / np.max(np.abs(u_r)))
    dofs = rl.K * lv.n_basis * 5 * 5
    out = {"config": name, "elements": rl.K, "p": p, "gpu_dof_updates_per_s": dofs / tg,
           "cpu_dof_updates_per_s": dofs / tc, "speedup": tc / tg, "gpu_ms_per_step": tg * 1e3,
           "cpu_ms_per_step": tc * 1e3, "cpu_threads": ref.num_threads(0), "step1_rel_err_vs_reference": err,
           "note": note}
    print(json.dumps(out), flush=True)


def body_level(mapping, dims, p, fs, with_ref=True):
    from paper_1208_4772_b200 import cases, refelem as R
    m, par = cases.ogrid_mesh(*dims, mapping)
    re = R.level_reference_element(p, True)
    nodes = cases.ogrid_nodes(par, re, mapping)
    rm = rl = None
    if with_ref:
        rm = ref.Mesh("arrays", arrays=cases.reference_arrays(m))
        rm.set_curved(p, np.arange(m.n_owned), nodes)
        rl = ref.Level(rm, p, bc_wall=0, bc_far=1)
        nodes = rl.nodes()[0]
    lv = gpu.GpuLevel(m, p, bc={"wall": "slip_wall", "farfield": "farfield", "symmetry": "symmetry"},
                      freestream=fs, curved=(np.arange(m.n_owned), nodes), re=re)
    return m, rm, rl, lv


def near_freestream(K, block, npb, fs, seed, amp=0.02):
    """freestream plus a small random perturbation of every nodal value
    (admissible; a state the body flows evolve from without blowing up)."""
    rng = np.random.default_rng(seed)
    u = np.zeros((K, 5, block))
    u[:, :, :npb] = fs[None, :, None] * (1.0 + amp * (rng.random((K, 5, npb)) - 0.5))
    u[:, 3, :npb] = fs[3] + amp * (rng.random((K, npb)) - 0.5)
    return u.reshape(-1)


def gpu_only(name, lv, cfg, u, steps, note):
    import torch
    lv.set_state(u)
    dt = 0.25 * lv.compute_timestep(gpu.run_config("llf"))
    lv.rk_steps(cfg, dt, 2)
    torch.cuda.synchronize()
    ext = torch.cuda.ExternalStream(lv.stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ext)
    lv.rk_steps(cfg, dt, steps)
    e1.record(ext)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) * 1e-3 / steps
    print(json.dumps({"config": name, "elements": lv.K, "p": lv.degree,
                      "gpu_dof_updates_per_s": lv.K * lv.n_basis * 25 / t, "gpu_ms_per_step": t * 1e3,
                      "note": note}), flush=True)


def main():
    from paper_1208_4772_b200 import cases
    if "--large-only" in sys.argv:
        return large()
    ref.num_threads(0)
    nthreads = ref.num_threads(__import__("os").cpu_count() or 1)
    # C1: periodic isentropic vortex
    L = 10.0
    mv = cases.periodic_cube(11, L)
    rm = ref.Mesh("cube", 11, scale=L)
    rl = ref.Level(rm, 3, bc_wall=0, bc_far=1)
    rl.make_periodic((L, L, L))
    fsv = cases.freestream(0.0)
    lv = gpu.GpuLevel(mv, 3, freestream=fsv)
    run("C1 isentropic vortex, periodic_cube(11), P=3, LLF", rm, rl, lv, gpu.run_config("llf"), ref.make_cfg("llf"),
        fsv, cases.vortex_store(mv, lv.re, lv.block), 3, 200, 3 if QUICK else 10,
        f"reference rk_step on {nthreads} host threads, periodic coupling (oracle/ref_periodic.cpp)")
    lv.close()
    # C2: NACA0012, M=0.8, alpha=1.25, P=4 curved, HLLC + AV (ramp)
    fs2 = cases.freestream(0.8, 1.25)
    visc = dict(enabled=True, eps0=0.02, kappa=4.0, s0_offset=2.0)
    m, rm, rl, lv = body_level(cases.naca0012_map(), (64, 12, 1), 4, fs2)
    run("C2 NACA0012 O-grid, all curved, P=4, M=0.8 a=1.25, HLLC + AV ramp", rm, rl, lv,
        gpu.run_config("hllc", viscosity=visc), ref.make_cfg("hllc", viscosity=visc), fs2,
        near_freestream(rl.K, rl.block, rl.n_basis, fs2, 5), 4, 20, 2 if QUICK else 3, "Persson-Peraire sensor + aux gradient + viscous "
                                                                "flux each stage")
    lv.close()
    # C3: cylinder, P = 1..6
    fs3 = cases.freestream(0.3)
    for p in ([4] if QUICK else [1, 2, 3, 4, 5, 6]):
        m, rm, rl, lv = body_level(cases.cylinder_map(), (32, 8, 2), p, fs3)
        run(f"C3 cylinder O-grid, all curved, P={p}, LLF", rm, rl, lv, gpu.run_config("llf"), ref.make_cfg("llf"),
            fs3, near_freestream(rl.K, rl.block, rl.n_basis, fs3, 5), p, 100, 2 if QUICK else 5,
            f"{rl.K} curved elements")
        lv.close()
    large()


def large():
    """C2 / C3 at GPU-filling sizes (GPU only)."""
    from paper_1208_4772_b200 import cases
    fs2, fs3 = cases.freestream(0.8, 1.25), cases.freestream(0.3)
    visc = dict(enabled=True, eps0=0.02, kappa=4.0, s0_offset=2.0)
    m, _, _, lv = body_level(cases.naca0012_map(), (256, 48, 4), 4, fs2, with_ref=False)
    u = near_freestream(lv.K, lv.block, lv.n_basis, fs2, 5)
    gpu_only("C2 NACA0012 O-grid 256x48x4, P=4, HLLC + AV ramp", lv, gpu.run_config("hllc", viscosity=visc), u,
             5, "all elements curved")
    gpu_only("C2 NACA0012 O-grid 256x48x4, P=4, HLLC inviscid", lv, gpu.run_config("hllc"), u, 5,
             "all elements curved")
    lv.close()
    m, _, _, lv = body_level(cases.cylinder_map(), (256, 48, 4), 4, fs3, with_ref=False)
    gpu_only("C3 cylinder O-grid 256x48x4, P=4, LLF", lv, gpu.run_config("llf"),
             near_freestream(lv.K, lv.block, lv.n_basis, fs3, 5),
             5, "all elements curved")
    lv.close()


if __name__ == "__main__":
    main()
