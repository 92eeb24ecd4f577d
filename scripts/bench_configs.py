"""Throughput of the BASELINE.json configs other than the headline (which is
bench.py): the GPU path (device-resident cdg_gpu_rk_steps) against the
reference's own rk_step (oracle/_ref, all host threads) on the SAME level and
state. Writes one JSON object per config to stdout.

  C1  make_cube_mesh(11) = 7,986 affine tets, P=3, LLF, farfield, smooth state
      (test_solver.cpp:44-59) -- the "isentropic vortex, ~8k affine, P=3" slot
  C2  curved sphere shell (make_sphere_shell_mesh(1,8,2,5) curved at P=4 by the
      reference's elasticity pipeline, 40% curved), HLLC, Persson-Peraire AV
      forced on -- the NACA0012 "curved P=4 + AV" kernel proxy
  C3  the same curved sphere at P=1..6, LLF -- the cylinder P=1..6 slot

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


def main():
    ref.num_threads(0)
    nthreads = ref.num_threads(__import__("os").cpu_count() or 1)
    fs = gpu.make_state(1.0, [0.4, 0.05, -0.1], 1.0)
    # C1
    rm = ref.Mesh("cube", 11)
    rl = ref.Level(rm, 3, bc_wall=1, bc_far=1)
    lv = gpu.GpuLevel(gpu_mesh(rm, ["wall", "farfield"]), 3, bc={"wall": 1, "farfield": 1}, freestream=fs)
    run("C1 cube(11) P=3 LLF farfield smooth", rm, rl, lv, gpu.run_config("llf"), ref.make_cfg("llf"), fs,
        smooth_state(rl), 3, 200, 3 if QUICK else 10, f"reference rk_step on {nthreads} host threads")
    # C2 / C3: the curved sphere at P (sphere_m038-like freestream)
    c = np.sqrt(1.4)
    fs2 = gpu.make_state(1.0, [0.38 * c, 0.0, 0.0], 1.0)
    visc = dict(enabled=True, eps0=0.3, kappa=4.0, s0_offset=-100.0)
    for p in ([4] if QUICK else [1, 2, 3, 4, 5]):
        rmc = ref.Mesh("sphere_curved", sphere=(2, 5, p, p))
        rlc = ref.Level(rmc, p, bc_wall=0, bc_far=1)
        nodes, curved = rlc.nodes()
        ids = np.nonzero(curved)[0]
        mesh = gpu_mesh(rmc, ["sphere", "farfield"])
        lvc = gpu.GpuLevel(mesh, p, bc={"sphere": 0, "farfield": 1}, freestream=fs2, curved=(ids, nodes[ids]))
        u = rlc.random_admissible_store(5)
        run(f"C3 curved sphere P={p} LLF", rmc, rlc, lvc, gpu.run_config("llf"), ref.make_cfg("llf"), fs2, u, p,
            100, 2 if QUICK else 5, f"{len(ids)} of {rlc.K} elements curved")
        if p == 4:
            run("C2 curved sphere P=4 HLLC + AV (NACA proxy)", rmc, rlc, lvc,
                gpu.run_config("hllc", viscosity=visc), ref.make_cfg("hllc", viscosity=visc), fs2, u, p,
                50, 2 if QUICK else 3, "AV forced on every element (s0_offset=-100): sensor + aux gradient + "
                                       "viscous flux each stage")
        lvc.close()


if __name__ == "__main__":
    main()
