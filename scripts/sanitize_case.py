"""Small cases for compute-sanitizer (racecheck / synccheck / memcheck /
initcheck) over the hot kernels: the fused P=4 kernel (fused traces, HLLC
and LLF), the p=1 neighbour-state kernel and the curved kernel with the grid
capped at 2 CTAs, so every CTA runs several tiles through the grid-stride
loop (the cross-tile shared-memory restaging and the fused-trace double
buffer are exercised), plus the curved viscous path and a 2-shard multi-rank
step.  usage: compute-sanitizer --tool racecheck python scripts/sanitize_case.py"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1208_4772_b200 import gpu, mesh as M, partition as P, refelem as R  # noqa: E402

fs = gpu.make_state(1.0, [0.3, 0.1, 0.0], 1.0)
m = M.cube_mesh(3)
for riemann in ("llf", "hllc"):
    lv = gpu.GpuLevel(m, 4, bc=0, freestream=fs)
    lv.set_max_ctas(2)
    lv.set_state(gpu.random_admissible_store(lv, seed=3))
    cfg = gpu.run_config(riemann)
    dt = 0.2 * lv.compute_timestep(cfg)
    lv.rk_steps(cfg, dt, 1)
    lv.compute_rhs(cfg)
    print("affine p=4", riemann, "fused", lv.fused_traces(), flush=True)
    lv.close()
for riemann in ("llf", "hllc"):  # p=1: the neighbour-state kernel (ping-pong state, no traces)
    lv = gpu.GpuLevel(m, 1, bc=1, freestream=fs)
    lv.set_max_ctas(2)
    lv.set_state(gpu.random_admissible_store(lv, seed=6))
    cfg = gpu.run_config(riemann)
    dt = 0.2 * lv.compute_timestep(cfg)
    lv.rk_steps(cfg, dt, 3)
    print("affine p=1", riemann, lv.rhs_kernel(), flush=True)
    lv.close()
re = R.level_reference_element(4, True)
ids = np.arange(m.n_owned)
X = M.warped_nodes(m, re)
for visc in (None, dict(enabled=True, eps0=0.01, kappa=4.0, s0_offset=-100.0)):
    lv = gpu.GpuLevel(m, 4, bc=0, freestream=fs, curved=(ids, X), re=re)
    lv.set_max_ctas(2)
    lv.set_state(gpu.random_admissible_store(lv, seed=4))
    cfg = gpu.run_config("llf", viscosity=visc)
    dt = 0.1 * lv.compute_timestep(gpu.run_config("llf"))
    lv.rk_steps(cfg, dt, 1)
    print("curved p=4 visc", visc is not None, flush=True)
    lv.close()
parts = [P.rank_part(3, 2, r) for r in range(2)]
levels = []
for pt in parts:
    L_ = gpu.GpuLevel(pt.mesh, 3, bc=1, freestream=fs)
    L_.set_state(gpu.random_admissible_store(L_, seed=5))
    L_.halo_define(pt.peers)
    levels.append(L_)
comm = gpu.GpuComm.local(levels)
comm.rk_steps(gpu.run_config("llf"), 1e-3, 1)
print("comm 2 shards ok", flush=True)
