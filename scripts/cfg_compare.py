"""Run a few RK steps of the bench workload (smaller mesh) under the kernel
config CDG_KCFG (env) and save the final state, so configs can be compared
on the GPU box. usage: python scripts/cfg_compare.py out.npy [n] [steps]"""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_1208_4772_b200 import gpu, mesh as M

out = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
fs = gpu.make_state(1.0, [0.35, 0.0, 0.0], 1.0)
lv = gpu.GpuLevel(M.cube_mesh(n), 4, bc=0, freestream=fs)
u0 = gpu.random_admissible_store(lv, seed=42)
lv.set_state(u0)
cfg = gpu.run_config("llf")
dt = 0.5 * lv.compute_timestep(cfg)
t0 = time.perf_counter()
lv.rk_steps(cfg, dt, steps)
u, res = lv.get_state()
print(f"K={lv.K} steps={steps} {time.perf_counter()-t0:.3f}s max|u|={np.abs(u).max():.6g} finite={np.isfinite(u).all()}")
np.save(out, u)
