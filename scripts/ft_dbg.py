import sys; sys.path.insert(0, ".")
import numpy as np
from paper_1208_4772_b200 import gpu, mesh as M
fs = gpu.make_state(1.0, [0.4, 0.05, -0.1], 1.0)
lv = gpu.GpuLevel(M.cube_mesh(2), 4, bc=1, freestream=fs)
u0 = gpu.random_admissible_store(lv, seed=7)
lv.set_state(u0)
cfg = gpu.run_config("llf")
lv.rk_steps(cfg, 1e-3, 1)
print("ok", np.abs(lv.get_state()[0]).max())
