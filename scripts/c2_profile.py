"""C2 proxy (curved sphere P=4, HLLC, AV forced) -- a few RK steps for ncu launch lists."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.argv.append("--quick")
from oracle import ref  # noqa: E402
from paper_1208_4772_b200 import gpu  # noqa: E402
import importlib.util
spec = importlib.util.spec_from_file_location("bc", "scripts/bench_configs.py")
bc = importlib.util.module_from_spec(spec)
spec.loader.exec_module(bc)
p = 4
c = np.sqrt(1.4)
fs2 = gpu.make_state(1.0, [0.38 * c, 0.0, 0.0], 1.0)
rmc = ref.Mesh("sphere_curved", sphere=(2, 5, p, p))
rlc = ref.Level(rmc, p, bc_wall=0, bc_far=1)
nodes, curved = rlc.nodes()
ids = np.nonzero(curved)[0]
lvc = gpu.GpuLevel(bc.gpu_mesh(rmc, ["sphere", "farfield"]), p, bc={"sphere": 0, "farfield": 1}, freestream=fs2,
                   curved=(ids, nodes[ids]))
u = rlc.random_admissible_store(5)
visc = dict(enabled=True, eps0=0.3, kappa=4.0, s0_offset=-100.0)
cfg = gpu.run_config("hllc", viscosity=visc)
lvc.set_state(u)
dt = 0.25 * lvc.compute_timestep(gpu.run_config("hllc"))
lvc.rk_steps(cfg, dt, 2)
print("ok")
