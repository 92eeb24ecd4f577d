"""BASELINE config 1 accuracy sweep: periodic isentropic vortex advected to
t = T on periodic_cube(n) (L = 10), p = 1..P; prints the L2 and max density
error against the exact (translated) vortex and the observed h-order.

    python scripts/vortex_accuracy.py [--ns 6 9 12] [--pmax 4] [--T 1.0]"""
import argparse
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1208_4772_b200 import cases, gpu  # noqa: E402

L = 10.0
FS = np.array([1.0, 1.0, 1.0, 0.0, 1.0 / 0.4 + 1.0])


def run(n, p, T, cfl=0.4):
    m = cases.periodic_cube(n, L)
    lv = gpu.GpuLevel(m, p, freestream=FS)
    lv.set_state(cases.vortex_store(m, lv.re, lv.block))
    cfg = gpu.run_config("llf", cfl=cfl)
    nsteps = int(np.ceil(T / lv.compute_timestep(cfg)))
    lv.rk_steps(cfg, T / nsteps, nsteps)
    u = lv.get_state()[0].reshape(lv.K, 5, lv.block)[:, 0, : lv.n_basis]
    exact = cases.isentropic_vortex(cases.element_nodes(m, lv.re), T)[..., 0]
    d = u - exact
    lv.close()
    return float(np.sqrt(np.mean(d * d))), float(np.max(np.abs(d))), nsteps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", type=int, nargs="+", default=[6, 9, 12])
    ap.add_argument("--pmax", type=int, default=4)
    ap.add_argument("--T", type=float, default=1.0)
    a = ap.parse_args()
    for p in range(1, a.pmax + 1):
        prev = None
        for n in a.ns:
            l2, mx, ns = run(n, p, a.T)
            order = None if prev is None else float(np.log(prev[1] / l2) / np.log(n / prev[0]))
            print(json.dumps({"p": p, "n": n, "tets": 6 * n ** 3, "steps": ns, "l2_rho": l2, "max_rho": mx,
                              "h_order_l2": order}), flush=True)
            prev = (n, l2)


if __name__ == "__main__":
    main()
