"""Generate the golden fixtures from the REAL reference (oracle/_ref: the
unmodified /root/reference/proj/core sources compiled in place). Run here,
where /root/reference exists; the .npz outputs are committed so the checks
travel to the GPU box without the reference.

    python tests/golden/make_golden.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import ref  # noqa: E402
from paper_1208_4772_b200 import refelem as R  # noqa: E402

OUT = Path(__file__).resolve().parent
FS = np.array([1.0, 0.4, 0.05, -0.1, 1.0 / 0.4 + 0.5 * (0.16 + 0.0025 + 0.01)])  # test_solver.cpp:24


def tables():
    for p in range(1, 9):
        for curved in (False, True):
            if curved and R.curved_volume_strength(p) == 2 * p + 1 and R.curved_face_strength(p) == 2 * p:
                continue
            co = (R.curved_volume_strength(p), R.curved_face_strength(p)) if curved else (0, 0)
            t = ref.refelem_tables(p, *co)
            name = f"refelem_p{p}{'_curved' if curved else ''}.npz"
            if p >= 5:
                # fingerprints only (full tables would be megabytes): nodes and
                # weights in full, matrices as row/column sums + 6 fixed rows
                fp = {}
                for k, v in t.items():
                    if v.ndim == 2 and v.shape[1] > 3:
                        rows = np.linspace(0, v.shape[0] - 1, 6).astype(int)
                        fp[k + "__rowsum"] = v.sum(axis=1)
                        fp[k + "__colsum"] = v.sum(axis=0)
                        fp[k + "__rows"] = v[rows]
                        fp[k + "__rowidx"] = rows
                    else:
                        fp[k] = v
                t = fp
            np.savez_compressed(OUT / name, **t)


def rhs_cases():
    cases = {}
    for p in (1, 2, 3, 4):
        for riem, bc_wall in (("llf", 0), ("hllc", 1)):  # slip wall / farfield on "wall"
            if True:
                mesh = ref.Mesh("cube", 2, 4.0)
                lv = ref.Level(mesh, p, bc_wall=bc_wall)
                u = lv.random_admissible_store(42)
                cfg = ref.make_cfg(riem)
                rhs = lv.compute_rhs(u, cfg, FS)
                dt = 0.25 * lv.compute_timestep(u, cfg)
                u2, res2 = lv.rk_steps(u, np.zeros_like(u), cfg, FS, dt, 2)
                key = f"p{p}_{riem}_bc{bc_wall}"
                cases[f"p{p}_u"] = u
                cases[key + "_rhs"] = rhs
                cases[key + "_dt"] = np.array([dt])
                cases[key + "_u2"] = u2
    np.savez_compressed(OUT / "rhs_cube2.npz", freestream=FS, **cases)


def viscous_cases():
    out = {}
    # test_solver.cpp:354-411 style: forced-on viscosity, p=2 on cube(3)
    mesh = ref.Mesh("cube", 3)
    lv = ref.Level(mesh, 2, bc_wall=1)
    u = lv.random_admissible_store(5)
    cfg = ref.make_cfg("llf", viscosity=dict(enabled=True, eps0=0.04, kappa=4.0, s0_offset=-100.0))
    out["forced_u"] = u
    out["forced_rhs"] = lv.compute_rhs(u, cfg, FS)
    eps, q = lv.last_viscosity()
    out["forced_eps"] = eps
    out["forced_q"] = q
    # default ramp with a noisy state: some elements on, some off
    cfg2 = ref.make_cfg("hllc", viscosity=dict(enabled=True, eps0=0.3, kappa=4.0, s0_offset=0.0))
    u2 = u.copy().reshape(lv.K, 5, lv.block)
    rng = np.random.default_rng(0)
    u2[::3, 0, : lv.n_basis] *= 1.0 + 0.2 * rng.uniform(-1, 1, size=u2[::3, 0, : lv.n_basis].shape)
    # elements 1::3 constant (only the mean mode): indicator 0 -> eps = 0 branch
    u2[1::3, :, : lv.n_basis] = u2[1::3, :, : lv.n_basis].mean(axis=2, keepdims=True)
    u2 = u2.reshape(-1)
    out["ramp_u"] = u2
    out["ramp_rhs"] = lv.compute_rhs(u2, cfg2, FS)
    eps2, q2 = lv.last_viscosity()
    out["ramp_eps"] = eps2
    out["ramp_rhs"] = out["ramp_rhs"]
    np.savez_compressed(OUT / "viscous_cube3_p2.npz", freestream=FS, **out)


def level_cases():
    out = {}
    for n, p in ((2, 3), (2, 4), (3, 2)):
        mesh = ref.Mesh("cube", n)
        lv = ref.Level(mesh, p)
        g = lv.geometry()
        ex = mesh.export()
        key = f"n{n}_p{p}"
        out[key + "_node_map"] = g["node_map"]
        out[key + "_neighbor"] = g["neighbor"]
        out[key + "_h"] = g["h"]
        out[key + "_tets"] = ex["tets"]
        out[key + "_metric0"] = g["cub_dr"][:, 0, :]
        out[key + "_jac0"] = g["cub_jac"][:, 0]
    np.savez_compressed(OUT / "level_geometry.npz", **out)


if __name__ == "__main__":
    tables()
    rhs_cases()
    viscous_cases()
    level_cases()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)
