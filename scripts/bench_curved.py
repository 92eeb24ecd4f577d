"""Throughput of the curved (isoparametric) RHS path at a size that fills the
GPU: make_cube_mesh(n) with every element (or a --frac subset) curved by a
smooth global map x -> x + A sin(2 pi y) sin(2 pi z) e_x + ... applied to the
physical collocation nodes (continuous across faces, so the face pairing is
unchanged). The curved sphere of the parity tests has 4,800 elements, too few
to load 148 SMs; this is the kernel-quality measurement for the curved path.

Per stage: trace kernel + k_rhs_curved (+ the affine row kernel for the
straight elements when --frac < 1). Model flops per curved element per stage
F(N_p, N_cub, N_f) from SURVEY §8d with the curved-mesh quadrature
(P=4: 70 / 56 / 224 -> 298,970 flop).

usage: python scripts/bench_curved.py [--n 24] [--p 4] [--frac 1.0] [--steps 4]
"""
import argparse
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1208_4772_b200 import gpu, mesh as M, refelem as R  # noqa: E402


def curved_nodes(mesh, re, amp):
    """Physical collocation nodes of every element under the smooth map."""
    lam = (re.colloc_nodes + 1.0) / 2.0                 # barycentric 1..3 of (r, s, t)
    bary = np.concatenate([1.0 - lam.sum(axis=1, keepdims=True), lam], axis=1)  # [N_p, 4]
    X = np.einsum("jv,kvd->kjd", bary, mesh.vertices[mesh.tets[:mesh.n_owned]])
    x, y, z = X[..., 0].copy(), X[..., 1].copy(), X[..., 2].copy()
    t = 2.0 * np.pi
    X[..., 0] = x + amp * np.sin(t * y) * np.sin(t * z)
    X[..., 1] = y + amp * np.sin(t * z) * np.sin(t * x)
    X[..., 2] = z + amp * np.sin(t * x) * np.sin(t * y)
    return X


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=24)
    ap.add_argument("--p", type=int, default=4)
    ap.add_argument("--frac", type=float, default=1.0)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--riemann", default="llf")
    ap.add_argument("--amp", type=float, default=0.02)
    ap.add_argument("--visc", action="store_true", help="Persson-Peraire AV forced on every element")
    ap.add_argument("--lib", default=None, help="a build.build_variant library (tuning)")
    args = ap.parse_args()
    import torch
    if args.lib:
        gpu.use_library(args.lib)

    mesh = M.cube_mesh(args.n)
    K = mesh.n_owned
    re = R.level_reference_element(args.p, True)
    X = curved_nodes(mesh, re, args.amp)
    # --frac < 1: the curved elements are the bottom z-slab of the mesh (a
    # curved wall layer; the cube mesh numbers elements z-slab by z-slab)
    ids = np.arange(int(round(min(args.frac, 1.0) * K)))
    lv = gpu.GpuLevel(mesh, args.p, bc=0, freestream=bench.freestream_state(), curved=(ids, X[ids]))
    cfg = gpu.run_config(args.riemann, cfl=0.5)
    if args.visc:
        cfg = gpu.run_config(args.riemann, cfl=0.5,
                             viscosity=dict(enabled=True, eps0=0.01, kappa=4.0, s0_offset=-100.0))
    npb = lv.n_basis
    u = np.zeros((K, 5, lv.block))
    g = np.random.default_rng(42)
    j = lambda: (g.random((K, npb)) - 0.5) * 0.1
    rho, vx, vy, vz, pr = 1.0 + j(), 0.3 + j(), j(), j(), 1.0 + j()
    u[:, 0, :npb], u[:, 1, :npb], u[:, 2, :npb], u[:, 3, :npb] = rho, rho * vx, rho * vy, rho * vz
    u[:, 4, :npb] = pr / 0.4 + 0.5 * rho * (vx * vx + vy * vy + vz * vz)
    lv.set_state(u.reshape(-1))
    dt = lv.compute_timestep(gpu.run_config(args.riemann, cfl=0.5)) * (0.2 if args.visc else 1.0)
    lv.rk_steps(cfg, dt, 3)  # warm-up
    torch.cuda.synchronize()
    lv.set_profiling(True)
    lv.rk_steps(cfg, dt, args.steps)
    lv.set_profiling(False)
    t_tr, t_rhs, nl = lv.last_profile()
    stages = 5 * args.steps
    lv.set_profiling(False)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ext = torch.cuda.ExternalStream(lv.stream())
    torch.cuda.synchronize()
    ev0.record(ext)
    lv.rk_steps(cfg, dt, args.steps)
    ev1.record(ext)
    torch.cuda.synchronize()
    ms_step = ev0.elapsed_time(ev1) / args.steps
    F, F_rhs, B = bench.model_flops_bytes(npb, re.n_cub, 4 * re.n_face_quad)
    peak = max(gpu.measure_fp64_peak(0))
    t_rhs_s = max(t_rhs, 1e-9) / stages * 1e-3  # (viscous steps run as one graph: no per-kernel split)
    t_tr_s = t_tr / stages * 1e-3
    Kc = len(ids)
    # the rhs time covers both kernels when --frac < 1; F_rhs is the same model
    # for both (curved-mesh quadrature on every element)
    F_k = F if lv.fused_traces() else F_rhs  # fused: the RHS kernels also write the next stage's traces
    ach = F_k * K / t_rhs_s / 1e12
    geo = 8 * (9 * re.n_cub + 4 * 4 * re.n_face_quad + npb * npb)
    out = {"config": f"make_cube_mesh({args.n}) = {K} tets, {Kc} curved (smooth map, amp {args.amp}), "
                     f"P={args.p} (N_cub={re.n_cub}, N_f={4 * re.n_face_quad}), {args.riemann.upper()}",
           "dof_updates_per_s": K * npb * 25 / (ms_step * 1e-3), "ms_per_step": ms_step,
           "rhs_kernel_ms": t_rhs_s * 1e3, "trace_kernel_ms": t_tr_s * 1e3,
           "rhs_model_flop_per_elem": F_k, "fused_traces": lv.fused_traces(), "rhs_tflops": ach, "fp64_peak_tflops": peak, "frac": ach / peak,
           "model_bytes_per_elem": B + geo * Kc / K,
           "hbm_gbs": (B + geo * Kc / K) * K / (t_rhs_s + t_tr_s) / 1e9}
    if t_rhs == 0:  # viscous steps run as one CUDA graph: no per-kernel split
        for k in ("rhs_kernel_ms", "trace_kernel_ms", "rhs_tflops", "frac", "hbm_gbs"):
            out[k] = None
    print(json.dumps(out), flush=True)
    lv.close()


if __name__ == "__main__":
    main()
