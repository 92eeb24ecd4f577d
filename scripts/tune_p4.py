"""Tuning harness (not the product): time the P=4 RK stage of one or more
builds of the C ABI side by side on the same synthetic workload.

    python scripts/tune_p4.py [--n 64] [--steps 6] [--riemann llf] LIB [LIB ...]

Each LIB (paper_1208_4772_b200/libcdg_gpu.so or a build.build_variant library,
optionally suffixed @traced / @generic for that kernel path) runs in its own
process. Per library: graph-replayed ms per RK step (CUDA
events on the level's stream), the profiled per-launch RHS-kernel time, the
FP64 fraction of the stage model, and a checksum of the state after the steps
(equal checksums: identical arithmetic)."""
import argparse
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def child(lib, n, steps, riemann, p, curved=False, visc=False):
    sys.path.insert(0, str(ROOT))
    import numpy as np
    import torch

    from paper_1208_4772_b200 import gpu, partition, refelem as R
    lib, _, path = str(lib).partition("@")  # LIB@traced|generic: that kernel path
    gpu.use_library(lib)
    import bench
    re = R.get_reference_element(p)
    part = partition.rank_part(n, 1, 0)
    if curved:  # every element curved by the smooth map (bench.py's curved block)
        from paper_1208_4772_b200 import mesh as M
        re = R.level_reference_element(p, True)
        lv = gpu.GpuLevel(part.mesh, p, bc=0, freestream=bench.freestream_state(), re=re,
                          curved=(np.arange(part.mesh.n_owned), M.warped_nodes(part.mesh, re)))
    else:
        lv = gpu.GpuLevel(part.mesh, p, bc=0, freestream=bench.freestream_state(), re=re)
    if path:
        lv.set_kernel_path(path)
    K, npb = lv.K, lv.n_basis
    g = np.random.default_rng(42)
    u = np.zeros((K, 5, lv.block))
    j = lambda: (g.random((K, npb)) - 0.5) * 0.1
    rho, vx, vy, vz, pr = 1.0 + j(), 0.3 + j(), j(), j(), 1.0 + j()
    u[:, 0, :npb], u[:, 1, :npb], u[:, 2, :npb], u[:, 3, :npb] = rho, rho * vx, rho * vy, rho * vz
    u[:, 4, :npb] = pr / 0.4 + 0.5 * rho * (vx * vx + vy * vy + vz * vz)
    lv.set_state(u.reshape(-1))
    cfg = gpu.run_config(riemann)
    dt = 0.5 * lv.compute_timestep(cfg)
    if visc:  # Persson-Peraire AV forced on every element (bench_curved.py --visc)
        cfg = gpu.run_config(riemann, viscosity=dict(enabled=True, eps0=0.01, kappa=4.0, s0_offset=-100.0))
        dt *= 0.4
    lv.rk_steps(cfg, dt, 2)
    torch.cuda.synchronize()
    ext = torch.cuda.ExternalStream(lv.stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ext)
    lv.rk_steps(cfg, dt, steps)
    e1.record(ext)
    torch.cuda.synchronize()
    ms_step = e0.elapsed_time(e1) / steps
    lv.set_profiling(True)
    lv.rk_steps(cfg, dt, steps)
    lv.set_profiling(False)
    t_tr, t_rhs, nl = lv.last_profile()
    F, F_rhs, _ = bench.model_flops_bytes(npb, re.n_cub, 4 * re.n_face_quad)
    if not lv.fused_traces():
        F = F_rhs
    peak = max(gpu.measure_fp64_peak(0))
    rhs_ms = t_rhs / (5 * steps)
    uu = lv.get_state()[0]
    print(json.dumps({"lib": str(lib) + ("@" + path if path else ""), "K": K, "ms_per_step": ms_step, "rhs_ms": rhs_ms,
                      "frac_graph": F * K / (ms_step / 5 * 1e-3) / 1e12 / peak,
                      "frac_rhs": F * K / (rhs_ms * 1e-3) / 1e12 / peak if rhs_ms > 0 else None, "peak": peak,
                      "checksum": float(np.sum(uu)), "fused": lv.fused_traces(), "trace_ms": t_tr / (5 * steps)}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--p", type=int, default=4)
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--riemann", default="llf")
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--curved", action="store_true")
    ap.add_argument("--visc", action="store_true")
    ap.add_argument("libs", nargs="+")
    a = ap.parse_args()
    if a.child:
        child(a.libs[0], a.n, a.steps, a.riemann, a.p, a.curved, a.visc)
        return
    for lib in a.libs:
        r = subprocess.run([sys.executable, __file__, "--child", "--n", str(a.n), "--p", str(a.p), "--steps",
                            str(a.steps), "--riemann", a.riemann, lib] + (["--curved"] if a.curved else []) + (["--visc"] if a.visc else []), capture_output=True, text=True, timeout=900)
        out = r.stdout.strip().splitlines()
        print(out[-1] if out else json.dumps({"lib": lib, "error": r.stderr[-800:]}), flush=True)


if __name__ == "__main__":
    main()
