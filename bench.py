"""Benchmark: DOF-updates/s of the fused RK-stage RHS + low-storage update.

Workload (BASELINE.json configs[4], the single-GPU-fitting headline config):
make_cube_mesh(88) = 4,088,832 straight tets, P=4 (N_p=35, N_cub=70, N_f=64),
LLF, slip walls, random admissible state (bench.cpp:22-40 recipe), FP64.
One "step" = one LSRK4 step = 5 fused RHS/update launches (each writes the
next stage's face traces). DOF-updates/s = K * N_p * 5 fields * 5 stages *
steps / time. The headline `value` is the graph-replayed production loop
(no per-kernel events); a second, profiled pass gives the kernel times of the
roofline. The `curved` object is the same metric on the curved
(isoparametric) path: make_cube_mesh(32) with every element curved by a
smooth map (196,608 curved tets, raised quadrature), LLF and HLLC, with its
own roofline.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N>1 (torchrun, one process per GPU): strong scaling over z-slab partitions of
the same mesh, driven by the library's multi-rank driver (cdg_gpu_comm, NCCL
inside the library; the unique id travels over torch.distributed).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

P_DEFAULT = 4
N_DEFAULT = 88
# BASELINE.json's metric (the reference is 3D: "curved-tri" reads as curved tets)
METRIC = "DOF-updates/sec (RK-stage RHS+update), curved-tri Euler P=4, 1/2/4/8 B200"


def workload_config(args, world: int) -> dict:
    """The `config` of both arms' JSON lines (no device needed)."""
    from paper_1208_4772_b200 import refelem as R
    re = R.get_reference_element(args.p)
    K = 6 * args.n ** 3
    npb, nf = re.n_basis, 4 * re.n_face_quad
    bp, tb = (npb + 15) // 16 * 16, (nf + 15) // 16 * 16
    return {"workload": f"make_cube_mesh({args.n}) = {K} straight tets, P={args.p} (N_p={npb}, N_cub={re.n_cub}, "
                        f"N_f={nf}), {args.riemann.upper()}, slip walls, random admissible state (bench.cpp:22-40)",
            "elements": K, "p": args.p, "riemann": args.riemann, "dof": K * npb * 5,
            "partition": f"{world} z-slab(s)" if args.partition == "slab" or world == 1 else f"{world} RCB parts",
            "l2": "working set ~%.0f GB >> 126 MB L2 (no flush needed)" % (K * (3 * 5 * bp + 5 * tb) * 8 / 1e9)}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--p", type=int, default=P_DEFAULT)
    ap.add_argument("--n", "--cube-n", dest="n", type=int, default=N_DEFAULT,
                    help="cube cells per side (6 n^3 tets); --cube-n under torchrun")
    ap.add_argument("--riemann", default="llf")
    ap.add_argument("--cfl", type=float, default=0.5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--partition", default="slab", choices=["slab", "rcb"],
                    help="N>1: z-slabs of the cube mesh, or recursive coordinate bisection (general meshes)")
    ap.add_argument("--curved-n", type=int, default=32,
                    help="cube cells per side of the curved block (6 n^3 curved tets; 0 = skip)")
    ap.add_argument("--cpu-n", type=int, default=CPU_N_DEFAULT,
                    help="cube cells per side of the reference CPU sample (6 n^3 tets)")
    return ap.parse_args()


def freestream_state(mach=0.3, alpha_deg=0.0, rho=1.0, p=1.0, gamma=1.4):
    """FreestreamConfig::state (config.cpp:12-24), the bench.cpp:155 state."""
    c = math.sqrt(gamma * p / rho)
    vmag = mach * c
    a = math.radians(alpha_deg)
    v = np.array([vmag * math.cos(a), 0.0, vmag * math.sin(a)])
    return np.array([rho, rho * v[0], rho * v[1], rho * v[2], p / (gamma - 1.0) + 0.5 * rho * v.dot(v)])


def model_flops_bytes(np_, ncub, nf):
    """SURVEY.md §8d / BASELINE.md §2 per-element-per-stage model."""
    F = 10 * (4 * np_ * ncub + 2 * np_ * nf + np_ * np_) + 30 * ncub + 130 * nf + 20 * np_
    F_rhs = F - 10 * np_ * nf            # minus the I_g trace GEMV (separate kernel)
    B = 160 * np_ + 80 * nf + 208 + 32
    return F, F_rhs, B


def kernel_flops_executed(np_, ncub, nf):
    """DMMA flops the kernels issue per element per stage (padding included)."""
    r4, r8 = (lambda x: (x + 3) // 4 * 4), (lambda x: (x + 7) // 8 * 8)
    kp, ncub8, np8, nf8 = r4(np_), r8(ncub), r8(np_), r8(nf)
    rhs = 2 * 5 * (ncub8 * kp + np8 * (3 * ncub8 + nf))
    tr = 2 * 5 * nf8 * kp
    return rhs, tr


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 4 + i and s[4 + i].lower().startswith("active")})
        power = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "power_w_max": max(power) if power else None, "samples": len(self.samples)}


CPU_N_DEFAULT = 30  # make_cube_mesh(30) = 162,000 tets: the largest cube sample whose reference DgLevel
                    # (~140 KB/element at P=4) fits comfortably in the GPU box's host RAM


def cpu_baseline(p, riemann, n_cpu=CPU_N_DEFAULT, steps=5, warmup=1, seconds_budget=60.0):
    """The reference's own rk_step (oracle/_ref built in place from the
    unmodified sources; the -O3 -march=native build of BASELINE.md §3 when this
    CPU runs it) on all host threads, on make_cube_mesh(n_cpu) -- a bounded
    sample of the same workload. Only the rk_step loop is timed (the store
    copies in and out of the reference's SolutionStore are outside the timer).
    Falls back to the C restatement (1 thread) without oracle/_ref."""
    try:
        from oracle import ref
        perf = ref.use_perf_build()
        if ref.available() or perf:
            nthreads = ref.num_threads(os.cpu_count() or 1)
            t0 = time.perf_counter()
            mesh = ref.Mesh("cube", n_cpu)
            lv = ref.Level(mesh, p, bc_wall=0, bc_far=1)
            setup = time.perf_counter() - t0
            cfg = ref.make_cfg(riemann)
            fs = freestream_state()
            u = lv.random_admissible_store(42)
            res = np.zeros_like(u)
            dt = 0.5 * lv.compute_timestep(u, cfg)
            if warmup:
                u, res, _ = lv.rk_steps_timed(u, res, cfg, fs, dt, warmup)
            times = []
            while len(times) < steps and sum(times) < seconds_budget:
                u, res, secs = lv.rk_steps_timed(u, res, cfg, fs, dt, 1)
                times.append(float(secs[0]))
            med = statistics.median(times)
            dofs = lv.K * lv.n_basis * 5 * 5
            build = ("-O3 -march=native build (BASELINE.md §3 flags)" if perf else
                     "-O3 -march=x86-64-v3 -ffp-contract=off build (bitwise-pinned oracle build)")
            return {"value": dofs / med, "unit": "DOF-updates/s", "cores": nthreads, "kind": "reference",
                    "cpu": ref.cpu_model(),
                    "sample": f"make_cube_mesh({n_cpu}) = {lv.K} tets, P={p}, {riemann.upper()}, "
                              f"{len(times)} timed rk_step after {warmup} warm-up (median {med:.3f} s; only the "
                              f"step loop timed, level setup {setup:.1f} s outside), oracle/_ref: the reference "
                              f"sources built in place, {build}, OpenMP {nthreads} threads",
                    "steps_timed": len(times), "median_step_s": med}
    except Exception as e:  # pragma: no cover - diagnostic path
        err = repr(e)
    else:
        err = "oracle/_ref not built"
    from oracle import port
    from paper_1208_4772_b200 import gpu, mesh as M, refelem as R
    m = M.cube_mesh(6)
    re = R.get_reference_element(p)
    ol = port.OracleLevel(m, re, bc=0, freestream=freestream_state())
    cfg = gpu.run_config(riemann)

    class _L:  # same recipe via the product helper on a shape-compatible object
        K, n_basis, block = ol.K, re.n_basis, ol.block
    u = gpu.random_admissible_store(_L, seed=42)
    dt = 0.5 * ol.compute_timestep(u, cfg)
    t0 = time.perf_counter()
    ol.rk_steps(u, np.zeros_like(u), cfg, dt, 1)
    t = time.perf_counter() - t0
    return {"value": ol.K * re.n_basis * 25 / t, "unit": "DOF-updates/s", "cores": 1, "kind": "port",
            "sample": f"make_cube_mesh(6) = {ol.K} tets, P={p}, 1 rk_step, C restatement ({err})"}


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU rk_step on this box's host cores,
    W warm-up + K timed steps of the bounded sample (at most ~2 min timed)."""
    if rank != 0:
        return
    cb = cpu_baseline(args.p, args.riemann, n_cpu=args.cpu_n, steps=args.steps, warmup=args.warmup,
                      seconds_budget=120.0)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"],
            "unit": "DOF-updates/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(args, world),
            "cpu_baseline": cb, "e2e": {"value": cb["value"], "unit": "DOF-updates/s",
                                        "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def synthetic_state(lv, seed):
    """bench.cpp:22-40's random admissible state, generated on the device."""
    import torch
    K, npb = lv.K, lv.n_basis
    g = torch.Generator(device="cuda").manual_seed(seed)
    u = torch.zeros((K, 5, lv.block), dtype=torch.float64, device="cuda")
    j = lambda: (torch.rand((K, npb), generator=g, dtype=torch.float64, device="cuda") - 0.5) * 0.1
    rho = 1.0 + j()
    vx, vy, vz = 0.3 + j(), j(), j()
    pr = 1.0 + j()
    u[:, 0, :npb] = rho
    u[:, 1, :npb] = rho * vx
    u[:, 2, :npb] = rho * vy
    u[:, 3, :npb] = rho * vz
    u[:, 4, :npb] = pr / 0.4 + 0.5 * rho * (vx * vx + vy * vy + vz * vz)
    del rho, vx, vy, vz, pr
    torch.cuda.synchronize()  # the level copies on its own (non-blocking) stream
    lv.set_state_device(u.data_ptr(), None)
    del u
    torch.cuda.empty_cache()


def time_steps(lv, run, steps):
    """device time (CUDA events on the level's stream) of run(steps)."""
    import torch
    ext = torch.cuda.ExternalStream(lv.stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(ext)
    run(steps)
    e1.record(ext)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def profile_steps(lv, cfg, dt, steps):
    """Per-kernel device times of `steps` RK steps (events around every launch
    on the level's stream; not the production mode, hence a separate pass)."""
    lv.set_profiling(True)
    lv.rk_steps(cfg, dt, steps)
    lv.set_profiling(False)
    t_tr, t_rhs, _ = lv.last_profile()
    return float(t_tr), float(t_rhs)


def curved_block(args, peak, hbm_peak):
    """The curved (isoparametric) path at a GPU-filling size: make_cube_mesh(n)
    with every element's collocation nodes moved by a smooth global map
    (mesh.warped_nodes), curved-mesh quadrature (P=4: N_cub 70, N_g 56), per-node
    metrics, M_e^-1 epilogue -- LLF and HLLC, graph-replayed steps, plus a
    profiled pass for the RHS kernel's roofline (F_rhs per curved element,
    SURVEY §8d with the curved quadrature)."""
    from paper_1208_4772_b200 import gpu, mesh as M, refelem as R
    t0 = time.perf_counter()
    p = args.p
    re = R.level_reference_element(p, True)
    mesh = M.cube_mesh(args.curved_n)
    X = M.warped_nodes(mesh, re)
    lv = gpu.GpuLevel(mesh, p, bc=0, freestream=freestream_state(), curved=(np.arange(mesh.n_owned), X), re=re)
    del X
    setup = time.perf_counter() - t0
    synthetic_state(lv, 7)
    K, npb, nf = lv.K, lv.n_basis, 4 * re.n_face_quad
    F, F_rhs, B = model_flops_bytes(npb, re.n_cub, nf)
    geo = 8 * (9 * re.n_cub + 4 * nf + npb * npb)  # per-node metric, per-face-node (n, sjac w), M_e^-1
    out = {"workload": f"make_cube_mesh({args.curved_n}) = {K} tets, ALL curved (smooth isoparametric map, "
                       f"amp 0.02), P={p} curved quadrature (N_cub={re.n_cub}, N_f={nf}), slip walls, random "
                       f"admissible state", "elements": K, "curved_elements": K, "setup_s": round(setup, 1)}
    for riemann in ("llf", "hllc"):
        cfg = gpu.run_config(riemann, cfl=args.cfl)
        dt = 0.5 * lv.compute_timestep(cfg)
        steps = max(3, args.steps // 2)
        lv.rk_steps(cfg, dt, 3)  # warm-up (graph capture)
        ms = time_steps(lv, lambda n: lv.rk_steps(cfg, dt, n), steps)
        t_tr, t_rhs = profile_steps(lv, cfg, dt, 2)
        t_rhs_s, t_tr_s = t_rhs / 10 * 1e-3, t_tr / 10 * 1e-3
        fused = lv.fused_traces()  # k_rhs_wac writes the next stage's traces: the whole stage F
        F_k = F if fused else F_rhs
        ach = F_k * K / t_rhs_s / 1e12
        r = {"value": K * npb * 25 * steps / (ms * 1e-3), "unit": "DOF-updates/s", "ms_per_step": ms / steps,
             "steps": steps, "rhs_kernel_ms": t_rhs_s * 1e3, "trace_kernel_ms": t_tr_s * 1e3,
             "roofline": {"bound": "tensor", "kernel": f"{lv.curved_kernel()}<P={p}> (curved: per-node metrics, fused "
                          "volume+surface+lift, M_e^-1 epilogue + LSRK update"
                          + (" + next-stage traces" if fused else "") + ")", "achieved": ach, "peak": peak,
                          "unit": "TFLOP/s", "frac": ach / peak, "algorithmic_flops_per_elem": F_k,
                          "fused_traces": fused,
                          "model_bytes_per_elem": B + geo,
                          "hbm_achieved_gbs": (B + geo) * K / t_rhs_s / 1e9, "hbm_peak_gbs": hbm_peak,
                          "stage_frac": F * K / (t_rhs_s + t_tr_s) / 1e12 / peak}}
        out[riemann] = r
    out["value"] = out["llf"]["value"]
    out["unit"] = "DOF-updates/s"
    lv.close()
    return out


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    from paper_1208_4772_b200 import gpu, partition, refelem as R

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    p = args.p
    re = R.get_reference_element(p)
    fs = freestream_state()
    t_setup = time.perf_counter()
    if args.partition == "rcb" and world > 1:
        from paper_1208_4772_b200 import mesh as M
        g_mesh = M.cube_mesh(args.n)
        part = partition.mesh_part(g_mesh, partition.rcb_owner(g_mesh, world), rank)
        del g_mesh
    else:
        part = partition.rank_part(args.n, world, rank)
    lv = gpu.GpuLevel(part.mesh, p, bc=0, freestream=fs, re=re, device=local_rank)
    cfg = gpu.run_config(args.riemann, cfl=args.cfl)
    K = lv.K
    npb = lv.n_basis
    synthetic_state(lv, 42 + rank)
    comm = None
    if world > 1:
        # the library's multi-rank driver: halo rows per peer, NCCL inside the
        # library; rank 0's unique id is broadcast over torch.distributed
        lv.halo_define(part.peers)
        uid = [gpu.GpuComm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = gpu.GpuComm.nccl(lv, uid[0], rank, world)
        dt = comm.compute_timestep(cfg)
    else:
        dt = lv.compute_timestep(cfg)
    setup_s = time.perf_counter() - t_setup

    def run_steps(n):
        if comm is not None:
            comm.rk_steps(cfg, dt, n)
        else:
            lv.rk_steps(cfg, dt, n)

    # ---- warm-up ------------------------------------------------------------
    run_steps(args.warmup)
    torch.cuda.synchronize()

    # ---- timed region: the production loop (graph replays on one GPU),
    # device events on the level's stream, max over ranks ----------------------
    ext = torch.cuda.ExternalStream(lv.stream())
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    launches0 = lv.launch_count()
    with ClockSampler(local_rank) as clk:
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(ext)
        run_steps(args.steps)
        ev1.record(ext)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
    launches = lv.launch_count() - launches0
    ms_total = ev0.elapsed_time(ev1)
    if dist is not None:
        t = torch.tensor([ms_total], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    K_global = 6 * args.n ** 3
    dofs_per_step = K_global * npb * 5 * 5
    value = dofs_per_step * args.steps / (ms_total * 1e-3)
    ms_per_step = ms_total / args.steps

    # ---- end-to-end through the public API with host buffers -----------------
    e2e = None
    if not args.no_e2e:
        # per step: snapshot + one RK step (dt/a/b H2D) + the residual's
        # inf-norm partials D2H (multi-rank: reduced over ranks inside the
        # library); wall clock, max over ranks -- run_steady's check loop
        steps = max(3, args.steps // 2)
        run_steps(1)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            if comm is not None:
                comm.snapshot()
                comm.rk_steps(cfg, dt, 1)
                r = comm.residual(dt, "inf")
            else:
                lv.snapshot()
                lv.rk_steps(cfg, dt, 1)
                r = lv.residual(dt, "inf")
        t_e2e = time.perf_counter() - t0
        if dist is not None:
            t = torch.tensor([t_e2e], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t_e2e = float(t.item())
        assert math.isfinite(r)
        e2e = {"value": dofs_per_step * steps / t_e2e, "unit": "DOF-updates/s",
               "h2d_bytes_per_step": world * 8 * 11, "d2h_bytes_per_step": world * 8 * 592,
               "what": "per step: snapshot + cdg_gpu_rk_steps(1) (dt/a/b H2D) + cdg_gpu_residual (inf-norm "
                       "partials D2H), wall clock, the run_steady check loop (solver.cpp:637-668)"
                       + ("; N>1: cdg_gpu_comm_* (halo exchange per stage, residual MAX over ranks)"
                          if world > 1 else "")}
        if world == 1:
            # reference rk_step adapter semantics: full state host->device->host every step
            u_host, res_host = lv.get_state()
            t0 = time.perf_counter()
            rt_steps = 2
            for _ in range(rt_steps):
                lv.set_state(u_host, res_host)
                lv.rk_steps(cfg, dt, 1)
                u_host, res_host = lv.get_state()
            t_rt = time.perf_counter() - t0
            e2e["roundtrip"] = {"value": dofs_per_step * rt_steps / t_rt, "unit": "DOF-updates/s",
                                "h2d_bytes_per_step": 2 * u_host.nbytes, "d2h_bytes_per_step": 2 * u_host.nbytes,
                                "what": "rk_step adapter: u,res H2D + 1 step + u,res D2H (pageable numpy)"}
            del u_host, res_host

    # ---- roofline (one GPU): a separate profiled pass for the kernel times ----
    F, F_rhs, B = model_flops_bytes(npb, re.n_cub, 4 * re.n_face_quad)
    ex_rhs, ex_tr = kernel_flops_executed(npb, re.n_cub, 4 * re.n_face_quad)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    roof = None
    peak = None
    if world == 1:
        fp64_dmma, fp64_dfma, fp64_k8, fp64_k16 = gpu.measure_fp64_peak(local_rank)
        peak = max(fp64_dmma, fp64_dfma, fp64_k8, fp64_k16)
        prof_steps = min(args.steps, 4)
        prof_tr, prof_rhs = profile_steps(lv, cfg, dt, prof_steps)
        launches_rhs = 5 * prof_steps
        t_rhs = prof_rhs / launches_rhs * 1e-3
        t_tr = prof_tr / launches_rhs * 1e-3
        kname = lv.rhs_kernel()
        ns = kname == "k_rhs_ns"
        fused = lv.fused_traces() or ns
        # the fused kernel also produces the next stage's traces: its work is the
        # whole stage model F (trace GEMM included); else F_rhs.
        # k_rhs_ns interpolates the face states itself (no stored traces): F, and
        # its bytes are the state (u, res read + write), one read of each
        # element's state as a neighbour, and the geometry -- no trace rows
        F_k = F if fused else F_rhs
        ex_k = ex_rhs + ex_tr if fused else ex_rhs
        if ns:
            B = 200 * npb + 208 + 32
        achieved = F_k * K / t_rhs / 1e12
        traffic = None
        ncu_file = ROOT / "profiles" / f"ncu_rhs_p{p}.json"
        if ncu_file.exists():
            traffic = json.loads(ncu_file.read_text()).get("dram_bytes_per_launch")
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": f"{kname}<P={p}> (fused volume+surface+lift+LSRK update"
                          + (" + face states interpolated from the nodal states (no stored traces)" if ns
                             else " + next-stage traces" if fused else "") + ", FP64 DMMA"
                          + (", warp-autonomous: 3 elements per warp, no CTA barrier" if kname == "k_rhs_wa" else "")
                          + ")",
                "fused_traces": fused,
                "algorithmic_flops_per_launch": F_k * K,
                "peak_source": "max of the FP64 DMMA (m16n8k4/k8/k16) and DFMA peaks measured live on this "
                               "GPU by cdg_gpu_measure_fp64_peak (the kernel uses DMMA m16n8k8); "
                               "MEASURED_PEAKS.json has no fp64 entry",
                "fp64_dmma_k4_tflops": fp64_dmma,
                "fp64_dfma_peak_tflops": fp64_dfma, "fp64_dmma_k8_tflops": fp64_k8,
                "fp64_dmma_k16_tflops": fp64_k16,
                "kernel_ms_avg": t_rhs * 1e3, "trace_kernel_ms_avg": t_tr * 1e3,
                "profiled_steps": prof_steps,
                "kernel_share_of_step": prof_rhs / prof_steps / ms_per_step,
                "executed_dmma_tflops": ex_k * K / t_rhs / 1e12,
                "model_bytes_per_element": B,
                "hbm_achieved_gbs": B * K / t_rhs / 1e9, "hbm_peak_gbs": hbm_peak,
                "hbm_frac": B * K / t_rhs / 1e9 / hbm_peak,
                "stage_model_tflops": F * K / ((t_rhs + t_tr)) / 1e12}

    clocks = clk.summary()
    line = {"metric": METRIC,
            "value": value, "unit": "DOF-updates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, world),
            "setup_s": round(setup_s, 1), "gpu_launches": launches, "clocks": clocks}
    if comm is not None:
        line["config"]["multi_rank"] = ("cdg_gpu_comm (NCCL inside the library): per stage pack -> "
                                        "ncclSend/Recv || interior tiles -> halo tiles")
    if e2e:
        line["e2e"] = e2e
    if roof:
        line["roofline"] = roof
    if comm is not None:
        comm.close()
    lv.close()
    if rank == 0 and world == 1 and args.curved_n > 0:
        line["curved"] = curved_block(args, peak, hbm_peak)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(p, args.riemann, n_cpu=args.cpu_n)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
