"""Overhead of the library's multi-rank driver, measured on ONE GPU: the same
mesh as 1 level and as R in-process shards (cdg_gpu_comm_create_local: per
stage pack -> peer copies || interior tiles -> unpack + halo tiles), same total
work, device-timed. The difference is the driver's cost (pack / unpack
kernels, copies, the interior / halo split of the grid, R x the launches);
on R GPUs the shards run concurrently and only this overhead plus the NVLink
transfer time remain on top of 1/R of the work.

usage: python scripts/bench_shards.py [--n 64] [--p 4] [--steps 5] [--ranks 2 4 8]"""
import argparse
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1208_4772_b200 import gpu, partition as P  # noqa: E402


def main():
    import torch
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--p", type=int, default=4)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--ranks", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--riemann", default="llf")
    a = ap.parse_args()
    fs = bench.freestream_state()
    cfg = gpu.run_config(a.riemann)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def timed(run, streams):
        torch.cuda.synchronize()
        e0, e1 = ev(), ev()
        e0.record()
        run()
        for s in streams:  # the levels' streams join the default stream
            torch.cuda.current_stream().wait_stream(torch.cuda.ExternalStream(s))
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    part = P.rank_part(a.n, 1, 0)
    lv = gpu.GpuLevel(part.mesh, a.p, bc=0, freestream=fs)
    u0 = gpu.random_admissible_store(lv, seed=3).reshape(lv.K, 5, lv.block)
    lv.set_state(u0.reshape(-1))
    dt = 0.4 * lv.compute_timestep(cfg)
    lv.rk_steps(cfg, dt, 2)
    t1 = timed(lambda: lv.rk_steps(cfg, dt, a.steps), [lv.stream()]) / a.steps
    K = lv.K
    dofs = K * lv.n_basis * 25
    out = {"workload": f"make_cube_mesh({a.n}) = {K} tets, P={a.p}, {a.riemann.upper()}", "steps": a.steps,
           "single_level_ms_per_step": t1, "single_level_dof_updates_per_s": dofs / (t1 * 1e-3), "shards": []}
    lv.close()
    for R in a.ranks:
        parts = [P.rank_part(a.n, R, r) for r in range(R)]
        levels = []
        for pt in parts:
            L = gpu.GpuLevel(pt.mesh, a.p, bc=0, freestream=fs)
            L.set_state(np.ascontiguousarray(u0[pt.elem_range[0]:pt.elem_range[1]]).reshape(-1))
            L.halo_define(pt.peers)
            levels.append(L)
        comm = gpu.GpuComm.local(levels)
        comm.rk_steps(cfg, dt, 2)
        tR = timed(lambda: comm.rk_steps(cfg, dt, a.steps), [L.stream() for L in levels]) / a.steps
        halo = sum(len(pe.recv_elem_face) for pt in parts for pe in pt.peers)
        out["shards"].append({"ranks": R, "ms_per_step": tR, "overhead_vs_single": tR / t1 - 1.0,
                              "halo_faces_total": halo,
                              "halo_bytes_per_stage": halo * 5 * levels[0].n_face_quad * 8})
        comm.close()
        for L in levels:
            L.close()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
