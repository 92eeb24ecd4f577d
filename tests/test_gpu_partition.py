"""Multi-rank code path on ONE GPU: the z-slab (and the general RCB) partition with the per-stage
halo exchange (cdg_gpu_rk_stage_phase + halo buffers), ranks emulated by
several levels on cuda:0 and the NCCL send/recv replaced by device copies.
Per-element arithmetic is partition independent, so the result must be
BITWISE identical to the single-level run."""
import numpy as np
import pytest

from paper_1208_4772_b200 import mesh as M, partition as P

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("R,p,overlap,kind", [(2, 3, False, "slab"), (3, 4, False, "slab"), (2, 3, True, "slab"),
                                               (3, 4, True, "slab"), (4, 2, True, "slab"), (3, 4, True, "rcb"),
                                               (5, 3, True, "rcb"), (4, 4, False, "rcb")])
def test_partitioned_rk_steps_bitwise_equal(gpu_lib, R, p, overlap, kind):
    """overlap=True: interior tiles (phase 2) run before the halo traces land,
    halo tiles (phase 3) after -- the comm/compute overlap of the multi-GPU
    stage; still bitwise identical."""
    import torch
    gpu = gpu_lib
    n = 4
    fs = gpu.make_state(1.0, [0.3, 0.1, 0.0], 1.0)
    cfg = gpu.run_config("llf")
    # single level reference run
    g = M.cube_mesh(n)
    lv = gpu.GpuLevel(g, p, bc=1, freestream=fs)
    u0 = gpu.random_admissible_store(lv, seed=21)
    lv.set_state(u0)
    dt = 0.2 * lv.compute_timestep(cfg)
    lv.rk_steps(cfg, dt, 3)
    u_ref = lv.get_state()[0].reshape(lv.K, 5, lv.block)
    u0 = u0.reshape(lv.K, 5, lv.block)
    # R "ranks" on the same device
    if kind == "slab":
        parts = [P.rank_part(n, R, r) for r in range(R)]
    else:  # general-mesh partition: recursive coordinate bisection
        owner = P.rcb_owner(g, R)
        parts = [P.mesh_part(g, owner, r) for r in range(R)]
    owned = [np.arange(*pt.elem_range) if pt.owned is None else pt.owned for pt in parts]
    levels, bufs = [], []
    per = 5 * lv.n_face_quad
    for pt, own in zip(parts, owned):
        L = gpu.GpuLevel(pt.mesh, p, bc=1, freestream=fs)
        L.set_state(np.ascontiguousarray(u0[own]).reshape(-1))
        send_all = np.concatenate([pe.send_elem_face for pe in pt.peers])
        recv_all = np.concatenate([pe.recv_elem_face for pe in pt.peers])
        sb = torch.zeros(len(send_all) * per, dtype=torch.float64, device="cuda")
        rb = torch.zeros(len(recv_all) * per, dtype=torch.float64, device="cuda")
        L.halo_setup(send_all, recv_all, sb.data_ptr(), rb.data_ptr())
        offs_s, offs_r, o_s, o_r = {}, {}, 0, 0
        for pe in pt.peers:
            offs_s[pe.rank] = (o_s, len(pe.send_elem_face) * per)
            offs_r[pe.rank] = (o_r, len(pe.recv_elem_face) * per)
            o_s += offs_s[pe.rank][1]
            o_r += offs_r[pe.rank][1]
        levels.append(L)
        bufs.append((sb, rb, offs_s, offs_r))
    for step in range(3):
        for stage in range(5):
            for L in levels:
                L.stage_phase(cfg, stage, 0, dt)
            torch.cuda.synchronize()
            if overlap:
                for L in levels:
                    L.stage_phase(cfg, stage, 2, dt)  # interior tiles before the exchange
                torch.cuda.synchronize()
            for r in range(R):
                sb_r, _, offs_s, _ = bufs[r]
                for s_rank, (o, nbytes) in offs_s.items():
                    _, rb_s, _, offs_r_s = bufs[s_rank]
                    o2, n2 = offs_r_s[r]
                    assert n2 == nbytes
                    rb_s[o2:o2 + n2].copy_(sb_r[o:o + nbytes])
            torch.cuda.synchronize()
            for L in levels:
                L.stage_phase(cfg, stage, 3 if overlap else 1, dt)
            torch.cuda.synchronize()
    out = np.empty_like(u_ref)
    for L, own in zip(levels, owned):
        out[own] = L.get_state()[0].reshape(L.K, 5, L.block)
    assert np.array_equal(out, u_ref)
