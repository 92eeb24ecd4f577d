"""Multi-GPU host logic on CPU: slab partition, canonical halo ordering and a
world_size-2 gloo exchange of face traces (computed by the oracle on the
global mesh) that must land exactly on the ghost faces each rank expects."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1208_4772_b200 import mesh as M, partition as P


@pytest.mark.parametrize("n,R", [(4, 2), (5, 3), (6, 4)])
def test_partition_consistency(n, R):
    g = M.cube_mesh(n)
    parts = [P.rank_part(n, R, r) for r in range(R)]
    assert sum(pt.mesh.n_owned for pt in parts) == g.n_owned
    for pt in parts:
        m, (lo, hi) = pt.mesh, pt.elem_range
        loc = np.where(m.neighbor >= 0, m.global_ids[np.maximum(m.neighbor, 0)], -1)
        assert np.array_equal(loc, g.neighbor[lo:hi])
        assert np.array_equal(m.neighbor_face, g.neighbor_face[lo:hi])
        assert np.array_equal(m.perm_code[m.neighbor >= 0], g.perm_code[lo:hi][m.neighbor >= 0])
        for peer in pt.peers:
            other = [q for q in parts[peer.rank].peers if q.rank == pt.rank][0]
            se, sf = peer.send_elem_face >> 2, peer.send_elem_face & 3
            re_, rf = other.recv_elem_face >> 2, other.recv_elem_face & 3
            assert np.array_equal(m.global_ids[se], parts[peer.rank].mesh.global_ids[re_])
            assert np.array_equal(sf, rf)


@pytest.mark.parametrize("n,R", [(4, 2), (5, 3), (5, 5), (6, 8)])
def test_rcb_partition_consistency(n, R):
    """General-mesh partition (recursive coordinate bisection): balanced,
    every element owned once, local connectivity == the global one, and the
    two sides of every rank pair enumerate their shared faces identically."""
    g = M.cube_mesh(n)
    owner = P.rcb_owner(g, R)
    counts = np.bincount(owner, minlength=R)
    assert counts.sum() == g.n_owned and counts.max() - counts.min() <= 1
    parts = [P.mesh_part(g, owner, r) for r in range(R)]
    for pt in parts:
        m = pt.mesh
        assert np.array_equal(m.global_ids[:m.n_owned], pt.owned)
        loc = np.where(m.neighbor >= 0, m.global_ids[np.maximum(m.neighbor, 0)], -1)
        assert np.array_equal(loc, g.neighbor[pt.owned])
        assert np.array_equal(m.neighbor_face, g.neighbor_face[pt.owned])
        assert (owner[m.global_ids[m.n_owned:]] != pt.rank).all()
        n_cut = 0
        for peer in pt.peers:
            other = [q for q in parts[peer.rank].peers if q.rank == pt.rank][0]
            se, sf = peer.send_elem_face >> 2, peer.send_elem_face & 3
            re_, rf = other.recv_elem_face >> 2, other.recv_elem_face & 3
            assert np.array_equal(m.global_ids[se], parts[peer.rank].mesh.global_ids[re_])
            assert np.array_equal(sf, rf)
            n_cut += len(se)
        # every face to a ghost is sent to exactly one peer
        assert n_cut == int((m.neighbor >= m.n_owned).sum())


def test_rcb_cube_cut_is_planar():
    """On the cube mesh RCB cuts between cell layers: a 2-way split shares
    exactly the 2 n^2 triangles of one lattice plane."""
    n = 4
    g = M.cube_mesh(n)
    owner = P.rcb_owner(g, 2)
    pt = P.mesh_part(g, owner, 0)
    assert sum(len(pe.send_elem_face) for pe in pt.peers) == 2 * n * n


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, q, kind="slab"):
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import port as oport
    from paper_1208_4772_b200 import gpu, refelem as R
    p = 2
    re = R.get_reference_element(p)
    g = M.cube_mesh(n)
    ol = oport.OracleLevel(g, re, bc=1, freestream=gpu.make_state(1, [0.3, 0, 0], 1))
    rng = np.random.default_rng(3)
    u = np.zeros((g.n_owned, 5, ol.block))
    u[:, :, : re.n_basis] = 1.0 + 0.1 * rng.uniform(-1, 1, size=(g.n_owned, 5, re.n_basis))
    traces = ol.interpolate_to_faces(u.reshape(-1)).reshape(g.n_owned, 5, ol.trace_block)
    pt = P.rank_part(n, world, rank) if kind == "slab" else P.mesh_part(g, P.rcb_owner(g, world), rank)
    m = pt.mesh
    ng = re.n_face_quad
    ok = True
    for peer in pt.peers:
        se = m.global_ids[peer.send_elem_face >> 2]
        sf = peer.send_elem_face & 3
        send = np.stack([traces[e, :, f * ng:(f + 1) * ng] for e, f in zip(se, sf)])
        recv = np.empty_like(send)
        st = torch.from_numpy(send.copy())
        rt = torch.from_numpy(recv)
        ops = [dist.P2POp(dist.isend, st, peer.rank), dist.P2POp(dist.irecv, rt, peer.rank)]
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        ge = m.global_ids[peer.recv_elem_face >> 2]
        gf = peer.recv_elem_face & 3
        expect = np.stack([traces[e, :, f * ng:(f + 1) * ng] for e, f in zip(ge, gf)])
        ok = ok and np.array_equal(rt.numpy(), expect)
    q.put((rank, ok, len(pt.peers)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,kind", [(2, "slab"), (2, "rcb")])
def test_gloo_halo_exchange(world, kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 4, q, kind)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    assert all(npeers == 1 for _, _, npeers in res)
