"""Multi-process (gloo, world_size 2 and 4, CPU) tests of the multi-GPU host
logic: slab arithmetic, the per-sweep exchange schedule stencil_run_dist
issues, the dist buffer layout, and the unique-id broadcast of make_comm.

The slab-decomposed algorithm is executed on CPU with the schedule of
paper_2103_09235_b200.dist.exchange_plan (ghost planes exchanged with gloo
send/recv each step) and the oracle stepping each slab; the gathered result
must equal the single-domain oracle bit for bit.  (On the GPU the same
schedule is checked by the emulated-rank tests.)"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, dims, shape, T, halo, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2103_09235_b200 import Plan
        from paper_2103_09235_b200.dist import exchange_plan, slab
        nd = len(dims)
        offs = oracle.taps(nd, 1, oracle.STAR if shape == "star" else oracle.BOX)
        w = synth.weights(len(offs), 1)
        lo, hi = slab(dims[0], rank, world)
        n0 = hi - lo
        # the library's dist layout agrees with the slab arithmetic
        plan = Plan(dims, 1, shape, w, "f64")
        L = plan.layout_dist(rank, world, halo)
        assert L.interior[0] == n0 and L.global_offset0 == lo and L.origin[0] == halo
        # local frame: planes [-halo, n0 + halo) of axis 0, ring elsewhere
        P = [n + 2 for n in dims]
        glo = max(0, lo - halo + 1)          # padded global index of local plane -halo
        ghi = min(P[0], hi + halo + 1)
        blk = synth.u0_block(dims, 1, [glo] + [0] * (nd - 1), [ghi] + P[1:], 2)
        off = glo - (lo - halo + 1)          # >0 only when clipped at the global start
        local = np.zeros([n0 + 2 * halo] + P[1:])
        local[off:off + blk.shape[0]] = blk
        for _ in range(T):
            # exchange 1 plane per side (fold_m = 1 steps), the library's schedule
            reqs = []
            for peer, (s0, s1), (r0, r1) in exchange_plan(n0, rank, world, 1):
                send = torch.from_numpy(np.ascontiguousarray(local[halo + s0:halo + s1]))
                recv = torch.empty_like(send)
                reqs.append((dist.isend(send, peer), dist.irecv(recv, peer), recv, r0, r1))
            for sr, rr, recv, r0, r1 in reqs:
                sr.wait()
                rr.wait()
                local[halo + r0:halo + r1] = recv.numpy()
            # one step on the slab (+1 ghost plane each side as its frozen-for-one-step ring)
            win = local[halo - 1:halo + n0 + 1]
            wdims = [n0] + list(dims[1:])
            stepped = oracle.run(wdims, 1, offs, w, win, 1)
            local[halo:halo + n0] = stepped[1:1 + n0]
        res = torch.from_numpy(np.ascontiguousarray(local[halo:halo + n0]))
        gathered = [torch.empty_like(res) for _ in range(world)]
        dist.all_gather(gathered, res)
        # the unique-id broadcast used by make_comm (bytes from rank 0 reach everyone)
        uid = bytes(range(128)) if rank == 0 else bytes(128)
        t = torch.tensor(list(uid), dtype=torch.uint8)
        dist.broadcast(t, src=0)
        assert bytes(t.tolist()) == bytes(range(128))
        if rank == 0:
            q.put(torch.cat(gathered).numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,dims,shape,T", [(2, (12, 9), "box", 5), (4, (16, 7, 6), "star", 4),
                                                (2, (10, 6, 5), "box", 3)])
def test_slab_exchange_schedule_matches_single_domain(world, dims, shape, T):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, shape, T, 2, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        got = q.get(timeout=120)
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for p in procs:
        assert p.exitcode == 0
    nd = len(dims)
    offs = oracle.taps(nd, 1, oracle.STAR if shape == "star" else oracle.BOX)
    ref = oracle.run(dims, 1, offs, synth.weights(len(offs), 1), synth.u0_frame(dims, 1, 2), T)
    inner = ref[(slice(1, -1),) + (slice(None),) * (nd - 1)]
    assert np.array_equal(got, inner)


def test_exchange_plan_and_slab():
    from paper_2103_09235_b200.dist import exchange_plan, slab
    assert slab(64, 0, 4) == (0, 16) and slab(64, 3, 4) == (48, 64)
    with pytest.raises(ValueError):
        slab(10, 0, 3)
    assert exchange_plan(16, 0, 1, 2) == []
    assert exchange_plan(16, 0, 4, 2) == [(1, (14, 16), (16, 18))]
    assert exchange_plan(16, 3, 4, 2) == [(2, (0, 2), (-2, 0))]
    assert exchange_plan(16, 1, 4, 2) == [(0, (0, 2), (-2, 0)), (2, (14, 16), (16, 18))]


def _gather_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2103_09235_b200.api import Comm
        from paper_2103_09235_b200.dist import all_gather_bytes
        # a stand-in for this rank's 3 peer records (IPC handle + offset each)
        rec = bytes((rank * 31 + i) % 256 for i in range(Comm.PEER_RECORD))
        got = all_gather_bytes(rec)
        ok = len(got) == world and all(
            g == bytes((r * 31 + i) % 256 for i in range(Comm.PEER_RECORD)) for r, g in enumerate(got))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_peer_records_all_gather(world):
    """make_peer_comm's bootstrap: every rank gets every rank's peer records in
    rank order (what stencil_comm_peer_attach expects)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_gather_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(60)
    assert all(res[r] for r in range(world)), res
