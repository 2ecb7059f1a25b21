"""Multi-GPU code paths that can run on ONE GPU (the pool gives one per call).

* The NCCL path end to end with a 1-rank communicator: stencil_comm_unique_id
  -> stencil_comm_create -> stencil_run_dist -> stencil_comm_wait
  (ncclCommGetAsyncError polling) -> destroy; equal to stencil_run bitwise.
* The fused peer-store exchange (NEXT-2) across TWO PROCESSES on the same
  GPU: real CUDA IPC handles exchanged through torch.distributed (gloo),
  cudaIpcOpenMemHandle in the other process, the sweep kernel's peer stores
  into the other process's allocation, cuStreamWriteValue32 into the peer's
  flag word and cuStreamWaitValue32 on this rank's own flags.  The ranks are
  HOST-SERIALISED (one run of one sweep per rank per turn, stream sync and a
  barrier in between), so every flag wait is already satisfied when it is
  enqueued: no kernel or stream on this GPU ever waits for work of another
  process that has not been submitted (B200_PROFILING.md forbids mutually
  waiting ranks on one GPU).  After K turns the slabs equal a 1-GPU run of
  K sweeps bitwise.
"""
import os
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
import synth

pytestmark = pytest.mark.gpu


def _plan(dims, shape, dtype):
    from paper_2103_09235_b200 import Plan
    offs = oracle.taps(len(dims), 1, oracle.STAR if shape == "star" else oracle.BOX)
    return Plan(dims, 1, shape, synth.weights(len(offs), 1), dtype)


@pytest.mark.parametrize("dims,shape,dtype,T,m", [((256, 300), "star", "f64", 9, 2),
                                                  ((40, 64, 96), "box", "f32", 6, 2)])
def test_nccl_single_rank_run_dist(dims, shape, dtype, T, m):
    from paper_2103_09235_b200.api import Comm
    plan = _plan(dims, shape, dtype)
    uid = Comm.unique_id()
    assert len(uid) == 128
    comm = Comm(uid, 0, 1)
    L = plan.layout_dist(0, 1, m)
    a, b, ws = plan.empty(layout=L), plan.empty(layout=L), plan.empty(layout=L)
    plan.fill_random_dist(0, 1, m, a, 2)
    plan.halo_exchange(comm, a, m)              # no neighbours: a no-op that must succeed
    plan.run_dist(comm, a, b, T, m, m, ws)
    comm.wait(timeout_ms=60000)
    a1, ref, rws = plan.empty(), plan.empty(), plan.empty()
    plan.fill_random(a1, 2)
    plan.run(a1, ref, T, m, workspace=rws)
    torch.cuda.synchronize()
    assert torch.equal(plan.interior_view(b, L), plan.interior_view(ref))
    comm.close()


@pytest.mark.parametrize("dims,shape,dtype,r", [((64, 300), "star", "f64", 1), ((64, 300), "box", "f32", 3),
                                                ((24, 40, 72), "star", "f64", 2),
                                                ((16, 33, 70), "box", "f32", 1)])
def test_nccl_send_recv_loopback(dims, shape, dtype, r):
    """Real ncclSend/ncclRecv through the library's per-sweep exchange (grouped
    calls, counts, datatype, plane addresses) with rank 0 as both neighbours:
    ghost planes [-halo, 0) <- planes [0, halo), [n0, n0+halo) <- [n0-halo, n0);
    nothing else in the buffer changes."""
    from paper_2103_09235_b200 import Plan
    from paper_2103_09235_b200.api import Comm
    offs = oracle.taps(len(dims), r, oracle.STAR if shape == "star" else oracle.BOX)
    plan = Plan(dims, r, shape, synth.weights(len(offs), 1), dtype)
    halo = r                                       # a 1-rank layout holds the r-ring outside the slab
    comm = Comm(Comm.unique_id(), 0, 1)
    with pytest.raises(Exception):
        plan.halo_exchange_loopback(comm, plan.empty(), r + 1)
    L = plan.layout_dist(0, 1, halo)
    a = plan.empty(layout=L)
    plan.fill_random_dist(0, 1, halo, a, 7)
    torch.cuda.synchronize()
    before = a.clone()
    plan.halo_exchange_loopback(comm, a, halo)
    comm.wait(timeout_ms=60000)
    torch.cuda.synchronize()
    n0 = dims[0]
    pl = L.stride[0]                               # elements per axis-0 plane
    o0 = L.origin[0]
    fa, fb = a.view(-1), before.view(-1)
    def planes(t, z0, z1):
        return t[(o0 + z0) * pl:(o0 + z1) * pl]
    assert torch.equal(planes(fa, -halo, 0), planes(fb, 0, halo))
    assert torch.equal(planes(fa, n0, n0 + halo), planes(fb, n0 - halo, n0))
    assert torch.equal(planes(fa, 0, n0), planes(fb, 0, n0))
    assert torch.equal(fa[:(o0 - halo) * pl], fb[:(o0 - halo) * pl])
    assert torch.equal(fa[(o0 + n0 + halo) * pl:], fb[(o0 + n0 + halo) * pl:])
    assert not torch.equal(planes(fa, -halo, 0), planes(fb, -halo, 0))   # the exchange did move data
    comm.close()


def _peer_worker(rank, world, port, outdir, dims, shape, dtype, m, K):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2103_09235_b200.dist import make_peer_comm
    plan = _plan(dims, shape, dtype)
    halo = m
    L = plan.layout_dist(rank, world, halo)
    a = plan.empty(layout=L)
    plan.fill_random_dist(rank, world, halo, a, 2)
    b, ws = plan.empty(layout=L), plan.empty(layout=L)
    comm = make_peer_comm(b, ws)                # real IPC handles across processes
    torch.cuda.synchronize()
    dist.barrier()
    for _ in range(K):
        for turn in range(world):
            if turn == rank:
                plan.run_dist(comm, a, b, m, m, halo, ws)   # one sweep; peer stores into the neighbours' b
                torch.cuda.synchronize()
            dist.barrier()
        a.copy_(b)                              # out, ghosts included, is the next input
        torch.cuda.synchronize()
        dist.barrier()
    np.save(os.path.join(outdir, "r%d.npy" % rank), plan.interior_view(b, L).double().cpu().numpy())
    comm.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("dims,shape,dtype,m,world", [((64, 300), "star", "f64", 2, 2),
                                                      ((24, 40, 72), "star", "f64", 2, 2),
                                                      ((96, 260), "box", "f32", 2, 3)])
def test_peer_exchange_two_processes_host_serialised(dims, shape, dtype, m, world):
    K = 4
    port = 29500 + (os.getpid() % 1000)
    with tempfile.TemporaryDirectory() as d:
        ctx = mp.get_context("spawn")
        procs = [ctx.Process(target=_peer_worker, args=(r, world, port, d, dims, shape, dtype, m, K))
                 for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(timeout=300)
        codes = [p.exitcode for p in procs]
        for p in procs:
            if p.is_alive():
                p.kill()
        assert codes == [0] * world, codes
        slabs = [np.load(os.path.join(d, "r%d.npy" % r)) for r in range(world)]
    plan = _plan(dims, shape, dtype)
    a, b, ws = plan.empty(), plan.empty(), plan.empty()
    plan.fill_random(a, 2)
    plan.run(a, b, K * m, m, workspace=ws)
    torch.cuda.synchronize()
    single = plan.interior_view(b).double().cpu().numpy()
    assert np.array_equal(np.concatenate(slabs, axis=0), single)
