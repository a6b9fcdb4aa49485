"""Row a10: the gradient all-reduce through the library's own NCCL communicator
(xmgn_comm_unique_id / xmgn_comm_init / xmgn_grad_reduce, "the
gradients from all partitions are aggregated").

CPU: argument validation and the unique id (no GPU needed).  GPU: a 1-rank
communicator leaves the gradient bitwise unchanged (a SUM over one rank), and --
where two GPUs are visible -- two ranks running their contiguous partition
blocks reproduce the 1-rank sum of all partitions."""
import os
import socket

import numpy as np
import pytest
import torch


@pytest.fixture(scope="module")
def xmgn():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2411_17164_b200 import xmgn as X
    return X


def test_comm_init_rejects_bad_arguments(xmgn):
    uid = bytes(128)
    for nranks, rank in [(0, 0), (2, 2), (2, -1)]:
        with pytest.raises(xmgn.XmgnError, match="EINVAL"):
            xmgn.Comm(uid, nranks, rank, 0)


def test_comm_unique_id(xmgn):
    try:
        a = xmgn.Comm.unique_id()
    except xmgn.XmgnError as e:      # no libnccl.so.2 on this host
        pytest.skip(str(e))
    b = xmgn.Comm.unique_id()
    assert len(a) == 128 and any(a) and a != b


@pytest.mark.gpu
def test_grad_reduce_single_rank_bitwise(xmgn):
    """nranks = 1: the in-place SUM all-reduce is the identity, bit for bit, on a
    gradient of the bench's size (H = 512, L = 15, m = 2: 35,466,240 floats)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    n = xmgn.param_count(xmgn.model_cfg(512, 15, 2))
    assert n == 35_466_240
    g = torch.randn(n, device="cuda") * 1e-3
    ref = g.clone()
    c = xmgn.Comm(xmgn.Comm.unique_id(), 1, 0, 0)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    c.grad_reduce(g, s)
    torch.cuda.synchronize()
    c.close()
    assert torch.equal(g.view(torch.int32), ref.view(torch.int32))


def _free_port():
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    p = so.getsockname()[1]
    so.close()
    return p


def _two_rank_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_2411_17164_b200 import xmgn
    from paper_2411_17164_b200.processor import Processor
    from xmgn_inputs import configs
    b = configs.custom((300, 1500), k=6, P=4, halo=3)
    H, L = 128, 3
    # this rank's contiguous block of partitions, gradients summed in order, then one all-reduce
    mine = bench.assign_parts(4, world, rank)
    pr = Processor(b, H, L, device=rank, parts=mine)
    params = pr.make_params()
    grad = torch.zeros(pr.n_params, device=f"cuda:{rank}")
    outs = {}
    for p in mine:
        h0, e0, g = pr.make_inputs(p)
        outs[p] = pr.forward(p, params, h0, e0).cpu()
        pr.backward(p, params, g, grad)
    uid = [xmgn.Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = xmgn.Comm(uid[0], world, rank, rank)
    comm.grad_reduce(grad, torch.cuda.current_stream())
    # inference gather: every rank's owned rows to rank 0, in rank order
    mine_rows = torch.cat([outs[p] for p in mine]).to(f"cuda:{rank}")
    oo = b["owned_offsets"]
    counts = [int(sum(oo[p + 1] - oo[p] for p in bench.assign_parts(4, world, r))) for r in range(world)]
    recv = torch.empty((sum(counts), H), device=f"cuda:{rank}") if rank == 0 else None
    comm.gather_rows(mine_rows, recv, counts if rank == 0 else None, torch.cuda.current_stream())
    torch.cuda.synchronize()
    comm.close()
    pr.close()
    # the 1-rank reference on this GPU: every partition in order, no all-reduce
    pr1 = Processor(b, H, L, device=rank)
    g1 = torch.zeros(pr1.n_params, device=f"cuda:{rank}")
    same = True
    all_outs = {}
    for p in pr1.parts:
        h0, e0, g = pr1.make_inputs(p)
        o = pr1.forward(p, params, h0, e0).cpu()
        all_outs[p] = o
        if p in outs:
            same = same and torch.equal(o, outs[p])
        pr1.backward(p, params, g, g1)
    torch.cuda.synchronize()
    rel = float((grad - g1).norm() / g1.norm())
    pr1.close()
    if rank == 0:   # the gathered rows are every partition's owned rows in partition order
        same = same and torch.equal(recv.cpu(), torch.cat([all_outs[p] for p in range(4)]))
    q.put((rank, same, rel))
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_gpu_grad_reduce_equals_one_rank_sum():
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_two_rank_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    for rank, same, rel in res:
        assert same, f"rank {rank}: forward outputs differ from the 1-rank run"
        assert rel <= 1e-5, f"rank {rank}: all-reduced gradient rel {rel:.2e} vs the 1-rank sum"
