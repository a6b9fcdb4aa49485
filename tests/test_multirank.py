"""Multi-rank host logic on CPU (gloo, world size 2): partitions are assigned in
contiguous blocks and the SUM all-reduce of per-rank gradients equals the
full-graph gradient -- the exchange xmgn_grad_reduce performs
with NCCL on GPUs."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from xmgn_inputs import configs, tensors
    b = configs.custom((200, 800), k=6, P=4, halo=2)
    H, L = 8, 2
    P = tensors.params(H, L).double().numpy()
    N = len(b["offsets"]) - 1
    g_full = tensors.upstream_grad(np.arange(N), H).double().numpy()
    G = np.zeros_like(P)
    oo = b["owned_offsets"]
    for p in bench.assign_parts(4, world, rank):
        lg = oracle.local_graph(b["offsets"], b["sources"], b["owned"][oo[p]:oo[p + 1]], L)
        f = oracle.forward(lg["offsets"], lg["sources"], P, tensors.node_features(lg["gid"], H).double().numpy(),
                           tensors.edge_features(lg["edge_gid"], H).double().numpy(), H, L)
        g = np.zeros((len(lg["gid"]), H))
        g[:lg["n_owned"]] = g_full[lg["gid"][:lg["n_owned"]]]
        G += oracle.backward(lg["offsets"], lg["sources"], P, f, g, H, L)["params"]
    t = torch.from_numpy(G)
    dist.all_reduce(t)
    if rank == 0:
        N, E = len(b["offsets"]) - 1, len(b["sources"])
        f = oracle.forward(b["offsets"], b["sources"], P, tensors.node_features(np.arange(N), H).double().numpy(),
                           tensors.edge_features(np.arange(E), H).double().numpy(), H, L)
        ref = oracle.backward(b["offsets"], b["sources"], P, f, g_full, H, L)["params"]
        q.put(float(np.abs(t.numpy() - ref).max() / np.abs(ref).max()))
    dist.destroy_process_group()


def test_assign_parts_blocks():
    for P, W in [(8, 1), (8, 2), (8, 8), (32, 8), (21, 4)]:
        got = [bench.assign_parts(P, W, r) for r in range(W)]
        assert sum(got, []) == list(range(P))
        assert max(map(len, got)) - min(map(len, got)) <= 1


def test_two_rank_gradient_sum_equals_full():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    err = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
    assert err < 1e-12
