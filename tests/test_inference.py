"""NEXT-3: the inference variant (Sec. III-D): forward only on each
partition with no activation checkpoints, halo predictions discarded, owned rows
gathered on rank 0 (xmgn_gather_rows) and placed at their global ids
(xmgn_scatter_rows).  Because the layers are the training forward's kernels, the
outputs are bitwise the training forward's, and -- partitioned = full graph
 -- bitwise independent of P_infer."""
import numpy as np
import pytest
import torch

from xmgn_inputs import configs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2411_17164_b200 import xmgn  # noqa: F401


def _assemble(b, H, L, P_parts, infer, prec=2):
    """Owned outputs of every partition in global order, via gather (1 rank) + scatter."""
    from paper_2411_17164_b200 import xmgn
    from paper_2411_17164_b200.processor import Processor
    pr = Processor(b, H, L, precision=prec, infer=infer)
    params = pr.make_params()
    inputs = {p: pr.make_inputs(p) for p in pr.parts}
    rows, gids = pr.infer(params, inputs)
    comm = xmgn.Comm(xmgn.Comm.unique_id(), 1, 0, 0)
    recv = torch.empty_like(rows)
    comm.gather_rows(rows, recv, [rows.shape[0]], torch.cuda.current_stream())
    comm.close()
    N = len(b["offsets"]) - 1
    full = torch.full((N, H), float("nan"), device="cuda")
    xmgn.scatter_rows(recv, torch.as_tensor(gids, device="cuda"), full)
    torch.cuda.synchronize()
    nb = pr.ws.nbytes()
    pr.close()
    return full.cpu(), nb


def test_inference_equals_training_forward_and_is_partition_invariant():
    H, L = 128, 6
    b4 = configs.custom((400, 2000), k=6, P=4, halo=L)
    b2 = configs.custom((400, 2000), k=6, P=2, halo=L)
    train4, nb_train = _assemble(b4, H, L, 4, infer=False)
    inf4, nb_inf = _assemble(b4, H, L, 4, infer=True)
    inf2, _ = _assemble(b2, H, L, 2, infer=True)
    assert not torch.isnan(train4).any()                     # every global row owned exactly once
    assert torch.equal(inf4, train4)                         # same kernels, same bits
    assert torch.equal(inf2, inf4)                           # P_infer != P_train: identical rows
    assert nb_inf * 2 < nb_train, (nb_inf, nb_train)         # no per-layer checkpoints


def test_inference_workspace_refuses_backward():
    from paper_2411_17164_b200 import xmgn
    from paper_2411_17164_b200.processor import Processor
    b = configs.custom((300,), k=6, P=2, halo=2)
    pr = Processor(b, 128, 2, infer=True)
    params = pr.make_params()
    h0, e0, g = pr.make_inputs(0)
    pr.forward(0, params, h0, e0)
    gp = torch.zeros(pr.n_params, device="cuda")
    with pytest.raises(xmgn.XmgnError, match="ESTATE"):
        pr.backward(0, params, g, gp)
    pr.close()


def test_cfg4_inference_memory_and_owned_rows():
    """The bench workload on one GPU with ONE inference partition holding the whole 2M-node
    graph would need the full graph's edge operands twice; instead: CFG4's 8 partitions
    through the inference workspace match the training forward bitwise on sampled rows,
    with a workspace a fraction of the training one."""
    from paper_2411_17164_b200.processor import Processor
    b = configs.load("cfg4")
    H, L = 512, 15
    pr = Processor(b, H, L, infer=True, parts=[0, 5])
    params = pr.make_params()
    inputs = {p: pr.make_inputs(p) for p in pr.parts}
    rows, gids = pr.infer(params, inputs)
    nb_inf = pr.ws.nbytes()
    del inputs
    pr.close()
    pt = Processor(b, H, L, parts=[0, 5])
    nb_train = pt.ws.nbytes()
    outs = []
    for p in pt.parts:
        h0, e0, _ = pt.make_inputs(p)
        outs.append(pt.forward(p, params, h0, e0))
    pt.close()
    assert torch.equal(rows, torch.cat(outs))
    assert nb_inf * 4 < nb_train, (nb_inf, nb_train)
