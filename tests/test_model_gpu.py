"""GPU parity of the full model (NEXT-1: encoders -> processor -> decoder -> owned-row MSE)
through the C-ABI (xmgn_model_fwd / xmgn_model_bwd) against the FP64 oracle
(oracle/model.py, pinned in tests/test_model_oracle.py).

Tolerances (north_star's forward bound, applied to the model output):
max |dy| <= 2e-2 x RMS(y_oracle) over all owned rows; loss relative 2e-2; every parameter
tensor (processor and IO) relative Frobenius <= 2e-2."""
import numpy as np
import pytest
import torch

import oracle
from oracle import model as M
from xmgn_inputs import configs, tensors
from gpu_util import max_over_rms, per_tensor_rel, rel_fro

pytestmark = pytest.mark.gpu
FP16, BF16 = 2, 0
TAU = 2e-2


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2411_17164_b200 import xmgn  # noqa: F401


def stats32(b):
    mean, std = M.feature_stats(b["positions"], b["normals"], b["offsets"], b["sources"])
    return np.concatenate([mean, std]).astype(np.float32)


def run_model_gpu(b, H, L, m=2, prec=FP16, infer=False, targets=True):
    from paper_2411_17164_b200.processor import Processor
    pr = Processor(b, H, L, m=m, precision=prec, infer=infer)
    params, io = pr.make_params(), pr.make_io_params()
    st = torch.as_tensor(stats32(b), device="cuda")
    N = len(b["offsets"]) - 1
    y = np.zeros((N, 4))
    loss = torch.zeros(1, device="cuda")
    gp = torch.zeros(pr.n_params, device="cuda")
    gio = torch.zeros_like(io)
    for p in pr.parts:
        inf = pr.info[p]
        pos, nrm, t = pr.make_model_inputs(p, b)
        pred = pr.model_forward(p, params, io, pos, nrm, st, t if targets else None, N, loss if targets else None)
        if targets and not infer:
            pr.model_backward(p, params, io, gp, gio)
        y[inf["gid"][:inf["n_owned"]]] = pred.double().cpu().numpy()
    torch.cuda.synchronize()
    out = dict(y=y, loss=float(loss.item()), params=gp.double().cpu().numpy(), io=gio.double().cpu().numpy())
    pr.close()
    return out


def run_model_oracle(b, H, L, m=2):
    N = len(b["offsets"]) - 1
    P = tensors.params(H, L, m).double().numpy()
    io = tensors.io_params(H, m).double().numpy()
    s = stats32(b).astype(np.float64)
    t = tensors.targets(np.arange(N)).double().numpy()
    pos, nrm = b["positions"].astype(np.float64), b["normals"].astype(np.float64)
    fw = M.forward(b["offsets"], b["sources"], pos, nrm, P, io, (s[:28], s[28:]), H, L, m, targets=t)
    bw = M.backward(b["offsets"], b["sources"], P, io, fw, H, L, m)
    return dict(y=fw["y"], loss=fw["loss"], params=bw["params"], io=bw["io"])


def io_per_tensor_rel(g, ref, H, m):
    lay, _ = M.io_layout(H, m)
    worst, name = 0.0, ""
    for blk, items in lay.items():
        for nm, o, s in items:
            n = int(np.prod(s))
            e = rel_fro(g[o:o + n], ref[o:o + n])
            if e > worst:
                worst, name = e, f"{blk}.{nm}"
    return worst, name


def _check(res, ref, H, L, m, tau=TAU):
    f = max_over_rms(res["y"], ref["y"])
    lr = abs(res["loss"] - ref["loss"]) / ref["loss"]
    gw, name = per_tensor_rel(res["params"], ref["params"], H, L, m)
    gi, iname = io_per_tensor_rel(res["io"], ref["io"], H, m)
    print(f"model: y max/RMS {f:.2e}  loss rel {lr:.2e}  proc grad {name} {gw:.2e}  io grad {iname} {gi:.2e}")
    assert f <= tau, f"prediction max/RMS {f:.3e}"
    assert lr <= tau, f"loss rel {lr:.3e}"
    assert gw <= tau, f"processor gradient {name} {gw:.3e}"
    assert gi <= tau, f"io gradient {iname} {gi:.3e}"


@pytest.mark.parametrize("H,L,m", [(128, 3, 2), (256, 2, 1), (512, 2, 2)])
def test_model_partitioned_vs_oracle(H, L, m):
    b = configs.custom((300, 1500), k=6, P=4, halo=L)
    _check(run_model_gpu(b, H, L, m), run_model_oracle(b, H, L, m), H, L, m)


def test_model_bf16_and_single_partition():
    b = configs.custom((400,), k=6, P=1, halo=2)
    _check(run_model_gpu(b, 128, 2, 2, prec=BF16), run_model_oracle(b, 128, 2, 2), 128, 2, 2)


def test_model_many_partitions_partial_tiles():
    """8 partitions of a 1,800-point graph: every chain program runs partial tiles."""
    b = configs.custom((300, 1800), k=6, P=8, halo=2)
    _check(run_model_gpu(b, 128, 2, 2), run_model_oracle(b, 128, 2, 2), 128, 2, 2)


def test_model_inference_workspace_matches_training_forward():
    """The inference workspace gives bitwise the training forward's predictions and the
    same loss (inference = the training forward without checkpoints)."""
    b = configs.custom((300, 1500), k=6, P=3, halo=2)
    tr = run_model_gpu(b, 128, 2, 2, infer=False)
    inf = run_model_gpu(b, 128, 2, 2, infer=True)
    assert np.array_equal(tr["y"], inf["y"])
    assert tr["loss"] == inf["loss"]


def test_model_deterministic_and_loss_additive():
    """Bitwise run-to-run, and the loss of P partitions = the full graph's MSE."""
    b = configs.custom((300, 1500), k=6, P=4, halo=2)
    r1, r2 = run_model_gpu(b, 128, 2, 2), run_model_gpu(b, 128, 2, 2)
    assert np.array_equal(r1["y"], r2["y"]) and np.array_equal(r1["io"], r2["io"])
    assert np.array_equal(r1["params"], r2["params"]) and r1["loss"] == r2["loss"]
    b1 = configs.custom((300, 1500), k=6, P=1, halo=2)
    full = run_model_gpu(b1, 128, 2, 2)
    assert abs(full["loss"] - r1["loss"]) <= 1e-5 * full["loss"]
    assert np.array_equal(full["y"], r1["y"])   # partitioned forward = full graph, bitwise


def test_model_errors():
    from paper_2411_17164_b200 import xmgn
    from paper_2411_17164_b200.processor import Processor
    b = configs.custom((200,), k=6, P=2, halo=2)
    pr = Processor(b, 128, 2)
    params, io = pr.make_params(), pr.make_io_params()
    gp, gio = torch.zeros(pr.n_params, device="cuda"), torch.zeros_like(io)
    with pytest.raises(xmgn.XmgnError, match="ESTATE"):
        pr.model_backward(0, params, io, gp, gio)            # no model forward yet
    pos, nrm, t = pr.make_model_inputs(0, b)
    st = torch.as_tensor(stats32(b), device="cuda")
    with pytest.raises(xmgn.XmgnError, match="EINVAL"):
        pr.model_forward(0, params, io, pos, nrm, st, t, 200, None)   # targets without loss
    pr.model_forward(0, params, io, pos, nrm, st)                    # prediction only
    with pytest.raises(xmgn.XmgnError, match="ESTATE"):
        pr.model_backward(0, params, io, gp, gio)            # that forward had no targets
    assert xmgn.io_param_count(pr.cfg) == M.io_param_count(128, 2)
    pr.close()
