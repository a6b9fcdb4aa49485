"""NEXT-2: the optimiser step after gradient aggregation (Sec. V-D).

CPU: the FP64 oracle (oracle/optim.py) pinned to the schedule's closed-form end
points, the clipping example of SPEC.md:380, torch.optim.Adam + clip_grad_norm_
in float64 (a library statement of the same update), and SPEC.md:470-472's
multi-step equivalence: partitioned training (halo = L, summed gradients) equals
full-graph training after 1 and 50 steps (FP64, <= 1e-9 / 1e-7 relative).
GPU: xmgn_adam_step against the oracle on the same inputs, and a 3-step GPU
training run against the oracle's."""
import math

import numpy as np
import pytest
import torch

import oracle
from oracle import optim
from xmgn_inputs import configs, tensors


def test_cosine_schedule_endpoints():
    T = 1000
    assert optim.cosine_lr(0, T) == pytest.approx(1e-3, rel=1e-15)
    assert optim.cosine_lr(T, T) == pytest.approx(1e-6, rel=1e-12)
    assert optim.cosine_lr(T // 2, T) == pytest.approx(0.5 * (1e-3 + 1e-6), rel=1e-12)
    assert optim.cosine_lr(5 * T, T) == optim.cosine_lr(T, T)       # clamped after the schedule
    lrs = [optim.cosine_lr(t, T) for t in range(T + 1)]
    assert all(a >= b for a, b in zip(lrs, lrs[1:]))                 # monotone decay


def test_clip_example_spec():
    """global norm 64 with threshold 32 -> every gradient scaled by 0.5."""
    g = np.full(16, 16.0)                                            # ||g|| = 64
    c, norm = optim.clip_global_norm(g, 32.0)
    assert norm == 64.0
    np.testing.assert_allclose(c, 8.0, rtol=1e-7)
    c2, _ = optim.clip_global_norm(g * 0.25, 32.0)                   # norm 16 < 32: unchanged
    np.testing.assert_array_equal(c2, g * 0.25)


def test_adam_matches_torch_float64():
    rng = np.random.default_rng(0)
    n, T = 5000, 30
    p0 = rng.standard_normal(n)
    grads = [rng.standard_normal(n) * (100.0 if t % 3 == 0 else 0.01) for t in range(T)]   # clip on / off
    tp = torch.tensor(p0, dtype=torch.float64, requires_grad=True)
    opt = torch.optim.Adam([tp], lr=1e-3, betas=(0.9, 0.999), eps=1e-8)
    sched = torch.optim.lr_scheduler.LambdaLR(opt, lambda t: optim.cosine_lr(t, T) / 1e-3)
    p, m, v = p0.copy(), np.zeros(n), np.zeros(n)
    for t in range(T):
        tp.grad = torch.tensor(grads[t], dtype=torch.float64)
        torch.nn.utils.clip_grad_norm_([tp], 32.0)
        opt.step()
        sched.step()
        p, m, v, _ = optim.adam_step(p, grads[t], m, v, t, T)
    np.testing.assert_allclose(p, tp.detach().numpy(), rtol=1e-12, atol=1e-14)


def _train(b, parts, steps, H=8, L=3):
    """`steps` FP64 training steps of the processor with an SSE loss over owned rows against
    hashed targets; partitions' gradients are summed, then one Adam step."""
    off, src = b["offsets"], b["sources"]
    N = len(off) - 1
    P = tensors.params(H, L).double().numpy()
    y = tensors.upstream_grad(np.arange(N), H).double().numpy()      # any fixed targets
    m, v = np.zeros_like(P), np.zeros_like(P)
    for t in range(steps):
        G = np.zeros_like(P)
        for owned in parts:
            lg = oracle.local_graph(off, src, owned, L)
            f = oracle.forward(lg["offsets"], lg["sources"], P, tensors.node_features(lg["gid"], H).double().numpy(),
                               tensors.edge_features(lg["edge_gid"], H).double().numpy(), H, L)
            g = np.zeros((len(lg["gid"]), H))
            no = lg["n_owned"]
            g[:no] = 2.0 * (f["h"][-1][:no] - y[lg["gid"][:no]])     # d SSE / d h^L, owned rows only
            G += oracle.backward(lg["offsets"], lg["sources"], P, f, g, H, L)["params"]
        P, m, v, _ = optim.adam_step(P, G, m, v, t, steps, grad_scale=1.0 / (N * H))
    return P


def test_partitioned_training_equals_full_graph_training():
    """SPEC.md:470-472 on the oracle: n = 500, k = 6, L = 3, P = 4, halo = 3, FP64."""
    b = configs.custom((500,), k=6, P=4, halo=3)
    oo = b["owned_offsets"]
    parts = [b["owned"][oo[p]:oo[p + 1]] for p in range(4)]
    full = [np.arange(len(b["offsets"]) - 1)]
    for steps, tol in ((1, 1e-9), (50, 1e-7)):
        a, c = _train(b, parts, steps), _train(b, full, steps)
        assert np.abs(a - c).max() / np.abs(c).max() <= tol, steps


@pytest.mark.gpu
def test_gpu_adam_step_matches_oracle():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2411_17164_b200 import xmgn
    rng = np.random.default_rng(1)
    n, T = 1_000_003, 5
    p = rng.standard_normal(n).astype(np.float32) * 0.05
    opt = xmgn.Adam(n, T)
    tp = torch.tensor(p, device="cuda")
    pr, m, v = p.astype(np.float64), np.zeros(n), np.zeros(n)
    for t in range(T):
        g = (rng.standard_normal(n) * (1e3 if t % 2 == 0 else 1e-3)).astype(np.float32)   # clip on / off
        opt.step(tp, torch.tensor(g, device="cuda"), grad_scale=0.5)
        pr, m, v, norm = optim.adam_step(pr, g.astype(np.float64), m, v, t, T, grad_scale=np.float32(0.5))
        torch.cuda.synchronize()
        assert abs(float(opt.norm.item()) - norm) <= 1e-6 * norm
        assert opt.lr(t) == pytest.approx(optim.cosine_lr(t, T), rel=1e-6)
    got = tp.double().cpu().numpy()
    assert np.abs(got - pr).max() <= 1e-6 * np.abs(pr).max()
    assert np.abs(opt.m.double().cpu().numpy() - m).max() <= 1e-5 * np.abs(m).max()


@pytest.mark.gpu
def test_gpu_training_steps_follow_oracle():
    """Three steps of partitioned GPU training (fwd + bwd per partition in FP16, gradients
    summed, MSE scale 1/(N d), xmgn_adam_step) against the oracle's FP64 training: the
    parameter updates point the same way (cosine > 0.99) and land within 2e-2 relative."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2411_17164_b200 import xmgn
    from paper_2411_17164_b200.processor import Processor
    H, L, T = 128, 3, 3
    b = configs.custom((300, 1500), k=6, P=4, halo=L)
    N = len(b["offsets"]) - 1
    pr_ = Processor(b, H, L)
    params = pr_.make_params()
    p0 = params.double().cpu().numpy()
    y = tensors.upstream_grad(np.arange(N), H).to("cuda")
    opt = xmgn.Adam(pr_.n_params, T)
    inputs = {p: pr_.make_inputs(p) for p in pr_.parts}
    for t in range(T):
        grad = torch.zeros(pr_.n_params, device="cuda")
        for p in pr_.parts:
            inf = pr_.info[p]
            h0, e0, _ = inputs[p]
            out = pr_.forward(p, params, h0, e0)
            g = 2.0 * (out - y[torch.as_tensor(inf["gid"][:inf["n_owned"]], device="cuda")])
            pr_.backward(p, params, g.contiguous(), grad)
        opt.step(params, grad, grad_scale=1.0 / (N * H))
    torch.cuda.synchronize()
    got = params.double().cpu().numpy()
    pr_.close()
    oo = b["owned_offsets"]
    ref = _train(b, [b["owned"][oo[p]:oo[p + 1]] for p in range(4)], T, H=H, L=L)
    du, dr = got - p0, ref - p0
    cos = float(du @ dr / (np.linalg.norm(du) * np.linalg.norm(dr)))
    rel = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    print(f"3-step training: update cosine {cos:.5f}, parameter rel {rel:.2e}")
    assert cos > 0.99 and rel <= 2e-2
