"""Brute-force dense-adjacency checker (TEST INFRASTRUCTURE ONLY), PyTorch FP64 CPU.

An independent second statement of the processor used to pin ``oracle.cpp``:
edges live in a dense N x N x H tensor (entry [i, j] = e_{j->i}), every MLP is
``torch.nn.functional.linear``/``silu``/``layer_norm`` over all N^2 pairs, the
aggregation is a masked dense sum a_i = sum_j A_ij e'_{j->i} (PAPER.md:134,
Eq. 2) and all gradients come from autograd.  For N <= 64 only.
"""
import torch
import torch.nn.functional as F


def _slices(params, H, L, m):
    """Views of the flat parameter vector in ABI order."""
    out, off = [], 0

    def take(*shape):
        nonlocal off
        n = 1
        for s in shape:
            n *= s
        t = params[off:off + n].view(*shape)
        off += n
        return t

    for _ in range(L):
        layer = []
        for kin in (3 * H, 2 * H):
            Ws, bs = [], []
            for j in range(m + 1):
                Ws.append(take(kin if j == 0 else H, H))
                bs.append(take(H))
            layer.append(dict(W=Ws, b=bs, gamma=take(H), beta=take(H)))
        out.append(layer)
    assert off == params.numel()
    return out


def _mlp_ln(x, blk, eps):
    z = F.linear(x, blk["W"][0].t(), blk["b"][0])
    for W, b in zip(blk["W"][1:], blk["b"][1:]):
        z = F.linear(F.silu(z), W.t(), b)
    return F.layer_norm(z, (z.shape[-1],), blk["gamma"], blk["beta"], eps)


def run(offsets, sources, params, h0, e0, g, H, L, m=2, eps=1e-5):
    """Returns dict(h=[L+1 x N x H], grads params/h0/e0) from dense autograd."""
    offsets = torch.as_tensor(offsets, dtype=torch.int64)
    sources = torch.as_tensor(sources, dtype=torch.int64)
    N = len(offsets) - 1
    dst = torch.repeat_interleave(torch.arange(N), offsets[1:] - offsets[:-1])
    A = torch.zeros(N, N, dtype=torch.float64)
    A[dst, sources] = 1.0
    P = torch.tensor(params, dtype=torch.float64, requires_grad=True)
    h = torch.tensor(h0, dtype=torch.float64, requires_grad=True)
    e0t = torch.tensor(e0, dtype=torch.float64, requires_grad=True)
    Ed = torch.zeros(N, N, H, dtype=torch.float64).index_put((dst, sources), e0t)
    blocks = _slices(P, H, L, m)
    hs = [h]
    hcur, Ecur = h, Ed
    for l in range(L):
        hi = hcur[:, None, :].expand(N, N, H)   # receiver i
        hj = hcur[None, :, :].expand(N, N, H)   # sender j
        Y = _mlp_ln(torch.cat([Ecur, hj, hi], -1), blocks[l][0], eps)
        Ecur = Ecur + Y * A[..., None]
        a = (A[..., None] * Ecur).sum(1)
        hcur = hcur + _mlp_ln(torch.cat([hcur, a], -1), blocks[l][1], eps)
        hs.append(hcur)
    loss = (torch.as_tensor(g, dtype=torch.float64) * hcur).sum()
    gP, gh, gE = torch.autograd.grad(loss, [P, h, e0t])
    return dict(h=torch.stack([x.detach() for x in hs]).numpy(), params=gP.numpy(),
                h0=gh.numpy(), e0=gE.numpy())


# ------------------------------------------------------------ the whole model (NEXT-1 pin)
def _io_slices(io, H, m, fn=24, fe=4, d=4):
    off = 0

    def take(*shape):
        nonlocal off
        n = 1
        for s in shape:
            n *= s
        t = io[off:off + n].view(*shape)
        off += n
        return t

    out = {}
    for name, fin in (("node", fn), ("edge", fe)):
        Ws, bs = [take(fin, H)], [take(H)]
        for _ in range(m):
            Ws.append(take(H, H)); bs.append(take(H))
        out[name] = dict(W=Ws, b=bs, gamma=take(H), beta=take(H))
    Ws, bs = [], []
    for j in range(m + 1):
        Ws.append(take(H, d if j == m else H)); bs.append(take(d if j == m else H))
    out["dec"] = dict(W=Ws, b=bs)
    assert off == io.numel()
    return out


def _mlp(x, blk):
    z = F.linear(x, blk["W"][0].t(), blk["b"][0])
    for W, b in zip(blk["W"][1:], blk["b"][1:]):
        z = F.linear(F.silu(z), W.t(), b)
    return z


def run_model(offsets, sources, pos, nrm, params, io, stats, targets, H, L, m=2, eps=1e-5, n_owned=None,
              n_global=None):
    """Dense-autograd statement of encoder -> processor -> decoder -> owned-row MSE
    (PAPER.md:161, 197, 219, 234).  Returns dict(y, loss, params, io) (gradients by autograd)."""
    offsets = torch.as_tensor(offsets, dtype=torch.int64)
    sources = torch.as_tensor(sources, dtype=torch.int64)
    N = len(offsets) - 1
    n_owned = N if n_owned is None else n_owned
    n_global = N if n_global is None else n_global
    dst = torch.repeat_interleave(torch.arange(N), offsets[1:] - offsets[:-1])
    A = torch.zeros(N, N, dtype=torch.float64)
    A[dst, sources] = 1.0
    x = torch.as_tensor(pos, dtype=torch.float64)
    nv = torch.as_tensor(nrm, dtype=torch.float64)
    mean = torch.as_tensor(stats[0], dtype=torch.float64)
    std = torch.as_tensor(stats[1], dtype=torch.float64)
    four = []
    for k in (1, 2, 4):
        ang = 2.0 * torch.pi * k * x          # [N, 3]
        four.append(torch.stack([torch.sin(ang), torch.cos(ang)], -1).reshape(N, 6))
    Xn = (torch.cat([x, nv] + four, 1) - mean[:24]) / std[:24]
    rel = x[sources] - x[dst]
    Xe = (torch.cat([rel, rel.norm(dim=1, keepdim=True)], 1) - mean[24:]) / std[24:]
    P = torch.tensor(params, dtype=torch.float64, requires_grad=True)
    IO = torch.tensor(io, dtype=torch.float64, requires_grad=True)
    S = _io_slices(IO, H, m)
    h = F.layer_norm(_mlp(Xn, S["node"]), (H,), S["node"]["gamma"], S["node"]["beta"], eps)
    e0 = F.layer_norm(_mlp(Xe, S["edge"]), (H,), S["edge"]["gamma"], S["edge"]["beta"], eps)
    Ecur = torch.zeros(N, N, H, dtype=torch.float64).index_put((dst, sources), e0)
    blocks = _slices(P, H, L, m)
    for l in range(L):
        hi = h[:, None, :].expand(N, N, H)
        hj = h[None, :, :].expand(N, N, H)
        Ecur = Ecur + _mlp_ln(torch.cat([Ecur, hj, hi], -1), blocks[l][0], eps) * A[..., None]
        a = (A[..., None] * Ecur).sum(1)
        h = h + _mlp_ln(torch.cat([h, a], -1), blocks[l][1], eps)
    y = _mlp(h, S["dec"])
    t = torch.as_tensor(targets, dtype=torch.float64)
    loss = F.mse_loss(y[:n_owned], t[:n_owned], reduction="sum") / (n_global * 4)
    gP, gIO = torch.autograd.grad(loss, [P, IO])
    return dict(y=y.detach().numpy(), loss=float(loss.detach()), params=gP.numpy(), io=gIO.numpy())
