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
