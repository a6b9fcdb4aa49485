"""FP64 oracle of the model AROUND the processor (NEXT-1) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module; the product never does.

What it computes, step by step in the paper's order:

* node inputs, 24 per point ("24 input features, including Fourier
  features with 3 different frequencies (i.e., 2pi, 4pi, 8pi)"
  "3D positions of surface points, surface normals, and Fourier features ...
  the sine and cosine of the position coordinates"): [x, n, then per frequency
  f (freq-major) and coordinate c (coordinate-minor) sin(f c), cos(f c)]
  (SPEC.md:134-141 fixes the column order);
* edge inputs, 4 per edge ("relative position vector x_j - x_i or the
  distance ||x_j - x_i||"): (x_src - x_dst, ||x_src - x_dst||),
  sender minus receiver;
* z-score normalisation with per-variable global mean / std;
* encoders: MLP (m hidden SiLU layers, linear output) + LayerNorm, no residual
  (SPEC.md "per-row layernorm after encoder and each processor MLP");
* the processor (oracle.forward / oracle.backward, Eqs. 1-4);
* decoder: MLP to d_out = 4 outputs (p, tau_x, tau_y, tau_z), no LN;
* loss: MSE over the owned rows only ("Halo nodes are filtered out
  before the loss computation", "mean squared error"), normalised by
  the GLOBAL N * d_out so per-partition losses and gradients sum to the full
  graph's (SPEC.md:468, 504 reading P15).

IO parameter layout (flat FP64 here; an independent restatement of include/xmgn.h
``xmgn_io_param_count``): node encoder [W1 (24 x H), b1, (Wj (H x H), bj) j=2..m+1,
gamma, beta], edge encoder [W1 (4 x H), b1, ..., gamma, beta], decoder [W1 (H x H),
b1, (Wj, bj) j=2..m, W_{m+1} (H x d_out), b_{m+1} (d_out)]; y = x W + b.

Backward: hand-written adjoints (Linear: dW = x^T dz, db = sum dz, dx = dz W^T;
SiLU' = s (1 + t (1 - s)); LN as in oracle.cpp), no autograd.  Pins:
tests/test_model_oracle.py (dense PyTorch-FP64 autograd of the whole model,
the SPEC feature examples, SSE additivity over partitions, finite differences).
"""
import math

import numpy as np

import oracle

FREQS = (2.0 * math.pi, 4.0 * math.pi, 8.0 * math.pi)
F_NODE, F_EDGE, D_OUT = 24, 4, 4


# ------------------------------------------------------------------ inputs
def node_inputs(pos, nrm):
    pos = np.asarray(pos, np.float64)
    nrm = np.asarray(nrm, np.float64)
    cols = [pos[:, 0], pos[:, 1], pos[:, 2], nrm[:, 0], nrm[:, 1], nrm[:, 2]]
    for f in FREQS:
        for c in range(3):
            cols.append(np.sin(f * pos[:, c]))
            cols.append(np.cos(f * pos[:, c]))
    return np.stack(cols, 1)


def edge_inputs(pos, offsets, sources):
    pos = np.asarray(pos, np.float64)
    offsets = np.asarray(offsets, np.int64)
    N = len(offsets) - 1
    dst = np.repeat(np.arange(N), np.diff(offsets))
    d = pos[np.asarray(sources, np.int64)] - pos[dst]
    return np.concatenate([d, np.sqrt((d * d).sum(1))[:, None]], 1)


def feature_stats(pos, nrm, offsets, sources):
    """Per-variable global mean and std (population) of the raw inputs: (mean, std) of
    the 24 node then the 4 edge columns.  A zero std is replaced by 1."""
    Xn, Xe = node_inputs(pos, nrm), edge_inputs(pos, offsets, sources)
    mean = np.concatenate([Xn.mean(0), Xe.mean(0)])
    std = np.concatenate([Xn.std(0), Xe.std(0)])
    std[std == 0] = 1.0
    return mean, std


def zscore(X, mean, std):
    return (X - mean) / std


# ------------------------------------------------------------------ layout
def io_layout(H, m=2, fn=F_NODE, fe=F_EDGE, d=D_OUT):
    """{block: [(name, offset, shape)]} and the total count."""
    out, off = {}, 0

    def add(blk, name, shape):
        nonlocal off
        out.setdefault(blk, []).append((name, off, shape))
        off += int(np.prod(shape))

    for blk, fin in (("node_enc", fn), ("edge_enc", fe)):
        add(blk, "W1", (fin, H)); add(blk, "b1", (H,))
        for j in range(2, m + 2):
            add(blk, f"W{j}", (H, H)); add(blk, f"b{j}", (H,))
        add(blk, "gamma", (H,)); add(blk, "beta", (H,))
    add("dec", "W1", (H, H)); add("dec", "b1", (H,))
    for j in range(2, m + 1):
        add("dec", f"W{j}", (H, H)); add("dec", f"b{j}", (H,))
    add("dec", f"W{m + 1}", (H, d)); add("dec", f"b{m + 1}", (d,))
    return out, off


def io_param_count(H, m=2):
    return io_layout(H, m)[1]


def _views(io, H, m):
    lay, n = io_layout(H, m)
    assert io.size == n, (io.size, n)
    return {blk: {name: io[o:o + int(np.prod(s))].reshape(s) for name, o, s in items}
            for blk, items in lay.items()}


# ------------------------------------------------------------------ MLPs
def _silu(t):
    return t / (1.0 + np.exp(-t))


def _dsilu(t):
    s = 1.0 / (1.0 + np.exp(-t))
    return s * (1.0 + t * (1.0 - s))


def _mlp_fwd(X, B, m, ln, eps):
    """z_1 = X W1 + b1, z_{j+1} = SiLU(z_j) W_{j+1} + b_{j+1}; optional LN(z_{m+1})."""
    zs = [X @ B["W1"] + B["b1"]]
    for j in range(2, m + 2):
        zs.append(_silu(zs[-1]) @ B[f"W{j}"] + B[f"b{j}"])
    out = zs[-1]
    if ln:
        mu = out.mean(1, keepdims=True)
        var = ((out - mu) ** 2).mean(1, keepdims=True)
        r = 1.0 / np.sqrt(var + eps)
        xh = (out - mu) * r
        out = B["gamma"] * xh + B["beta"]
        return out, dict(zs=zs, xh=xh, r=r)
    return out, dict(zs=zs)


def _mlp_bwd(X, B, m, ln, cache, dY, G):
    """Adjoint of _mlp_fwd: accumulates parameter gradients into the views G."""
    zs = cache["zs"]
    if ln:
        xh, r = cache["xh"], cache["r"]
        G["gamma"] += (dY * xh).sum(0)
        G["beta"] += dY.sum(0)
        dxh = dY * B["gamma"]
        dz = r * (dxh - dxh.mean(1, keepdims=True) - xh * (dxh * xh).mean(1, keepdims=True))
    else:
        dz = dY
    for j in range(m + 1, 1, -1):
        a = _silu(zs[j - 2])
        G[f"W{j}"] += a.T @ dz
        G[f"b{j}"] += dz.sum(0)
        dz = (dz @ B[f"W{j}"].T) * _dsilu(zs[j - 2])
    G["W1"] += X.T @ dz
    G["b1"] += dz.sum(0)
    return dz @ B["W1"].T


# ------------------------------------------------------------------ the model
def forward(offsets, sources, pos, nrm, params, io, stats, H, L, m=2, eps=1e-5, targets=None, n_owned=None,
            n_global=None):
    """Encoder -> processor -> decoder on one (local or full) graph.

    Returns dict(y = predictions of every row [N, 4], loss = SSE over the owned prefix
    / (n_global * 4) (None without targets), and the caches the backward needs)."""
    mean, std = stats
    N = len(offsets) - 1
    n_owned = N if n_owned is None else n_owned
    n_global = N if n_global is None else n_global
    V = _views(np.asarray(io, np.float64), H, m)
    Xn = zscore(node_inputs(pos, nrm), mean[:F_NODE], std[:F_NODE])
    Xe = zscore(edge_inputs(pos, offsets, sources), mean[F_NODE:], std[F_NODE:])
    h0, cn = _mlp_fwd(Xn, V["node_enc"], m, True, eps)
    e0, ce = _mlp_fwd(Xe, V["edge_enc"], m, True, eps)
    f = oracle.forward(offsets, sources, params, h0, e0, H, L, m, eps)
    y, cd = _mlp_fwd(f["h"][-1], V["dec"], m, False, eps)
    loss = None
    if targets is not None:
        t = np.asarray(targets, np.float64)
        diff = y[:n_owned] - t[:n_owned]
        loss = float((diff * diff).sum()) / (n_global * D_OUT)
    return dict(y=y, loss=loss, Xn=Xn, Xe=Xe, cn=cn, ce=ce, cd=cd, proc=f, n_owned=n_owned, n_global=n_global,
                targets=targets)


def backward(offsets, sources, params, io, fw, H, L, m=2, eps=1e-5):
    """Gradients of fw's loss: dict(params = processor gradient, io = IO gradient)."""
    io = np.asarray(io, np.float64)
    V = _views(io, H, m)
    gio = np.zeros_like(io)
    GV = _views(gio, H, m)
    y, n_owned = fw["y"], fw["n_owned"]
    t = np.asarray(fw["targets"], np.float64)
    dy = np.zeros_like(y)
    dy[:n_owned] = 2.0 * (y[:n_owned] - t[:n_owned]) / (fw["n_global"] * D_OUT)
    g = _mlp_bwd(fw["proc"]["h"][-1], V["dec"], m, False, fw["cd"], dy, GV["dec"])
    b = oracle.backward(offsets, sources, params, fw["proc"], g, H, L, m, eps)
    _mlp_bwd(fw["Xn"], V["node_enc"], m, True, fw["cn"], b["h0"], GV["node_enc"])
    _mlp_bwd(fw["Xe"], V["edge_enc"], m, True, fw["ce"], b["e0"], GV["edge_enc"])
    return dict(params=b["params"], io=gio, g=g)
