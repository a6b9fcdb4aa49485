"""Shared helpers for the GPU parity tests: run the CUDA path through the C-ABI
on a bundle and gather owned outputs / summed gradients in global order, and
the matching oracle computations (full graph or probe balls)."""
import numpy as np
import torch

import oracle
from xmgn_inputs import tensors


def run_gpu(bundle, H, L, prec, m=2, g_rows=None, want_inputs=True, halo_depth=None, param_fn=None, g_scale=1.0):
    """Returns dict(h [N,H] owned outputs in global order, params grad, h0/e0 grads
    scatter-added over partitions).  g_rows: optional bool mask of global rows
    where the upstream gradient is non-zero (else all); param_fn(params: np.ndarray
    FP64) -> modified params (BF16-representable values); g_scale multiplies g."""
    from paper_2411_17164_b200.processor import Processor
    pr = Processor(bundle, H, L, m=m, precision=prec, halo_depth=halo_depth)
    params = pr.make_params()
    if param_fn is not None:
        params = torch.as_tensor(param_fn(params.double().cpu().numpy()), dtype=torch.float32, device="cuda")
    N, E = len(bundle["offsets"]) - 1, len(bundle["sources"])
    gp = torch.zeros(pr.n_params, device="cuda")
    h = np.zeros((N, H))
    gh = np.zeros((N, H)) if want_inputs else None
    ge = np.zeros((E, H)) if want_inputs else None
    for p in pr.parts:
        inf = pr.info[p]
        h0, e0, g = pr.make_inputs(p)
        if g_rows is not None:
            g = g * torch.as_tensor(g_rows[inf["gid"][:inf["n_owned"]]], device="cuda", dtype=torch.float32)[:, None]
        if g_scale != 1.0:
            g = (g.double() * g_scale).float()
        out = pr.forward(p, params, h0, e0)
        a, b = pr.backward(p, params, g, gp, want_inputs=want_inputs)
        h[inf["gid"][:inf["n_owned"]]] = out.double().cpu().numpy()
        if want_inputs:
            np.add.at(gh, inf["gid"], a.double().cpu().numpy())
            np.add.at(ge, inf["edge_gid"], b.double().cpu().numpy())
    torch.cuda.synchronize()
    res = dict(h=h, params=gp.double().cpu().numpy(), h0=gh, e0=ge, raw_params=params)
    pr.close()
    return res


def oracle_full(bundle, H, L, m=2, g_rows=None, param_fn=None, g_scale=1.0):
    off, src = bundle["offsets"], bundle["sources"]
    N, E = len(off) - 1, len(src)
    P = tensors.params(H, L, m).double().numpy()
    if param_fn is not None:
        P = param_fn(P)
    h0 = tensors.node_features(np.arange(N), H).double().numpy()
    e0 = tensors.edge_features(np.arange(E), H).double().numpy()
    g = tensors.upstream_grad(np.arange(N), H).double().numpy()
    if g_rows is not None:
        g = g * g_rows[:, None]
    if g_scale != 1.0:   # the FP32 values the GPU receives
        g = (g * g_scale).astype(np.float32).astype(np.float64)
    f = oracle.forward(off, src, P, h0, e0, H, L, m)
    b = oracle.backward(off, src, P, f, g, H, L, m)
    return dict(h=f["h"][-1], params=b["params"], h0=b["h0"], e0=b["e0"])


def oracle_probe(bundle, probe, H, L, m=2, with_grad=True):
    """Oracle on the L-hop ball of one probe node (itself a halo partition
    with one owned node): h^L of the probe, and the gradient of
    <g_probe, h^L_probe> (parameters, and h0/e0 scattered to global ids)."""
    off, src = bundle["offsets"], bundle["sources"]
    lg = oracle.local_graph(off, src, np.array([probe]), L)
    P = tensors.params(H, L, m).double().numpy()
    h0 = tensors.node_features(lg["gid"], H).double().numpy()
    e0 = tensors.edge_features(lg["edge_gid"], H).double().numpy()
    f = oracle.forward(lg["offsets"], lg["sources"], P, h0, e0, H, L, m)
    out = dict(h=f["h"][-1][0], gid=lg["gid"], edge_gid=lg["edge_gid"])
    if with_grad:
        g = np.zeros((len(lg["gid"]), H))
        g[0] = tensors.upstream_grad(np.array([probe]), H).double().numpy()[0]
        b = oracle.backward(lg["offsets"], lg["sources"], P, f, g, H, L, m)
        out.update(params=b["params"], h0=b["h0"], e0=b["e0"])
    return out


def max_over_rms(a, ref):
    return float(np.abs(a - ref).max() / np.sqrt((ref ** 2).mean()))


def row_max_over_rms(a, ref):
    """max over rows i of ||a_i - ref_i||_2 / RMS_i(||ref_i||_2): a wrong or missing
    row shows up as O(1) even when the whole-tensor Frobenius error stays small."""
    rn = np.sqrt(((ref ** 2).sum(axis=1)).mean())
    return float(np.sqrt(((a - ref) ** 2).sum(axis=1)).max() / max(rn, 1e-300))


def rel_fro(a, ref):
    return float(np.linalg.norm(a - ref) / max(np.linalg.norm(ref), 1e-300))


def per_tensor_rel(gp, ref, H, L, m=2):
    lay, _ = tensors.param_layout(H, L, m)
    worst, name = 0.0, ""
    for nm, l, blk, slot, o, shape, fan in lay:
        n = int(np.prod(shape))
        e = rel_fro(gp[o:o + n], ref[o:o + n])
        if e > worst:
            worst, name = e, f"{nm}[l={l},{'edge' if blk == 0 else 'node'}]"
    return worst, name
