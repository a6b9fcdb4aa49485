"""Host-side convenience layer over the C-ABI (argument marshalling only).

``Processor`` owns one graph handle + one workspace on one GPU and runs the
partitions assigned to this rank sequentially (several partitions
per GPU), accumulating parameter gradients in fixed partition order
(PAPER.md:176).  Synthetic per-partition inputs are hashed from GLOBAL ids by
``xmgn_inputs.tensors`` so every partition sees exactly the full graph's values.
All arithmetic of the method runs inside libxmgn.so.
"""
import numpy as np
import torch

from . import xmgn
from xmgn_inputs import tensors


class Processor:
    def __init__(self, bundle, H, L, m=2, precision=xmgn.PREC_FP16, device=0, parts=None, halo_depth=None,
                 ln_eps=1e-5, infer=False):
        torch.cuda.set_device(device)
        self.device = torch.device("cuda", device)
        self.H, self.L, self.m = H, L, m
        depth = L if halo_depth is None else halo_depth
        self.graph = xmgn.Graph.from_bundle(bundle, depth, device)
        self.cfg = xmgn.model_cfg(H, L, m, precision, ln_eps)
        self.ws = xmgn.Workspace(self.graph, self.cfg, infer=infer)
        self.parts = list(range(self.graph.n_parts)) if parts is None else list(parts)
        self.info = {p: self.graph.export(p) for p in self.parts}
        self.n_params = xmgn.param_count(self.cfg)

    # ------------------------------------------------------------------ inputs
    def make_inputs(self, p):
        """h0 [n_local,H], e0 [e_local,H], g [n_owned,H] on the device (hash of global ids)."""
        inf = self.info[p]
        gid = torch.as_tensor(inf["gid"], device=self.device)
        egid = torch.as_tensor(inf["edge_gid"], device=self.device)
        h0 = tensors.node_features(gid, self.H, self.device)
        e0 = tensors.edge_features(egid, self.H, self.device)
        g = tensors.upstream_grad(gid[:inf["n_owned"]], self.H, self.device)
        return h0, e0, g

    def make_params(self):
        return tensors.params(self.H, self.L, self.m, self.device)

    # ------------------------------------------------------------------ compute
    def forward(self, p, params, h0, e0, stream=None):
        out = torch.empty((self.info[p]["n_owned"], self.H), dtype=torch.float32, device=self.device)
        self.ws.forward(p, params, h0, e0, out, stream)
        return out

    def backward(self, p, params, g, grad_params, want_inputs=False, stream=None):
        gh0 = ge0 = None
        if want_inputs:
            gh0 = torch.empty((self.info[p]["n_local"], self.H), dtype=torch.float32, device=self.device)
            ge0 = torch.empty((self.info[p]["e_local"], self.H), dtype=torch.float32, device=self.device)
        self.ws.backward(p, params, g, grad_params, gh0, ge0, stream)
        return gh0, ge0

    def step(self, params, grad_params, inputs, stream=None):
        """fwd + bwd of every local partition (gradients summed in order)."""
        outs = []
        for p in self.parts:
            h0, e0, g = inputs[p]
            outs.append(self.forward(p, params, h0, e0, stream))
            self.backward(p, params, g, grad_params, stream=stream)
        return outs

    def infer(self, params, inputs, stream=None):
        """Forward of every local partition; returns (rows [sum n_owned, H], global ids) of the
        owned rows in partition order -- halo predictions are never returned."""
        outs, gids = [], []
        for p in self.parts:
            h0, e0 = inputs[p][0], inputs[p][1]
            outs.append(self.forward(p, params, h0, e0, stream))
            gids.append(self.info[p]["gid"][:self.info[p]["n_owned"]])
        return torch.cat(outs), np.concatenate(gids)

    # ------------------------------------------------------------------ the full model (NEXT-1)
    def make_model_inputs(self, p, bundle):
        """pos, nrm [n_local, 3] (local order) and z-scored targets [n_owned, 4] on the device."""
        inf = self.info[p]
        gid = inf["gid"]
        pos = torch.as_tensor(np.ascontiguousarray(bundle["positions"][gid], np.float32), device=self.device)
        nrm = torch.as_tensor(np.ascontiguousarray(bundle["normals"][gid], np.float32), device=self.device)
        t = tensors.targets(torch.as_tensor(gid[:inf["n_owned"]], device=self.device), self.device)
        return pos, nrm, t

    def make_io_params(self):
        return tensors.io_params(self.H, self.m, self.device)

    def model_forward(self, p, params, io_params, pos, nrm, stats, targets=None, n_global=0, loss=None, stream=None):
        pred = torch.empty((self.info[p]["n_owned"], xmgn.IO_DOUT), dtype=torch.float32, device=self.device)
        self.ws.model_forward(p, params, io_params, pos, nrm, stats, pred, targets, n_global, loss, stream)
        return pred

    def model_backward(self, p, params, io_params, grad_params, grad_io, stream=None):
        self.ws.model_backward(p, params, io_params, grad_params, grad_io, stream)

    def close(self):
        self.ws.close()
        self.graph.close()
